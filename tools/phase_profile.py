"""Per-phase device time of the persistent engine (RGDBEK_PHASE_TIMING=1).

usage: python tools/phase_profile.py C2c [steps] [grid]
Prints one JSON line: phase -> microseconds per iteration, plus it/s with and
without the instrumentation (the timer reads are by one thread of CTA 0).
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

PHASES = {1: "passT", 2: "s_v_colkeys_L1", 3: "colsel_L2", 4: "colsel_L3", 5: "mask_x_update",
          6: "passN", 7: "stop_z_rowkeys_L1", 8: "rowsel_L2", 9: "rowsel_L3", 10: "row_mask",
          0: "bookkeeping", 11: "dense_P2_columns", 12: "dense_P2_flush_sum",
          13: "colsel_local_L1", 14: "colsel_local_L2L3", 15: "rowsel_local"}


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C2c"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 500
    if len(sys.argv) > 3:
        os.environ["RGDBEK_GRID"] = sys.argv[3]
    from workloads import by_name
    from paper_2509_19267_b200 import Solver
    w = by_name(name)
    out = {"workload": name, "steps": steps}
    for timing in (0, 1):
        os.environ["RGDBEK_PHASE_TIMING"] = str(timing)
        s = (Solver(w.A, w.b, eta=w.eta) if w.dense else
             Solver.from_scipy(w.A, w.b, eta=w.eta, symmetric=w.symmetric))
        s.reset(0)
        s.step(5)
        s.reset(0)
        r = s.step(steps)
        out["engine_ctas"] = s.engine_info()[1]
        out[f"it_per_s_timing{timing}"] = steps / r["seconds"]
        if timing:
            t = s.phase_times()
            iters = steps + 5 + 2   # phase timers accumulate over every launch on the handle
            out["us_per_iter"] = {PHASES[i]: round(t[i] / 1e3 / iters, 2) for i in PHASES}
            out["us_per_iter_total"] = round(sum(t[i] for i in PHASES) / 1e3 / iters, 2)
            if len(t) > 17:
                out["local_sel_overflows"] = {"col": int(t[16]), "row": int(t[17])}
            if len(t) > 21:
                out["rowsel_local_split_us"] = {k: round(t[18 + i] / 1e3 / iters, 2) for i, k in
                                                enumerate(["gather", "level2", "level3", "rank"])}
        s.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
