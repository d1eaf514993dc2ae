"""A/B of create-time env settings in ONE process (one workload build, solvers side by side,
interleaved timing) — for workloads too large to rebuild per variant (C5).

usage: python tools/ab_pf.py C5c "RGDBEK_TILE_PF=0" "RGDBEK_TILE_PF=T" [--steps 50 --reps 3]
"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    argv = sys.argv[1:]
    steps, reps = 50, 3
    if "--steps" in argv:
        i = argv.index("--steps"); steps = int(argv[i + 1]); del argv[i:i + 2]
    if "--reps" in argv:
        i = argv.index("--reps"); reps = int(argv[i + 1]); del argv[i:i + 2]
    from workloads import by_name
    from paper_2509_19267_b200 import Solver
    for wl in argv[0].split(","):
        w = by_name(wl)
        ss = []
        for v in argv[1:]:
            kv = dict(x.split("=", 1) for x in v.split(",")) if v != "base" else {}
            old = {k: os.environ.get(k) for k in kv}
            os.environ.update(kv)
            s = Solver(w.A, w.b, eta=w.eta) if w.dense else \
                Solver.from_scipy(w.A, w.b, eta=w.eta, symmetric=w.symmetric)
            for k, o in old.items():
                if o is None:
                    os.environ.pop(k)
                else:
                    os.environ[k] = o
            ss.append((v, s))
        res = {}
        for _ in range(reps):
            for v, s in ss:
                s.reset(0)
                s.step(3)
                r = s.step(steps)
                res.setdefault(v, []).append(steps / r["seconds"])
        xs0 = None
        for v, s in ss:
            xs = res[v]
            print(json.dumps({"workload": wl, "variant": v, "it_s": round(statistics.median(xs), 2),
                              "all": [round(x, 2) for x in xs]}), flush=True)
            s.close()
        del w


if __name__ == "__main__":
    main()
