"""Cost of the peer-sharded protocol on ONE GPU: it/s of the single-rank persistent kernel
vs R emulated ranks (rgdbek_group_create: one cooperative launch of R x G CTAs over the
same HBM).  The ranks share one GPU's bandwidth, so this measures the exchange protocol's
overhead (extra barriers, owner reduces, halo copies), not a speedup.
usage: python tools/sharded_probe.py C3 [steps]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    from workloads import by_name
    from paper_2509_19267_b200 import Solver, ShardGroup
    from paper_2509_19267_b200.dist import partition_rows, shard_csr
    name = sys.argv[1]
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
    w = by_name(name)
    m, n = w.shape
    out = {"workload": name, "steps": steps}
    s = Solver(w.A, w.b, eta=w.eta) if w.dense else Solver.from_scipy(w.A, w.b, eta=w.eta, symmetric=w.symmetric)
    s.reset(0); s.step(3); s.reset(0)
    r = s.step(steps)
    out["single_it_s"] = round(steps / r["seconds"], 1)
    s.close()
    for R in (2, 4, 8):
        parts = partition_rows(m if w.dense else w.A.indptr, R)
        ss = []
        for (r0, r1) in parts:
            if w.dense:
                ss.append(Solver(w.A[r0:r1], w.b[r0:r1], eta=w.eta, m=m, row_range=(r0, r1)))
            else:
                rp, ci, val = shard_csr(*w.csr_arrays(), r0, r1)
                ss.append(Solver.from_csr(m, n, rp, ci, val, w.b[r0:r1], eta=w.eta, row_range=(r0, r1)))
        g = ShardGroup(ss)
        g.reset(0); g.step(3); g.reset(0)
        r = g.step(steps)
        out[f"R{R}_it_s"] = round(steps / r["seconds"], 1)
        wins = [tuple(x.peer_window()[:2]) for x in ss]
        out[f"R{R}_windows"] = wins
        g.close()
        for x in ss:
            x.close()
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
