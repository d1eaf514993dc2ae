"""Break the e2e (host-buffer) path into create / reset / step / get_x wall times.

usage: python tools/e2e_probe.py C1 [steps] [reps]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    from workloads import by_name
    from paper_2509_19267_b200 import Solver
    name = sys.argv[1] if len(sys.argv) > 1 else "C1"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 4
    w = by_name(name)
    A_h = torch.from_numpy(np.ascontiguousarray(w.A)).pin_memory()
    b_h = torch.from_numpy(w.b).pin_memory()
    x_h = torch.empty(w.A.shape[1], dtype=torch.float64).pin_memory()
    for r in range(reps):
        torch.cuda.synchronize()
        t = [time.perf_counter()]
        s = Solver(A_h, b_h, eta=w.eta)
        t.append(time.perf_counter())
        s.reset(0)
        t.append(time.perf_counter())
        s.step(steps)
        t.append(time.perf_counter())
        s.x(out=x_h)
        t.append(time.perf_counter())
        s.close()
        t.append(time.perf_counter())
        d = [round((b - a) * 1e3, 3) for a, b in zip(t, t[1:])]
        print(json.dumps({"rep": r, "ms": dict(zip(["create", "reset", "step", "get_x", "close"], d)),
                          "e2e_it_s": round(steps / (t[4] - t[0]), 1)}))


if __name__ == "__main__":
    main()
