"""Algorithm 2 (lazy averaging) on the paper's parallel test problems (tab:parSpeedupsm,
P:507-540): scipy.sparse.rand m x 20000 with 99 % sparsity (stored dense here: the
lazy mode is dense-only), x_true = rand, b = A x_true, eta = 0.1, stop at RSE <= 1e-4,
for P = 1, 2, 4, 8 logical processes.  Prints one JSON line per (m, P).

usage: python tools/lazy_paper_table.py [m ...]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import scipy.sparse as sp
    from paper_2509_19267_b200 import Solver
    ms = [int(a) for a in sys.argv[1:]] or [10000, 20000]
    n = 20000
    for m in ms:
        rng = np.random.default_rng(m)
        A = sp.random(m, n, density=0.01, format="csr", random_state=rng).toarray()
        xt = rng.random(n)
        b = A @ xt
        for P in (0, 1, 2, 4, 8):
            s = Solver(A, b, eta=0.1, stop="rse")
            if P:
                s.set_lazy(P)
            res = s.solve(1e-4, 20000, 0)
            print(json.dumps({"m": m, "n": n, "processes": P, "iters": res["iters"],
                              "outcome": res["outcome"], "rse": res["rse"],
                              "seconds": round(res["seconds"], 4)}), flush=True)
            s.close()


if __name__ == "__main__":
    main()
