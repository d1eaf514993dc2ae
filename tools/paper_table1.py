"""The paper's sequential random-matrix experiments (tab:fatmatrices P:312-335,
tab:tallmatrices P:337-359) on the GPU library: MATLAB-sprandn-like A at 99 %
sparsity (standard normal values), x_true = randn, b = A x_true, x0 = 0, z0 = b,
eta = 0.5, stop at RSE <= 1e-6.  Both updates: the paper's exact
projections (inner CGLS, rgdbek_set_mode 1) and the pseudoinverse-free sweep.
One JSON line per (shape, update), mean over `reps` seeds.

usage: python tools/paper_table1.py [reps]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SHAPES = [(500, 8000), (1000, 8000), (1500, 8000), (2000, 8000), (2500, 8000),
          (8000, 500), (8000, 1000), (8000, 1500), (8000, 2000), (8000, 2500)]
PAPER = {(500, 8000): (12.0, 0.360229), (1000, 8000): (14.0, 0.941294),
         (1500, 8000): (17.1, 2.434340), (2000, 8000): (20.9, 4.563865),
         (2500, 8000): (25.5, 6.927544), (8000, 500): (11.8, 0.401969),
         (8000, 1000): (14.1, 0.965721), (8000, 1500): (17.0, 2.304293),
         (8000, 2000): (20.6, 4.766493), (8000, 2500): (24.9, 8.396985)}


def main():
    import numpy as np
    import scipy.sparse as sp
    from paper_2509_19267_b200 import Solver
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    for (m, n) in SHAPES:
        for update in ("exact", "pinv_free"):
            its, secs = [], []
            for seed in range(reps):
                rng = np.random.default_rng(1000 * m + n + seed)
                A = sp.random(m, n, density=0.01, format="csr", random_state=rng,
                              data_rvs=rng.standard_normal)
                A.sort_indices()
                b = A @ rng.standard_normal(n)
                s = Solver.from_scipy(A, b, eta=0.5, stop="rse")
                if update == "exact":
                    s.set_mode("exact", inner_tol=1e-8, inner_max=200)
                res = s.solve(1e-6, 400000, seed)
                s.close()
                its.append(res["iters"])
                secs.append(res["seconds"])
            pi, pt = PAPER[(m, n)]
            print(json.dumps({"m": m, "n": n, "update": update, "iters": float(np.mean(its)),
                              "seconds": float(np.mean(secs)), "paper_iters": pi,
                              "paper_cpu_seconds": pt}), flush=True)


if __name__ == "__main__":
    main()
