"""Small runs of every kernel family for compute-sanitizer (one tool per gpurun call).

usage: python tools/sanitize_cases.py [grid]
Runs a few iterations of the persistent kernel (Alg. 1, sparse and dense), the
exact-projection kernel, the Algorithm 2 kernel and the graph engine on the C1,
C2s, C3s and C5t twins, each checked against nothing (the sanitizer is the check).
grid = CTAs of the persistent kernels (1 makes the grid barrier a no-op, which the
serialising race / sync checkers need).
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
grid = sys.argv[1] if len(sys.argv) > 1 else "2"
os.environ["RGDBEK_GRID"] = grid

from workloads import by_name
from paper_2509_19267_b200 import Solver


def mk(w):
    if w.dense:
        return Solver(w.A, w.b, eta=w.eta)
    return Solver.from_scipy(w.A, w.b, eta=w.eta, symmetric=w.symmetric)


for name in ("C1", "C2s", "C3s", "C5t"):
    w = by_name(name)
    s = mk(w)
    s.reset(0); r = s.step(3); print(name, "persistent", r["iters"], flush=True)
    s.set_mode("exact", inner_tol=1e-10, inner_max=4)
    s.reset(0); r = s.step(2); print(name, "exact", r["iters"], flush=True)
    s.set_mode("pinv_free")
    s.set_selection("greedy")
    s.reset(0); r = s.step(2); print(name, "greedy", r["iters"], flush=True)
    s.set_selection("random")
    if w.dense and int(grid) >= 2:
        s.set_lazy(2)
        s.reset(0); r = s.step(2); print(name, "lazy2", r["iters"], flush=True)
        s.set_lazy(0)
    s.close()
os.environ["RGDBEK_ENGINE"] = "graph"
for name in ("C1", "C3s"):
    w = by_name(name)
    s = mk(w)
    s.reset(0); r = s.step(2); print(name, "graph", r["iters"], flush=True)
    s.close()
print("sanitize cases done")
