"""Subprocess driver of tests/test_gpu_selection_paths.py (run with RGDBEK_LIB pointing at
the selection-stress build): trajectory parity vs the oracle while every overflow and
slow path of the exact selection runs.  Prints one JSON line."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np

from oracle import Oracle
from paper_2509_19267_b200 import Solver, _native
from workloads import by_name


def solver(w):
    if w.dense:
        return Solver(w.A, w.b, eta=w.eta)
    return Solver.from_scipy(w.A, w.b, eta=w.eta, symmetric=w.symmetric)


def run(name, iters, seed):
    w = by_name(name)
    s = solver(w)
    s.set_capture(True)
    o = Oracle(w.A, w.b, w.eta)
    s.reset(seed)
    bn = np.linalg.norm(w.b)
    for k in range(iters):
        rec = o.iterate(seed, keep_blocks=True)
        s.step(1)
        U, J = s.block_lists()
        assert np.array_equal(U, rec.U) and np.array_equal(J, rec.J), (name, k)
        assert np.linalg.norm(s.x() - o.x) <= 1e-10 * max(np.linalg.norm(o.x), 1e-300), (name, k)
        assert np.linalg.norm(s.z() - o.z) <= 1e-10 * bn, (name, k)
    st = s.selection_stats()
    s.close()
    return st


info = _native.rgdbek_build_info()
out = {"lib": os.environ.get("RGDBEK_LIB"), "build_info": info, "runs": {}}
engine = os.environ.get("RGDBEK_ENGINE", "persistent")
for name in sys.argv[1:]:
    out["runs"][f"{name}/{engine}"] = run(name, 12, seed=5)
print(json.dumps(out))
