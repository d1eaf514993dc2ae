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


def run_sharded(name, R, iters, seed):
    """The peer-sharded engine (R emulated ranks) under the stress build: the distributed
    slow path (x_sel_slow) resolves every selection; full lists vs the oracle."""
    from paper_2509_19267_b200 import ShardGroup
    from paper_2509_19267_b200.dist import partition_rows, shard_csr
    w = by_name(name)
    m, n = w.shape
    parts = partition_rows(m if w.dense else w.A.indptr, R)
    ss = []
    for (r0, r1) in parts:
        if w.dense:
            x = Solver(w.A[r0:r1], w.b[r0:r1], eta=w.eta, m=m, row_range=(r0, r1))
        else:
            rp, ci, val = shard_csr(*w.csr_arrays(), r0, r1)
            x = Solver.from_csr(m, n, rp, ci, val, w.b[r0:r1], eta=w.eta, row_range=(r0, r1))
        x.set_capture(True)
        ss.append(x)
    g = ShardGroup(ss)
    o = Oracle(w.A, w.b, w.eta)
    g.reset(seed)
    bn = np.linalg.norm(w.b)
    for k in range(iters):
        rec = o.iterate(seed, keep_blocks=True)
        g.step(1)
        U = np.sort(np.concatenate([x.block_lists()[0] for x in ss]))
        J = np.sort(np.concatenate([x.block_lists()[1] for x in ss]))
        assert np.array_equal(U, rec.U) and np.array_equal(J, rec.J), (name, R, k)
        assert np.linalg.norm(ss[0].x() - o.x) <= 1e-10 * max(np.linalg.norm(o.x), 1e-300), (name, R, k)
        z = np.concatenate([x.z() for x in ss])
        assert np.linalg.norm(z - o.z) <= 1e-10 * bn, (name, R, k)
    st = ss[0].selection_stats()
    g.close()
    for x in ss:
        x.close()
    return st


info = _native.rgdbek_build_info()
out = {"lib": os.environ.get("RGDBEK_LIB"), "build_info": info, "runs": {}}
engine = os.environ.get("RGDBEK_ENGINE", "persistent")
for name in sys.argv[1:]:
    if name.startswith("sharded:"):
        _, wl, R = name.split(":")
        out["runs"][name] = run_sharded(wl, int(R), 8, seed=5)
    else:
        out["runs"][f"{name}/{engine}"] = run(name, 12, seed=5)
print(json.dumps(out))
