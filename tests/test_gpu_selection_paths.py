"""The exact selection's rarely-taken paths, forced (p_sel_slow, the local
smem-overflow fallback, the grid-wide dense selection and the graph engine's
k_select_slow were never executed by a test).

* A test-only build of the same sources (paper_2509_19267_b200/_build.py VARIANTS
  "selstress": LOCAL_SEL_MAX 64, LCAND_CAP 4, CAND_CAP 0, FINAL_CAP 0) runs the
  oracle parity protocol with FULL index lists; rgdbek_selection_stats proves the
  overflow and slow paths ran.
* The production build on a dense system with m > 32768 rows (grid-wide row selection
  of the dense persistent kernel).
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _variant_run(engine, names):
    from paper_2509_19267_b200 import _build
    lib = _build.build_variant("selstress")
    env = dict(os.environ, RGDBEK_LIB=lib, RGDBEK_ENGINE=engine)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "_selstress_driver.py"), *names],
                       env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_persistent_overflow_and_slow_paths():
    out = _variant_run("persistent", ["C1", "C2s", "C3s", "C5t"])
    assert out["build_info"]["local_sel_max"] == 64 and out["build_info"]["final_cap"] == 0
    tot = np.sum([v for v in out["runs"].values()], axis=0)
    assert tot[0] > 0, out        # local selections fell back after a smem-list overflow
    assert tot[1] > 0, out        # the exact slow path resolved selections


def test_sharded_distributed_slow_path():
    """The peer-sharded engine's distributed slow path (x_sel_slow: one radix level per
    global exchange over every rank's keys) under the stress build, R = 2 and 4, dense and
    sparse: full lists, x and z vs the oracle; the counter proves it ran."""
    out = _variant_run("persistent", ["sharded:C5t:2", "sharded:C2s:4", "sharded:C3s:2"])
    tot = np.sum([v for v in out["runs"].values()], axis=0)
    assert tot[1] > 0, out


def test_graph_engine_slow_path():
    out = _variant_run("graph", ["C1", "C3s"])
    tot = np.sum([v for v in out["runs"].values()], axis=0)
    assert tot[2] > 0, out        # k_select_slow resolved selections


def test_dense_tall_grid_wide_selection():
    """m = 40000 > LOCAL_SEL_MAX rows: the dense kernel's grid-wide row selection
    (levels 2 and 3 over all CTAs), full U / J lists vs the oracle."""
    from oracle import Oracle
    from paper_2509_19267_b200 import Solver, _native
    from workloads import dense_gaussian
    assert 40000 > _native.rgdbek_build_info()["local_sel_max"]
    w = dense_gaussian(40000, 120, seed=7, noise=0.05)
    s = Solver(w.A, w.b, eta=0.5)
    s.set_capture(True)
    o = Oracle(w.A, w.b, 0.5)
    s.reset(2)
    bn = np.linalg.norm(w.b)
    for k in range(15):
        rec = o.iterate(2, keep_blocks=True)
        s.step(1)
        U, J = s.block_lists()
        assert np.array_equal(U, rec.U) and np.array_equal(J, rec.J), k
        assert np.linalg.norm(s.x() - o.x) <= 1e-10 * np.linalg.norm(o.x), k
        assert np.linalg.norm(s.z() - o.z) <= 1e-10 * bn, k
    s.close()
