"""Pins of the oracle's GDBEK greedy selection."""
import numpy as np
import pytest

from oracle import Oracle, STOP_REL_ERR, STOP_RSE, OUTCOME_CONVERGED
from oracle.rgdbek import greedy_block
from workloads import dense_gaussian, sparse_random

pytestmark = pytest.mark.filterwarnings("error")


def test_greedy_block_examples():
    # threshold eta * max with a closed comparison: the argmax is always in
    assert greedy_block(np.array([3.0, 1.0, 0.5, 0.0]), 0.5).tolist() == [0]
    assert greedy_block(np.array([3.0, 1.0, 0.5, 0.0]), 0.3).tolist() == [0, 1]
    assert greedy_block(np.array([2.0, 1.0]), 0.5).tolist() == [0, 1]      # 1 >= 0.5 * 2
    assert greedy_block(np.zeros(4), 0.5).tolist() == []
    eps = np.random.default_rng(0).random(1000)
    blk = greedy_block(eps, 0.9)
    assert int(np.argmax(eps)) in blk.tolist()
    assert len(blk) == int(np.count_nonzero(eps >= 0.9 * eps.max()))


@pytest.mark.parametrize("update", ["pinv_free", "exact_lstsq"])
def test_gdbek_converges(update):
    w = dense_gaussian(200, 50, seed=4, noise=0.1)
    o = Oracle(w.A, w.b, 0.5, update=update, select="greedy")
    out, it, rse, rel = o.solve(1e-8, 20000, 0, stop=STOP_REL_ERR, xstar=w.xstar)
    assert out == OUTCOME_CONVERGED
    np.testing.assert_allclose(o.z, w.rvec, atol=1e-5 * np.linalg.norm(w.b))


def test_greedy_is_seed_free():
    w = dense_gaussian(120, 40, seed=2)
    a = Oracle(w.A, w.b, 0.5, select="greedy")
    b = Oracle(w.A, w.b, 0.5, select="greedy")
    for _ in range(10):
        ra, rb = a.iterate(1), b.iterate(999)
        assert (ra.hash_u, ra.hash_j) == (rb.hash_u, rb.hash_j)
    np.testing.assert_array_equal(a.x, b.x)


def test_rgdbek_needs_fewer_iterations_than_gdbek():
    # tab:fatmatrices: RGDBEK 12.0 vs GDBEK 34.3 iterations at 500 x 8000,
    # 99 % sparse, eta = 0.5, RSE <= 1e-6 (exact-projection updates)
    w = sparse_random(500, 8000, density=0.01, seed=0)
    r = Oracle(w.A, w.b, 0.5, update="exact_lstsq", select="random")
    g = Oracle(w.A, w.b, 0.5, update="exact_lstsq", select="greedy")
    out_r, it_r, _, _ = r.solve(1e-6, 500, 1, stop=STOP_RSE)
    out_g, it_g, _, _ = g.solve(1e-6, 500, 1, stop=STOP_RSE)
    assert out_r == OUTCOME_CONVERGED
    assert it_r < it_g
