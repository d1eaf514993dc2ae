"""Pins of the Algorithm 2 oracle (oracle/lazy.py, reading R28):
special cases that reduce to something fixed independently of its code."""
import numpy as np
import pytest
import scipy.sparse as sp

from oracle import Oracle, STOP_REL_ERR, OUTCOME_CONVERGED
from oracle.lazy import LazyOracle, partition_bounds


def _dense(seed, m, n, noise=0.0):
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((m, n))
    xs = rng.standard_normal(n)
    b = A @ xs + noise * rng.standard_normal(m)
    return A, b, xs


def test_partition_bounds_cover_rows_in_order():
    for m, P in [(10, 3), (200, 7), (5, 5)]:
        bd = partition_bounds(m, P)
        assert bd[0][0] == 0 and bd[-1][1] == m
        assert all(bd[i][1] == bd[i + 1][0] for i in range(P - 1))
        assert all(r1 - r0 in (m // P, m // P + 1) for r0, r1 in bd)


@pytest.mark.parametrize("sparse", [False, True])
def test_one_process_is_algorithm_1(sparse):
    """P = 1: Algorithm 2 is Algorithm 1 (one process holds every row)."""
    A, b, _ = _dense(3, 60, 25, noise=0.2)
    if sparse:
        A[np.abs(A) < 0.8] = 0.0
        A = sp.csr_matrix(A)
    o1, o2 = Oracle(A, b, 0.5), LazyOracle(A, b, 0.5, parts=1)
    for _ in range(20):
        r1, r2 = o1.iterate(7), o2.iterate(7)
        assert (r1.kp, r1.hash_u, r1.kpp, r1.hash_j) == (r2.kp, r2.hash_u, r2.kpp, r2.hash_j)
        assert (r1.Z, r1.W, r1.X, r1.V) == (r2.Z, r2.W, r2.X, r2.V)
        assert np.array_equal(o1.x, o2.x) and np.array_equal(o1.z, o2.z)


def test_one_row_per_process_is_cimmino():
    """P = m: every local z-problem min ||a_i,U y - z_i|| is solved exactly by its
    first iterate, so z_1 = 0; every process selects its own row, and the lazy
    average of the row projections is one Cimmino step with weights 1/m."""
    A, b, _ = _dense(5, 40, 12)
    m = A.shape[0]
    o = LazyOracle(A, b, 0.5, parts=m)
    o.iterate(1)
    assert np.linalg.norm(o.z) <= 1e-12 * np.linalg.norm(b)
    r = b                                          # r = b - z_1 - A x_0 with z_1 ~ 0, x_0 = 0
    cimmino = (A.T @ (r / np.sum(A * A, axis=1))) / m
    assert np.linalg.norm(o.x - cimmino) <= 1e-10 * np.linalg.norm(cimmino)


def test_block_sizes_per_process():
    """Each process samples round(eta * d_p) of its own rows (reading R2 per process)."""
    A, b, _ = _dense(2, 103, 20, noise=0.1)
    o = LazyOracle(A, b, 0.3, parts=4)
    rec = o.iterate(0, keep_blocks=True)
    want = sum(max(1, int(np.floor(0.3 * (r1 - r0) + 0.5))) for r0, r1 in o.bounds)
    assert rec.kpp == want == len(rec.J)
    for r0, r1 in o.bounds:                        # every process picks only its own rows
        inside = (rec.J >= r0) & (rec.J < r1)
        assert inside.sum() == max(1, int(np.floor(0.3 * (r1 - r0) + 0.5)))


@pytest.mark.parametrize("P", [2, 4, 7])
def test_local_z_steps_never_increase_the_local_residual(P):
    """Each process's z-step is the first CGLS iterate of its own problem, so
    ||z^(p)_{k+1}||^2 = ||z^(p)_k||^2 - Z_p^2 / W_p <= ||z^(p)_k||^2 (the per-process
    form of eq:res_norm_evolve).  (Convergence of Algorithm 2 itself is
    not a pin: with a global U and local residuals it can stall — P = 4 on this
    system stops near rel. error 1e-4.)"""
    A, b, _ = _dense(11, 120, 30, noise=0.3)
    o = LazyOracle(A, b, 0.5, parts=P)
    for _ in range(30):
        before = [float(np.linalg.norm(o.z[r0:r1])) for r0, r1 in o.bounds]
        o.iterate(0)
        after = [float(np.linalg.norm(o.z[r0:r1])) for r0, r1 in o.bounds]
        assert all(a2 <= a1 * (1 + 1e-13) + 1e-300 for a1, a2 in zip(before, after))


def test_two_processes_converge_on_this_consistent_system():
    """A smoke check of the trajectory (not a mathematical pin): P = 2 reaches
    rel. error 1e-8 on the 120 x 30 Gaussian system used above."""
    A, b, xs = _dense(11, 120, 30)
    o = LazyOracle(A, b, 0.5, parts=2)
    out, iters, rse, rel = o.solve(1e-8, 20000, 0, stop=STOP_REL_ERR, xstar=xs)
    assert out == OUTCOME_CONVERGED and rel <= 1e-8


def test_explicit_bounds_equal_the_default_partition():
    from workloads import dense_gaussian
    w = dense_gaussian(90, 20, seed=4)
    a = LazyOracle(w.A, w.b, 0.5, parts=3)
    b = LazyOracle(w.A, w.b, 0.5, bounds=[(0, 30), (30, 60), (60, 90)])
    for _ in range(5):
        ra, rb = a.iterate(2), b.iterate(2)
        assert (ra.hash_u, ra.hash_j) == (rb.hash_u, rb.hash_j)
    assert np.array_equal(a.x, b.x) and np.array_equal(a.z, b.z)
    with pytest.raises(ValueError):
        LazyOracle(w.A, w.b, 0.5, bounds=[(0, 30), (31, 90)])
