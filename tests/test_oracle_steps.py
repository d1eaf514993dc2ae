"""Pins of the oracle's column step, row step and whole sweep.

Each check is fixed by the paper or by mathematics, not by re-typing the
oracle's formula:
  * eq:res_norm_evolve: ||z_{k+1} - r||^2 = ||z_k - r||^2 - ||P e_k||^2,
    which for the rank-one projector onto w = A zeta gives Z^2 / W (reading R1).
  * The z-step equals the first iterate of textbook CGLS on min ||A_U y - z_k||
    (the paper's subproblem, P:117 / Alg. 2); the x-step equals the
    first iterate of Craig's method on A^J y = r^J.
  * Block size 1 reduces to REK's column step and the Kaczmarz/REK row
    step.
  * Updates are exact projections: w^T z_{k+1} = 0, xi^T (b - z_{k+1} - A x_{k+1}) = 0.
  * Aug. with r in null(A^T): same selections and x, z shifted by r (Theorem 1's
    decomposition).
  * Limits x_k -> A^+ b, z_k -> (I - A A^+) b (Theorem 1) by SVD brute force.
"""
import numpy as np
import pytest
import scipy.sparse as sp

from oracle.rgdbek import (Oracle, STOP_REL_ERR, STOP_RSE, OUTCOME_CONVERGED,
                           OUTCOME_MAX_ITER, OUTCOME_STALLED, block_hash)
from workloads import dense_gaussian, sparse_random, popmodel

pytestmark = pytest.mark.filterwarnings("error")


def _cgls(A, rhs, iters):
    """Textbook CGLS (Hestenes-Stiefel on the normal equations), from y = 0."""
    y = np.zeros(A.shape[1])
    r = rhs.copy()
    s = A.T @ r
    p = s.copy()
    gamma = s @ s
    for _ in range(iters):
        q = A @ p
        alpha = gamma / (q @ q)
        y = y + alpha * p
        r = r - alpha * q
        s = A.T @ r
        gnew = s @ s
        p = s + (gnew / gamma) * p
        gamma = gnew
    return y


def _craig(A, rhs, iters):
    """Craig's method (CGNE: CG on A A^T u = rhs, y = A^T u), from y = 0."""
    y = np.zeros(A.shape[1])
    r = rhs.copy()
    p = A.T @ r
    rr = r @ r
    for _ in range(iters):
        alpha = rr / (p @ p)
        y = y + alpha * p
        r = r - alpha * (A @ p)
        rnew = r @ r
        p = A.T @ r + (rnew / rr) * p
        rr = rnew
    return y


def _run_column_step(o, seed):
    z_old = o.z.copy()
    kp, U, Z, W = o.column_step(seed)
    return z_old, kp, U, Z, W


@pytest.mark.parametrize("noise", [0.0, 0.1])
def test_column_step_pythagoras_and_orthogonality(noise):
    w = dense_gaussian(300, 60, seed=3, noise=noise)
    o = Oracle(w.A, w.b, 0.5)
    for k in range(8):
        z_old, kp, U, Z, W = _run_column_step(o, seed=5)
        e_old, e_new = z_old - w.rvec, o.z - w.rvec
        # eq:res_norm_evolve with the rank-one projector onto w = A zeta
        assert abs((e_old @ e_old - e_new @ e_new) - Z * Z / W) <= 1e-11 * (e_old @ e_old)
        wv = w.A[:, U] @ (w.A[:, U].T @ z_old)
        assert abs(wv @ o.z) <= 1e-12 * np.linalg.norm(wv) * np.linalg.norm(z_old)
        o.row_step(seed=5)
        o.k += 1


def test_column_step_is_first_cgls_iterate():
    w = dense_gaussian(120, 40, seed=4, noise=0.1)
    o = Oracle(w.A, w.b, 0.3)
    z_old, kp, U, Z, W = _run_column_step(o, seed=1)
    AU = w.A[:, U]
    y1 = _cgls(AU, z_old, 1)
    np.testing.assert_allclose(o.z, z_old - AU @ y1, rtol=0, atol=1e-12 * np.linalg.norm(z_old))
    # and it is NOT the exact projection of P:117 (that is the many-iteration limit)
    y_exact = np.linalg.lstsq(AU, z_old, rcond=None)[0]
    assert np.linalg.norm(o.z - (z_old - AU @ y_exact)) > 1e-6 * np.linalg.norm(z_old)
    y_many = _cgls(AU, z_old, 60)
    np.testing.assert_allclose(AU @ y_many, AU @ y_exact, atol=1e-8 * np.linalg.norm(z_old))


def test_row_step_is_first_craig_iterate_and_projection():
    w = dense_gaussian(150, 50, seed=6, noise=0.1)
    o = Oracle(w.A, w.b, 0.2)
    o.column_step(seed=2)
    x_old = o.x.copy()
    r = w.b - o.z - w.A @ x_old
    kpp, J, X, V = o.row_step(seed=2)
    AJ = w.A[J, :]
    y1 = _craig(AJ, r[J], 1)
    np.testing.assert_allclose(o.x, x_old + y1, rtol=0, atol=1e-13 * max(1.0, np.linalg.norm(y1)))
    # projection: xi^T (b - z_{k+1} - A x_{k+1}) = 0 for xi = r on J
    xi = np.zeros(len(r)); xi[J] = r[J]
    res_new = w.b - o.z - w.A @ o.x
    assert abs(xi @ res_new) <= 1e-12 * np.linalg.norm(xi) * np.linalg.norm(r)


def test_block_size_one_reduces_to_rek_and_kaczmarz():
    # eta small enough that k_c = k_r = 1: REK column step and the
    # Kaczmarz row step with the z correction (P:47 when z = 0)
    w = dense_gaussian(40, 10, seed=8, noise=0.1)
    o = Oracle(w.A, w.b, 0.01)
    assert o.kc == 1 and o.kr == 1
    for k in range(5):
        z_old, x_old = o.z.copy(), o.x.copy()
        kp, U, Z, W = o.column_step(seed=9)
        j = U[0]
        a_j = w.A[:, j]
        z_rek = z_old - (a_j @ z_old) / (a_j @ a_j) * a_j
        np.testing.assert_allclose(o.z, z_rek, rtol=0, atol=1e-13 * np.linalg.norm(z_old))
        kpp, J, X, V = o.row_step(seed=9)
        i = J[0]
        a_i = w.A[i, :]
        x_k = x_old + (w.b[i] - o.z[i] - a_i @ x_old) / (a_i @ a_i) * a_i
        np.testing.assert_allclose(o.x, x_k, rtol=0, atol=1e-13 * max(1, np.linalg.norm(x_k)))
        o.k += 1


def test_inconsistent_shift_invariance_and_monotone_z_error():
    # b and b + r (A^T r = 0) give the same s, w, r-vector, hence identical
    # blocks and x, with z shifted by r exactly
    w = dense_gaussian(400, 100, seed=0, noise=0.1)
    b_cons = w.b - w.rvec
    oi, oc = Oracle(w.A, w.b, 0.5), Oracle(w.A, b_cons, 0.5)
    prev = np.inf
    for k in range(50):
        ri, rc = oi.iterate(31), oc.iterate(31)
        assert (ri.kp, ri.hash_u, ri.kpp, ri.hash_j) == (rc.kp, rc.hash_u, rc.kpp, rc.hash_j)
        assert np.linalg.norm(oi.x - oc.x) <= 1e-12 * np.linalg.norm(oc.x)
        assert np.linalg.norm((oi.z - w.rvec) - oc.z) <= 1e-12 * np.linalg.norm(w.b)
        e = np.linalg.norm(oi.z - w.rvec)
        assert e <= prev * (1 + 1e-14)
        prev = e


def test_range_invariant_for_fat_system():
    # x_0 = 0 and every update is a multiple of A^T xi, so x_k in range(A^T) (reading R24)
    w = sparse_random(30, 80, density=0.3, seed=2)
    o = Oracle(w.A, w.b, 0.5)
    for _ in range(20):
        o.iterate(4)
    Ad = w.A.toarray()
    _, s, Vt = np.linalg.svd(Ad)
    rank = int(np.sum(s > 1e-10 * s[0]))
    null_part = Vt[rank:] @ o.x
    assert np.linalg.norm(null_part) <= 1e-12 * np.linalg.norm(o.x)


@pytest.mark.parametrize("case", ["tall_consistent", "tall_inconsistent", "fat", "sparse_tall"])
def test_limits_against_svd_brute_force(case):
    if case == "tall_consistent":
        w = dense_gaussian(60, 20, seed=1)
    elif case == "tall_inconsistent":
        w = dense_gaussian(60, 20, seed=1, noise=0.3)
    elif case == "fat":
        w = sparse_random(20, 45, density=0.4, seed=3)
    else:
        w = sparse_random(80, 25, density=0.3, seed=5, consistent=False)
    Ad = w.A if w.dense else w.A.toarray()
    U, s, Vt = np.linalg.svd(Ad, full_matrices=False)
    keep = s > 1e-12 * s[0]
    xstar = Vt[keep].T @ ((U[:, keep].T @ w.b) / s[keep])      # A^+ b
    rstar = w.b - Ad @ xstar                                    # (I - A A^+) b
    o = Oracle(w.A, w.b, 0.5)
    out, iters, rse, rel = o.solve(1e-10, 20000, 7, stop=STOP_REL_ERR, xstar=xstar)
    assert out == OUTCOME_CONVERGED
    assert np.linalg.norm(o.x - xstar) <= 1e-10 * np.linalg.norm(xstar)
    assert np.linalg.norm(o.z - rstar) <= 1e-6 * np.linalg.norm(w.b)


def test_normal_equations_on_consistent_full_rank():
    w = dense_gaussian(200, 50, seed=0)
    xs = np.linalg.solve(w.A.T @ w.A, w.A.T @ w.b)
    o = Oracle(w.A, w.b, 0.5)
    out, iters, rse, rel = o.solve(1e-6, 10000, 0, stop=STOP_REL_ERR, xstar=xs)
    assert out == OUTCOME_CONVERGED
    assert 40 <= iters <= 90          # SURVEY V7 range 56-61 over seeds; sanity band
    assert rse < 1e-10


def test_rse_stop_and_spec_identity_example():
    # A = 10x10 identity, b = ones -> x = ones, converged
    A = np.eye(10)
    o = Oracle(A, np.ones(10), 0.5)
    out, iters, rse, rel = o.solve(1e-12, 1000, 0, stop=STOP_RSE)
    assert out == OUTCOME_CONVERGED and rse <= 1e-12
    np.testing.assert_allclose(o.x, np.ones(10), atol=1e-6)
    # RSE scale invariance (A, b) -> (cA, cb)
    o2 = Oracle(3.0 * A, 3.0 * np.ones(10), 0.5)
    o2.x = o.x.copy()
    assert abs(o2.rse() - o.rse()) <= 1e-15


def test_max_iter_and_stall():
    w = dense_gaussian(60, 20, seed=1)
    o = Oracle(w.A, w.b, 0.5)
    out, iters, _, _ = o.solve(1e-300, 7, 0, stop=STOP_RSE)
    assert out == OUTCOME_MAX_ITER and iters == 7
    # b = 0 is rejected by the ABI; a zero-score start (b in null(A^T) AND b with
    # A x = b unreachable) stalls: A = [[1,0],[0,0]], b = (0, 1): z_0 = b gives s = 0
    # (no column mass) and r = b - z_1 - A x = 0 (no row mass).
    o = Oracle(np.array([[1.0, 0.0], [0.0, 0.0]]), np.array([0.0, 1.0]), 0.5)
    out, iters, rse, _ = o.solve(1e-12, 100, 0, stop=STOP_RSE)
    assert out == OUTCOME_STALLED and iters == 1 and rse == 1.0


def test_empty_rows_and_columns_never_selected():
    A = sp.csr_matrix(np.array([[1.0, 0, 2, 0], [0, 0, 0, 0], [3.0, 0, 0, 1], [0, 0, 1, 1]]))
    o = Oracle(A, np.array([1.0, 2.0, 3.0, 4.0]), 0.9)
    for _ in range(10):
        rec = o.iterate(3, keep_blocks=True)
        assert 1 not in rec.U.tolist()        # zero column (gamma = 0)
        assert 1 not in rec.J.tolist()        # zero row (rho = 0)
        assert rec.hash_u == block_hash(rec.U)


def test_popmodel_twin_converges_in_band():
    # C5s-shaped systems converge in ~thousands of iterations; here a
    # smaller twin (5000x500) must reach 1e-6 and x -> x* with z -> r
    w = popmodel(5000, 500, seed=0)      # kappa ~ 29.7, like C5s (29.5)
    o = Oracle(w.A, w.b, 0.5)
    out, iters, rse, rel = o.solve(1e-6, 20000, 0, stop=STOP_REL_ERR, xstar=w.xstar)
    assert out == OUTCOME_CONVERGED
    assert np.linalg.norm(o.z - w.rvec) <= 1e-4 * np.linalg.norm(w.b)
