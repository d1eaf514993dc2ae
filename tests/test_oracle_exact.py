"""Pins of the oracle's exact-projection mode (Alg. 1's pseudoinverse updates,
P:117 and P:122), against what the mathematics fixes:
  * the z-step is the orthogonal projection onto range(A_U)^perp: A_U^T z_{k+1} = 0,
    idempotent, and Pythagoras (eq:res_norm_evolve) with P_U = A_U A_U^+;
  * the x-step is the minimum-norm least-squares correction: (A^J)^T residual = 0 on J,
    the correction lies in range(A^J^T), and for |J| <= n with full row rank
    the selected equations hold exactly;
  * the limit of many CGLS iterations (a textbook implementation) equals the step;
  * the paper's claim that exact projections need fewer outer iterations
    (6 vs 15 on a sprandn-like 500 x 8000).
"""
import numpy as np
import pytest

from oracle import Oracle, STOP_REL_ERR, STOP_RSE, OUTCOME_CONVERGED
from workloads import dense_gaussian, sparse_random

pytestmark = pytest.mark.filterwarnings("error")


def _cgls(A, rhs, iters):
    y = np.zeros(A.shape[1]); r = rhs.copy(); s = A.T @ r; p = s.copy(); g = s @ s
    for _ in range(iters):
        q = A @ p; al = g / (q @ q); y += al * p; r -= al * q; s = A.T @ r
        gn = s @ s
        if gn < 1e-30 * (rhs @ rhs):
            break
        p = s + (gn / g) * p; g = gn
    return y


@pytest.mark.parametrize("noise", [0.0, 0.2])
def test_exact_z_step_is_orthogonal_projection(noise):
    w = dense_gaussian(120, 30, seed=3, noise=noise)
    o = Oracle(w.A, w.b, 0.4, update="exact_lstsq")
    for _ in range(4):
        z_old = o.z.copy()
        kp, U, Z, W = o.column_step(seed=2)
        AU = w.A[:, U]
        assert np.linalg.norm(AU.T @ o.z) <= 1e-10 * np.linalg.norm(AU) * np.linalg.norm(z_old)
        P = AU @ np.linalg.pinv(AU)
        np.testing.assert_allclose(o.z, z_old - P @ z_old, atol=1e-10 * np.linalg.norm(z_old))
        e0, e1 = z_old - w.rvec, o.z - w.rvec
        assert abs((e0 @ e0 - e1 @ e1) - (P @ e0) @ (P @ e0)) <= 1e-9 * (e0 @ e0)
        y = _cgls(AU, z_old, 200)
        np.testing.assert_allclose(z_old - AU @ y, o.z, atol=1e-8 * np.linalg.norm(z_old))
        o.row_step(seed=2)
        o.k += 1


def test_exact_x_step_min_norm_fat_block():
    # |J| < n: A^J has full row rank, the selected equations are solved exactly
    w = dense_gaussian(60, 40, seed=5)
    o = Oracle(w.A, w.b, 0.3, update="exact_lstsq")
    o.column_step(seed=1)
    x0 = o.x.copy()
    r = w.b - o.z - w.A @ x0
    kpp, J, X, V = o.row_step(seed=1)
    assert kpp < w.A.shape[1]
    AJ = w.A[J]
    dx = o.x - x0
    np.testing.assert_allclose(AJ @ o.x, (w.b - o.z)[J], atol=1e-10 * np.linalg.norm(w.b))
    # minimum norm: dx in range(A^J^T)
    Q, _ = np.linalg.qr(AJ.T)
    assert np.linalg.norm(dx - Q @ (Q.T @ dx)) <= 1e-10 * np.linalg.norm(dx)
    np.testing.assert_allclose(dx, _cgls(AJ, r[J], 500), atol=1e-8 * np.linalg.norm(dx))


def test_exact_x_step_least_squares_tall_block():
    # |J| > n: the correction is the least-squares solution, normal equations hold on J
    w = dense_gaussian(200, 20, seed=6, noise=0.3)
    o = Oracle(w.A, w.b, 0.5, update="exact_lstsq")
    o.column_step(seed=4)
    x0 = o.x.copy()
    kpp, J, X, V = o.row_step(seed=4)
    assert kpp > w.A.shape[1]
    AJ = w.A[J]
    res = (w.b - o.z)[J] - AJ @ o.x
    assert np.linalg.norm(AJ.T @ res) <= 1e-10 * np.linalg.norm(AJ) ** 2 * np.linalg.norm(o.x - x0)


def test_exact_mode_limits_and_fewer_iterations():
    w = dense_gaussian(300, 60, seed=1, noise=0.1)
    oe = Oracle(w.A, w.b, 0.5, update="exact_lstsq")
    out, it_e, _, _ = oe.solve(1e-10, 2000, 3, stop=STOP_REL_ERR, xstar=w.xstar)
    assert out == OUTCOME_CONVERGED
    np.testing.assert_allclose(oe.z, w.rvec, atol=1e-8 * np.linalg.norm(w.b))
    op = Oracle(w.A, w.b, 0.5)
    out, it_p, _, _ = op.solve(1e-10, 20000, 3, stop=STOP_REL_ERR, xstar=w.xstar)
    assert out == OUTCOME_CONVERGED
    assert it_e < it_p


@pytest.mark.parametrize("noise", [0.0, 0.2])
def test_inner_cgls_mode_converges_to_the_projection(noise):
    # the paper's route (inner LSQR-equivalent CGLS, update="exact") reaches the
    # pseudoinverse updates (update="exact_lstsq") on well-conditioned blocks
    w = dense_gaussian(150, 40, seed=9, noise=noise)
    oc = Oracle(w.A, w.b, 0.5, update="exact", inner_tol=1e-14, inner_max=300)
    ol = Oracle(w.A, w.b, 0.5, update="exact_lstsq")
    for _ in range(6):
        rc, rl = oc.iterate(8), ol.iterate(8)
        assert (rc.hash_u, rc.hash_j) == (rl.hash_u, rl.hash_j)
        assert np.linalg.norm(oc.x - ol.x) <= 1e-10 * np.linalg.norm(ol.x)
        assert np.linalg.norm(oc.z - ol.z) <= 1e-10 * np.linalg.norm(w.b)
    # one inner iteration of the z-solve is exactly the pseudoinverse-free z-step
    o1 = Oracle(w.A, w.b, 0.5, update="exact", inner_max=1)
    op = Oracle(w.A, w.b, 0.5)
    o1.column_step(2)
    op.column_step(2)
    np.testing.assert_array_equal(o1.z, op.z)


def test_exact_mode_sprandn_fat_iteration_count():
    # on a 1 %-dense 500 x 8000 sprandn-like system at eta = 0.5, RSE <= 1e-6,
    # exact projections took 6 iterations against 15 for the pinv-free sweep (paper: 12.0)
    w = sparse_random(500, 8000, density=0.01, seed=0)
    oe = Oracle(w.A, w.b, 0.5, update="exact_lstsq")
    out, it_e, rse, _ = oe.solve(1e-6, 200, 1, stop=STOP_RSE)
    op = Oracle(w.A, w.b, 0.5)
    out2, it_p, rse2, _ = op.solve(1e-6, 500, 1, stop=STOP_RSE)
    assert out == out2 == OUTCOME_CONVERGED
    assert it_e < it_p
    assert 3 <= it_e <= 12 and 8 <= it_p <= 30
