"""Pins of the oracle's norm caches rho_i = ||A^(i)||^2 and gamma_j = ||A_(j)||^2
(the denominators of the row / column scores, Alg. 1 lines 5 and 10),
and of the way column_step / row_step compose them with the sampler.

What fixes them (none of these re-types the oracle's formula):
  * the paper's printed Frobenius norm of its FEM Poisson matrix
    (tab:poisson_helmholtz: ||A||_F = 1.028786e2), since
    sum_i rho_i = sum_j gamma_j = ||A||_F^2;
  * the closed form of a rank-one matrix A = u v^T: rho_i = u_i^2 ||v||^2,
    gamma_j = v_j^2 ||u||^2 (distinguishes rows from columns on non-square A);
  * sum rho = sum gamma = ||A||_F^2 from numpy's Frobenius norm (a library routine),
    which an unsquared norm fails;
  * the selection law P(j) = eps_j / sum eps at block size 1, measured
    through Oracle.column_step / Oracle.row_step on systems whose scores have a
    closed form that does NOT contain the norms: A = Q D with orthonormal Q makes
    eps^z_j = (Q^T z)_j^2 whatever the column scaling D, so a dropped, unsquared
    or swapped denominator changes the frequencies.
"""
import numpy as np
import pytest
import scipy.sparse as sp

from oracle.rgdbek import Oracle, col_sq_norms, row_sq_norms
from workloads import poisson_fem_paper

from conftest import read_golden_kv

pytestmark = pytest.mark.filterwarnings("error")


def test_norm_caches_match_the_papers_poisson_frobenius_norm():
    g = read_golden_kv("poisson_fem_625.txt")
    A = poisson_fem_paper(25)
    rho, gam = row_sq_norms(A), col_sq_norms(A)
    assert rho.shape == (625,) and gam.shape == (625,)
    # printed to 7 significant digits
    assert abs(np.sqrt(rho.sum()) - float(g["frobenius_norm"])) <= 5e-5
    assert abs(np.sqrt(gam.sum()) - float(g["frobenius_norm"])) <= 5e-5


@pytest.mark.parametrize("sparse", [False, True])
def test_rank_one_closed_form_rows_vs_columns(sparse):
    rng = np.random.default_rng(4)
    u = rng.standard_normal(7) * np.arange(1, 8)      # unequal row norms
    v = rng.standard_normal(4) * np.array([0.1, 1.0, 3.0, 10.0])   # unequal column norms
    A = np.outer(u, v)
    M = sp.csr_matrix(A) if sparse else A
    np.testing.assert_allclose(row_sq_norms(M), u ** 2 * (v @ v), rtol=1e-13)
    np.testing.assert_allclose(col_sq_norms(M), v ** 2 * (u @ u), rtol=1e-13)


@pytest.mark.parametrize("sparse", [False, True])
def test_sums_equal_frobenius_and_scale_quadratically(sparse):
    rng = np.random.default_rng(5)
    A = rng.standard_normal((30, 11)) * rng.uniform(0.1, 5.0, size=11)
    A[rng.random(A.shape) < 0.4] = 0.0
    M = sp.csr_matrix(A) if sparse else A
    f2 = np.linalg.norm(A, "fro") ** 2
    assert abs(row_sq_norms(M).sum() - f2) <= 1e-12 * f2
    assert abs(col_sq_norms(M).sum() - f2) <= 1e-12 * f2
    M3 = 3.0 * M
    np.testing.assert_allclose(row_sq_norms(M3), 9.0 * row_sq_norms(M), rtol=1e-14)
    np.testing.assert_allclose(col_sq_norms(M3), 9.0 * col_sq_norms(M), rtol=1e-14)
    # an empty row / column has norm 0 (reading R6: never selected)
    A[2, :] = 0.0
    A[:, 5] = 0.0
    M = sp.csr_matrix(A) if sparse else A
    assert row_sq_norms(M)[2] == 0.0 and col_sq_norms(M)[5] == 0.0


def _orthonormal(rows, cols, seed):
    q, _ = np.linalg.qr(np.random.default_rng(seed).standard_normal((rows, cols)))
    return q


def _frequencies(draw, n, trials):
    cnt = np.zeros(n)
    for seed in range(trials):
        sel = draw(seed)
        assert len(sel) == 1
        cnt[sel[0]] += 1
    return cnt / trials


@pytest.mark.parametrize("m", [12, 5])
def test_k1_column_step_frequency_is_normalised_score(m):
    """Alg. 1 lines 5-7 through Oracle.column_step, block size 1, on an
    m x 5 system A = Q D (orthonormal Q, very unequal column norms D; m = 5 is square,
    where row norms != column norms): with z_0 = b,
    eps_j = (A^T b)_j^2 / ||A_j||^2 = (Q^T b)_j^2, independent of D."""
    n, trials = 5, 6000
    Q = _orthonormal(m, n, 1)
    D = np.array([0.05, 1.0, 7.0, 0.3, 20.0])
    c = np.array([3.0, 2.0, 1.0, 1.0, 0.5])
    b = Q @ c + 0.4 * (np.eye(m) - Q @ Q.T) @ np.random.default_rng(2).standard_normal(m)
    A = Q * D

    def draw(seed):
        o = Oracle(A, b, eta=0.01)                       # k_c = max(1, floor(0.05 + 0.5)) = 1
        assert o.kc == 1
        kp, U, Z, W = o.column_step(seed)
        return U

    f = _frequencies(draw, n, trials)
    p = c ** 2 / np.sum(c ** 2)
    se = np.sqrt(p * (1 - p) / trials)
    assert np.all(np.abs(f - p) <= 4.5 * se + 1e-12), (f, p)


@pytest.mark.parametrize("n", [12, 5])
def test_k1_row_step_frequency_is_normalised_score(n):
    """Alg. 1 lines 10-12 through Oracle.row_step, block size 1, on a
    5 x n system A = D Q^T (orthonormal rows scaled by D; n = 5 is square) with x = 0,
    z = 0: r = b, eps_i = b_i^2 / ||A^(i)||^2 = (b_i / D_i)^2; b = D c gives eps = c^2."""
    m, trials = 5, 6000
    Q = _orthonormal(n, m, 3)
    D = np.array([0.05, 1.0, 7.0, 0.3, 20.0])
    c = np.array([0.5, 3.0, 1.0, 2.0, 1.0])
    A = D[:, None] * Q.T
    b = D * c

    def draw(seed):
        o = Oracle(A, b, eta=0.01)
        assert o.kr == 1
        o.z = np.zeros(m)                                # state after a column step that
        kpp, J, X, V = o.row_step(seed)                  # reached z = 0, with x = 0
        return J

    f = _frequencies(draw, m, trials)
    p = c ** 2 / np.sum(c ** 2)
    se = np.sqrt(p * (1 - p) / trials)
    assert np.all(np.abs(f - p) <= 4.5 * se + 1e-12), (f, p)
