"""Pins of the synthetic workload generators against the paper's printed values."""
import numpy as np
import pytest
import scipy.sparse as sp

from conftest import read_golden_kv
from workloads import (dense_gaussian, poisson2d, poisson_fem_paper, popmodel,
                       toeplitz_blur)
from workloads.gen import pps_trajectory


def test_poisson_fem_matches_paper_table():
    # tab:poisson_helmholtz: sparsity 99.32 %, kappa 2.327776e2, ||A||_F 1.028786e2
    g = read_golden_kv("poisson_fem_625.txt")
    A = poisson_fem_paper(25)
    N = int(g["nodes"])
    assert A.shape == (N, N)
    assert round(100 * (1 - A.nnz / N ** 2), 2) == float(g["sparsity_percent"])
    assert abs(np.sqrt((A.data ** 2).sum()) - float(g["frobenius_norm"])) < 5e-5
    assert abs(np.linalg.cond(A.toarray()) - float(g["condition_number"])) < 5e-4
    # 2 * 24 * 24 = 1152 P1 triangles on the structured 25x25 grid
    assert 2 * (25 - 1) ** 2 == int(g["elements"])


def test_c3_stencil_is_the_papers_interior_block():
    A = poisson_fem_paper(25).toarray()
    interior = [i * 25 + j for i in range(1, 24) for j in range(1, 24)]
    B = poisson2d(23).A.toarray()
    np.testing.assert_array_equal(A[np.ix_(interior, interior)], B)
    w = poisson2d(23)
    assert w.symmetric and (abs(w.A - w.A.T)).nnz == 0
    np.testing.assert_allclose(w.A @ w.xstar, w.b)


def test_c3_full_size_counts():
    # 2000^2 interior grid -> 4,000,000 unknowns, 19,992,000 nnz
    N = 2000
    assert 5 * N * N - 4 * N == 19_992_000


def test_toeplitz_psf_values():
    g = read_golden_kv("toeplitz_psf.txt")
    w = toeplitz_blur(40 * 40)
    A = w.A
    assert abs(A[500, 500] - float(g["diagonal"])) < 1e-18
    assert A[500].nnz == int(g["nnz_per_interior_row"])
    assert (abs(A - A.T)).nnz == 0
    s = float(g["sigma"])
    assert abs(A[500, 507] - np.exp(-49 / (2 * s * s)) / (s * np.sqrt(2 * np.pi))) < 1e-18
    assert A[500, 521] == 0.0
    assert w.b.shape == (1600,) and np.all(np.isfinite(w.b))


def test_pps_trajectory_positive():
    # eq:predpreyscav with tab:param and x0,y0,z0 = 4,3,2 keeps populations positive
    traj = pps_trajectory()
    assert traj.shape == (2001, 3)
    assert np.all(traj > 0)


def test_popmodel_structure_and_null_residual():
    w = popmodel(5000, 500, seed=0)
    A = w.A
    assert A.shape == (5000, 500) and A.nnz == 5000 * 20
    assert np.all(np.diff(A.indptr) == 20)
    Ad = A.toarray()
    cols = [np.flatnonzero(Ad[i]) for i in (0, 2500, 4999)]
    for c in cols:
        assert np.array_equal(c, np.arange(c[0], c[0] + 20))
    assert cols[2][-1] == 499
    # r in null(A^T) (P:185 r = (I - A A^+) b): A^T r = 0 to rounding
    assert np.linalg.norm(A.T @ w.rvec) <= 1e-14 * np.linalg.norm(Ad, 2) * np.linalg.norm(w.rvec)
    np.testing.assert_allclose(np.linalg.norm(w.rvec), 0.1 * np.linalg.norm(A @ w.xstar), rtol=1e-12)


def test_dense_inconsistent_residual_orthogonal():
    w = dense_gaussian(500, 100, seed=2, noise=0.1)
    assert np.linalg.norm(w.A.T @ w.rvec) <= 1e-12 * np.linalg.norm(w.A) * np.linalg.norm(w.rvec)
    np.testing.assert_allclose(w.b - w.rvec, w.A @ w.xstar, rtol=1e-12, atol=1e-12)


def test_generators_are_seeded():
    a, b = dense_gaussian(50, 10, seed=4), dense_gaussian(50, 10, seed=4)
    assert np.array_equal(a.A, b.A) and np.array_equal(a.b, b.b)
    p, q = popmodel(3000, 300, seed=1), popmodel(3000, 300, seed=1)
    assert (p.A != q.A).nnz == 0 and np.array_equal(p.b, q.b)
