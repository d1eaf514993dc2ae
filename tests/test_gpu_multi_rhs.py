"""Several right-hand sides sharing A (multi.cuh; the paper's 3-channel
deblurring solves A x_i = b_i with one blur operator; reading R29).

Bar: right-hand side q of one multi-RHS solve follows the single-RHS oracle of
(A, b_q) with seed + q exactly — blocks (|U|, |J| and their hashes) every iteration,
x and z within 1e-10 — so every pass over A serves nrhs independent solves.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    from paper_2509_19267_b200 import _build
    _build.build()


def _rhs_set(w, nr, seed=0):
    """nr right-hand sides for w's matrix: b itself and b of other synthetic solutions."""
    rng = np.random.default_rng(seed)
    B = [w.b]
    for q in range(1, nr):
        xq = rng.standard_normal(w.shape[1])
        B.append(w.A @ xq + (0.05 * rng.standard_normal(w.shape[0]) if q % 2 else 0.0))
    return np.array(B)


@pytest.mark.parametrize("nr", [2, 3, 4])
@pytest.mark.parametrize("name", ["C4s", "C5t", "C3s"])
def test_multi_rhs_follows_independent_solves(name, nr):
    from oracle import Oracle
    from paper_2509_19267_b200 import Solver
    from workloads import by_name
    w = by_name(name)
    B = _rhs_set(w, nr)
    s = Solver.from_scipy_multi(w.A, B, eta=w.eta)
    assert s.nrhs == nr
    orcs = [Oracle(w.A, B[q], w.eta) for q in range(nr)]
    s.reset(7)
    for k in range(25):
        recs = [orcs[q].iterate(7 + q) for q in range(nr)]
        s.step(1)
        for q in range(nr):
            t = s.trace_rhs(q)[-1]
            rec = recs[q]
            assert (t["k"], t["kp"], t["hash_u"], t["kpp"], t["hash_j"]) == \
                   (k, rec.kp, rec.hash_u, rec.kpp, rec.hash_j), (k, q)
            for f in ("Z", "W", "X", "V"):
                assert abs(t[f] - getattr(rec, f)) <= 1e-9 * max(abs(getattr(rec, f)), 1e-300), (k, q, f)
        if k % 6 == 5 or k == 24:
            for q in range(nr):
                o = orcs[q]
                assert np.linalg.norm(s.x_rhs(q) - o.x) <= 1e-10 * max(np.linalg.norm(o.x), 1e-300), (k, q)
                assert np.linalg.norm(s.z_rhs(q) - o.z) <= 1e-10 * np.linalg.norm(B[q]), (k, q)
    s.close()


def test_three_channel_deblurring_parity():
    """The paper's deblurring shape: ONE Gaussian Toeplitz blur (eq:toeplitz,
    sigma = r = 20) of a 48 x 48 synthetic colour image, the three channels as three
    right-hand sides of one solve: each channel follows its own single-RHS oracle."""
    import scipy.sparse as sp
    from apps.drivers import synthetic_rgb
    from oracle import Oracle
    from paper_2509_19267_b200 import Solver
    side, sigma, radius = 48, 20.0, 20
    N = side * side
    offs = np.arange(-radius, radius + 1)
    coef = np.exp(-(offs.astype(np.float64) ** 2) / (2.0 * sigma * sigma)) / (sigma * np.sqrt(2.0 * np.pi))
    A = sp.diags([np.full(N - abs(o), c) for o, c in zip(offs, coef)], offs, shape=(N, N), format="csr")
    img = synthetic_rgb(side, 0)
    B = np.array([A @ img[:, :, c].ravel() for c in range(3)])
    s = Solver.from_scipy_multi(A, B, eta=0.5)
    orcs = [Oracle(A.tocsr(), B[c], 0.5) for c in range(3)]
    s.reset(11)
    for k in range(30):
        recs = [orcs[c].iterate(11 + c) for c in range(3)]
        s.step(1)
        for c in range(3):
            t = s.trace_rhs(c)[-1]
            assert (t["kp"], t["hash_u"], t["kpp"], t["hash_j"]) == \
                   (recs[c].kp, recs[c].hash_u, recs[c].kpp, recs[c].hash_j), (k, c)
    for c in range(3):
        assert np.linalg.norm(s.x_rhs(c) - orcs[c].x) <= 1e-10 * np.linalg.norm(orcs[c].x)
    s.close()


def test_multi_rhs_time_to_tolerance():
    """Three consistent right-hand sides on the population-model twin (C5t): iterations to
    ||x_q - x*_q|| / ||x*_q|| <= 1e-6 — the solve stops when the last channel meets it,
    each channel's first crossing within 2 % of its single-RHS oracle's count."""
    from oracle import Oracle, STOP_REL_ERR
    from paper_2509_19267_b200 import Solver, RGDBEK_CONVERGED
    from workloads import by_name
    w = by_name("C5t")
    rng = np.random.default_rng(5)
    X = [w.xstar] + [rng.standard_normal(w.shape[1]) for _ in range(2)]
    B = np.array([w.A @ xq for xq in X])
    s = Solver.from_scipy_multi(w.A, B, eta=w.eta, stop="rel_err", trace_capacity=1 << 16)
    for q in range(3):
        s.set_reference_rhs(q, X[q])
    res = s.solve(1e-6, 100000, 0)
    its = []
    for q in range(3):
        o = Oracle(w.A, B[q], w.eta)
        out, iters, _, _ = o.solve(1e-6, 100000, q, stop=STOP_REL_ERR, xstar=X[q])
        assert out == 0
        its.append(iters)
    assert res["outcome"] == RGDBEK_CONVERGED
    assert abs(res["iters"] - max(its)) <= max(1, int(0.02 * max(its))), (res["iters"], its)
    for q in range(3):
        assert np.linalg.norm(s.x_rhs(q) - X[q]) <= 1e-6 * np.linalg.norm(X[q])
    s.close()


def test_multi_rhs_argument_checks():
    from paper_2509_19267_b200 import Solver, RgdbekError
    from workloads import by_name
    w = by_name("C5t")
    B = _rhs_set(w, 2)
    s = Solver.from_scipy_multi(w.A, B, eta=w.eta)
    with pytest.raises(RgdbekError):
        s.set_mode("exact")
    with pytest.raises(RgdbekError):
        s.set_selection("greedy")
    with pytest.raises(RgdbekError):
        s.x_rhs(2)
    s.close()
    with pytest.raises(RgdbekError):
        Solver.from_scipy_multi(w.A, np.vstack([B, B, B]), eta=w.eta)      # 6 > 4
    with pytest.raises(RgdbekError):
        Solver.from_scipy_multi(w.A, np.vstack([B[0], 0 * B[1]]), eta=w.eta)  # zero RHS
