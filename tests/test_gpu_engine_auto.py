"""Engine choice at create (runtime.cu setup_persistent): a sparse system with
nnz >= 2^26 on one GPU runs the multi-kernel graph engine (its 2-deep tile rings fit 48
tile warps per SM), everything else the persistent kernel; a feature only the persistent
kernels implement (exact mode, greedy sets, Algorithm 2, several right-hand sides)
switches an automatically chosen graph engine back.  The threshold is lowered with
RGDBEK_GRAPH_NNZ so small systems exercise the same decisions; the trajectory stays the
oracle's (full parity bars of test_gpu_parity.py) on either engine.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    from paper_2509_19267_b200 import _build
    _build.build()


def _sparse(name="C3s"):
    from paper_2509_19267_b200 import Solver
    from workloads import by_name
    w = by_name(name)
    return w, Solver.from_scipy(w.A, w.b, eta=w.eta, symmetric=w.symmetric)


def test_large_sparse_picks_graph_engine_and_keeps_parity(monkeypatch):
    from oracle import Oracle
    monkeypatch.delenv("RGDBEK_ENGINE", raising=False)
    monkeypatch.setenv("RGDBEK_GRAPH_NNZ", "1000")
    w, s = _sparse("C3s")
    assert s.engine_info()[0] == 1
    o = Oracle(w.A, w.b, w.eta)
    s.reset(5)
    for k in range(20):
        rec = o.iterate(5)
        s.step(1)
        t = s.trace()[-1]
        assert (t["kp"], t["hash_u"], t["kpp"], t["hash_j"]) == (rec.kp, rec.hash_u, rec.kpp, rec.hash_j), k
    assert np.linalg.norm(s.x() - o.x) <= 1e-10 * np.linalg.norm(o.x)
    s.close()


def test_below_threshold_and_dense_stay_persistent(monkeypatch):
    from paper_2509_19267_b200 import Solver
    from workloads import by_name
    monkeypatch.delenv("RGDBEK_ENGINE", raising=False)
    monkeypatch.delenv("RGDBEK_GRAPH_NNZ", raising=False)
    w, s = _sparse("C3s")
    assert s.engine_info()[0] == 0
    s.close()
    monkeypatch.setenv("RGDBEK_GRAPH_NNZ", "1000")
    wd = by_name("C1")
    sd = Solver(wd.A, wd.b, eta=wd.eta)
    assert sd.engine_info()[0] == 0
    sd.close()
    monkeypatch.setenv("RGDBEK_ENGINE", "persistent")       # explicit choice wins
    w, s = _sparse("C3s")
    assert s.engine_info()[0] == 0
    s.close()


@pytest.mark.parametrize("feature", ["exact", "greedy"])
def test_persistent_only_features_switch_back(feature, monkeypatch):
    """set_mode('exact') / set_selection('greedy') on an automatically chosen graph engine
    move the handle to the persistent kernel, which then matches the oracle."""
    from oracle import Oracle
    monkeypatch.delenv("RGDBEK_ENGINE", raising=False)
    monkeypatch.setenv("RGDBEK_GRAPH_NNZ", "1000")
    w, s = _sparse("C3s")
    assert s.engine_info()[0] == 1
    if feature == "exact":
        s.set_mode("exact", inner_tol=1e-13, inner_max=60)
        o = Oracle(w.A, w.b, w.eta, update="exact", inner_tol=1e-13, inner_max=60)
    else:
        s.set_selection("greedy")
        o = Oracle(w.A, w.b, w.eta, select="greedy")
    assert s.engine_info()[0] == 0
    s.reset(1)
    for k in range(8):
        rec = o.iterate(1)
        s.step(1)
        t = s.trace()[-1]
        assert (t["kp"], t["kpp"]) == (rec.kp, rec.kpp), k
    assert np.linalg.norm(s.x() - o.x) <= 1e-8 * np.linalg.norm(o.x)
    s.close()


def test_explicit_graph_engine_refuses_persistent_only_features(monkeypatch):
    """An explicitly requested graph engine is not switched: exact mode is refused."""
    from paper_2509_19267_b200 import RgdbekError
    monkeypatch.setenv("RGDBEK_ENGINE", "graph")
    w, s = _sparse("C3s")
    assert s.engine_info()[0] == 1
    with pytest.raises(RgdbekError):
        s.set_mode("exact")
    s.close()


def test_multi_rhs_on_a_large_system_runs_persistent(monkeypatch):
    from paper_2509_19267_b200 import Solver
    from workloads import by_name
    monkeypatch.delenv("RGDBEK_ENGINE", raising=False)
    monkeypatch.setenv("RGDBEK_GRAPH_NNZ", "1000")
    w = by_name("C3s")
    B = np.stack([w.b, 0.5 * w.b])
    s = Solver.from_scipy_multi(w.A, B, eta=w.eta)
    assert s.engine_info()[0] == 0 and s.nrhs == 2
    s.close()
