"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, same seeded inputs.

Bars (BASELINE.json north_star):
  * block index sets identical for the first 50 iterations: |U_k|, |J_k| and
    their 64-bit hashes equal, iteration by iteration;
  * x and z within relative 1e-10 (x normalised by ||x_oracle||, z by ||b||,
    reading R18) after every one of those iterations;
  * iterations to ||x - x*||/||x*|| <= 1e-6 within +/-2% of the oracle's.
"""
import os
import re

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL_X = 1e-10
TOL_Z = 1e-10
TOL_SCAL = 1e-9


@pytest.fixture(scope="module", autouse=True)
def _lib():
    from paper_2509_19267_b200 import _build
    _build.build()


def _solver(w, **kw):
    from paper_2509_19267_b200 import Solver
    if w.dense:
        return Solver(w.A, w.b, eta=w.eta, **kw)
    return Solver.from_scipy(w.A, w.b, eta=w.eta, symmetric=w.symmetric, **kw)


def _oracle(w):
    from oracle import Oracle
    return Oracle(w.A, w.b, w.eta)


def _run_parity(w, iters=50, seed=0, every=1, lazy=0, oracle=None):
    """Step both sides one iteration at a time; compare blocks, scalars, x and z."""
    s = _solver(w)
    if lazy:
        s.set_lazy(lazy)
    o = oracle if oracle is not None else _oracle(w)
    s.reset(seed)
    bn = np.linalg.norm(w.b)
    for k in range(iters):
        rec = o.iterate(seed)
        s.step(1)
        if (k + 1) % every and k + 1 != iters:
            continue
        g = s.trace()[-1]
        assert g["k"] == k
        assert (g["kp"], g["hash_u"]) == (rec.kp, rec.hash_u), f"U differs at k={k}"
        assert (g["kpp"], g["hash_j"]) == (rec.kpp, rec.hash_j), f"J differs at k={k}"
        for f in ("Z", "W", "X", "V"):
            a, b = g[f], getattr(rec, f)
            assert abs(a - b) <= TOL_SCAL * max(abs(b), 1e-300), (k, f, a, b)
        x = s.x()
        assert np.linalg.norm(x - o.x) <= TOL_X * max(np.linalg.norm(o.x), 1e-300), k
        assert np.linalg.norm(s.z() - o.z) <= TOL_Z * bn, k
        nu, hu, nj, hj = s.blocks()
        assert (nu, hu, nj, hj) == (rec.kp, rec.hash_u, rec.kpp, rec.hash_j)
    s.close()
    return o


@pytest.mark.parametrize("name,eta", [("C1", 0.5), ("C1", 0.1), ("C2s", 0.5), ("C2s", 0.1),
                                      ("C2si", 0.5)])
def test_dense_50_iterations(name, eta):
    from workloads import by_name
    w = by_name(name)
    w.eta = eta
    _run_parity(w, 50, seed=3)


@pytest.mark.parametrize("engine,grid", [("graph", None), ("persistent", "1"), ("persistent", "7")])
@pytest.mark.parametrize("name", ["C1", "C2si", "C3s", "C5t"])
def test_engines_and_grid_sizes(name, engine, grid, monkeypatch):
    """Both engines (multi-kernel CUDA graph, persistent cooperative kernel) and
    persistent grids of 1 and 7 CTAs give the oracle's trajectory."""
    from workloads import by_name
    monkeypatch.setenv("RGDBEK_ENGINE", engine)
    if grid:
        monkeypatch.setenv("RGDBEK_GRID", grid)
    _run_parity(by_name(name), 20, seed=4)


@pytest.mark.parametrize("name", ["C3s", "C4s", "C5t"])
def test_sparse_50_iterations(name):
    from workloads import by_name
    _run_parity(by_name(name), 50, seed=1)


def test_sparse_random_with_empty_rows_and_columns():
    import scipy.sparse as sp
    from workloads import sparse_random
    w = sparse_random(700, 300, density=0.01, seed=9, consistent=False)
    A = w.A.tolil()
    A[:, 7] = 0.0
    A[:, 150] = 0.0
    A[3, :] = 0.0
    A = A.tocsr()
    A.eliminate_zeros()
    A.sort_indices()
    w.A = A
    assert (np.diff(A.indptr) == 0).any()                            # empty rows
    assert (np.bincount(A.indices, minlength=300) == 0).any()        # empty columns
    _run_parity(w, 30, seed=2)


def _tile_geometry():
    """The loaded library's own tile geometry (rgdbek_build_info), so a -D variant build
    loaded through RGDBEK_LIB is tested against ITS tiles."""
    from paper_2509_19267_b200 import _build, _native
    _build.build()
    info = _native.rgdbek_build_info()
    return info["tile_nnz"], info["tile_rows"]


def _tile_edge_matrix(seed=11):
    TILE_NNZ, TILE_ROWS = _tile_geometry()
    """Row and column lengths around the sparse tile limits (csr_tiles.cuh:
    TILE_NNZ nonzeros, TILE_ROWS rows per tile): rows / columns longer than a tile
    (the group-wide path, both passes), a row of exactly TILE_NNZ, a run of 1-nnz
    rows longer than TILE_ROWS (row-limited tiles), empty rows, short rows elsewhere."""
    import scipy.sparse as sp
    from workloads.gen import Workload
    rng = np.random.default_rng(seed)
    m, n = 3000, 2400
    rows, cols = [], []
    def add_row(i, cnt):
        c = rng.choice(n, size=cnt, replace=False)
        rows.extend([i] * cnt); cols.extend(c.tolist())
    for i in range(m):
        if i in (5, 1500, 2999):
            add_row(i, TILE_NNZ + 300)        # longer than a tile
        elif i == 800:
            add_row(i, TILE_NNZ)              # exactly a tile
        elif 1000 <= i < 1000 + TILE_ROWS + 60:
            add_row(i, 1)                     # tiles limited by rows, not nonzeros
        elif i % 97 == 0:
            continue                          # empty rows
        else:
            add_row(i, int(rng.integers(2, 9)))
    for j in (3, 777):                        # columns longer than a tile (pass T); row 800 stays exact
        extra = rng.choice(np.delete(np.arange(m), 800), size=TILE_NNZ + 500, replace=False)
        rows.extend(extra.tolist()); cols.extend([j] * len(extra))
    A = sp.coo_matrix((rng.standard_normal(len(rows)), (rows, cols)), shape=(m, n)).tocsr()
    A.sum_duplicates(); A.sort_indices(); A.eliminate_zeros()
    b = A @ rng.standard_normal(n) + 0.05 * rng.standard_normal(m)
    return Workload("tile_edges", A, b, None, None, eta=0.5, meta={"seed": seed})


@pytest.mark.parametrize("engine", ["persistent", "graph"])
def test_sparse_tile_edges(engine, monkeypatch):
    """Long rows / columns (> one tile), a full tile, row-limited tiles and
    empty rows, through both engines' TMA-fed tile passes."""
    monkeypatch.setenv("RGDBEK_ENGINE", engine)
    w = _tile_edge_matrix()
    TILE_NNZ, TILE_ROWS = _tile_geometry()
    lens = np.diff(w.A.indptr)
    assert lens.max() > TILE_NNZ and (lens == TILE_NNZ).any() and (lens == 0).any()
    assert np.bincount(w.A.indices, minlength=w.A.shape[1]).max() > TILE_NNZ
    _run_parity(w, 25, seed=6)


@pytest.mark.parametrize("name,P", [("C2s", 2), ("C2s", 3), ("C2s", 4), ("C2s", 8),
                                    ("C2si", 4), ("C1", 2)])
def test_lazy_algorithm_2(name, P):
    """The paper's parallel Algorithm 2 with P logical processes (rgdbek_set_lazy)
    against oracle/lazy.py: global U, per-process J, x/z, summed scalars."""
    from oracle.lazy import LazyOracle
    from workloads import by_name
    w = by_name(name)
    _run_parity(w, 30, seed=2, lazy=P, oracle=LazyOracle(w.A, w.b, w.eta, parts=P))


@pytest.mark.parametrize("P", [2, 8])
def test_lazy_time_to_tolerance_matches_oracle(P):
    """Algorithm 2 on the C2 twin: iterations to rel. error 1e-6 within +-2 % of the
    Algorithm 2 oracle's (191 at P = 2, 154 at P = 8 vs 62 for Algorithm 1 there)."""
    from oracle import STOP_REL_ERR
    from oracle.lazy import LazyOracle
    from paper_2509_19267_b200 import RGDBEK_CONVERGED
    from workloads import by_name
    w = by_name("C2s")
    s = _solver(w, stop="rel_err")
    s.set_lazy(P)
    s.set_reference(w.xstar)
    res = s.solve(1e-6, 5000, 0)
    o = LazyOracle(w.A, w.b, w.eta, parts=P)
    out, iters, rse, rel = o.solve(1e-6, 5000, 0, stop=STOP_REL_ERR, xstar=w.xstar)
    assert res["outcome"] == RGDBEK_CONVERGED == out
    assert abs(res["iters"] - iters) <= max(1, int(0.02 * iters)), (res["iters"], iters)
    s.close()


@pytest.mark.parametrize("name", ["C2s", "C2si"])
def test_lazy_one_process_is_algorithm_1(name):
    """set_lazy(1) runs the Algorithm 2 kernel with one process: Algorithm 1's oracle."""
    from workloads import by_name
    _run_parity(by_name(name), 30, seed=5, lazy=1)


def test_lazy_argument_checks():
    from paper_2509_19267_b200 import RgdbekError
    from workloads import by_name
    w = by_name("C3s")                                # sparse: not supported
    s = _solver(w)
    with pytest.raises(RgdbekError):
        s.set_lazy(2)
    s.close()
    d = _solver(by_name("C1"))
    with pytest.raises(RgdbekError):
        d.set_lazy(9)
    d.set_selection("greedy")
    with pytest.raises(RgdbekError):
        d.set_lazy(2)
    d.set_selection("random")
    d.set_lazy(2)
    with pytest.raises(RgdbekError):
        d.set_mode("exact")
    d.set_lazy(0)                                     # back to Algorithm 1
    d.close()


def test_fat_sparse_system():
    from workloads import sparse_random
    w = sparse_random(200, 900, density=0.02, seed=4)
    _run_parity(w, 30, seed=5)


def test_block_size_one_and_large_eta():
    from workloads import dense_gaussian
    w = dense_gaussian(300, 80, seed=2, noise=0.1)
    w.eta = 0.001            # k_c = k_r = 1: REK-type steps
    _run_parity(w, 25, seed=1)
    w.eta = 0.97
    _run_parity(w, 25, seed=1)


@pytest.mark.parametrize("name,seeds", [("C1", [0, 1, 2, 3]), ("C2s", [0, 1]), ("C5t", [0])])
def test_time_to_tolerance_matches_oracle(name, seeds):
    from oracle import STOP_REL_ERR
    from paper_2509_19267_b200 import RGDBEK_CONVERGED
    from workloads import by_name
    w = by_name(name)
    for seed in seeds:
        s = _solver(w, stop="rel_err")
        s.set_reference(w.xstar)
        res = s.solve(1e-6, 100000, seed)
        o = _oracle(w)
        out, iters, rse, rel = o.solve(1e-6, 100000, seed, stop=STOP_REL_ERR, xstar=w.xstar)
        assert res["outcome"] == RGDBEK_CONVERGED == out
        assert abs(res["iters"] - iters) <= max(1, int(0.02 * iters)), (seed, res["iters"], iters)
        assert res["rel_err"] <= 1e-6
        s.close()


def test_rse_stop_spec_identity():
    from paper_2509_19267_b200 import Solver, RGDBEK_CONVERGED
    s = Solver(np.eye(10), np.ones(10), eta=0.5, stop="rse")
    res = s.solve(1e-12, 1000, 0)
    assert res["outcome"] == RGDBEK_CONVERGED and res["rse"] <= 1e-12
    np.testing.assert_allclose(s.x(), np.ones(10), atol=1e-6)


def test_stall_and_max_iter():
    from paper_2509_19267_b200 import Solver, RGDBEK_STALLED, RGDBEK_MAX_ITER
    s = Solver(np.array([[1.0, 0.0], [0.0, 0.0]]), np.array([0.0, 1.0]), eta=0.5)
    res = s.solve(1e-12, 100, 0)
    assert res["outcome"] == RGDBEK_STALLED and res["iters"] == 1 and res["rse"] == 1.0
    from workloads import dense_gaussian
    w = dense_gaussian(60, 20, seed=1)
    s = Solver(w.A, w.b, eta=0.5)
    res = s.solve(1e-300, 7, 0)
    assert res["outcome"] == RGDBEK_MAX_ITER and res["iters"] == 7


def test_inconsistent_shift_invariance_on_gpu():
    from workloads import by_name
    w = by_name("C2si")
    from paper_2509_19267_b200 import Solver
    a = Solver(w.A, w.b, eta=0.5)
    c = Solver(w.A, w.b - w.rvec, eta=0.5)
    a.reset(7); c.reset(7)
    a.step(40); c.step(40)
    ta, tc = a.trace(), c.trace()
    assert [(t["hash_u"], t["hash_j"]) for t in ta] == [(t["hash_u"], t["hash_j"]) for t in tc]
    assert np.linalg.norm(a.x() - c.x()) <= 1e-12 * np.linalg.norm(c.x())
    assert np.linalg.norm((a.z() - w.rvec) - c.z()) <= 1e-12 * np.linalg.norm(w.b)


def test_step_chunks_equal_one_run_and_resume():
    from workloads import by_name
    w = by_name("C2s")
    from paper_2509_19267_b200 import Solver
    a = Solver(w.A, w.b)
    b = Solver(w.A, w.b)
    a.reset(11); b.reset(11)
    a.step(30)
    b.step(7); b.step(0); b.step(13); b.step(10)
    assert np.array_equal(a.x(), b.x()) and np.array_equal(a.z(), b.z())
    # resume from a saved state
    c = Solver(w.A, w.b)
    c.reset(11)
    c.set_state(b.x(), b.z(), 30)
    a.step(5); c.step(5)
    assert np.array_equal(a.x(), c.x()) and np.array_equal(a.z(), c.z())


def test_step_zero_reports_rse_of_current_iterate():
    from workloads import by_name
    w = by_name("C1")
    s = _solver(w)
    s.reset(0)
    r = s.step(0)
    assert r["iters"] == 0 and abs(r["rse"] - 1.0) < 1e-15
    r = s.step(4)
    o = _oracle(w)
    for _ in range(4):
        rec = o.iterate(0)
    assert r["iters"] == 4 and abs(r["rse"] - rec.rse) <= 1e-9 * rec.rse


def test_create_errors():
    import scipy.sparse as sp
    from paper_2509_19267_b200 import Solver, RgdbekError
    with pytest.raises(RgdbekError) as e:
        Solver(np.eye(3), np.zeros(3))
    assert e.value.code == -4
    A = np.eye(3); A[1, 1] = np.nan
    with pytest.raises(RgdbekError) as e:
        Solver(A, np.ones(3))
    assert e.value.code == -5
    # columns not strictly increasing
    with pytest.raises(RgdbekError) as e:
        Solver.from_csr(2, 3, np.array([0, 2, 3]), np.array([2, 1, 0], dtype=np.int32),
                        np.ones(3), np.ones(2))
    assert e.value.code == -3
    with pytest.raises(RgdbekError) as e:
        Solver.from_csr(2, 3, np.array([0, 2, 3]), np.array([0, 5, 0], dtype=np.int32),
                        np.ones(3), np.ones(2))
    assert e.value.code == -3
    with pytest.raises(RgdbekError) as e:
        Solver.from_scipy(sp.csr_matrix(np.array([[1.0, 2.0], [0.0, 1.0]])), np.ones(2),
                          symmetric=True)
    assert e.value.code == -1


def test_torch_cuda_tensors_as_inputs():
    import torch
    from workloads import by_name
    from paper_2509_19267_b200 import Solver
    w = by_name("C1")
    At = torch.from_numpy(w.A).cuda()
    bt = torch.from_numpy(w.b).cuda()
    s = Solver(At, bt, eta=0.5, stream=torch.cuda.current_stream().cuda_stream)
    s.reset(0)
    s.step(10)
    xo = torch.empty(w.A.shape[1], dtype=torch.float64, device="cuda")
    s.x(out=xo)
    o = _oracle(w)
    for _ in range(10):
        o.iterate(0)
    assert np.linalg.norm(xo.cpu().numpy() - o.x) <= 1e-10 * np.linalg.norm(o.x)


@pytest.mark.parametrize("name", ["C2c", "C2i"])
def test_full_size_dense_bench_configuration(name):
    """BASELINE configs[1] at full size, in bench.py's launch configuration:
    5 iterations compared element-wise (oracle takes seconds per iteration)."""
    from workloads import by_name
    w = by_name(name)
    _run_parity(w, 5, seed=0)


def test_full_size_c3_sampled():
    """C3 (4M unknowns) at full size: 3 iterations vs the oracle on sampled rows."""
    from workloads import by_name
    w = by_name("C3")
    s = _solver(w)
    o = _oracle(w)
    s.reset(0)
    recs = [o.iterate(0) for _ in range(3)]
    s.step(3)
    t = s.trace()
    assert [(r["kp"], r["hash_u"], r["kpp"], r["hash_j"]) for r in t] == \
           [(r.kp, r.hash_u, r.kpp, r.hash_j) for r in recs]
    rng = np.random.default_rng(0)
    idx = rng.choice(w.A.shape[1], 4096, replace=False)
    x = s.x()
    assert np.max(np.abs(x[idx] - o.x[idx])) <= 1e-10 * np.max(np.abs(o.x))
    assert np.linalg.norm(s.z() - o.z) <= 1e-10 * np.linalg.norm(w.b)


def test_full_size_c4_sampled():
    """C4 (1M-pixel Toeplitz blur, 43M nnz) at full size, in bench.py's launch
    configuration: 3 iterations, blocks identical, x / z within 1e-10."""
    from workloads import by_name
    w = by_name("C4")
    s = _solver(w)
    o = _oracle(w)
    s.reset(0)
    recs = [o.iterate(0) for _ in range(3)]
    s.step(3)
    t = s.trace()
    assert [(r["kp"], r["hash_u"], r["kpp"], r["hash_j"]) for r in t] == \
           [(r.kp, r.hash_u, r.kpp, r.hash_j) for r in recs]
    assert np.linalg.norm(s.x() - o.x) <= 1e-10 * np.linalg.norm(o.x)
    assert np.linalg.norm(s.z() - o.z) <= 1e-10 * np.linalg.norm(w.b)


@pytest.mark.parametrize("eta", [0.5, 0.1])
def test_full_size_c2c_time_to_tolerance(eta):
    """The headline metric's second half at full size (20000 x 5000): iterations
    to relative error 1e-6 within +-2 % of the oracle's own count (SURVEY V13
    quotes 62 at eta = 0.5 and 165 at eta = 0.1 from an independent run)."""
    from oracle import STOP_REL_ERR
    from paper_2509_19267_b200 import RGDBEK_CONVERGED
    from workloads import by_name
    w = by_name("C2c")
    w.eta = eta
    s = _solver(w, stop="rel_err")
    s.set_reference(w.xstar)
    res = s.solve(1e-6, 100000, 0)
    o = _oracle(w)
    out, iters, rse, rel = o.solve(1e-6, 100000, 0, stop=STOP_REL_ERR, xstar=w.xstar)
    assert res["outcome"] == RGDBEK_CONVERGED == out
    assert abs(res["iters"] - iters) <= max(1, int(0.02 * iters)), (res["iters"], iters)
    assert res["rel_err"] <= 1e-6
    s.close()


@pytest.mark.parametrize("name", ["C2si", "C5t", "C3s"])
def test_sharded_code_path_world1_nccl(name):
    """The row-sharded (NCCL) code path of the library on one GPU: a world of 1
    rank runs every allreduce / allgather, finalize and survivor kernel of the
    multi-GPU plan; its trajectory must still be the oracle's."""
    import socket
    import torch
    import torch.distributed as dist
    from paper_2509_19267_b200.dist import init_nccl_comm, destroy_nccl_comm
    from workloads import by_name
    import bench
    sock = socket.socket(); sock.bind(("127.0.0.1", 0)); port = sock.getsockname()[1]; sock.close()
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        comm = init_nccl_comm(0)
        w = by_name(name)
        s = bench.make_solver(w, 0, None, (0, w.shape[0]), comm)
        assert s.engine_info()[0] == 1
        o = _oracle(w)
        s.reset(2)
        bn = np.linalg.norm(w.b)
        for k in range(20):
            rec = o.iterate(2)
            s.step(1)
            g = s.trace()[-1]
            assert (g["kp"], g["hash_u"], g["kpp"], g["hash_j"]) == (rec.kp, rec.hash_u, rec.kpp, rec.hash_j), k
            assert np.linalg.norm(s.x() - o.x) <= TOL_X * np.linalg.norm(o.x)
            assert np.linalg.norm(s.z() - o.z) <= TOL_Z * bn
        s.close()
        destroy_nccl_comm(comm)
    finally:
        dist.destroy_process_group()


def test_time_to_tolerance_c5s_scaled_twin():
    """C5s (50000x5000, 1e6 nnz, the oracle-feasible twin of C5): iterations to
    ||x - x*||/||x*|| <= 1e-6 within 2 % of the oracle's (~5.7k iterations)."""
    from oracle import STOP_REL_ERR
    from workloads import by_name
    w = by_name("C5s")
    s = _solver(w, stop="rel_err")
    s.set_reference(w.xstar)
    res = s.solve(1e-6, 100000, 0)
    o = _oracle(w)
    out, iters, _, _ = o.solve(1e-6, 100000, 0, stop=STOP_REL_ERR, xstar=w.xstar)
    assert abs(res["iters"] - iters) <= int(0.02 * iters), (res["iters"], iters)
    s.close()


@pytest.mark.parametrize("name,inner_max", [("C2s", 200), ("C2si", 200), ("C5t", 2000), ("C3s", 60)])
def test_exact_projection_mode(name, inner_max):
    """NEXT #1: Alg. 1's exact projections by inner CGLS (the paper's
    LSQR route), same stopping rule on both sides: identical blocks every
    iteration, x and z to 1e-8.  inner_max lets the inner solves converge
    (C5t's row blocks have kappa ~ 43, so CGLS needs ~10^3 iterations to 1e-13):
    an UNconverged Krylov iterate on an ill-conditioned block amplifies the
    two sides' different summation orders, so only converged solves are compared
    (C3s runs a fixed 60 inner iterations on well-separated blocks)."""
    from oracle import Oracle
    from workloads import by_name
    w = by_name(name)
    s = _solver(w)
    s.set_mode("exact", inner_tol=1e-13, inner_max=inner_max)
    o = Oracle(w.A, w.b, w.eta, update="exact", inner_tol=1e-13, inner_max=inner_max)
    s.reset(5)
    bn = np.linalg.norm(w.b)
    for k in range(8):
        rec = o.iterate(5)
        s.step(1)
        g = s.trace()[-1]
        assert (g["kp"], g["hash_u"], g["kpp"], g["hash_j"]) == (rec.kp, rec.hash_u, rec.kpp, rec.hash_j), k
        assert abs(g["Z"] - rec.Z) <= 1e-9 * rec.Z and abs(g["X"] - rec.X) <= 1e-8 * rec.X
        assert np.linalg.norm(s.x() - o.x) <= 1e-8 * np.linalg.norm(o.x), k
        assert np.linalg.norm(s.z() - o.z) <= 1e-8 * bn, k
    s.close()


def test_exact_mode_time_to_tolerance():
    from oracle import Oracle, STOP_REL_ERR
    from paper_2509_19267_b200 import RGDBEK_CONVERGED
    from workloads import by_name
    w = by_name("C2s")
    s = _solver(w, stop="rel_err")
    s.set_mode("exact", inner_tol=1e-13, inner_max=200)
    s.set_reference(w.xstar)
    res = s.solve(1e-6, 1000, 0)
    o = Oracle(w.A, w.b, w.eta, update="exact", inner_tol=1e-13, inner_max=200)
    out, iters, _, _ = o.solve(1e-6, 1000, 0, stop=STOP_REL_ERR, xstar=w.xstar)
    assert res["outcome"] == RGDBEK_CONVERGED == out
    assert abs(res["iters"] - iters) <= max(1, int(0.02 * iters)), (res["iters"], iters)


@pytest.mark.parametrize("name,update", [("C2s", "pinv_free"), ("C5t", "pinv_free"),
                                         ("C3s", "pinv_free"), ("C2si", "exact")])
def test_greedy_gdbek_selection(name, update):
    """NEXT #2: GDBEK's threshold sets on the GPU (pinv-free and exact
    updates) vs the oracle: identical blocks, x and z to 1e-10 (1e-8 exact)."""
    from oracle import Oracle
    from workloads import by_name
    w = by_name(name)
    s = _solver(w)
    s.set_selection("greedy")
    kw = {}
    if update == "exact":
        s.set_mode("exact", inner_tol=1e-13, inner_max=200)
        kw = dict(update="exact", inner_tol=1e-13, inner_max=200)
    o = Oracle(w.A, w.b, w.eta, select="greedy", **kw)
    tol = 1e-8 if update == "exact" else TOL_X
    s.reset(0)
    for k in range(12):
        rec = o.iterate(0)
        s.step(1)
        g = s.trace()[-1]
        assert (g["kp"], g["hash_u"], g["kpp"], g["hash_j"]) == (rec.kp, rec.hash_u, rec.kpp, rec.hash_j), k
        assert np.linalg.norm(s.x() - o.x) <= tol * np.linalg.norm(o.x), k
        assert np.linalg.norm(s.z() - o.z) <= tol * np.linalg.norm(w.b), k
    s.close()


@pytest.mark.parametrize("name", ["C1", "C2s", "C2si"])
def test_exact_mode_matches_lstsq_definition(name):
    """NEXT #1 against the DEFINITION of Alg. 1's updates, not the CGLS
    route: the oracle's update="exact_lstsq" (numpy minimum-norm lstsq on the extracted
    A_U, A^J).  With converged inner solves (reading R1b) the GPU gives the same blocks
    every iteration and x, z to 1e-8.  (Well-conditioned dense blocks: on C3s's
    ill-conditioned Poisson blocks 400 CGLS steps stop ~2e-8 short of the projection,
    which the CGLS-route comparison test_exact_projection_mode covers.)"""
    from oracle import Oracle
    from workloads import by_name
    w = by_name(name)
    s = _solver(w)
    s.set_mode("exact", inner_tol=1e-14, inner_max=400)
    o = Oracle(w.A, w.b, w.eta, update="exact_lstsq")
    s.reset(3)
    bn = np.linalg.norm(w.b)
    for k in range(6):
        rec = o.iterate(3)
        s.step(1)
        g = s.trace()[-1]
        assert (g["kp"], g["hash_u"], g["kpp"], g["hash_j"]) == (rec.kp, rec.hash_u, rec.kpp, rec.hash_j), k
        assert np.linalg.norm(s.x() - o.x) <= 1e-8 * np.linalg.norm(o.x), k
        assert np.linalg.norm(s.z() - o.z) <= 1e-8 * bn, k
    s.close()


@pytest.mark.parametrize("name,engine,mode", [("C1", "persistent", "pinv_free"),
                                              ("C2s", "persistent", "pinv_free"),
                                              ("C5t", "persistent", "pinv_free"),
                                              ("C3s", "persistent", "pinv_free"),
                                              ("C2si", "graph", "pinv_free"),
                                              ("C5t", "graph", "pinv_free"),
                                              ("C2s", "persistent", "exact")])
def test_full_block_lists_every_iteration(name, engine, mode, monkeypatch):
    """SURVEY §8(c) parity protocol: the FULL index lists U_k, J_k (rgdbek_set_capture +
    rgdbek_get_blocks) equal the oracle's, every iteration, on C1 / C2 / C5 twins."""
    from oracle import Oracle
    from workloads import by_name
    monkeypatch.setenv("RGDBEK_ENGINE", engine)
    w = by_name(name)
    s = _solver(w)
    s.set_capture(True)
    kw = {}
    if mode == "exact":
        s.set_mode("exact", inner_tol=1e-13, inner_max=200)
        kw = dict(update="exact", inner_tol=1e-13, inner_max=200)
    o = Oracle(w.A, w.b, w.eta, **kw)
    s.reset(4)
    iters = 30 if mode == "pinv_free" else 6
    for k in range(iters):
        rec = o.iterate(4, keep_blocks=True)
        s.step(1)
        U, J = s.block_lists()
        assert np.array_equal(U, rec.U), f"U differs at k={k}"
        assert np.array_equal(J, rec.J), f"J differs at k={k}"
    s.close()


def test_block_lists_need_capture():
    from paper_2509_19267_b200 import RgdbekError
    from workloads import by_name
    s = _solver(by_name("C1"))
    s.reset(0)
    s.step(2)
    with pytest.raises(RgdbekError) as e:
        s.block_lists()
    assert e.value.code == -6
    s.close()


def test_lazy_wide_columns_per_cta(monkeypatch):
    """Algorithm 2 with more than 1024 columns per CTA (the column-sum phase
    looped only over the first 1024): 2 CTAs, n = 2300, P = 2 vs oracle/lazy.py."""
    from oracle.lazy import LazyOracle
    from workloads import dense_gaussian
    monkeypatch.setenv("RGDBEK_GRID", "2")
    w = dense_gaussian(600, 2300, seed=3)
    _run_parity(w, 12, seed=1, lazy=2, oracle=LazyOracle(w.A, w.b, w.eta, parts=2))


def test_output_buffers_are_checked():
    from workloads import by_name
    w = by_name("C1")
    s = _solver(w)
    s.reset(0)
    s.step(1)
    for bad in (np.empty(w.A.shape[1], dtype=np.float32), np.empty(w.A.shape[1] - 1),
                np.empty(2 * w.A.shape[1])[::2]):
        with pytest.raises(ValueError):
            s.x(out=bad)
    with pytest.raises(ValueError):
        s.z(out=np.empty(3))
    s.close()
