"""B200-native RGDBEK hot path (arXiv 2509.19267) — Python front end.

The solver runs in librgdbek.so (hand-written sm_100a CUDA behind the C ABI
of include/rgdbek.h).  This package only marshals arguments: numpy arrays or
torch tensors (host or CUDA) become pointers; torch is used for device
memory, streams and process groups, never for the method's arithmetic.
"""
import ctypes as C

import numpy as np

from . import _native as N
from ._native import (RgdbekError, RGDBEK_CONVERGED, RGDBEK_MAX_ITER, RGDBEK_STALLED,
                      RGDBEK_STOP_RSE, RGDBEK_STOP_REL_ERR, RGDBEK_STOP_NONE)

__all__ = ["Solver", "ShardGroup", "RgdbekError", "RGDBEK_CONVERGED", "RGDBEK_MAX_ITER", "RGDBEK_STALLED",
           "RGDBEK_STOP_RSE", "RGDBEK_STOP_REL_ERR", "RGDBEK_STOP_NONE", "library_path"]

library_path = N.LIB_PATH
_STOP = {"rse": RGDBEK_STOP_RSE, "rel_err": RGDBEK_STOP_REL_ERR, "none": RGDBEK_STOP_NONE}


def _ptr(a, dtype):
    """(pointer, keepalive) of a contiguous array of `dtype` (numpy or torch, host or CUDA)."""
    if hasattr(a, "data_ptr"):                       # torch tensor
        import torch
        tdt = {np.float64: torch.float64, np.int64: torch.int64, np.int32: torch.int32}[dtype]
        t = a.contiguous()
        if t.dtype != tdt:
            t = t.to(tdt)
        return C.c_void_p(t.data_ptr()), t
    arr = np.ascontiguousarray(a, dtype=dtype)
    return C.c_void_p(arr.ctypes.data), arr


class Solver:
    """One RGDBEK problem resident on one GPU (one rank of a row-sharded solve).

    Solver(A, b, eta=0.5) with A a dense (m, n) array, or
    Solver.from_csr(m, n, row_ptr, col_idx, val, b, ...) for sparse A.
    """

    def __init__(self, A=None, b=None, eta=0.5, stop="rse", device=0, stream=None,
                 symmetric=False, trace_capacity=4096, row_range=None, m=None, nccl_comm=None,
                 _handle=None, _shape=None):
        self._h = None
        self._opts = N.rgdbek_options_default()
        self._opts.eta = float(eta)
        self._opts.stop = _STOP[stop] if isinstance(stop, str) else int(stop)
        self._opts.device = int(device)
        self._opts.stream = stream
        self._opts.symmetric = 1 if symmetric else 0
        self._opts.trace_capacity = int(trace_capacity)
        if nccl_comm is not None:
            self._opts.nccl_comm = nccl_comm
        if row_range is not None:
            self._opts.row_begin, self._opts.row_end = int(row_range[0]), int(row_range[1])
        if _handle is not None:
            self._h = _handle
            self.m, self.n, self.m_local = _shape
            return
        if A is None or b is None:
            raise ValueError("A and b are required")
        m_loc, n = A.shape
        self.m = int(m) if m is not None else m_loc
        self.n = n
        self.m_local = m_loc
        pa, ka = _ptr(A, np.float64)
        pb, kb = _ptr(b, np.float64)
        self._h = N.rgdbek_create_dense(self.m, n, pa, n, pb, self._opts)
        del ka, kb

    @classmethod
    def from_csr(cls, m, n, row_ptr, col_idx, val, b, eta=0.5, stop="rse", device=0, stream=None,
                 symmetric=False, trace_capacity=4096, row_range=None, nccl_comm=None):
        self = cls.__new__(cls)
        Solver.__init__(self, eta=eta, stop=stop, device=device, stream=stream,
                        symmetric=symmetric, trace_capacity=trace_capacity, row_range=row_range,
                        nccl_comm=nccl_comm, _handle=0, _shape=(m, n, 0))
        self._h = None
        m_loc = len(row_ptr) - 1
        prp, k1 = _ptr(row_ptr, np.int64)
        pci, k2 = _ptr(col_idx, np.int32)
        pv, k3 = _ptr(val, np.float64)
        pb, k4 = _ptr(b, np.float64)
        self._h = N.rgdbek_create_csr(int(m), int(n), int(len(val)), prp, pci, pv, pb, self._opts)
        self.m, self.n, self.m_local = int(m), int(n), m_loc
        return self

    @classmethod
    def from_scipy_multi(cls, A, B, eta=0.5, stop="rse", device=0, stream=None, trace_capacity=4096):
        """Several right-hand sides sharing sparse A (rgdbek_create_csr_multi): B is
        (nrhs, m); right-hand side q follows the single-RHS solve with seed + q."""
        A = A.tocsr(copy=True)
        A.sort_indices()
        B = np.ascontiguousarray(B, dtype=np.float64)
        if B.ndim != 2 or B.shape[1] != A.shape[0]:
            raise ValueError("B must be (nrhs, m)")
        self = cls.__new__(cls)
        Solver.__init__(self, eta=eta, stop=stop, device=device, stream=stream,
                        trace_capacity=trace_capacity, _handle=0, _shape=(A.shape[0], A.shape[1], 0))
        self._h = None
        prp, k1 = _ptr(A.indptr.astype(np.int64), np.int64)
        pci, k2 = _ptr(A.indices.astype(np.int32), np.int32)
        pv, k3 = _ptr(A.data.astype(np.float64), np.float64)
        pb, k4 = _ptr(B, np.float64)
        self._h = N.rgdbek_create_csr_multi(A.shape[0], A.shape[1], A.nnz, prp, pci, pv, pb,
                                            B.shape[0], self._opts)
        self.m, self.n, self.m_local = A.shape[0], A.shape[1], A.shape[0]
        return self

    @property
    def nrhs(self):
        return N.rgdbek_rhs_count(self._h)

    def x_rhs(self, rhs):
        out = np.empty(self.n)
        N.rgdbek_get_x_rhs(self._h, int(rhs), _out_ptr(out, self.n))
        return out

    def z_rhs(self, rhs):
        out = np.empty(self.m_local)
        N.rgdbek_get_z_rhs(self._h, int(rhs), _out_ptr(out, self.m_local))
        return out

    def set_reference_rhs(self, rhs, xstar):
        p, keep = _ptr(xstar, np.float64)
        N.rgdbek_set_reference_rhs(self._h, int(rhs), p)

    def trace_rhs(self, rhs, max_records=1 << 20):
        recs = N.rgdbek_get_trace_rhs(self._h, int(rhs), max_records)
        return [dict(k=r.k, kp=r.kp, hash_u=r.hash_u, Z=r.Z, W=r.W, kpp=r.kpp, hash_j=r.hash_j,
                     X=r.X, V=r.V, rse=r.rse) for r in recs]

    @classmethod
    def from_scipy(cls, A, b, **kw):
        A = A.tocsr(copy=True)                       # never reorder the caller's matrix
        A.sort_indices()
        return cls.from_csr(A.shape[0], A.shape[1], A.indptr.astype(np.int64),
                            A.indices.astype(np.int32), A.data.astype(np.float64), b, **kw)

    # ---- calls --------------------------------------------------------------------
    def reset(self, seed=0):
        N.rgdbek_reset(self._h, int(seed))

    def step(self, n_iter):
        return _res(N.rgdbek_step(self._h, int(n_iter)))

    def solve(self, tol=1e-6, max_iter=100000, seed=0):
        return _res(N.rgdbek_solve(self._h, float(tol), int(max_iter), int(seed)))

    def set_stop(self, stop):
        N.rgdbek_set_stop(self._h, _STOP[stop] if isinstance(stop, str) else int(stop))

    def set_reference(self, xstar):
        p, keep = _ptr(xstar, np.float64)
        N.rgdbek_set_reference(self._h, p)

    def set_state(self, x, z_local, k):
        px, kx = _ptr(x, np.float64)
        pz, kz = _ptr(z_local, np.float64)
        N.rgdbek_set_state(self._h, px, pz, int(k))

    def x(self, out=None):
        out = np.empty(self.n) if out is None else out
        N.rgdbek_get_x(self._h, _out_ptr(out, self.n))
        return out

    def z(self, out=None):
        out = np.empty(self.m_local) if out is None else out
        N.rgdbek_get_z(self._h, _out_ptr(out, self.m_local))
        return out

    def blocks(self):
        """(|U|, hash U, |J|, hash J) of the last completed iteration."""
        return N.rgdbek_get_blocks(self._h)

    def set_capture(self, enable=True):
        """Record the U / J masks of every iteration (needed by block_lists())."""
        N.rgdbek_set_capture(self._h, 1 if enable else 0)

    def block_lists(self):
        """(U, J) sorted index arrays of the last completed iteration (J: global rows of
        this rank); needs set_capture() before the iterations."""
        U = np.empty(self.n, dtype=np.int32)
        J = np.empty(max(self.m_local, 1), dtype=np.int32)
        nu, _, nj, _ = N.rgdbek_get_blocks(self._h, C.c_void_p(U.ctypes.data),
                                           C.c_void_p(J.ctypes.data))
        return U[:nu].copy(), J[:nj].copy()

    def selection_stats(self):
        """[local smem overflows, persistent slow-path selections, graph slow-path selections, 0]."""
        return N.rgdbek_selection_stats(self._h)

    def trace(self, max_records=1 << 20):
        recs = N.rgdbek_get_trace(self._h, max_records)
        return [dict(k=r.k, kp=r.kp, hash_u=r.hash_u, Z=r.Z, W=r.W, kpp=r.kpp, hash_j=r.hash_j,
                     X=r.X, V=r.V, rse=r.rse) for r in recs]

    def launch_kernel(self, kernel, reps):
        return N.rgdbek_launch_kernel(self._h, int(kernel), int(reps))

    def phase_times(self):
        """Per-phase device ns of the persistent engine (RGDBEK_PHASE_TIMING=1), else []."""
        return N.rgdbek_phase_times(self._h)

    def set_mode(self, mode, inner_tol=1e-12, inner_max=50):
        """'pinv_free' (default) or 'exact' (Alg. 1's projections via inner CGLS)."""
        m = {"pinv_free": 0, "exact": 1}[mode] if isinstance(mode, str) else int(mode)
        N.rgdbek_set_mode(self._h, m, inner_tol, inner_max)

    def set_selection(self, rule):
        """'random' (RGDBEK sampling, default) or 'greedy' (GDBEK threshold sets)."""
        r = {"random": 0, "greedy": 1}[rule] if isinstance(rule, str) else int(rule)
        N.rgdbek_set_selection(self._h, r)

    def set_lazy(self, processes):
        """The paper's parallel Algorithm 2 with `processes` logical row processes
        (lazily averaged x-update); 0 returns to Algorithm 1."""
        N.rgdbek_set_lazy(self._h, int(processes))

    def peer_window(self):
        """(window begin, window end, first row, end row) of a peer-sharded rank."""
        return tuple(N.rgdbek_peer_window(self._h))

    def passes(self):
        """Full passes over A since the last reset (persistent engine)."""
        return N.rgdbek_get_counters(self._h)

    def a_bytes(self):
        """Exact mode: algorithmic bytes of A read since the last reset."""
        return N.rgdbek_get_a_bytes(self._h)

    def engine_info(self):
        """(engine, ctas): engine 0 = persistent kernel, 1 = CUDA-graph engine."""
        return N.rgdbek_engine_info(self._h)

    def launches_per_iteration(self):
        return N.rgdbek_launches_per_iteration(self._h)

    @property
    def stream(self):
        return N.rgdbek_stream(self._h)

    def close(self):
        if self._h:
            N.rgdbek_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class ShardGroup:
    """R peer-sharded ranks (Solvers created with row_range=..., m=..., no nccl_comm) on ONE
    GPU, run as one cooperative launch (rgdbek_group_create): the multi-GPU decomposition
    emulated for tests.  Per-rank state stays readable through the member Solvers."""

    def __init__(self, solvers):
        self.solvers = list(solvers)
        self._g = N.rgdbek_group_create([s._h for s in self.solvers])

    def reset(self, seed=0):
        N.rgdbek_group_reset(self._g, int(seed), self.solvers[0]._h)

    def step(self, n_iter):
        return _res(N.rgdbek_group_step(self._g, int(n_iter), self.solvers[0]._h))

    def solve(self, tol=1e-6, max_iter=100000, seed=0):
        return _res(N.rgdbek_group_solve(self._g, float(tol), int(max_iter), int(seed),
                                         self.solvers[0]._h))

    def close(self):
        if self._g:
            N.rgdbek_group_destroy(self._g)
            self._g = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _out_ptr(out, count):
    """Pointer of a caller's output buffer after checking it can take `count` float64
    values contiguously (the C call writes exactly count * 8 bytes)."""
    if hasattr(out, "data_ptr"):                     # torch tensor
        import torch
        if out.dtype != torch.float64 or not out.is_contiguous() or out.numel() != count:
            raise ValueError(f"out must be a contiguous float64 tensor of {count} elements")
        return C.c_void_p(out.data_ptr())
    if (not isinstance(out, np.ndarray) or out.dtype != np.float64
            or not out.flags["C_CONTIGUOUS"] or out.size != count):
        raise ValueError(f"out must be a C-contiguous float64 array of {count} elements")
    return C.c_void_p(out.ctypes.data)


def _res(r):
    return dict(outcome=r.outcome, iters=r.iters, rse=r.rse, rel_err=r.rel_err, seconds=r.seconds)
