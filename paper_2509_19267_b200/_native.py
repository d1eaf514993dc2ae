"""ctypes binding of include/rgdbek.h — argument marshalling only.

Every function here has the name of the C entry point it calls.  No step of
the method runs in Python: if librgdbek.so is missing or cannot find an
sm_100 GPU, the calls fail loudly (there is no CPU fallback).
"""
import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "librgdbek.so")

RGDBEK_OK = 0
STATUS_NAMES = {0: "OK", -1: "E_ARG", -2: "E_DIM", -3: "E_CSR", -4: "E_ZERO_RHS",
                -5: "E_NONFINITE", -6: "E_STATE", -7: "E_CUDA", -8: "E_NCCL", -9: "E_OOM",
                -10: "E_INTERNAL"}
RGDBEK_CONVERGED, RGDBEK_MAX_ITER, RGDBEK_STALLED = 0, 2, 3
RGDBEK_STOP_RSE, RGDBEK_STOP_REL_ERR, RGDBEK_STOP_NONE = 0, 1, 2

EXPORTED = [
    "rgdbek_abi_version", "rgdbek_options_default", "rgdbek_create_csr", "rgdbek_create_dense",
    "rgdbek_reset", "rgdbek_step", "rgdbek_solve", "rgdbek_set_stop", "rgdbek_set_reference",
    "rgdbek_get_x", "rgdbek_get_z", "rgdbek_get_blocks", "rgdbek_get_trace", "rgdbek_set_state",
    "rgdbek_launch_kernel", "rgdbek_launches_per_iteration", "rgdbek_stream",
    "rgdbek_phase_times", "rgdbek_engine_info", "rgdbek_set_mode", "rgdbek_get_counters",
    "rgdbek_set_selection", "rgdbek_set_lazy", "rgdbek_set_capture", "rgdbek_selection_stats",
    "rgdbek_build_info", "rgdbek_get_a_bytes", "rgdbek_plan_ownership", "rgdbek_peer_window", "rgdbek_group_create",
    "rgdbek_group_reset", "rgdbek_group_step", "rgdbek_group_solve", "rgdbek_group_destroy",
    "rgdbek_peer_export", "rgdbek_peer_connect", "rgdbek_create_csr_multi", "rgdbek_rhs_count",
    "rgdbek_get_x_rhs", "rgdbek_get_z_rhs", "rgdbek_set_reference_rhs", "rgdbek_get_trace_rhs",
    "rgdbek_nccl_unique_id", "rgdbek_nccl_comm_init", "rgdbek_nccl_comm_destroy",
    "rgdbek_last_error", "rgdbek_destroy",
]


class rgdbek_options(C.Structure):
    _fields_ = [("eta", C.c_double), ("stop", C.c_int32), ("device", C.c_int32),
                ("stream", C.c_void_p), ("nccl_comm", C.c_void_p),
                ("row_begin", C.c_int64), ("row_end", C.c_int64),
                ("symmetric", C.c_int32), ("trace_capacity", C.c_int32)]


class rgdbek_result(C.Structure):
    _fields_ = [("outcome", C.c_int32), ("pad_", C.c_int32), ("iters", C.c_int64),
                ("rse", C.c_double), ("rel_err", C.c_double), ("seconds", C.c_double)]


class rgdbek_trace_record(C.Structure):
    _fields_ = [("k", C.c_int64), ("kp", C.c_int64), ("hash_u", C.c_uint64),
                ("Z", C.c_double), ("W", C.c_double), ("kpp", C.c_int64),
                ("hash_j", C.c_uint64), ("X", C.c_double), ("V", C.c_double),
                ("rse", C.c_double)]


class RgdbekError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"rgdbek {STATUS_NAMES.get(code, code)} ({code}): {msg}")
        self.code = code


_lib = None


def load(path=None):
    """Load librgdbek.so (in-tree).  Raises if it is missing: no fallback."""
    global _lib
    if _lib is not None:
        return _lib
    # RGDBEK_LIB: an explicitly built variant of the library (tools/ab_variants.py)
    path = path or os.environ.get("RGDBEK_LIB") or LIB_PATH
    if not os.path.exists(path):
        raise RuntimeError(f"{path} is missing: build it with __graft_entry__.build() "
                           "(there is no CPU fallback)")
    lib = C.CDLL(path, mode=C.RTLD_GLOBAL)
    H = C.c_void_p
    P = C.c_void_p
    sig = {
        "rgdbek_abi_version": (C.c_int32, []),
        "rgdbek_options_default": (None, [C.POINTER(rgdbek_options)]),
        "rgdbek_create_csr": (C.c_int, [C.POINTER(H), C.c_int64, C.c_int64, C.c_int64, P, P, P, P,
                                        C.POINTER(rgdbek_options)]),
        "rgdbek_create_dense": (C.c_int, [C.POINTER(H), C.c_int64, C.c_int64, P, C.c_int64, P,
                                          C.POINTER(rgdbek_options)]),
        "rgdbek_reset": (C.c_int, [H, C.c_uint64]),
        "rgdbek_step": (C.c_int, [H, C.c_int64, C.POINTER(rgdbek_result)]),
        "rgdbek_solve": (C.c_int, [H, C.c_double, C.c_int64, C.c_uint64, C.POINTER(rgdbek_result)]),
        "rgdbek_set_stop": (C.c_int, [H, C.c_int32]),
        "rgdbek_set_reference": (C.c_int, [H, P]),
        "rgdbek_get_x": (C.c_int, [H, P]),
        "rgdbek_get_z": (C.c_int, [H, P]),
        "rgdbek_get_blocks": (C.c_int, [H, C.POINTER(C.c_int64), C.POINTER(C.c_uint64), P,
                                        C.POINTER(C.c_int64), C.POINTER(C.c_uint64), P]),
        "rgdbek_get_trace": (C.c_int, [H, C.POINTER(rgdbek_trace_record), C.c_int64,
                                       C.POINTER(C.c_int64)]),
        "rgdbek_set_state": (C.c_int, [H, P, P, C.c_int64]),
        "rgdbek_launch_kernel": (C.c_int, [H, C.c_int32, C.c_int32, C.POINTER(C.c_double)]),
        "rgdbek_launches_per_iteration": (C.c_int, [H, C.POINTER(C.c_int64)]),
        "rgdbek_stream": (C.c_void_p, [H]),
        "rgdbek_phase_times": (C.c_int, [H, C.POINTER(C.c_double), C.c_int32,
                                         C.POINTER(C.c_int32)]),
        "rgdbek_engine_info": (C.c_int, [H, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
        "rgdbek_set_mode": (C.c_int, [H, C.c_int32, C.c_double, C.c_int32]),
        "rgdbek_get_counters": (C.c_int, [H, C.POINTER(C.c_int64)]),
        "rgdbek_get_a_bytes": (C.c_int, [H, C.POINTER(C.c_double)]),
        "rgdbek_set_selection": (C.c_int, [H, C.c_int32]),
        "rgdbek_set_lazy": (C.c_int, [H, C.c_int32]),
        "rgdbek_set_capture": (C.c_int, [H, C.c_int32]),
        "rgdbek_selection_stats": (C.c_int, [H, C.POINTER(C.c_int64)]),
        "rgdbek_build_info": (C.c_int32, [C.POINTER(C.c_int32), C.c_int32]),
        "rgdbek_plan_ownership": (C.c_int, [C.c_int32, C.POINTER(C.c_int64), C.c_int64,
                                            C.POINTER(C.c_int64)]),
        "rgdbek_peer_window": (C.c_int, [H, C.POINTER(C.c_int64)]),
        "rgdbek_group_create": (C.c_int, [C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), C.c_int32]),
        "rgdbek_group_reset": (C.c_int, [C.c_void_p, C.c_uint64]),
        "rgdbek_group_step": (C.c_int, [C.c_void_p, C.c_int64, C.POINTER(rgdbek_result)]),
        "rgdbek_group_solve": (C.c_int, [C.c_void_p, C.c_double, C.c_int64, C.c_uint64,
                                         C.POINTER(rgdbek_result)]),
        "rgdbek_group_destroy": (None, [C.c_void_p]),
        "rgdbek_peer_export": (C.c_int, [H, P]),
        "rgdbek_create_csr_multi": (C.c_int, [C.POINTER(H), C.c_int64, C.c_int64, C.c_int64, P, P, P,
                                              P, C.c_int32, C.POINTER(rgdbek_options)]),
        "rgdbek_rhs_count": (C.c_int32, [H]),
        "rgdbek_get_x_rhs": (C.c_int, [H, C.c_int32, P]),
        "rgdbek_get_z_rhs": (C.c_int, [H, C.c_int32, P]),
        "rgdbek_set_reference_rhs": (C.c_int, [H, C.c_int32, P]),
        "rgdbek_get_trace_rhs": (C.c_int, [H, C.c_int32, C.POINTER(rgdbek_trace_record), C.c_int64,
                                           C.POINTER(C.c_int64)]),
        "rgdbek_peer_connect": (C.c_int, [H, C.c_int32, C.c_int32, P, C.POINTER(C.c_int64)]),
        "rgdbek_nccl_unique_id": (C.c_int, [P]),
        "rgdbek_nccl_comm_init": (C.c_int, [C.POINTER(C.c_void_p), C.c_int32, C.c_int32, P,
                                            C.c_int32]),
        "rgdbek_nccl_comm_destroy": (C.c_int, [C.c_void_p]),
        "rgdbek_last_error": (C.c_char_p, [H]),
        "rgdbek_destroy": (None, [H]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def check(code, handle=None):
    if code != RGDBEK_OK:
        lib = load()
        msg = lib.rgdbek_last_error(handle)
        raise RgdbekError(code, msg.decode() if msg else "")
    return code


# ---- thin wrappers with the C names ------------------------------------------------

def rgdbek_abi_version():
    return load().rgdbek_abi_version()


def rgdbek_options_default():
    o = rgdbek_options()
    load().rgdbek_options_default(C.byref(o))
    return o


def rgdbek_create_dense(m, n, A_ptr, lda, b_ptr, opts):
    h = C.c_void_p()
    check(load().rgdbek_create_dense(C.byref(h), m, n, A_ptr, lda, b_ptr, C.byref(opts)), None)
    return h


def rgdbek_create_csr(m, n, nnz, row_ptr, col_idx, val, b_ptr, opts):
    h = C.c_void_p()
    check(load().rgdbek_create_csr(C.byref(h), m, n, nnz, row_ptr, col_idx, val, b_ptr,
                                   C.byref(opts)), None)
    return h


def rgdbek_create_csr_multi(m, n, nnz, row_ptr, col_idx, val, b_all, nrhs, opts):
    h = C.c_void_p()
    check(load().rgdbek_create_csr_multi(C.byref(h), m, n, nnz, row_ptr, col_idx, val, b_all, nrhs,
                                         C.byref(opts)), None)
    return h


def rgdbek_rhs_count(h):
    return load().rgdbek_rhs_count(h)


def rgdbek_get_x_rhs(h, rhs, out_ptr):
    check(load().rgdbek_get_x_rhs(h, rhs, out_ptr), h)


def rgdbek_get_z_rhs(h, rhs, out_ptr):
    check(load().rgdbek_get_z_rhs(h, rhs, out_ptr), h)


def rgdbek_set_reference_rhs(h, rhs, ptr):
    check(load().rgdbek_set_reference_rhs(h, rhs, ptr), h)


def rgdbek_get_trace_rhs(h, rhs, max_records):
    buf = (rgdbek_trace_record * max(int(max_records), 1))()
    cnt = C.c_int64()
    check(load().rgdbek_get_trace_rhs(h, rhs, buf, max_records, C.byref(cnt)), h)
    return [buf[i] for i in range(cnt.value)]


def rgdbek_reset(h, seed):
    check(load().rgdbek_reset(h, seed), h)


def rgdbek_step(h, n_iter):
    r = rgdbek_result()
    check(load().rgdbek_step(h, n_iter, C.byref(r)), h)
    return r


def rgdbek_solve(h, tol, max_iter, seed):
    r = rgdbek_result()
    check(load().rgdbek_solve(h, tol, max_iter, seed, C.byref(r)), h)
    return r


def rgdbek_set_stop(h, mode):
    check(load().rgdbek_set_stop(h, mode), h)


def rgdbek_set_reference(h, xstar_ptr):
    check(load().rgdbek_set_reference(h, xstar_ptr), h)


def rgdbek_get_x(h, out_ptr):
    check(load().rgdbek_get_x(h, out_ptr), h)


def rgdbek_get_z(h, out_ptr):
    check(load().rgdbek_get_z(h, out_ptr), h)


def rgdbek_get_blocks(h, U_ptr=None, J_ptr=None):
    nu, nj = C.c_int64(), C.c_int64()
    hu, hj = C.c_uint64(), C.c_uint64()
    check(load().rgdbek_get_blocks(h, C.byref(nu), C.byref(hu), U_ptr, C.byref(nj), C.byref(hj),
                                   J_ptr), h)
    return nu.value, hu.value, nj.value, hj.value


def rgdbek_get_trace(h, max_records):
    buf = (rgdbek_trace_record * max(int(max_records), 1))()
    cnt = C.c_int64()
    check(load().rgdbek_get_trace(h, buf, max_records, C.byref(cnt)), h)
    return [buf[i] for i in range(cnt.value)]


def rgdbek_set_state(h, x_ptr, z_ptr, k):
    check(load().rgdbek_set_state(h, x_ptr, z_ptr, k), h)


def rgdbek_launch_kernel(h, kernel, reps):
    b = C.c_double()
    check(load().rgdbek_launch_kernel(h, kernel, reps, C.byref(b)), h)
    return b.value


def rgdbek_launches_per_iteration(h):
    v = C.c_int64()
    check(load().rgdbek_launches_per_iteration(h, C.byref(v)), h)
    return v.value


def rgdbek_stream(h):
    return load().rgdbek_stream(h)


def rgdbek_phase_times(h):
    buf = (C.c_double * 24)()
    cnt = C.c_int32()
    check(load().rgdbek_phase_times(h, buf, 24, C.byref(cnt)), h)
    return [buf[i] for i in range(cnt.value)]


def rgdbek_set_mode(h, mode, inner_tol=1e-12, inner_max=50):
    check(load().rgdbek_set_mode(h, int(mode), float(inner_tol), int(inner_max)), h)


def rgdbek_set_selection(h, selection):
    check(load().rgdbek_set_selection(h, int(selection)), h)


def rgdbek_set_lazy(h, processes):
    check(load().rgdbek_set_lazy(h, int(processes)), h)


def rgdbek_set_capture(h, enable):
    check(load().rgdbek_set_capture(h, int(enable)), h)


def rgdbek_selection_stats(h):
    buf = (C.c_int64 * 4)()
    check(load().rgdbek_selection_stats(h, buf), h)
    return [buf[i] for i in range(4)]


def rgdbek_build_info():
    lib = load()
    cnt = lib.rgdbek_build_info(None, 0)
    buf = (C.c_int32 * cnt)()
    lib.rgdbek_build_info(buf, cnt)
    keys = ["tile_nnz", "tile_rows", "local_sel_max", "lcand_cap", "cand_cap", "final_cap",
            "persistent_threads", "tile_group_threads"]
    return dict(zip(keys, [buf[i] for i in range(cnt)]))


PEER_HANDLE_BYTES = 64


def rgdbek_plan_ownership(windows, n):
    """Owned-column boundaries [R + 1] for rank windows [(lo, hi), ...] (host-only call)."""
    R = len(windows)
    w = (C.c_int64 * (2 * R))(*[int(v) for lohi in windows for v in lohi])
    ob = (C.c_int64 * (R + 1))()
    check(load().rgdbek_plan_ownership(R, w, int(n), ob), None)
    return [ob[i] for i in range(R + 1)]


def rgdbek_peer_window(h):
    out = (C.c_int64 * 4)()
    check(load().rgdbek_peer_window(h, out), h)
    return [out[i] for i in range(4)]


def rgdbek_group_create(handles):
    arr = (C.c_void_p * len(handles))(*[h.value if isinstance(h, C.c_void_p) else h for h in handles])
    g = C.c_void_p()
    check(load().rgdbek_group_create(C.byref(g), arr, len(handles)), None)
    return g


def rgdbek_group_reset(g, seed, h0=None):
    check(load().rgdbek_group_reset(g, seed), h0)


def rgdbek_group_step(g, n_iter, h0=None):
    r = rgdbek_result()
    check(load().rgdbek_group_step(g, n_iter, C.byref(r)), h0)
    return r


def rgdbek_group_solve(g, tol, max_iter, seed, h0=None):
    r = rgdbek_result()
    check(load().rgdbek_group_solve(g, tol, max_iter, seed, C.byref(r)), h0)
    return r


def rgdbek_group_destroy(g):
    load().rgdbek_group_destroy(g)


def rgdbek_peer_export(h):
    buf = (C.c_char * PEER_HANDLE_BYTES)()
    check(load().rgdbek_peer_export(h, buf), h)
    return bytes(buf)


def rgdbek_peer_connect(h, nranks, rank, handles, windows):
    hb = (C.c_char * (PEER_HANDLE_BYTES * nranks)).from_buffer_copy(b"".join(handles))
    w = (C.c_int64 * (2 * nranks))(*[int(v) for lohi in windows for v in lohi])
    check(load().rgdbek_peer_connect(h, nranks, rank, hb, w), h)


def rgdbek_get_counters(h):
    v = C.c_int64()
    check(load().rgdbek_get_counters(h, C.byref(v)), h)
    return v.value


def rgdbek_get_a_bytes(h):
    v = C.c_double()
    check(load().rgdbek_get_a_bytes(h, C.byref(v)), h)
    return v.value


def rgdbek_engine_info(h):
    e, c = C.c_int32(), C.c_int32()
    check(load().rgdbek_engine_info(h, C.byref(e), C.byref(c)), h)
    return e.value, c.value


def rgdbek_nccl_unique_id():
    buf = (C.c_char * 128)()
    check(load().rgdbek_nccl_unique_id(buf), None)
    return bytes(buf)


def rgdbek_nccl_comm_init(nranks, rank, uid, device):
    comm = C.c_void_p()
    idb = (C.c_char * 128).from_buffer_copy(uid)
    check(load().rgdbek_nccl_comm_init(C.byref(comm), nranks, rank, idb, device), None)
    return comm


def rgdbek_nccl_comm_destroy(comm):
    check(load().rgdbek_nccl_comm_destroy(comm), None)


def rgdbek_last_error(h=None):
    m = load().rgdbek_last_error(h)
    return m.decode() if m else ""


def rgdbek_destroy(h):
    load().rgdbek_destroy(h)
