"""Device memory of the handles (runtime.cu pool_alloc / rgdbek_destroy): every buffer comes
from the device's stream-ordered pool, so a destroyed handle's memory is reused by the next
create in the process instead of growing the footprint, and a failing allocation reports
RGDBEK_E_OOM instead of corrupting state.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    from paper_2509_19267_b200 import _build
    _build.build()


def _free_bytes():
    import torch
    torch.cuda.synchronize()
    return torch.cuda.mem_get_info()[0]


@pytest.mark.parametrize("name", ["C2s", "C3s"])
def test_create_destroy_cycles_reuse_the_pool(name):
    """Ten create / step / destroy cycles hold no more device memory than the first one
    (the pool keeps one handle's worth mapped), and every cycle's trajectory is the same."""
    from paper_2509_19267_b200 import Solver
    from workloads import by_name
    w = by_name(name)

    def make():
        if w.dense:
            return Solver(w.A, w.b, eta=w.eta)
        return Solver.from_scipy(w.A, w.b, eta=w.eta, symmetric=w.symmetric)

    s = make()
    s.reset(1)
    s.step(5)
    x0 = s.x()
    s.close()
    after_first = _free_bytes()
    for _ in range(10):
        s = make()
        s.reset(1)
        s.step(5)
        assert np.array_equal(s.x(), x0)
        s.close()
    # allow a little slack for allocator granularity / other allocations of the process
    assert _free_bytes() >= after_first - (64 << 20)


def test_oversized_create_reports_oom():
    """A dense system far beyond HBM fails cleanly with RGDBEK_E_OOM (-9): the device
    allocation fails before any copy touches the (tiny) host buffers, and the library
    stays usable afterwards."""
    import ctypes
    from paper_2509_19267_b200 import _native as N, Solver
    from workloads import by_name
    m, n = 1 << 20, 1 << 20                    # 8 TiB of fp64: cannot be allocated
    h = ctypes.c_void_p()
    opts = N.rgdbek_options_default()
    A = np.zeros(4, dtype=np.float64)
    b = np.zeros(4, dtype=np.float64)
    st = N.load().rgdbek_create_dense(ctypes.byref(h), m, n, A.ctypes.data, n,
                                      b.ctypes.data, ctypes.byref(opts))
    assert st == -9
    w = by_name("C1")
    s = Solver(w.A, w.b, eta=w.eta)
    s.reset(0)
    s.step(3)
    s.close()
