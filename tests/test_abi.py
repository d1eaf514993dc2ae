"""CPU checks of the boundary: the C-ABI library builds, loads and exports every
symbol include/rgdbek.h declares; without a GPU it fails loudly (no CPU fallback)."""
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "rgdbek.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rgdbek_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2509_19267_b200 import _build, _native
    _build.build()
    return _native.load()


def test_header_declares_the_north_star_calls():
    names = _declared()
    for must in ("rgdbek_create_csr", "rgdbek_create_dense", "rgdbek_solve", "rgdbek_step"):
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    from paper_2509_19267_b200 import _native
    so = _native.LIB_PATH
    out = subprocess.run(["nm", "-D", "--defined-only", so], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (rgdbek_[a-z0-9_]+)", out))
    missing = [n for n in _declared() if n not in exported]
    assert not missing, missing
    for n in _declared():
        assert hasattr(lib, n)
    assert set(_native.EXPORTED) == set(_declared())


def test_library_is_sm100a(lib):
    from paper_2509_19267_b200 import _native
    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_abi_version_and_defaults(lib):
    from paper_2509_19267_b200 import _native as N
    assert N.rgdbek_abi_version() == 1
    o = N.rgdbek_options_default()
    assert o.eta == 0.5 and o.stop == N.RGDBEK_STOP_RSE and o.row_begin == -1
    assert o.trace_capacity == 4096


def test_struct_layouts_match_header(lib):
    import ctypes as C
    from paper_2509_19267_b200 import _native as N
    assert C.sizeof(N.rgdbek_result) == 40
    assert C.sizeof(N.rgdbek_trace_record) == 80
    assert C.sizeof(N.rgdbek_options) == 56


@pytest.mark.skipif(os.path.exists("/dev/nvidia0"), reason="a GPU is present")
def test_no_gpu_fails_loudly(lib):
    import paper_2509_19267_b200 as P
    with pytest.raises(P.RgdbekError) as e:
        P.Solver(np.eye(4), np.ones(4))
    assert e.value.code == -7 and "no CPU fallback" in str(e.value)


def test_argument_errors_before_device(lib):
    import ctypes as C
    from paper_2509_19267_b200 import _native as N
    o = N.rgdbek_options_default()
    o.eta = 1.5
    h = C.c_void_p()
    A = np.eye(3)
    b = np.ones(3)
    code = lib.rgdbek_create_dense(C.byref(h), 3, 3, A.ctypes.data, 3, b.ctypes.data, C.byref(o))
    assert code == -1 and "eta" in N.rgdbek_last_error(None)
    code = lib.rgdbek_create_dense(C.byref(h), 3, 3, None, 3, b.ctypes.data, C.byref(o))
    assert code == -1
    o.eta = 0.5
    code = lib.rgdbek_create_dense(C.byref(h), 0, 3, A.ctypes.data, 3, b.ctypes.data, C.byref(o))
    assert code == -2


def test_product_package_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2509_19267_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f


def test_build_info_reports_the_compiled_geometry(lib):
    """rgdbek_build_info needs no device: the tile / selection geometry tests use."""
    from paper_2509_19267_b200 import _native
    info = _native.rgdbek_build_info()
    assert info["tile_nnz"] >= info["tile_rows"] > 0
    assert info["local_sel_max"] == 32768 and info["final_cap"] == 1024
    assert info["persistent_threads"] == 1024 and info["tile_group_threads"] == 256


def test_plan_ownership_host_only(lib):
    """rgdbek_plan_ownership (no device): owned-column boundaries partition [0, n); banded
    windows (strictly increasing) are split at the midpoint of each overlap, so every owned
    column lies in its owner's window; identical windows (dense A) give equal slices."""
    from paper_2509_19267_b200 import _native as N
    n = 1000
    wins = [(0, 270), (240, 520), (500, 760), (740, 1000)]
    ob = N.rgdbek_plan_ownership(wins, n)
    assert ob[0] == 0 and ob[-1] == n and all(ob[i] <= ob[i + 1] for i in range(4))
    for r, (lo, hi) in enumerate(wins):
        assert lo <= ob[r] and ob[r + 1] <= hi, (r, ob)
    assert ob[1] == (240 + 270) // 2
    assert N.rgdbek_plan_ownership([(0, n)] * 4, n) == [0, 250, 500, 750, 1000]
    assert N.rgdbek_plan_ownership([(0, n)], n) == [0, n]
