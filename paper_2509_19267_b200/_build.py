"""Build the in-tree C-ABI library librgdbek.so for sm_100a (nvcc, no JIT cache)."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "librgdbek.so")
SOURCES = ["runtime.cu"]
HEADERS = ["common.cuh", "select.cuh", "kernels.cuh", "persistent.cuh", "csr_tiles.cuh", "exact.cuh"]

NVCC_FLAGS = [
    "-O3", "-std=c++17", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC", "-shared",
    "-Xptxas", "-v",
]


# Test-only variants of the same sources (tests/test_gpu_selection_paths.py): the
# selection-stress build shrinks every candidate capacity so that all overflow and
# slow paths of the exact selection run on small systems.
VARIANTS = {
    "selstress": ["-DRG_LOCAL_SEL_MAX=64", "-DRG_LCAND_CAP=4", "-DRG_CAND_CAP=0",
                  "-DRG_FINAL_CAP=0"],
}


def variant_path(name):
    return os.path.join(HERE, f"librgdbek_{name}.so")


def _stale(lib=LIB):
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(ROOT, "include", "rgdbek.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def _nvcc(out, defines=()):
    nvcc = os.environ.get("NVCC", "nvcc")
    cmd = [nvcc, *NVCC_FLAGS, *defines, "-I", os.path.join(ROOT, "include"), "-o", out + ".tmp",
           *[os.path.join(CSRC, s) for s in SOURCES], "-ldl"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"nvcc failed building {os.path.basename(out)}")
    os.replace(out + ".tmp", out)
    return res.stderr


def build(force=False, verbose=False):
    if not force and not _stale():
        return LIB
    report = _nvcc(LIB)
    if verbose:
        sys.stderr.write(report)
    with open(os.path.join(HERE, "ptxas_report.txt"), "w") as f:
        f.write(report)
    return LIB


def build_variant(name, force=False):
    """Build a test-only variant library (VARIANTS[name]) next to librgdbek.so."""
    out = variant_path(name)
    if force or _stale(out):
        _nvcc(out, VARIANTS[name])
    return out


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
