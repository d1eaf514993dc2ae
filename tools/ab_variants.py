"""Build A/B variants of librgdbek.so with -D overrides (experiments only).

usage: python tools/ab_variants.py NAME "-DRG_TBUF=2 -DRG_PEND=128" [NAME2 "FLAGS2" ...]
Writes build_ab/librgdbek_NAME.so; load one with RGDBEK_LIB=<path>.
"""
import os
import shlex
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2509_19267_b200 import _build as B  # noqa: E402


def main():
    args = sys.argv[1:]
    os.makedirs(os.path.join(ROOT, "build_ab"), exist_ok=True)
    for name, flags in zip(args[0::2], args[1::2]):
        out = os.path.join(ROOT, "build_ab", f"librgdbek_{name}.so")
        cmd = [os.environ.get("NVCC", "nvcc"), *B.NVCC_FLAGS, *shlex.split(flags), "-I",
               os.path.join(ROOT, "include"), "-o", out,
               *[os.path.join(B.CSRC, s) for s in B.SOURCES], "-ldl"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode:
            sys.stderr.write(res.stderr)
            raise SystemExit(f"variant {name} failed")
        print(out)


if __name__ == "__main__":
    main()
