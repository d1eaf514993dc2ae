#!/bin/bash
# Build librgdbek.so from a git revision into build_ab/librgdbek_NAME.so (A/B baseline).
# usage: bash tools/build_rev.sh REV NAME
REV=${1:-HEAD}; NAME=${2:-head}
ROOT=$(cd "$(dirname "$0")/.." && pwd)
WT=$(mktemp -d /tmp/rg_wt_XXXX)
git -C "$ROOT" worktree add -f "$WT" "$REV" -q || exit 1
mkdir -p "$ROOT/build_ab"
(cd "$WT" && nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC \
   -shared -I include -o "$ROOT/build_ab/librgdbek_$NAME.so" paper_2509_19267_b200/csrc/runtime.cu -ldl)
rc=$?
git -C "$ROOT" worktree remove --force "$WT"
exit $rc
