#!/bin/bash
# Speculative column level 2 in the sparse persistent kernel: parity (incl. the selection-stress
# build, whose tiny LOCAL_SEL_MAX sends every system through the grid-wide path), then A/B.
mkdir -p gpurun_out
timeout 1500 python -m pytest -x -q tests/test_gpu_parity.py tests/test_gpu_selection_paths.py tests/test_gpu_multi_rhs.py -k "sparse or C3 or C4 or C5 or c3 or c4 or c5 or selstress or tile or engines" > gpurun_out/tests_specu.log 2>&1; echo tests=$?
tail -2 gpurun_out/tests_specu.log
timeout 1500 python tools/ab_run.py C3,C4,C3s,C5s base build_ab/librgdbek_nospecu.so --steps 300 --reps 3 > gpurun_out/ab_specu.jsonl 2> gpurun_out/ab_specu.err; echo ab=$?
cat gpurun_out/ab_specu.jsonl
