#!/bin/bash
# Warp-local pass-T key batching: parity, then A/B against -DRG_WPEND=0 (group-wide list).
mkdir -p gpurun_out
timeout 900 python -m pytest -x -q tests/test_gpu_parity.py tests/test_gpu_selection_paths.py tests/test_gpu_sharded.py -k "sparse or C3 or C5 or c3 or c5 or selstress or sharded" > gpurun_out/tests_wpend.log 2>&1; echo tests=$?
tail -2 gpurun_out/tests_wpend.log
timeout 1200 python tools/ab_run.py C3,C4,C5m,C5s,C3s base build_ab/librgdbek_grouppend.so build_ab/librgdbek_warponly.so --steps 300 --reps 3 > gpurun_out/ab_wpend_small.jsonl 2> gpurun_out/ab_wpend_small.err; echo ab_small=$?
cat gpurun_out/ab_wpend_small.jsonl
