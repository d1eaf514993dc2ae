#!/bin/bash
# Early buffer release for one-row-per-warp tiles: parity, then A/B against -DRG_EARLY_REL=0.
mkdir -p gpurun_out
timeout 900 python -m pytest -x -q tests/test_gpu_parity.py tests/test_gpu_selection_paths.py -k "sparse or C3 or C5 or c3 or c5 or selstress" > gpurun_out/tests_early.log 2>&1; echo tests=$?
tail -2 gpurun_out/tests_early.log
timeout 900 python tools/ab_pass.py C5m,C5s,C3,C4 base build_ab/librgdbek_noearly.so --reps 3 > gpurun_out/ab_early_small.jsonl 2> gpurun_out/ab_early_small.err; echo ab_small=$?
cat gpurun_out/ab_early_small.jsonl
timeout 2400 python tools/ab_run.py C5c base build_ab/librgdbek_noearly.so --steps 40 --reps 2 > gpurun_out/ab_early_c5.jsonl 2> gpurun_out/ab_early_c5.err; echo ab_c5=$?
cat gpurun_out/ab_early_c5.jsonl
