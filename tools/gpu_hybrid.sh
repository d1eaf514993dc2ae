#!/bin/bash
# Hybrid engine: parity (engine tests + sparse 50-iteration runs under RGDBEK_ENGINE=hybrid), then A/B.
mkdir -p gpurun_out
timeout 600 python -m pytest -x -q tests/test_gpu_parity.py -k "engines_and_grid" > gpurun_out/tests_hyb.log 2>&1; echo tests_engines=$?
tail -3 gpurun_out/tests_hyb.log
RGDBEK_ENGINE=hybrid timeout 900 python -m pytest -x -q tests/test_gpu_parity.py -k "sparse or C3 or C4 or c3 or c4 or tile" > gpurun_out/tests_hyb2.log 2>&1; echo tests_sparse_hybrid=$?
tail -3 gpurun_out/tests_hyb2.log
timeout 1500 python tools/ab_run.py C3,C4,C5m,C5s base "env:RGDBEK_ENGINE=hybrid" "env:RGDBEK_ENGINE=graph" --steps 300 --reps 2 > gpurun_out/ab_hyb.jsonl 2> gpurun_out/ab_hyb.err; echo ab=$?
cat gpurun_out/ab_hyb.jsonl; tail -3 gpurun_out/ab_hyb.err
