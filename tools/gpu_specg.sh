#!/bin/bash
# Speculative level 2 in the graph engine (C5's engine): parity, then A/B on C5c / C5m.
mkdir -p gpurun_out
timeout 1500 python -m pytest -x -q tests/test_gpu_parity.py tests/test_gpu_selection_paths.py tests/test_gpu_engine_auto.py -k "engine or graph or auto or selstress or nccl or world" > gpurun_out/tests_specg.log 2>&1; echo tests=$?
tail -2 gpurun_out/tests_specg.log
RGDBEK_ENGINE=graph timeout 1500 python -m pytest -x -q tests/test_gpu_parity.py -k "sparse_50 or C5t or c5t or time_to" > gpurun_out/tests_specg2.log 2>&1; echo tests_graph=$?
tail -2 gpurun_out/tests_specg2.log
timeout 2400 python tools/ab_run.py C5c,C5m base build_ab/librgdbek_head2.so --steps 40 --reps 2 > gpurun_out/ab_specg.jsonl 2> gpurun_out/ab_specg.err; echo ab=$?
cat gpurun_out/ab_specg.jsonl
