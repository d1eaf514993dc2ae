#!/bin/bash
# Graph-engine vector kernels with 4 loads in flight per thread: parity (graph engine) + C5 A/B.
mkdir -p gpurun_out
timeout 900 python -m pytest -x -q tests/test_gpu_parity.py tests/test_gpu_selection_paths.py tests/test_gpu_engine_auto.py -k "engine or graph or auto or selstress or nccl" > gpurun_out/tests_unroll.log 2>&1; echo tests=$?
tail -2 gpurun_out/tests_unroll.log
timeout 2400 python tools/ab_run.py C5c,C5m base build_ab/librgdbek_prev.so --steps 40 --reps 2 > gpurun_out/ab_unroll.jsonl 2> gpurun_out/ab_unroll.err; echo ab=$?
cat gpurun_out/ab_unroll.jsonl
