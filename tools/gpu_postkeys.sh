#!/bin/bash
# Column keys after sparse pass T (grid-stride sweep) vs fused into the tile epilogue.
mkdir -p gpurun_out
timeout 1500 python -m pytest -x -q tests/test_gpu_parity.py tests/test_gpu_selection_paths.py tests/test_gpu_multi_rhs.py tests/test_gpu_engine_auto.py -k "sparse or C3 or C4 or C5 or c3 or c4 or c5 or selstress or auto or rhs" > gpurun_out/tests_postkeys.log 2>&1; echo tests=$?
tail -2 gpurun_out/tests_postkeys.log
timeout 1500 python tools/ab_run.py C3,C4,C5s,C3s,C4s base build_ab/librgdbek_fusedkeys.so --steps 300 --reps 3 > gpurun_out/ab_postkeys.jsonl 2> gpurun_out/ab_postkeys.err; echo ab=$?
cat gpurun_out/ab_postkeys.jsonl
