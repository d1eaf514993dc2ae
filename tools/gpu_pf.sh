#!/bin/bash
# L2 prefetch of tile gather windows: parity with it forced on, then A/B (one process per workload).
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build_pf.log 2>&1 || { tail -30 gpurun_out/build_pf.log; exit 1; }
RGDBEK_TILE_PF=1 timeout 900 python -m pytest -x -q tests/test_gpu_parity.py tests/test_gpu_sharded.py -k "sparse or C3 or C5 or c3 or c5 or sharded" > gpurun_out/tests_pf.log 2>&1; echo tests=$?
tail -2 gpurun_out/tests_pf.log
timeout 1200 python tools/ab_pf.py C5m,C3,C4 RGDBEK_TILE_PF=0 RGDBEK_TILE_PF=T RGDBEK_TILE_PF=N RGDBEK_TILE_PF=1 --steps 300 --reps 3 > gpurun_out/ab_pf_small.jsonl 2> gpurun_out/ab_pf_small.err; echo ab_small=$?
cat gpurun_out/ab_pf_small.jsonl
timeout 1800 python tools/ab_pf.py C5c RGDBEK_TILE_PF=0 RGDBEK_TILE_PF=T RGDBEK_TILE_PF=1 --steps 40 --reps 3 > gpurun_out/ab_pf_c5.jsonl 2> gpurun_out/ab_pf_c5.err; echo ab_c5=$?
cat gpurun_out/ab_pf_c5.jsonl; tail -3 gpurun_out/ab_pf_c5.err
