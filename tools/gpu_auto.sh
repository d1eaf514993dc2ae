#!/bin/bash
# Automatic engine choice (graph engine for nnz >= 2^26, 2-deep rings in its tile kernel):
# tests, then the C5 bench line on the new default.
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build_auto.log 2>&1 || { tail -30 gpurun_out/build_auto.log; exit 1; }
timeout 1500 python -m pytest -x -q tests/test_gpu_engine_auto.py tests/test_gpu_parity.py tests/test_gpu_selection_paths.py -k "engine or auto or graph or sparse or selstress or nccl or world" > gpurun_out/tests_auto.log 2>&1; echo tests=$?
tail -3 gpurun_out/tests_auto.log
timeout 1500 python tools/ab_run.py C3,C4 base "env:RGDBEK_ENGINE=graph" --steps 300 --reps 2 > gpurun_out/ab_auto_small.jsonl 2>&1; echo ab=$?
cat gpurun_out/ab_auto_small.jsonl
timeout 2400 python bench.py --workload C5 --steps 200 --warmup 3 --skip-cpu --skip-sparse > gpurun_out/auto_bench_C5.json 2> gpurun_out/auto_bench_C5.err; echo bench_C5=$?
python -c "
import json; d=json.loads(open('gpurun_out/auto_bench_C5.json').read().strip().splitlines()[-1])
print({k: d.get(k) for k in ('value','ms_per_step','gpu_launches')}, d['config'].get('engine'), {k: d['roofline'].get(k) for k in ('kernel','frac','iteration_frac')}, d['roofline'].get('standalone_kernels'), d.get('e2e'))"
