#!/bin/bash
# End-of-round check: build, full GPU suite, smoke, default bench line.
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build_fc.log 2>&1 || { tail -30 gpurun_out/build_fc.log; exit 1; }
timeout 3000 python -m pytest -q -m gpu tests > gpurun_out/tests_fc.log 2>&1; echo tests=$?
tail -3 gpurun_out/tests_fc.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_fc.log 2>&1; echo smoke=$?
tail -2 gpurun_out/smoke_fc.log
timeout 900 python bench.py > gpurun_out/bench_fc.json 2> gpurun_out/bench_fc.err; echo bench=$?
python -c "
import json; d=json.loads(open('gpurun_out/bench_fc.json').read().strip().splitlines()[-1])
print(d['value'], d['roofline']['frac'], d['e2e']['value'], d['clocks'], d['sparse']['value'], d['sparse']['multi_rhs']['rhs_iterations_per_s'], d['cpu_baseline']['value'])"
