#!/bin/bash
# Stream-ordered pool allocation: full GPU suite, then the e2e create breakdown on C4 / C5s.
mkdir -p gpurun_out
timeout 3000 python -m pytest -q -m gpu tests > gpurun_out/tests_pool.log 2>&1; echo tests=$?
tail -3 gpurun_out/tests_pool.log
for w in C4 C5s C4; do
  RGDBEK_CREATE_TIMING=1 timeout 600 python bench.py --workload $w --steps 300 --skip-cpu --skip-ttt --skip-phases --skip-sparse > gpurun_out/pool_$w.json 2> gpurun_out/pool_$w.err; echo $w=$?
  grep -E "^e2e:" gpurun_out/pool_$w.err
  python -c "import json; d=json.loads(open('gpurun_out/pool_$w.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'])"
done
