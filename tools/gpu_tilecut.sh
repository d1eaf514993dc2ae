#!/bin/bash
# Batched row-pointer loads in the device tiling: parity + create timing.
mkdir -p gpurun_out
timeout 1200 python -m pytest -x -q tests/test_gpu_parity.py tests/test_gpu_sharded.py tests/test_gpu_multi_rhs.py -k "sparse or tile or C3 or C4 or C5 or c3 or c4 or c5 or sharded or rhs" > gpurun_out/tests_tilecut.log 2>&1; echo tests=$?
tail -2 gpurun_out/tests_tilecut.log
for w in C3 C4; do
  RGDBEK_CREATE_TIMING=1 timeout 600 python bench.py --workload $w --steps 1000 --skip-cpu --skip-ttt --skip-phases --skip-sparse > gpurun_out/tilecut_$w.json 2> gpurun_out/tilecut_$w.err; echo $w=$?
  grep -E "^create: tiles|^e2e:" gpurun_out/tilecut_$w.err | tail -4
  python -c "import json; d=json.loads(open('gpurun_out/tilecut_$w.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'])"
done
