#!/bin/bash
# Sweep the dense pass-N warp-unit count (RGDBEK_PN_UNITS) and smem staging on C2c.
mkdir -p gpurun_out
for u in 16 8 32 64 4; do
  for rep in 1 2; do
  RGDBEK_PN_UNITS=$u timeout 120 python bench.py --workload C2c --steps 2000 --warmup 5 --skip-ttt --skip-cpu --skip-e2e --skip-phases 2>/dev/null | python -c "import sys,json;d=json.loads(sys.stdin.readline());print('units',$u,d['value'],d['roofline']['frac'])" >> gpurun_out/pn_sweep.log
  done
done
RGDBEK_PN_SMEM=1 timeout 120 python bench.py --workload C2c --steps 2000 --warmup 5 --skip-ttt --skip-cpu --skip-e2e --skip-phases 2>/dev/null | python -c "import sys,json;d=json.loads(sys.stdin.readline());print('smem',d['value'],d['roofline']['frac'])" >> gpurun_out/pn_sweep.log
cat gpurun_out/pn_sweep.log
