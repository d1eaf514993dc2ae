#!/bin/bash
# Create-time phase breakdown (RGDBEK_CREATE_TIMING) through the bench's e2e path.
mkdir -p gpurun_out
for w in C4 C4; do
  RGDBEK_CREATE_TIMING=1 timeout 600 python bench.py --workload $w --steps 300 --skip-cpu --skip-ttt --skip-phases --skip-sparse > gpurun_out/create_$w.json 2> gpurun_out/create_$w.err; echo $w=$?
  grep -E "^create:|^e2e:" gpurun_out/create_$w.err | head -40
done
