#!/bin/bash
# ncu --set full of the graph engine's k_csr_tiles (pass N / pass T) on one workload.
W=${1:-C4}
mkdir -p gpurun_out
python paper_2509_19267_b200/_build.py > gpurun_out/build.log 2>&1 || exit 1
export RGDBEK_ENGINE=graph RGDBEK_GRAPH=plain
timeout 300 python tools/run_steps.py $W 2 > gpurun_out/tiles_plain_$W.log 2>&1 || { cat gpurun_out/tiles_plain_$W.log; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_csr_tiles -s 2 -c 2 \
  -o gpurun_out/prof_tiles_$W python tools/run_steps.py $W 2 > gpurun_out/ncu_tiles_$W.log 2>&1; echo ncu=$?
