#!/bin/bash
# Launch list of the graph engine on C3 / C4 (eager launches so ncu sees every kernel).
mkdir -p gpurun_out
export RGDBEK_ENGINE=graph RGDBEK_GRAPH=eager
for w in C3 C4; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/graph_launches_$w.csv python tools/run_steps.py $w 4 > gpurun_out/graph_launch_$w.log 2>&1; echo $w=$?
  python tools/launch_shares.py gpurun_out/graph_launches_$w.csv | head -30
done
