#!/bin/bash
# Quick GPU check: build, C1 bench (e2e breakdown on stderr), phase profiles.
mkdir -p gpurun_out
python paper_2509_19267_b200/_build.py > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 300 python bench.py --workload C1 --steps 1000 --warmup 3 --skip-ttt > gpurun_out/q_C1.json 2> gpurun_out/q_C1.err
for w in ${@:-C2c C3}; do timeout 300 python tools/phase_profile.py $w 300 >> gpurun_out/q_phases.jsonl 2>&1; done
cat gpurun_out/q_C1.json; grep e2e gpurun_out/q_C1.err; cat gpurun_out/q_phases.jsonl
