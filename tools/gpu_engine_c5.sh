#!/bin/bash
# Engine choice on the largest system: persistent vs graph (3- and 2-deep tile rings).
mkdir -p gpurun_out
timeout 3000 python tools/ab_run.py C5c,C5m base "env:RGDBEK_ENGINE=graph" "build_ab/librgdbek_tbuf2.so|RGDBEK_ENGINE=graph" --steps 40 --reps 2 > gpurun_out/ab_engine_c5.jsonl 2> gpurun_out/ab_engine_c5.err; echo ab=$?
cat gpurun_out/ab_engine_c5.jsonl; tail -3 gpurun_out/ab_engine_c5.err
