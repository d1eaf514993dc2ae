#!/bin/bash
# Graph-engine tile kernel: committed tree vs pending-list-free smem vs register budgets.
mkdir -p gpurun_out
timeout 1200 python tools/ab_pass.py C5m,C4 build_ab/librgdbek_head.so build_ab/librgdbek_nolb.so build_ab/librgdbek_gtb5.so base --reps 2 > gpurun_out/ab_gtb_pass.jsonl 2> gpurun_out/ab_gtb_pass.err; echo ab_pass=$?
cat gpurun_out/ab_gtb_pass.jsonl
timeout 2400 python tools/ab_run.py C5c build_ab/librgdbek_head.so build_ab/librgdbek_nolb.so build_ab/librgdbek_gtb5.so --steps 40 --reps 2 > gpurun_out/ab_gtb_c5.jsonl 2> gpurun_out/ab_gtb_c5.err; echo ab_c5=$?
cat gpurun_out/ab_gtb_c5.jsonl
