#!/bin/bash
# Sparse-path check: build, GPU parity, phase profiles, short sparse bench lines,
# then one ncu --set full capture of the persistent kernel on C3 (source imported).
mkdir -p gpurun_out
python paper_2509_19267_b200/_build.py > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "sparse or fat or c3 or c5s or C3 or C4" > gpurun_out/sp_pytest.log 2>&1
rc=$?; echo "sparse pytest rc=$rc" >> gpurun_out/sp_pytest.log; tail -3 gpurun_out/sp_pytest.log
[ $rc -ne 0 ] && exit 1
rm -f gpurun_out/sp_phases.jsonl
for w in C3 C4 C5s; do timeout 300 python tools/phase_profile.py $w 300 >> gpurun_out/sp_phases.jsonl 2>&1; done
cat gpurun_out/sp_phases.jsonl
for w in C3 C4 C5s; do timeout 300 python bench.py --workload $w --steps 500 --warmup 3 --skip-cpu --skip-ttt --skip-e2e > gpurun_out/sp_bench_$w.json 2> gpurun_out/sp_bench_$w.err; python -c "
import json; d=json.loads(open('gpurun_out/sp_bench_$w.json').read().strip().splitlines()[-1]); r=d['roofline']; print('$w', d['value'], r['frac'], {k:(v['frac'], v['us_per_launch']) for k,v in r.get('standalone_kernels',{}).items()})"; done
if [ "$NCU" = 1 ]; then
timeout 300 python tools/run_steps.py ${NCU_W:-C3} 3 > gpurun_out/c3_p.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_persistent -c 1 -o gpurun_out/prof_persist_${NCU_W:-C3}_v3 python tools/run_steps.py ${NCU_W:-C3} 3 > gpurun_out/ncu_pc3.log 2>&1; echo ncu=$?
fi
