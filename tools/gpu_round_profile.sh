# Round profile: bench (C2c default line), launch list of the same command, ncu --set full of
# k_persistent on short runs of every workload, phase breakdowns.
# usage: bash tools/gpu_round_profile.sh TAG [workloads for ncu]
TAG=${1:-r1}; shift
NW=${@:-C2c C3 C4 C5s}
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench_exit=$?
cat gpurun_out/bench_$TAG.json
S="python bench.py --steps 50 --warmup 3 --skip-cpu --skip-e2e --skip-ttt --skip-phases"
$S > gpurun_out/short_$TAG.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $S > gpurun_out/ncu_launch_$TAG.log 2>&1; echo ncu_launch=$?
for w in $NW; do
  timeout 300 python tools/run_steps.py $w 4 > /dev/null 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_persistent -c 1 -o gpurun_out/prof_persist_${TAG}_$w python tools/run_steps.py $w 4 > gpurun_out/ncu_full_${TAG}_$w.log 2>&1; echo ncu_full_$w=$?
done
for w in C1 C2c C2i C3 C4 C5s; do timeout 300 python tools/phase_profile.py $w 200; done > gpurun_out/phases_$TAG.jsonl 2>&1
cat gpurun_out/phases_$TAG.jsonl
