# Bench every workload once (N=1).  usage: bash tools/gpu_bench_all.sh TAG [workloads...]
TAG=${1:-r1}; shift
WL=${@:-C1 C2c C2i C3 C4 C5s}
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
for w in $WL; do
  timeout 900 python bench.py --workload $w --steps ${STEPS:-1000} --cpu-budget 15 > gpurun_out/bench_${TAG}_$w.json 2> gpurun_out/bench_${TAG}_$w.err
  echo "$w exit=$?"; cat gpurun_out/bench_${TAG}_$w.json; tail -2 gpurun_out/bench_${TAG}_$w.err
done
