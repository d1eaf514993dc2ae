# One GPU call: build, parity subset, bench (C2c), launch list (plain graph), ncu of a hot kernel.
# usage: bash tools/gpu_profile_dense.sh <kernel-regex> [tag]
K=${1:-k_dense_passN}
TAG=${2:-r1}
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { echo build failed; tail gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo tests_exit=$?; tail -3 gpurun_out/gpu_tests.log
python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench_exit=$?
cat gpurun_out/bench_$TAG.json
S="python bench.py --steps 5 --warmup 3 --skip-cpu --skip-e2e --skip-ttt"
export RGDBEK_GRAPH=plain
$S > gpurun_out/bench_short.json 2> gpurun_out/bench_short.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $S > gpurun_out/ncu_launches.log 2>&1; echo ncu1=$?
ncu --set full --clock-control none --import-source on -k regex:$K -s ${SKIP:-30} -c 1 -o gpurun_out/prof_$TAG $S > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?
