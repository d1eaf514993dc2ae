# Round-2 baseline: ncu --set full of k_persistent on the sparse configs (final r1 tree),
# plus per-phase device times.  usage: bash tools/gpu_ncu_r2.sh TAG [workloads]
TAG=${1:-r2a}; shift
NW=${@:-C3 C4 C5c}
python __graft_entry__.py > gpurun_out/build_$TAG.log 2>&1 || { tail gpurun_out/build_$TAG.log; exit 1; }
for w in $NW; do
  timeout 300 python tools/phase_profile.py $w 100 >> gpurun_out/phases_$TAG.jsonl 2>&1
done
cat gpurun_out/phases_$TAG.jsonl
for w in $NW; do
  K=4; [ "$w" = "C5c" ] && K=2
  timeout 600 python tools/run_steps.py $w $K > gpurun_out/plain_${TAG}_$w.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_persistent -c 1 \
     -o gpurun_out/prof_${TAG}_$w python tools/run_steps.py $w $K > gpurun_out/ncu_${TAG}_$w.log 2>&1
  echo ncu_$w=$?
done
