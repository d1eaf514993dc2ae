# Round-2 final measurements: bench lines, launch list of the default command, ncu --set full
# of k_persistent (summarised to text on the box; large reports removed: gpurun returns
# at most 64 MiB).  usage: bash tools/gpu_final_r2.sh TAG [part: bench|ncu]
T=${1:-r2g}; PART=${2:-bench}
python __graft_entry__.py > gpurun_out/build_$T.log 2>&1 || { tail -30 gpurun_out/build_$T.log; exit 1; }
summ() {  # summarise one report to text, drop the report if large
  python tools/ncu_summary.py $1.ncu-rep > $1_summary.txt 2>&1
  python tools/ncu_lines.py $1.ncu-rep 30 > $1_lines.txt 2>&1
  [ -f $1.ncu-rep ] && [ $(stat -c %s $1.ncu-rep) -gt 8000000 ] && rm -f $1.ncu-rep
}
if [ "$PART" = "bench" ]; then
  python bench.py > gpurun_out/${T}_bench_C2c.json 2> gpurun_out/${T}_bench_C2c.err; echo bench_default=$?
  python bench.py > gpurun_out/${T}_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_default.csv python bench.py > gpurun_out/${T}_ncu_launch.log 2>&1; echo ncu_launch=$?
  for w in C1 C2i C3 C4 C5s; do
    timeout 900 python bench.py --workload $w --steps 1000 --skip-sparse > gpurun_out/${T}_bench_$w.json 2> gpurun_out/${T}_bench_$w.err; echo bench_$w=$?
  done
  timeout 2400 python bench.py --workload C5 --steps 200 --warmup 3 --skip-cpu --skip-sparse > gpurun_out/${T}_bench_C5.json 2> gpurun_out/${T}_bench_C5.err; echo bench_C5=$?
elif [ "$PART" = "ncu" ]; then
  for w in C2c C3 C4; do
    timeout 300 python tools/run_steps.py $w 4 > /dev/null 2>&1 && \
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_persistent -c 1 -o gpurun_out/prof_${T}_$w python tools/run_steps.py $w 4 > gpurun_out/ncu_${T}_$w.log 2>&1; echo ncu_$w=$?
    summ gpurun_out/prof_${T}_$w
  done
  # C5 runs the graph engine (nnz >= 2^26): its two tile kernels (pass T, pass N), and the
  # launch list of a few iterations for the kernels' shares; eager launches (RGDBEK_GRAPH=eager:
  # ncu does not profile kernels inside a graph with conditional nodes)
  export RGDBEK_GRAPH=eager
  timeout 900 python tools/run_steps.py C5c 2 > /dev/null 2>&1 && \
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_csr_tiles -c 2 -o gpurun_out/prof_${T}_C5c python tools/run_steps.py C5c 2 > gpurun_out/ncu_${T}_C5c.log 2>&1; echo ncu_C5c=$?
  summ gpurun_out/prof_${T}_C5c
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_C5c.csv python tools/run_steps.py C5c 3 > gpurun_out/ncu_${T}_C5c_launch.log 2>&1; echo ncu_C5c_launch=$?
fi
if [ "$PART" = "ncu5" ]; then                     # the C5 (graph engine) captures alone
  export RGDBEK_GRAPH=eager
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_csr_tiles -c 2 -o gpurun_out/prof_${T}_C5c python tools/run_steps.py C5c 2 > gpurun_out/ncu_${T}_C5c.log 2>&1; echo ncu_C5c=$?
  summ gpurun_out/prof_${T}_C5c
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_C5c.csv python tools/run_steps.py C5c 3 > gpurun_out/ncu_${T}_C5c_launch.log 2>&1; echo ncu_C5c_launch=$?
fi
du -sh gpurun_out
