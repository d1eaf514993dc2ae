python __graft_entry__.py > gpurun_out/build_r2i.log 2>&1 || { tail -30 gpurun_out/build_r2i.log; exit 1; }
timeout 1200 python -m pytest -x -q tests/test_gpu_parity.py tests/test_gpu_sharded.py tests/test_gpu_multi_rhs.py -k "sparse or tile or c3 or c4 or C5 or c5 or sharded or multi or rhs or deblur" > gpurun_out/tests_r2i.log 2>&1; echo tests=$?
tail -3 gpurun_out/tests_r2i.log
for w in C3 C4; do timeout 900 python bench.py --workload $w --steps 1000 --skip-sparse --skip-cpu > gpurun_out/r2i_bench_$w.json 2>gpurun_out/r2i_bench_$w.err; echo bench_$w=$?; done
timeout 2400 python bench.py --workload C5 --steps 200 --warmup 3 --skip-cpu --skip-sparse > gpurun_out/r2i_bench_C5.json 2> gpurun_out/r2i_bench_C5.err; echo bench_C5=$?
grep "e2e:" gpurun_out/r2i_bench_C5.err | head -3
