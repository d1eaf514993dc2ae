python __graft_entry__.py > gpurun_out/build_r2f.log 2>&1 || { tail -30 gpurun_out/build_r2f.log; exit 1; }
timeout 900 python -m pytest -x -q tests/test_gpu_parity.py -k "exact or greedy" > gpurun_out/tests_r2f_exact.log 2>&1; echo exact=$?
tail -5 gpurun_out/tests_r2f_exact.log
python bench.py > gpurun_out/bench_r2_default.json 2> gpurun_out/bench_r2_default.err; echo bench=$?
cat gpurun_out/bench_r2_default.json
python bench.py --mode exact --steps 20 --warmup 3 --skip-cpu --skip-e2e --skip-sparse > gpurun_out/bench_r2_exact_C2c.json 2> gpurun_out/bench_r2_exact_C2c.err; echo exact_bench=$?
cat gpurun_out/bench_r2_exact_C2c.json
