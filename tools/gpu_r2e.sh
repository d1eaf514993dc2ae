python __graft_entry__.py > gpurun_out/build_r2e.log 2>&1 || { tail -30 gpurun_out/build_r2e.log; exit 1; }
timeout 900 python -m pytest -x -q tests/test_gpu_multi_rhs.py > gpurun_out/tests_r2e_multi.log 2>&1; echo multi=$?
tail -30 gpurun_out/tests_r2e_multi.log
