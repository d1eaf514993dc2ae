python __graft_entry__.py > gpurun_out/build_r2d.log 2>&1 || { tail -30 gpurun_out/build_r2d.log; exit 1; }
timeout 900 python -m pytest -x -q tests/test_gpu_sharded.py > gpurun_out/tests_r2d_sharded.log 2>&1; echo sharded=$?
tail -30 gpurun_out/tests_r2d_sharded.log
timeout 600 python -m pytest -x -q tests/test_gpu_parity.py -k "sparse or tile or c5s or engines" > gpurun_out/tests_r2d_sparse.log 2>&1; echo sparse=$?
tail -5 gpurun_out/tests_r2d_sparse.log
