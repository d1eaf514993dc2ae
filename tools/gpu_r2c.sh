python __graft_entry__.py > gpurun_out/build_r2c.log 2>&1 || { tail -30 gpurun_out/build_r2c.log; exit 1; }
timeout 600 python -m pytest -x -q tests/test_gpu_sharded.py > gpurun_out/tests_r2c_sharded.log 2>&1; echo sharded=$?
tail -30 gpurun_out/tests_r2c_sharded.log
timeout 1200 python -m pytest -x -q -m gpu tests --deselect tests/test_gpu_sharded.py > gpurun_out/tests_r2c_all.log 2>&1; echo all=$?
tail -15 gpurun_out/tests_r2c_all.log
