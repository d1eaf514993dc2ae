python __graft_entry__.py > gpurun_out/build_spec.log 2>&1 || { tail -20 gpurun_out/build_spec.log; exit 1; }
timeout 900 python -m pytest -x -q tests/test_gpu_parity.py -k "sparse or tile or c3 or c4 or c5s" tests/test_gpu_selection_paths.py > gpurun_out/tests_spec.log 2>&1; echo tests=$?; tail -3 gpurun_out/tests_spec.log
python tools/ab_run.py "C3,C4,C5m" base build_ab/librgdbek_prespec.so --steps 500 --reps 3 > gpurun_out/ab_spec.log 2>&1; cat gpurun_out/ab_spec.log
