python __graft_entry__.py > gpurun_out/build_r2b.log 2>&1 || { tail -30 gpurun_out/build_r2b.log; exit 1; }
timeout 900 python -m pytest -x -q tests/test_gpu_selection_paths.py tests/test_gpu_parity.py -k "block_lists or selection or lazy_wide or output_buffers or tall or lstsq or tile_edges" > gpurun_out/tests_r2b.log 2>&1; echo tests=$?
tail -15 gpurun_out/tests_r2b.log
for w in C2c C3; do timeout 300 python tools/phase_profile.py $w 200; done > gpurun_out/phases_r2b.jsonl 2>&1
cat gpurun_out/phases_r2b.jsonl | cut -c1-400
