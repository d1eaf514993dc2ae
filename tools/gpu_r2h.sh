python __graft_entry__.py > gpurun_out/build_r2h.log 2>&1 || { tail -30 gpurun_out/build_r2h.log; exit 1; }
timeout 900 python -m pytest -x -q tests/test_gpu_sharded.py tests/test_gpu_peer_ipc.py > gpurun_out/tests_r2h_sharded.log 2>&1; echo sharded=$?
tail -4 gpurun_out/tests_r2h_sharded.log
for w in C2c C3 C4 C5s; do timeout 600 python tools/sharded_probe.py $w 200; done > gpurun_out/sharded_probe_r2h.jsonl 2>&1
cut -c1-160 gpurun_out/sharded_probe_r2h.jsonl
