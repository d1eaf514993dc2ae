for w in C5s C4; do timeout 600 python tools/sharded_probe.py $w 200; done > gpurun_out/probe_base.jsonl 2>&1
for w in C5s C4; do RGDBEK_LIB=build_ab/librgdbek_xgpu.so timeout 600 python tools/sharded_probe.py $w 200; done > gpurun_out/probe_xgpu.jsonl 2>&1
cat gpurun_out/probe_base.jsonl gpurun_out/probe_xgpu.jsonl | cut -c1-200
