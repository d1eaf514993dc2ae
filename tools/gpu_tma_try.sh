#!/bin/bash
# Opt-in TMA pass-N experiment: parity subset + phase profile with and without it.
mkdir -p gpurun_out
python paper_2509_19267_b200/_build.py > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 240 python tools/e2e_probe.py C1 1000 4 > gpurun_out/e2e_probe_C1.jsonl 2>&1
timeout 240 python tools/e2e_probe.py C2c 2000 2 > gpurun_out/e2e_probe_C2c.jsonl 2>&1
RGDBEK_PN_TMA=1 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu \
  -k "dense_50 or full_size_dense or time_to_tolerance_matches or step_chunks or engines" \
  > gpurun_out/tma_pytest.log 2>&1; echo "tma pytest rc=$?" >> gpurun_out/tma_pytest.log
RGDBEK_PN_TMA=1 timeout 300 python tools/phase_profile.py C2c 500 > gpurun_out/tma_phase.json 2>&1
timeout 300 python tools/phase_profile.py C2c 500 > gpurun_out/notma_phase.json 2>&1
tail -3 gpurun_out/tma_pytest.log; cat gpurun_out/tma_phase.json gpurun_out/notma_phase.json gpurun_out/e2e_probe_C1.jsonl gpurun_out/e2e_probe_C2c.jsonl
