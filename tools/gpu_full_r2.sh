#!/bin/bash
# Full GPU suite + smoke on the current tree.
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build_full.log 2>&1 || { tail -30 gpurun_out/build_full.log; exit 1; }
timeout 3000 python -m pytest -q -m gpu tests > gpurun_out/tests_full.log 2>&1; echo tests=$?
tail -5 gpurun_out/tests_full.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_full.log 2>&1; echo smoke=$?
tail -2 gpurun_out/smoke_full.log
