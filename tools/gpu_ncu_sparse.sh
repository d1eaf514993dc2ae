python __graft_entry__.py > gpurun_out/build.log 2>&1
export RGDBEK_ENGINE=graph RGDBEK_GRAPH=plain
python tools/run_steps.py C3 2 > gpurun_out/c3_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_csr_tiles -s 2 -c 2 -o gpurun_out/prof_tiles_C3 python tools/run_steps.py C3 2 > gpurun_out/ncu_tiles.log 2>&1; echo ncu1=$?
unset RGDBEK_ENGINE RGDBEK_GRAPH
python tools/run_steps.py C3 2 > gpurun_out/c3_p.log 2>&1 && \
ncu --set full --clock-control none -k regex:k_persistent -c 1 -o gpurun_out/prof_persist_C3 python tools/run_steps.py C3 2 > gpurun_out/ncu_pc3.log 2>&1; echo ncu2=$?
