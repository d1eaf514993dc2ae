python __graft_entry__.py > gpurun_out/build_nm.log 2>&1 || exit 1
timeout 300 python tools/run_multi.py C4 3 3 > gpurun_out/nm_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_multi -c 1 -o gpurun_out/prof_multi_C4 python tools/run_multi.py C4 3 3 > gpurun_out/ncu_multi.log 2>&1; echo ncu=$?
python tools/ncu_summary.py gpurun_out/prof_multi_C4.ncu-rep > gpurun_out/prof_multi_C4_summary.txt 2>&1
python tools/ncu_lines.py gpurun_out/prof_multi_C4.ncu-rep 30 > gpurun_out/prof_multi_C4_lines.txt 2>&1
rm -f gpurun_out/prof_multi_C4.ncu-rep
