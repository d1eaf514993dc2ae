python tools/ab_run.py "C3,C4,C5m" base build_ab/librgdbek_tbuf2.so --steps 300 --reps 2 > gpurun_out/ab_engine_persist.log 2>&1
RGDBEK_ENGINE=graph python tools/ab_run.py "C3,C4,C5m" base build_ab/librgdbek_tbuf2.so --steps 300 --reps 2 > gpurun_out/ab_engine_graph.log 2>&1
echo persistent; cat gpurun_out/ab_engine_persist.log; echo graph; cat gpurun_out/ab_engine_graph.log
