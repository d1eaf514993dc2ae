# One compute-sanitizer tool per call (B200_PROFILING.md): bash tools/gpu_sanitize.sh TOOL GRID TAG
TOOL=${1:-memcheck}; GRID=${2:-2}; TAG=${3:-r2}
python __graft_entry__.py > gpurun_out/build_san.log 2>&1 || { tail gpurun_out/build_san.log; exit 1; }
timeout 300 python tools/sanitize_cases.py $GRID > gpurun_out/san_plain_$TOOL.log 2>&1; echo plain=$?
[ -s gpurun_out/san_plain_$TOOL.log ] && tail -2 gpurun_out/san_plain_$TOOL.log
timeout 1500 compute-sanitizer --tool $TOOL --print-limit 50 --error-exitcode 9 \
   python tools/sanitize_cases.py $GRID > gpurun_out/sanitize_${TAG}_$TOOL.log 2>&1
echo sanitizer_$TOOL=$?
tail -5 gpurun_out/sanitize_${TAG}_$TOOL.log
