# one compute-sanitizer tool per call (B200_PROFILING.md): plain run first, then the tool
T=${1:-memcheck}
timeout 600 python tools/sanitize_cases.py > gpurun_out/sanitize_plain.log 2>&1 && \
timeout 2400 compute-sanitizer --tool $T --print-limit 20 python tools/sanitize_cases.py > gpurun_out/sanitize_$T.log 2>&1
echo "exit $?"; tail -25 gpurun_out/sanitize_$T.log
