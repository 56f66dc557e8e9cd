# cfg5 Q6 bench line (no profiler), then one ncu --set full capture of k_apply_tc at Q6 64^3
set -x
mkdir -p gpurun_out
timeout 900 python bench.py --config cfg5q6 --steps 5 --warmup 3 > gpurun_out/tc_bench_cfg5q6.json 2> gpurun_out/tc_bench.err; tail -3 gpurun_out/tc_bench.err
cat gpurun_out/tc_bench_cfg5q6.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_apply_tc -c 1 -f -o gpurun_out/tc_q6 \
  python tools/time_apply.py --cells 64 --degree 6 --reps 2 > gpurun_out/tc_ncu.log 2>&1; tail -3 gpurun_out/tc_ncu.log
