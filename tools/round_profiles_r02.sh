#!/bin/bash
# Round-2 evidence for the headline kernel (arg1 = tag, e.g. r02_v2): the default bench line,
# the launch list of the bench command, an ncu metrics pass (DRAM bytes + predicated-on FP64
# instruction counts + duration) and one ncu --set full capture of the halo kernel on cfg 3,
# and the sha1 of the library they were taken with.
cd "$(dirname "$0")/.."
T=${1:-r02_vX}
O=gpurun_out
sha1sum paper_1910_13247_b200/libmf_b200.so | cut -c1-12 > $O/${T}_build.txt
python bench.py > $O/${T}_bench.json 2> $O/${T}_bench.err; echo "bench rc=$?"
python bench.py --solve --steps 20 --warmup 3 --no-cpu-baseline > $O/${T}_solve_cfg3.json 2>> $O/${T}_bench.err; echo "solve rc=$?"
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${T}_cfg3_launches.csv \
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "launches rc=$?"
python tools/prof_apply.py > /dev/null 2>&1 && \
  ncu --clock-control none -k regex:k_apply_halo -s 2 -c 1 --csv --log-file $O/${T}_halo_cfg3_metrics.csv \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__inst_executed.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active \
  python tools/prof_apply.py > /dev/null 2>&1; echo "metrics rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_apply_halo -s 2 -c 1 -o $O/${T}_halo_cfg3 \
  python tools/prof_apply.py > /dev/null 2>&1; echo "ncu full rc=$?"
# ---- the DMMA kernel (k = 5..7, cfg 5 Q6): bench line, a 256^3 metrics pass (DRAM bytes, FP64
# and DMMA counts of the timed kernel) and one --set full capture at 64^3
python bench.py --config cfg5q6 --steps 5 --warmup 3 > $O/${T}_bench_cfg5q6.json 2>> $O/${T}_bench.err; echo "cfg5q6 bench rc=$?"
python tools/prof_apply.py --config cfg5q6 --reps 2 > /dev/null 2>&1 && \
  ncu --clock-control none -k regex:k_apply_tc -c 1 --csv --log-file $O/${T}_tc_cfg5q6_metrics.csv \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__ops_path_tensor_src_fp64.sum,smsp__inst_executed.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active \
  python tools/prof_apply.py --config cfg5q6 --reps 2 > /dev/null 2>&1; echo "tc metrics rc=$?"
python tools/prof_apply.py --config cfg5q6 --cells 64 > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_apply_tc -s 1 -c 1 -o $O/${T}_tc_q6_64 \
  python tools/prof_apply.py --config cfg5q6 --cells 64 > /dev/null 2>&1; echo "tc ncu full rc=$?"
