# atomic cost: reductions vs plain stores (timing only), 64^3 and 256^3 Q6; ncu of the 256^3 launch
set -x
for lib in paper_1910_13247_b200/libmf_b200.so paper_1910_13247_b200/lib_store.so; do
  MF_LIB_PATH=$lib timeout 120 python tools/time_apply.py --cells 64 --degree 6
  MF_LIB_PATH=$lib timeout 300 python tools/time_apply.py --cells 256 --degree 6 --reps 3
done
timeout 900 ncu --section SpeedOfLight --section MemoryWorkloadAnalysis --section WarpStateStats --section LaunchStats --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_red.sum,lts__t_requests_op_red.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,lts__t_sectors_srcunit_tex_op_red_lookup_miss.sum --clock-control none -k regex:k_apply_tc -c 1 -f -o gpurun_out/tc_q6_256 python tools/time_apply.py --cells 256 --degree 6 --reps 1 > gpurun_out/tc_ncu256.log 2>&1; tail -2 gpurun_out/tc_ncu256.log
