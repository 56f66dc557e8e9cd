./tools/micro/cluster_launch 2>&1 | tee gpurun_out/cluster_launch.log
for sh in 64,64,64 32,64,128; do
  for v in halo; do timeout 120 python tools/time_apply.py --shape $sh --degree 4 --variant $v --reps 50; done
done 2>&1 | tee gpurun_out/halo_time3.log
