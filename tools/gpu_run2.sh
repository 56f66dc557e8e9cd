for sh in 64,64,64 32,64,128 32,128,64 64,32,128; do
  for v in halo plane; do timeout 120 python tools/time_apply.py --shape $sh --degree 4 --variant $v --reps 50; done
done 2>&1 | tee gpurun_out/halo_time2.log
bash tools/gpu_ncu_halo.sh
python tools/ncu_summary.py gpurun_out/prof_halo.ncu-rep > gpurun_out/prof_halo_summary.txt 2>&1 || true
