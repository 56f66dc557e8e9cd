set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python -m pytest tests/test_gpu_halo.py -x -q 2>&1 | tail -30 > gpurun_out/halo_tests.log
cat gpurun_out/halo_tests.log
for v in halo plane; do timeout 120 python tools/time_apply.py --cells 64 --degree 4 --variant $v --reps 100; done 2>&1 | tee gpurun_out/halo_time.log
