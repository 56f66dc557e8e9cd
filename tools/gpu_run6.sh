timeout 300 python -m pytest tests/test_gpu_halo.py -x -q 2>&1 | tail -1
for sh in 64,64,64 32,32,256; do
  timeout 60 python tools/time_apply.py --shape $sh --degree 4 --variant halo --reps 30 2>&1 | tail -1
done
