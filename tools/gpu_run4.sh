timeout 600 python -m pytest tests/test_gpu_halo.py -x -q 2>&1 | tail -2
MF_HALO_PROF=1 timeout 120 python tools/time_apply.py --shape 64,64,64 --degree 4 --variant halo --reps 1 2>&1 | tail -36
timeout 120 python tools/time_apply.py --shape 64,64,64 --degree 4 --variant halo --reps 50 2>&1 | tail -1
