# DMMA kernel: shared-memory slice staging (MF_TC_SMEMU) vs the register prefetch, Q6 64^3 / 256^3, Q5
set -x
MF_LIB_PATH=paper_1910_13247_b200/lib_su384.so timeout 600 python -m pytest tests/test_gpu_tc.py -x -q 2>&1 | tail -2
for lib in paper_1910_13247_b200/libmf_b200.so paper_1910_13247_b200/lib_su384.so paper_1910_13247_b200/lib_su448.so; do
  echo $lib
  MF_LIB_PATH=$lib timeout 120 python tools/time_apply.py --cells 64 --degree 6
  MF_LIB_PATH=$lib timeout 120 python tools/time_apply.py --cells 64 --degree 5
  MF_LIB_PATH=$lib timeout 300 python tools/time_apply.py --cells 256 --degree 6 --reps 3
done
