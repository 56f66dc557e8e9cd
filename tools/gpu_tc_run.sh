# DMMA kernel: non-volatile mma asm (lib_nv) vs the current library
set -x
MF_LIB_PATH=paper_1910_13247_b200/lib_nv.so timeout 600 python -m pytest tests/test_gpu_tc.py -x -q 2>&1 | tail -2
for lib in paper_1910_13247_b200/libmf_b200.so paper_1910_13247_b200/lib_nv.so; do
  echo $lib
  MF_LIB_PATH=$lib timeout 120 python tools/time_apply.py --cells 64 --degree 6
  MF_LIB_PATH=$lib timeout 120 python tools/time_apply.py --cells 64 --degree 5
  MF_LIB_PATH=$lib timeout 120 python tools/time_apply.py --cells 48 --degree 7
  MF_LIB_PATH=$lib timeout 300 python tools/time_apply.py --cells 256 --degree 6 --reps 3
done
