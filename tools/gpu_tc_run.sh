# detached-slab decomposition (apply, diagonal) + the >= 2-GPU NCCL test (skips on one GPU)
set -x
timeout 900 python -m pytest tests/test_gpu_slabs.py tests/test_gpu_multi.py -q -rs 2>&1 | tail -12
