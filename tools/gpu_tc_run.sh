# detached-slab decomposition parity + the apply suites that share its paths
set -x
timeout 900 python -m pytest tests/test_gpu_slabs.py tests/test_gpu_halo.py tests/test_gpu_tc.py -x -q 2>&1 | tail -15
