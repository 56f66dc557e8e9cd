timeout 900 python -m pytest tests/test_gpu_guards.py -x -q 2>&1 | grep -E "Error|error|assert|FAILED|passed|failed" | head -20
MF_LIB_PATH=$PWD/paper_1910_13247_b200/lib_checked.so timeout 900 python -m pytest tests/test_gpu_halo.py -x -q 2>&1 | grep -E "Error|error|assert|FAILED|passed|failed" | head -20
