set -x
timeout 600 python -m pytest tests/test_gpu_tc.py -x -q 2>&1 | tail -15
timeout 120 python tools/time_apply.py --cells 64 --degree 6
MF_NO_TC=1 timeout 120 python tools/time_apply.py --cells 64 --degree 6
timeout 120 python tools/time_apply.py --cells 64 --degree 5
MF_NO_TC=1 timeout 120 python tools/time_apply.py --cells 64 --degree 5
timeout 120 python tools/time_apply.py --cells 48 --degree 7
MF_NO_TC=1 timeout 120 python tools/time_apply.py --cells 48 --degree 7
