timeout 900 python -m pytest tests/test_gpu_solver.py tests/test_gpu_mg.py tests/test_gpu_dg.py tests/test_gpu_hex.py -x -q 2>&1 | tail -3
timeout 300 python bench.py --solve --steps 20 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps(d['solve']))"
timeout 300 python bench.py --config cfg4 --solve --steps 20 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps(d['solve']))"
