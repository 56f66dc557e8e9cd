# solver: parity (iteration counts = oracle) and cfg3 Chebyshev-PCG timing with the three-term Chebyshev step
set -x
timeout 1200 python -m pytest tests/test_gpu_solver.py tests/test_gpu_mg.py -x -q 2>&1 | tail -2
timeout 600 python bench.py --solve --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/solve3.json 2> gpurun_out/solve3.err; tail -2 gpurun_out/solve3.err
python -c "
import json; d=json.load(open('gpurun_out/solve3.json')); s=d.get('solve') or {}
print(json.dumps({k: d[k] for k in d if 'solve' in k}, indent=0)[:1500])"
