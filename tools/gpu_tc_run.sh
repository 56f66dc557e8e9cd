# solver with the closed-form Jacobi diagonal: parity and cfg3 Chebyshev-PCG timing (vs the stored vector)
set -x
timeout 1200 python -m pytest tests/test_gpu_solver.py tests/test_gpu_mg.py -x -q 2>&1 | tail -2
for v in "" 1; do
  env ${v:+MF_DINV_VECTOR=1} timeout 600 python bench.py --solve --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/solve3.json 2> gpurun_out/solve3.err; tail -1 gpurun_out/solve3.err
  python -c "import json; d=json.load(open('gpurun_out/solve3.json')); print('dinv_vector=$v', d['solve']['iterations'], d['solve']['seconds'], d['solve']['mixed'])"
done
