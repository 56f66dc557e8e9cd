#!/bin/bash
# solver parity tests, then the cfg3 / cfg4 Chebyshev-PCG solve with fused and unfused Chebyshev steps
cd "$(dirname "$0")/.."
python -m pytest tests/test_gpu_solver.py -q -x 2>&1 | tail -2
for cfg in ${@:-cfg3}; do for f in 0; do
  MF_CHEB_FUSED=$f python bench.py --steps 20 --warmup 3 --no-cpu-baseline --solve --config $cfg > gpurun_out/solve_${cfg}_$f.log 2>&1
  python -c "import json;d=json.load(open('gpurun_out/solve_${cfg}_$f.log'));s=d['solve'];print('$cfg fused=$f its',s['iterations'],'s %.3f ms/it %.3f'%(s['seconds'],1e3*s['seconds']/s['iterations']))" || tail -3 gpurun_out/solve_${cfg}_$f.log
done; done
