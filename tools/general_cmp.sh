#!/bin/bash
# general-kernel parity (all apply tests), then cfg4 bench with the v2 (default) and v1 3D kernels
cd "$(dirname "$0")/.."
python -m pytest tests/test_gpu_apply.py -q -x 2>&1 | tail -1
for v in 2 1; do
  if [ $v = 1 ]; then export MF_GENERAL_V1=1; fi
  python bench.py --steps 100 --warmup 10 --no-cpu-baseline --config cfg4 > gpurun_out/g4_v$v.log 2>&1
  python -c "import json;d=json.load(open('gpurun_out/g4_v$v.log'));print('cfg4 v$v GDoF/s %.2f  kernel_us %.1f frac %.3f'%(d['value']/1e9,d['roofline']['kernel_ms']*1e3,d['roofline']['frac']))" || tail -3 gpurun_out/g4_v$v.log
done
