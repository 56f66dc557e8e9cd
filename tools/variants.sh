#!/bin/bash
# parity of the Cartesian variants + bench of each variant on cfg3
cd "$(dirname "$0")/.."
python -m pytest tests/test_gpu_apply.py -q -x -k "variants or cfg3" 2>&1 | tail -1
for v in ${@:-plane tile}; do
  python bench.py --steps 300 --warmup 20 --no-cpu-baseline --variant $v > gpurun_out/b_$v.log 2>&1
  python -c "import json;d=json.load(open('gpurun_out/b_$v.log'));print('$v GDoF/s %.1f  kernel_us %.1f frac %.3f'%(d['value']/1e9,d['roofline']['kernel_ms']*1e3,d['roofline']['frac']))" || tail -3 gpurun_out/b_$v.log
done
