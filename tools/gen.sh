#!/bin/bash
cd "$(dirname "$0")/.."
python -m pytest tests/test_gpu_apply.py -q -x -k "matches_assembled or cfg4 or general" 2>&1 | tail -1
python bench.py --config cfg4 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/b_cfg4.log 2>&1
python -c "import json;d=json.load(open('gpurun_out/b_cfg4.log'));print('cfg4 GDoF/s %.2f kernel_us %.1f frac %.3f'%(d['value']/1e9,d['roofline']['kernel_ms']*1e3,d['roofline']['frac']))" || tail -3 gpurun_out/b_cfg4.log
