#!/bin/bash
cd "$(dirname "$0")/.."
for s in 8x4 16x2; do
  MF_TILE=$s python -m pytest tests/test_gpu_apply.py -q -x -k "variants and plane" 2>&1 | tail -1
  MF_TILE=$s python bench.py --steps 300 --warmup 20 --no-cpu-baseline --variant plane > gpurun_out/b_$s.log 2>&1
  python -c "import json;d=json.load(open('gpurun_out/b_$s.log'));print('$s GDoF/s %.1f  kernel_us %.1f'%(d['value']/1e9,d['roofline']['kernel_ms']*1e3))"
  MF_TILE=$s python tools/prof_apply.py --variant plane > gpurun_out/plain.log 2>&1 && MF_TILE=$s ncu --metrics gpu__time_duration.sum --clock-control none -c 6 --csv --log-file gpurun_out/launches_$s.csv python tools/prof_apply.py --variant plane > /dev/null 2>&1
  grep -E "k_tile_init|k_apply_plane" gpurun_out/launches_$s.csv | tail -2 | awk -F'","' '{print substr($5,1,30), $NF}'
done
