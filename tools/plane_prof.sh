#!/bin/bash
# parity of the Cartesian variants, bench of the default path on cfg3, launch list (init + main kernel)
cd "$(dirname "$0")/.."
python -m pytest tests/test_gpu_apply.py -q -x -k "variants or cfg3" 2>&1 | tail -1
python bench.py --steps 300 --warmup 20 --no-cpu-baseline > gpurun_out/b_plane.log 2>&1
python -c "import json;d=json.load(open('gpurun_out/b_plane.log'));print('GDoF/s %.1f  kernel_us %.1f frac %.3f'%(d['value']/1e9,d['roofline']['kernel_ms']*1e3,d['roofline']['frac']))" || tail -3 gpurun_out/b_plane.log
python tools/prof_apply.py > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 6 --csv --log-file gpurun_out/launches_plane.csv python tools/prof_apply.py > /dev/null 2>&1
grep -E "k_tile_init|k_apply_plane" gpurun_out/launches_plane.csv | tail -2 | awk -F'","' '{print substr($5,1,30), $NF}'
