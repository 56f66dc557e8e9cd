#!/bin/bash
# quick GPU iteration: tile/cfg3 parity tests, bench, optional ncu of the tile kernel (arg1 = report name)
cd "$(dirname "$0")/.."
python -m pytest tests/test_gpu_apply.py -q -x -k "variants or cfg3" > gpurun_out/tile_tests.log 2>&1
tail -2 gpurun_out/tile_tests.log
python bench.py --steps 500 --warmup 20 --no-cpu-baseline > gpurun_out/bench_tile.log 2>&1
python -c "import json;d=json.load(open('gpurun_out/bench_tile.log'));print('GDoF/s %.1f  kernel_us %.1f  frac %.3f'%(d['value']/1e9,d['roofline']['kernel_ms']*1e3,d['roofline']['frac']))"
if [ -n "$1" ]; then
  python tools/prof_apply.py > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_apply_tile -s 2 -c 1 -o gpurun_out/$1 python tools/prof_apply.py > gpurun_out/ncu_tile.log 2>&1
  echo "ncu rc=$?"
fi
