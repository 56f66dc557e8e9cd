# one bench line per config on the current build (no profiler), for the round's record
mkdir -p gpurun_out
for c in cfg2 cfg4 cfg5q4 hex3 dg4; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/final_bench_$c.json 2> gpurun_out/final_bench_$c.err
  echo "$c rc=$?"; python -c "import json; d=json.load(open('gpurun_out/final_bench_$c.json')); print('$c', d['value']/1e9, d['ms_per_step'], d['roofline']['frac'], d['clocks']['reasons'])"
done
