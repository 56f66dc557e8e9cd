#!/bin/bash
# bench lines (cfg3 default incl. cpu_baseline, cfg4, hex3, dg4, cfg3 solve), launch lists and one
# ncu --set full capture of each dominant kernel; arg1 = tag (e.g. r01_v7)
cd "$(dirname "$0")/.."
T=${1:-rXX}
python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?"
for c in cfg4 hex3 dg4; do
  python bench.py --config $c > gpurun_out/${T}_bench_$c.json 2>> gpurun_out/${T}_bench.err; echo "$c rc=$?"
done
python bench.py --solve --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_solve_cfg3.json 2>> gpurun_out/${T}_bench.err; echo "solve rc=$?"
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_plane_cfg3_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "launches rc=$?"
for c in cfg4 hex3 dg4; do
  python tools/prof_apply.py --config $c > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_${c}_launches.csv python tools/prof_apply.py --config $c > /dev/null 2>&1; echo "launches $c rc=$?"
done
python tools/prof_apply.py > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_apply_plane -s 2 -c 1 -o gpurun_out/${T}_plane_cfg3 python tools/prof_apply.py > /dev/null 2>&1; echo "ncu3 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_apply_cell3 -s 2 -c 1 -o gpurun_out/${T}_general_cfg4 python tools/prof_apply.py --config cfg4 > /dev/null 2>&1; echo "ncu4 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_apply_cell3 -s 2 -c 1 -o gpurun_out/${T}_hex3 python tools/prof_apply.py --config hex3 > /dev/null 2>&1; echo "ncuhex rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_apply_dg -s 2 -c 1 -o gpurun_out/${T}_dg4 python tools/prof_apply.py --config dg4 > /dev/null 2>&1; echo "ncudg rc=$?"
ncu --set full --clock-control none -k regex:k_tile_init -s 2 -c 1 -o gpurun_out/${T}_init_cfg3 python tools/prof_apply.py > /dev/null 2>&1; echo "ncuinit rc=$?"
