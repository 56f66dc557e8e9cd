#!/bin/bash
# one ncu --set full capture of the cfg3 main kernel (arg1 = report name), after a plain run exits 0
cd "$(dirname "$0")/.."
python tools/prof_apply.py > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:${2:-k_apply_plane} -s 2 -c 1 -o gpurun_out/$1 python tools/prof_apply.py > gpurun_out/ncu_$1.log 2>&1
echo "ncu rc=$?"
