# ncu --set full of one apply kernel (default: the halo kernel on cfg 3)
K=${1:-k_apply_halo}; V=${2:-halo}; C=${3:-64}; D=${4:-4}
python tools/time_apply.py --cells $C --degree $D --variant $V --reps 3 > gpurun_out/plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 -o gpurun_out/prof_$V python tools/time_apply.py --cells $C --degree $D --variant $V --reps 3 > gpurun_out/ncu_$V.log 2>&1
tail -3 gpurun_out/ncu_$V.log
