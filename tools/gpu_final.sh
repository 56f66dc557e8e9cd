# round-end evidence: the full GPU suite, smoke, default bench, then the profile set (arg: tag)
T=${1:-r02_vX}
mkdir -p gpurun_out
bash tools/gpu_full.sh gpurun_out
bash tools/round_profiles_r02.sh $T
ls -la gpurun_out | tail -30
