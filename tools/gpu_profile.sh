# ncu evidence for one bench step: launch list (serialised, cold) + --set full of every kernel in one step.
# usage: bash tools/gpu_profile.sh <tag> <workload>
set -x
TAG=${1:-r1}; WL=${2:-kg}
mkdir -p gpurun_out
timeout 900 ncu --nvtx --nvtx-include "embc_step/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_${TAG}_${WL}.csv python bench.py --workload $WL --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_${TAG}_${WL}.log 2>&1
timeout 1500 ncu --nvtx --nvtx-include "embc_step/" --set full --clock-control none --import-source on -c 12 -f \
  -o gpurun_out/full_${TAG}_${WL} python bench.py --workload $WL --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_${TAG}_${WL}.log 2>&1
