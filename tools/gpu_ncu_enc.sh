# ncu --set full of selected kernels in one bench step: bash tools/gpu_ncu_enc.sh <tag> <workload> <kernel-regex>
TAG=$1; WL=$2; K=$3
mkdir -p gpurun_out
timeout 1500 ncu --nvtx --nvtx-include "embc_step/" -k "regex:$K" --set full --clock-control none --import-source on -c 4 -f \
  -o gpurun_out/full_${TAG}_${WL} python bench.py --workload $WL --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_${TAG}_${WL}.log 2>&1
tail -3 gpurun_out/ncu_full_${TAG}_${WL}.log
