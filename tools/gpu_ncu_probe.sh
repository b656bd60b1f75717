# ncu --set full (source counters, fine sampling) of one k_dec_main / k_encode launch of a probe workload.
# usage: bash tools/gpu_ncu_probe.sh TAG WORKLOAD MODE TABLES KERNEL
TAG=${1:-np}; WL=${2:-kg}; MODE=${3:-huffman}; T=${4:-26}; K=${5:-k_dec_main}
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none --warp-sampling-interval 0 -k regex:$K --launch-skip 6 -c 1 -f \
  -o gpurun_out/${TAG} python tools/probe_codec.py $WL $MODE --tables $T > gpurun_out/${TAG}_run.log 2>&1
python tools/ncu_lines.py gpurun_out/${TAG}.ncu-rep $K 60 > gpurun_out/${TAG}_lines.txt 2>&1
ncu -i gpurun_out/${TAG}.ncu-rep --page details --csv > gpurun_out/${TAG}_details.csv 2>&1
head -70 gpurun_out/${TAG}_lines.txt
