# bench lines on the GPU box: bash tools/gpu_bench.sh <tag> [workloads...]
TAG=${1:-x}; shift
WLS=${@:-kg tb}
mkdir -p gpurun_out
for w in $WLS; do
  timeout 900 python bench.py --workload $w --steps 50 --warmup 5 > gpurun_out/bench_${w}_${TAG}.log 2>&1
  echo "== $w rc=$?"; tail -c 600 gpurun_out/bench_${w}_${TAG}.log | grep -v '^{' | tail -5
  python tools/show_bench.py gpurun_out/bench_${w}_${TAG}.log
done
exit 0
