# KG bench under a list of env settings: bash tools/gpu_kg_env.sh tag "VAR=a" "VAR=b" ...
TAG=$1; shift
mkdir -p gpurun_out
for e in "$@"; do
  env $e timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_kg_${TAG}_${e//=/_}.log 2>&1
  echo "$e"; python tools/show_bench.py gpurun_out/bench_kg_${TAG}_${e//=/_}.log
done
exit 0
