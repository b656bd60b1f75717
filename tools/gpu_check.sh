# parity + bench on the GPU box: bash tools/gpu_check.sh [tag]
TAG=${1:-x}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -40 > gpurun_out/pytest_gpu_${TAG}.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_kg_${TAG}.log 2>&1
timeout 600 python bench.py --workload tb --no-cpu-baseline > gpurun_out/bench_tb_${TAG}.log 2>&1
tail -5 gpurun_out/pytest_gpu_${TAG}.log; tail -2 gpurun_out/smoke_${TAG}.log
python tools/show_bench.py gpurun_out/bench_kg_${TAG}.log gpurun_out/bench_tb_${TAG}.log; exit 0
import json,sys
t=open(sys.argv[1]).read().strip().splitlines()
try:
    d=json.loads(t[-1]); print(sys.argv[1], "value", d["value"], "ms", d["ms_per_step"], "e2e", d["e2e"]["value"], "kernels", d["kernels_ms"])
except Exception: print("\n".join(t[-15:]))
PY
done
