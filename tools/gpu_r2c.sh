# Round-2 evidence: GPU tests, smoke, bench lines for every workload, reference arm,
# ncu launch lists (KG, TB) and --set full captures of one KG and one TB step.
TAG=${1:-r2j}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1200 python -m pytest tests -q -m gpu -x --timeout 300 2>&1 | tail -30 > gpurun_out/ev_${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev_${TAG}_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/ev_${TAG}_bench_kg.log 2>&1
timeout 600 python bench.py --workload tb --no-cpu-baseline > gpurun_out/ev_${TAG}_bench_tb.log 2>&1
timeout 600 python bench.py --workload sc --no-cpu-baseline > gpurun_out/ev_${TAG}_bench_sc.log 2>&1
timeout 600 python bench.py --workload cfg1 --no-cpu-baseline > gpurun_out/ev_${TAG}_bench_cfg1.log 2>&1
timeout 600 python bench.py --workload tb --exchange-step --no-cpu-baseline > gpurun_out/ev_${TAG}_bench_tbx.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ev_${TAG}_bench_ref.log 2>&1
for WL in kg tb; do
  timeout 900 ncu --nvtx --nvtx-include "embc_step/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/ev_${TAG}_launches_${WL}.csv python bench.py --workload $WL --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
done
timeout 1500 ncu --nvtx --nvtx-include "embc_step/" --set full --clock-control none --import-source on -c 5 -f \
  -o gpurun_out/ev_${TAG}_full_tb python bench.py --workload tb --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --nvtx --nvtx-include "embc_step/" --set full --clock-control none --import-source on -c 2 -f \
  -o gpurun_out/ev_${TAG}_full_kg python bench.py --workload kg --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
tail -3 gpurun_out/ev_${TAG}_pytest_gpu.log; tail -1 gpurun_out/ev_${TAG}_smoke.log
python tools/show_bench.py gpurun_out/ev_${TAG}_bench_*.log
