mkdir -p gpurun_out
timeout 900 ncu --nvtx --nvtx-include "embc_step/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none --csv \
    --log-file gpurun_out/cc_launches_tb.csv python bench.py --workload tb --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/cc_launches_tb.csv
bash tools/gpu_tl.sh tlsc sc
