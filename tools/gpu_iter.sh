# debug timings (TB, KG) then parity + bench
bash tools/gpu_dbg.sh tb 80 | grep -E "D1|k_emit:|k_stats:|^job" | tail -32
bash tools/gpu_dbg.sh kg 80 | grep -E "D1|k_emit:|k_stats:" | tail -6
bash tools/gpu_check.sh ${1:-x}
