# A/B of the KG / TB bench: round-start worktree (tools/ab_r2a) vs the current tree, interleaved.
TAG=${1:-ab}
mkdir -p gpurun_out
for i in 1 2; do
  (cd tools/ab_r2a && timeout 300 python bench.py --no-cpu-baseline --steps 100) > gpurun_out/${TAG}_old_kg_$i.log 2>&1
  timeout 300 python bench.py --no-cpu-baseline --steps 100 > gpurun_out/${TAG}_new_kg_$i.log 2>&1
done
(cd tools/ab_r2a && timeout 300 python bench.py --workload tb --no-cpu-baseline) > gpurun_out/${TAG}_old_tb.log 2>&1
timeout 300 python bench.py --workload tb --no-cpu-baseline > gpurun_out/${TAG}_new_tb.log 2>&1
for f in gpurun_out/${TAG}_*.log; do echo "$f $(python -c "import json,sys; d=json.loads([l for l in open('$f') if l.startswith('{')][-1]); print(d['ms_per_step'], d['kernels_ms'])")"; done
