# A/B of the KG / TB bench: a base worktree (tools/ab_base, built in place) vs the current tree, interleaved.
TAG=${1:-ab}; WLS=${2:-kg tb}
mkdir -p gpurun_out
for i in 1 2; do
  for WL in $WLS; do
    (cd tools/ab_base && timeout 300 python bench.py --workload $WL --no-cpu-baseline --steps 100 --schedule serial) > gpurun_out/${TAG}_old_${WL}_$i.log 2>&1
    timeout 300 python bench.py --workload $WL --no-cpu-baseline --steps 100 --schedule serial > gpurun_out/${TAG}_new_${WL}_$i.log 2>&1
  done
done
for f in gpurun_out/${TAG}_*.log; do echo "$f $(python -c "import json,sys; d=json.loads([l for l in open('$f') if l.startswith('{')][-1]); print(d['ms_per_step'], d['kernels_ms'])")"; done
