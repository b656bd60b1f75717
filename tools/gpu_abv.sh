# A/B over library variants (EMBC_LIB): base worktree, current tree, tools/ablibs/lib_*.so; serial KG / TB bench.
TAG=${1:-abv}; WLS=${2:-kg tb}
mkdir -p gpurun_out
for i in 1 2; do
  for WL in $WLS; do
    (cd tools/ab_base && timeout 300 python bench.py --workload $WL --no-cpu-baseline --steps 100 --schedule serial) > gpurun_out/${TAG}_base_${WL}_$i.log 2>&1
    timeout 300 python bench.py --workload $WL --no-cpu-baseline --steps 100 --schedule serial > gpurun_out/${TAG}_cur_${WL}_$i.log 2>&1
    for L in tools/ablibs/lib_*.so; do
      n=$(basename $L .so)
      EMBC_LIB=$PWD/$L timeout 300 python bench.py --workload $WL --no-cpu-baseline --steps 100 --schedule serial > gpurun_out/${TAG}_${n}_${WL}_$i.log 2>&1
    done
  done
done
for f in gpurun_out/${TAG}_*.log; do echo "$f $(python -c "import json,sys; d=json.loads([l for l in open('$f') if l.startswith('{')][-1]); print(d['ms_per_step'], d['kernels_ms'])" 2>&1 | tail -1)"; done
