# CTA-count knobs on the pipelined / serial Kaggle-shaped bench
for cfg in ${@:-296:8192 148:8192 296:16384 148:32768}; do
  D=${cfg%%:*}; V=${cfg#*:}
  EMBC_TILE_DIV=$D EMBC_CT_VALS=$V timeout 300 python bench.py --no-cpu-baseline --steps 200 > gpurun_out/ctas_${D}_${V}.log 2>&1
  echo "div=$D ctvals=$V $(python -c "import json; d=json.loads([l for l in open('gpurun_out/ctas_${D}_${V}.log') if l.startswith('{')][-1]); m=d['method']; print(d['value'], d['ms_per_step'], m['ms_per_step_serial'], d['kernels_ms'], d['e2e']['value'])" 2>&1 | tail -1)"
done
