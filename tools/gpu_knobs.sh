# Decode knob sweep (EMBC_SEG vlz segment bytes, EMBC_HSUB huffman subsequences per small-call block); serial KG / TB bench.
TAG=${1:-kn}
mkdir -p gpurun_out
EMBC_SEG=256 EMBC_HSUB=128 timeout 600 python -m pytest tests -q -m gpu -x --timeout 120 -k "codec or edges or bench_parity" 2>&1 | tail -2
for WL in kg tb; do
  for S in 1024 512 256; do
    for H in 256 128; do
      [ $WL = tb ] && [ $H = 128 ] && continue
      EMBC_SEG=$S EMBC_HSUB=$H timeout 300 python bench.py --workload $WL --no-cpu-baseline --steps 100 --schedule serial > gpurun_out/${TAG}_${WL}_s${S}_h${H}.log 2>&1
      echo "$WL seg=$S hsub=$H $(python -c "import json; d=json.loads([l for l in open('gpurun_out/${TAG}_${WL}_s${S}_h${H}.log') if l.startswith('{')][-1]); print(d['ms_per_step'], d['kernels_ms'])" 2>&1 | tail -1)"
    done
  done
done
