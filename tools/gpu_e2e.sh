# e2e pipeline sweep: bash tools/gpu_e2e.sh SLOTS:MULT ...
for cfg in ${@:-3:8 4:24}; do
  S=${cfg%%:*}; M=${cfg#*:}
  EMBC_E2E_SLOTS=$S EMBC_E2E_MULT=$M timeout 300 python bench.py --no-cpu-baseline --steps 200 > gpurun_out/e2e_${S}_${M}.log 2>&1
  echo "slots=$S mult=$M $(python -c "import json; d=json.loads([l for l in open('gpurun_out/e2e_${S}_${M}.log') if l.startswith('{')][-1]); e=d['e2e']; print(d['value'], e['value'], e['ms_per_step'], e.get('pin_memory_value'), e.get('eager_value'))" 2>&1 | tail -1)"
done
