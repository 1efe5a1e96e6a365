# resident trainer with 1 / 2 / 4 CTAs per family: parity (fit + bench workloads) and the C2 bench
for cl in 2 4; do
  echo "== parity FAMSEER_RES_CLUSTER=$cl"
  FAMSEER_RES_CLUSTER=$cl timeout 900 python -m pytest tests/test_fit_gpu.py tests/test_bench_parity_gpu.py tests/test_store_gpu.py -x -q 2>&1 | tail -3
done
for cl in 1 2 4; do
  FAMSEER_RES_CLUSTER=$cl timeout 600 python bench.py --no-cpu --no-e2e ${BENCH_ARGS} > gpurun_out/ab.json 2> gpurun_out/ab.err || tail -5 gpurun_out/ab.err
  python - "$cl" <<'PY'
import json, sys
d = json.load(open('gpurun_out/ab.json'))
print('cluster', sys.argv[1], 'value', round(d['value']), 'ms', round(d['ms_per_step'], 3), 'fit_resident', d['kernel_ms_one_step'].get('fit_resident'))
print('  phases', d['device_counters'].get('resident_phase_cycles_cta0'))
PY
done
