# A/B: the default build and every var/<name>/libfamseer.so on the C2 bench (no CPU / e2e legs),
# printing value, fit ms and the resident per-phase cycle counters of each.
# Optional: AB_TESTS=1 also runs the fit/bench parity tests against each variant.
for lib in paper_2201_00194_b200/libfamseer.so var/*/libfamseer.so; do
  [ -f "$lib" ] || continue
  echo "== $lib"
  if [ -n "$AB_TESTS" ]; then
    FAMSEER_LIB=$PWD/$lib timeout 900 python -m pytest tests/test_fit_gpu.py tests/test_bench_parity_gpu.py -x -q 2>&1 | tail -2
  fi
  FAMSEER_LIB=$PWD/$lib timeout 600 python bench.py --no-cpu --no-e2e ${BENCH_ARGS} > gpurun_out/ab.json 2> gpurun_out/ab.err || tail -5 gpurun_out/ab.err
  python - <<'PY'
import json
d = json.load(open('gpurun_out/ab.json'))
c = d['device_counters']
ph = c.get('resident_phase_cycles_cta0')
print('value', round(d['value']), 'ms', round(d['ms_per_step'], 3), 'kernels', {k: round(v, 3) for k, v in d['kernel_ms_one_step'].items() if v > 0.05})
print('phases', ph)
PY
done
