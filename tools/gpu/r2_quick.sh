# quick loop: fit parity (resident + multi, cluster variants), then phase counters and a C2 bench
set -x
timeout 1200 python -m pytest tests/test_fit_gpu.py tests/test_bench_parity_gpu.py tests/test_store_gpu.py tests/test_engine_e2e.py -x -q ${PYTEST_ARGS} 2>&1 | tail -8
timeout 300 python tools/phase_probe.py c2 2>&1 | tail -3
timeout 600 python bench.py --no-cpu --no-e2e --no-secondary ${BENCH_ARGS} > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err; echo bench=$?
tail -3 gpurun_out/bench_quick.err
python - <<'PY'
import json
d=json.load(open('gpurun_out/bench_quick.json'))
print('value', round(d['value']), 'ms', round(d['ms_per_step'],3), 'phases', d['phases_ms'])
print('kernels', d['kernel_ms_one_step'])
PY
