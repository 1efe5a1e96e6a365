# quick loop: parity (fit + bench-workload parity), smoke, C2 bench without CPU/e2e
set -x
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_fit_gpu.py tests/test_bench_parity_gpu.py -x -q 2>&1 | tail -15
timeout 600 python bench.py --no-cpu --no-e2e ${BENCH_ARGS} > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err; echo bench=$?
python - <<'PY'
import json
d=json.load(open('gpurun_out/bench_quick.json'))
print('value', round(d['value']), 'ms', round(d['ms_per_step'],3), 'phases', d['phases_ms'])
print('kernels', d['kernel_ms_one_step'])
print('nodes', d['fit_nodes'], 'ctr', d['device_counters'])
PY
