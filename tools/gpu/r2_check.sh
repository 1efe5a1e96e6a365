# round-2 loop: full GPU suite (minus pending goldens), smoke, quick C2 bench
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} 2>&1 | tail -25
timeout 600 python bench.py --no-cpu --no-e2e ${BENCH_ARGS} > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err; echo bench=$?
tail -3 gpurun_out/bench_quick.err
python - <<'PY'
import json
d=json.load(open('gpurun_out/bench_quick.json'))
print('value', round(d['value']), 'ms', round(d['ms_per_step'],3), 'phases', d['phases_ms'])
print('kernels', d['kernel_ms_one_step'])
PY
