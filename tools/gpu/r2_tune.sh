set -x
timeout 900 python -m pytest tests/test_tune_step_gpu.py tests/test_bench_parity_gpu.py tests/test_score_index_gpu.py -x -q 2>&1 | tail -3
for f in "" "--no-overlap"; do
  timeout 600 python bench.py --no-cpu --no-secondary $f > gpurun_out/bt.json 2> gpurun_out/bt.err; echo rc=$?
  tail -2 gpurun_out/bt.err
  python -c "
import json; d=json.load(open('gpurun_out/bt.json')); print('$f', 'value', round(d['value']), 'ms', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value']), round(d['e2e']['ms_per_step'],3), d['e2e']['api'])"
done
