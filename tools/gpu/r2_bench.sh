# default bench line (C2 + secondary C5 block + CPU baseline + e2e), then the 2-rank family-sharded
# path on the box's one GPU (FAMSEER_BENCH_SHARE_GPU=1: ranks share it, gloo) - per-family model
# digests must equal the 1-rank run's
set -x
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench=$?
FAMSEER_BENCH_SHARE_GPU=1 timeout 600 python bench.py --gpus 2 --no-cpu --no-e2e --no-secondary > gpurun_out/bench_n2_shared.json 2> gpurun_out/bench_n2_shared.err; echo bench2=$?
tail -5 gpurun_out/bench_default.err gpurun_out/bench_n2_shared.err
python - <<'PY'
import json
a=json.load(open('gpurun_out/bench_default.json'))
print('value', round(a['value']), 'ms', round(a['ms_per_step'],3), 'e2e', a['e2e'] and round(a['e2e']['value']), 'phases', a['phases_ms'])
print('roofline', {k: a['roofline'].get(k) for k in ('kernel','achieved','frac','frac_s8d')})
print('kernels', a['kernel_ms_one_step'])
print('secondary', json.dumps(a.get('secondary_c5'))[:1500])
print('cpu', a.get('cpu_baseline'))
b=json.load(open('gpurun_out/bench_n2_shared.json'))
print('n2', b['n_gpus'], b['scaling'], b['parallelism'], round(b['value']), b['family_ids'])
print('digests equal:', a['family_model_sha'] == b['family_model_sha'], a['family_model_sha'], b['family_model_sha'])
PY
