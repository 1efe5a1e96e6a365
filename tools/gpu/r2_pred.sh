# predict A/B: parity (predict / score / golden), roofline probe FP64 walk vs coded kernel, C2 bench
set -x
timeout 1200 python -m pytest tests/test_predict_gpu.py tests/test_bench_parity_gpu.py tests/test_featurize_gpu.py tests/test_rank_gpu.py tests/test_pairwise_gpu.py tests/test_full_golden_gpu.py tests/test_capi.py -x -q 2>&1 | tail -4
timeout 600 python tools/roofline_probe.py --families 8 --rows 65536 --trees 1000 > gpurun_out/roofline_new.json 2> gpurun_out/roofline_new.err; echo probe=$?
FAMSEER_LIB=$PWD/var/orig/libfamseer.so timeout 600 python tools/roofline_probe.py --families 8 --rows 65536 --trees 1000 > gpurun_out/roofline_orig.json 2> gpurun_out/roofline_orig.err; echo probe2=$?
python - <<'PY'
import json
for f in ('roofline_new', 'roofline_orig'):
    d = json.load(open('gpurun_out/%s.json' % f))
    print(f, {k: (round(v['ms'], 4), round(v['gbs'], 1), round(v.get('node_visits_per_s', 0) / 1e9, 1)) for k, v in d.items() if isinstance(v, dict) and 'gbs' in v})
PY
timeout 600 python bench.py --no-cpu --no-secondary > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err; echo bench=$?
python -c "
import json; d=json.load(open('gpurun_out/bench_quick.json')); print('value', round(d['value']), 'ms', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value']), d['kernel_ms_one_step'])"
