timeout 1500 python -m pytest tests/test_full_golden_gpu.py tests/test_fit_gpu.py tests/test_bench_parity_gpu.py -x -q 2>&1 | tail -2
for c in c4 c5; do
timeout 1500 python bench.py --config $c --steps 2 --warmup 3 --no-cpu --no-e2e --no-secondary > gpurun_out/b.json 2> gpurun_out/b.err
python -c "
import json; d=json.load(open('gpurun_out/b.json')); k=d['kernel_ms_one_step']; print('$c', round(d['ms_per_step'],1), 'hist', k.get('fit_hist_build'), 'exact', k.get('fit_exact'), 'screen', k.get('fit_screen'), 'nodes', d.get('fit_nodes'), 'roof', d['roofline'].get('frac'), d['roofline'].get('frac_s8d'))"
done
