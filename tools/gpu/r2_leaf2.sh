timeout 1500 python -m pytest tests/test_full_golden_gpu.py tests/test_fit_gpu.py -x -q 2>&1 | tail -2
timeout 900 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu --no-e2e --no-secondary > gpurun_out/b4.json 2> gpurun_out/b4.err
python -c "
import json; d=json.load(open('gpurun_out/b4.json')); k=d['kernel_ms_one_step']; print('c4', round(d['ms_per_step'],2), 'leaf', k.get('fit_leaf'), 'exact', k.get('fit_exact'))"
timeout 1500 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu --no-e2e --no-secondary > gpurun_out/b5.json 2> gpurun_out/b5.err
python -c "
import json; d=json.load(open('gpurun_out/b5.json')); k=d['kernel_ms_one_step']; print('c5', round(d['ms_per_step'],1), 'leaf', k.get('fit_leaf'), 'exact', k.get('fit_exact'))"
