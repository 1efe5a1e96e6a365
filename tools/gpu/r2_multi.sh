set -x
timeout 1500 python -m pytest tests/test_fit_gpu.py tests/test_full_golden_gpu.py tests/test_bench_parity_gpu.py tests/test_store_gpu.py -x -q 2>&1 | tail -3
timeout 900 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu --no-e2e --no-secondary > gpurun_out/b4.json 2> gpurun_out/b4.err; echo c4=$?
python -c "
import json; d=json.load(open('gpurun_out/b4.json')); print('c4', round(d['value']), round(d['ms_per_step'],2), d['kernel_ms_one_step'])"
timeout 1500 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu --no-e2e --no-secondary > gpurun_out/b5.json 2> gpurun_out/b5.err; echo c5=$?
python -c "
import json; d=json.load(open('gpurun_out/b5.json')); print('c5', round(d['value']), round(d['ms_per_step'],1), d['kernel_ms_one_step'])"
