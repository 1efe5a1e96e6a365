# multi-kernel path: fit parity (all trainer shapes) + C4 quick bench
set -x
timeout 900 python -m pytest tests/test_fit_gpu.py tests/test_bench_parity_gpu.py -x -q 2>&1 | tail -3
timeout 900 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_c4q.json 2> gpurun_out/bench_c4q.err
python -c "import json; d=json.load(open('gpurun_out/bench_c4q.json')); print(d['ms_per_step'], d['kernel_ms_one_step'])"
