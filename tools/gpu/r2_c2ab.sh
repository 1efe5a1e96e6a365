# C2 resident A/B: parity suites that reach the resident trainer, then phase counters + bench
set -x
timeout 900 python -m pytest tests/test_fit_gpu.py tests/test_full_golden_gpu.py tests/test_bench_parity_gpu.py tests/test_store_gpu.py -x -q 2>&1 | tail -2
bash tools/gpu/r2_ab.sh
