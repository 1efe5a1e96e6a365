# PDL A/B for the multi-kernel round (C4, C5): parity first, then bench with and without PDL.
set -x
timeout 1500 python -m pytest tests/test_fit_gpu.py tests/test_full_golden_gpu.py tests/test_bench_parity_gpu.py tests/test_store_gpu.py -x -q 2>&1 | tail -3
for mode in pdl nopdl pdl nopdl; do
  if [ $mode = nopdl ]; then export FAMSEER_NO_PDL=1; else unset FAMSEER_NO_PDL; fi
  timeout 900 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu --no-e2e --no-secondary > gpurun_out/b4_$mode.json 2> gpurun_out/b4_$mode.err
  python -c "
import json; d=json.load(open('gpurun_out/b4_$mode.json')); print('c4 $mode', round(d['value']), round(d['ms_per_step'],2))"
done
for mode in pdl nopdl; do
  if [ $mode = nopdl ]; then export FAMSEER_NO_PDL=1; else unset FAMSEER_NO_PDL; fi
  timeout 1500 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu --no-e2e --no-secondary > gpurun_out/b5_$mode.json 2> gpurun_out/b5_$mode.err
  python -c "
import json; d=json.load(open('gpurun_out/b5_$mode.json')); print('c5 $mode', round(d['value']), round(d['ms_per_step'],1))"
done
