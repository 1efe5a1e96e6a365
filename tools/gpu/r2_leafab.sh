for e in "" "FAMSEER_LEAF_WARP=1"; do
  env $e timeout 900 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu --no-e2e --no-secondary > gpurun_out/b4.json 2> gpurun_out/b4.err
  python -c "
import json; d=json.load(open('gpurun_out/b4.json')); k=d['kernel_ms_one_step']; print('c4 [$e]', round(d['ms_per_step'],2), 'leaf', k.get('fit_leaf'))"
  env $e timeout 1500 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu --no-e2e --no-secondary > gpurun_out/b5.json 2> gpurun_out/b5.err
  python -c "
import json; d=json.load(open('gpurun_out/b5.json')); k=d['kernel_ms_one_step']; print('c5 [$e]', round(d['ms_per_step'],1), 'leaf', k.get('fit_leaf'))"
done
