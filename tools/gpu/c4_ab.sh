for lib in var/prev/libfamseer.so paper_2201_00194_b200/libfamseer.so var/prev/libfamseer.so paper_2201_00194_b200/libfamseer.so; do
  FAMSEER_LIB=$PWD/$lib timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/c4.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/c4.json')); print('$lib', round(d['ms_per_step'],2), round(d['kernel_ms_one_step']['fit_rounds'],2))"
done
