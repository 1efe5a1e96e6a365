# multi-kernel histogram variants: roofline probe (8 families x 65,536 rows, C5-like) and the C4 bench
for lib in var/p0/libfamseer.so paper_2201_00194_b200/libfamseer.so var/p2m1/libfamseer.so var/p3m1/libfamseer.so; do
  echo "== $lib"
  FAMSEER_LIB=$PWD/$lib timeout 600 python tools/roofline_probe.py --families 8 --rows 65536 --trees 200 > gpurun_out/rp.json 2> gpurun_out/rp.err || tail -3 gpurun_out/rp.err
  python -c "
import json; d=json.load(open('gpurun_out/rp.json')); print('probe hist_build', d['hist_build'], 'fit_kernels', {k: round(v,2) for k,v in d.get('fit_kernels_ms',{}).items()})"
  FAMSEER_LIB=$PWD/$lib timeout 600 python bench.py --config c4 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/c4.json 2> gpurun_out/c4.err || tail -3 gpurun_out/c4.err
  python -c "
import json; d=json.load(open('gpurun_out/c4.json')); print('c4 ms', round(d['ms_per_step'],2), 'hist', d['kernel_ms_one_step'].get('fit_hist_build'))"
done
