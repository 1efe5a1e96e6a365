# C4/C5 bench for the default build and every var/*/libfamseer.so variant
for lib in ${VAB_LIBS:-paper_2201_00194_b200/libfamseer.so var/*/libfamseer.so}; do
  for c in c4 c5; do
    st=3; [ $c = c5 ] && st=2
    FAMSEER_LIB=$PWD/$lib timeout 1500 python bench.py --config $c --steps $st --warmup 3 --no-cpu --no-e2e --no-secondary > gpurun_out/vab.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/vab.json')); k=d['kernel_ms_one_step']; print('$lib $c', round(d['value']), round(d['ms_per_step'],1), 'leaf', k.get('fit_leaf'), 'exact', k.get('fit_exact'))"
  done
done
