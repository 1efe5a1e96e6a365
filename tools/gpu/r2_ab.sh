# A/B of the resident trainer: phase counters + C2 bench value for the default build, var/* builds
# and AB_ENVS (space-separated VAR=value settings run on the default build)
abrun() {
  echo "== $1 $2"
  env FAMSEER_LIB=$PWD/$1 $2 timeout 300 python tools/phase_probe.py c2 2>&1 | head -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['resident_phase_cycles_cta0']; print({k: round(v/100) for k,v in p.items()}, 'sum', round(sum(p.values())/100))"
  env FAMSEER_LIB=$PWD/$1 $2 timeout 600 python bench.py --no-cpu --no-e2e --no-secondary ${BENCH_ARGS} > gpurun_out/ab.json 2> gpurun_out/ab.err || tail -3 gpurun_out/ab.err
  python -c "
import json; d=json.load(open('gpurun_out/ab.json')); print('value', round(d['value']), 'ms', round(d['ms_per_step'],3), 'fit_resident', d['kernel_ms_one_step'].get('fit_resident'))"
}
for lib in paper_2201_00194_b200/libfamseer.so var/*/libfamseer.so; do [ -f "$lib" ] && abrun $lib ""; done
for e in ${AB_ENVS}; do abrun paper_2201_00194_b200/libfamseer.so "$e"; done
