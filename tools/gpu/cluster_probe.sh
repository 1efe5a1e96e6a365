for cl in 1 2 4; do
  FAMSEER_RES_CLUSTER=$cl FAMSEER_LIB=$PWD/var/hprobe/libfamseer.so timeout 600 python bench.py --no-cpu --no-e2e --steps 3 > gpurun_out/ab.json 2> gpurun_out/ab.err || tail -5 gpurun_out/ab.err
  python - "$cl" <<'PY'
import json, sys
d = json.load(open('gpurun_out/ab.json'))
c = d['device_counters']
pr = c.get('probe'); ph = c.get('resident_phase_cycles_cta0')
passes = pr[3]
print('cluster', sys.argv[1], 'passes', passes, 'max warp loop/pass', pr[0], 'mean warp loop/pass', round(pr[1] / passes / 16), 'hist/pass', round(ph['hist'] / passes))
PY
done
