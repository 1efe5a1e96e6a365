# Probes: resident phase counters under the A/B probe builds (var/*), roofline probe at T=100/1000.
set -x
for lib in paper_2201_00194_b200/libfamseer.so var/*/libfamseer.so; do
  echo "== $lib"; FAMSEER_LIB=$PWD/$lib timeout 300 python tools/phase_probe.py c2 2>&1 | tail -3
done
timeout 600 python tools/roofline_probe.py --families 8 --rows 65536 --trees 1000 > gpurun_out/roofline_r2.json 2> gpurun_out/roofline_r2.err; echo probe=$?
cat gpurun_out/roofline_r2.json; tail -3 gpurun_out/roofline_r2.err
