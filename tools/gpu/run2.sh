set -x
for c in c1 c3; do timeout 600 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo $c=$?; done
timeout 900 python bench.py --config c4 --steps 3 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo c4=$?
timeout 600 python tools/roofline_probe.py --families 8 --rows 65536 --trees 1000 > gpurun_out/roofline_probe.json 2> gpurun_out/roofline_probe.err; echo probe=$?
timeout 1500 python bench.py --config c5 --steps 3 --warmup 3 --no-e2e > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo c5=$?
tail -c 3000 gpurun_out/bench_c5.err
