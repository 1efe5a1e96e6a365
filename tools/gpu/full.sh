# Full measurement pass (round evidence): benches per config, reference arm, launch list, ncu captures.
set -x
nvidia-smi --query-gpu=name,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo c2=$?
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_c2.json 2> gpurun_out/bench_ref_c2.err; echo ref=$?
for c in c1 c3; do timeout 600 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo $c=$?; done
timeout 900 python bench.py --config c4 --steps 3 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo c4=$?
timeout 1800 python bench.py --config c5 --steps 3 --warmup 3 --no-e2e > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo c5=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$?
bash tools/gpu/prof_resident.sh
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hist_build_atomic -c 1 -f -o gpurun_out/prof_hist_c5 python tools/fit_once.py c5 2 > gpurun_out/ncu_hist.log 2>&1; echo ncu3=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:predict_heap -c 1 -f -o gpurun_out/prof_score_c2 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_score.log 2>&1; echo ncu4=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4_fit.csv python tools/fit_once.py c4 20 > /dev/null 2>&1; echo ncu5=$?
timeout 600 python tools/roofline_probe.py --families 8 --rows 65536 --trees 1000 > gpurun_out/roofline_probe.json 2> gpurun_out/roofline_probe.err; echo probe=$?
