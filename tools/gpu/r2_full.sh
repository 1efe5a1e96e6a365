# Round-2 evidence pass: smoke, GPU suite, bench lines per config, reference arm, 2-rank
# family-sharded run, launch lists, ncu --set full of the dominant kernels, roofline probe.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo c2=$?
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_c2.json 2> gpurun_out/bench_ref_c2.err; echo ref=$?
for c in c1 c3; do timeout 600 python bench.py --config $c --no-secondary > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo $c=$?; done
timeout 900 python bench.py --config c4 --steps 3 --warmup 3 --no-secondary > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo c4=$?
timeout 1500 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu --no-e2e --no-secondary > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo c5=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4_fit20.csv python tools/fit_once.py c4 20 > /dev/null 2>&1; echo ncu_c4=$?
FAMSEER_BENCH_SHARE_GPU=1 timeout 600 python bench.py --gpus 2 --no-cpu --no-e2e --no-secondary > gpurun_out/bench_n2_shared.json 2> gpurun_out/bench_n2_shared.err; echo n2=$?
timeout 600 python tools/roofline_probe.py --families 8 --rows 65536 --trees 1000 > gpurun_out/roofline_probe.json 2> gpurun_out/roofline_probe.err; echo probe=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-secondary > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$?
bash tools/gpu/prof_resident.sh
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hist_build_atomic -c 1 -f -o gpurun_out/prof_hist_c5 python tools/fit_once.py c5 2 > gpurun_out/ncu_hist.log 2>&1; echo ncu3=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:predict_kernel -s 1 -c 1 -f -o gpurun_out/prof_predict python tools/roofline_probe.py --families 8 --rows 65536 --trees 1000 --reps 1 > gpurun_out/ncu_pred.log 2>&1; echo ncu4=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:predict_kernel -c 1 -f -o gpurun_out/prof_score_c2 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-secondary > gpurun_out/ncu_score.log 2>&1; echo ncu5=$?
for r in prof_fit_resident prof_hist_c5 prof_predict prof_score_c2; do ncu -i gpurun_out/$r.ncu-rep --page details --csv > gpurun_out/${r}_details.csv 2>/dev/null; ncu -i gpurun_out/$r.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum > gpurun_out/${r}_dram.csv 2>/dev/null; done
cat gpurun_out/bench_c2.json
