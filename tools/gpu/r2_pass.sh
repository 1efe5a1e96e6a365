# Round-2 evidence pass: smoke, full GPU suite, default bench line, reference arm, 2-rank family
# sharded run on the one GPU, launch list of the C2 step.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 2400 python -m pytest tests -m gpu -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -15 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo bench=$?
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_c2.json 2> gpurun_out/bench_ref_c2.err; echo ref=$?
FAMSEER_BENCH_SHARE_GPU=1 timeout 600 python bench.py --gpus 2 --no-cpu --no-e2e --no-secondary > gpurun_out/bench_n2_shared.json 2> gpurun_out/bench_n2_shared.err; echo bench2=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-secondary > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$?
tail -3 gpurun_out/bench_c2.err gpurun_out/bench_n2_shared.err
cat gpurun_out/bench_c2.json gpurun_out/bench_ref_c2.json
