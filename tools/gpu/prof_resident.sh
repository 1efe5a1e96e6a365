# ncu full capture (with source) of one fit_resident launch at the bench's C2 workload
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fit_resident -c 1 -f -o gpurun_out/prof_fit_resident python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_full.log 2>&1; echo ncu=$?
