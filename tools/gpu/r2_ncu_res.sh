# ncu --set full with source counters of the C2 resident trainer (one launch)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fit_resident -s 1 -c 1 -f -o gpurun_out/prof_res_c2 python tools/phase_probe.py c2 > gpurun_out/ncu_res.log 2>&1; echo ncu=$?
ncu -i gpurun_out/prof_res_c2.ncu-rep --page source --csv --print-source sass > gpurun_out/res_src_sass.csv 2>/dev/null; echo src=$?
ncu -i gpurun_out/prof_res_c2.ncu-rep --page source --csv --print-source cuda > gpurun_out/res_src_cuda.csv 2>/dev/null; echo src2=$?
ls -la gpurun_out/
