timeout 900 ncu --set full --clock-control none --import-source on -k regex:leaf_cta -s 2 -c 1 -f -o gpurun_out/prof_leaf_c5 python tools/fit_once.py c5 3 > /dev/null 2>&1; echo ncu=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:partition -s 4 -c 2 -f -o gpurun_out/prof_part_c5 python tools/fit_once.py c5 3 > /dev/null 2>&1; echo ncu=$?
for r in prof_leaf_c5 prof_part_c5; do ncu -i gpurun_out/$r.ncu-rep --page source --csv --print-source sass > gpurun_out/${r}_src.csv 2>/dev/null; ncu -i gpurun_out/$r.ncu-rep --page details --csv > gpurun_out/${r}_details.csv 2>/dev/null; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5_fit3.csv python tools/fit_once.py c5 3 > /dev/null 2>&1; echo ncu=$?
