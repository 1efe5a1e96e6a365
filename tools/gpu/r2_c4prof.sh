# C4 multi-kernel round: launch list (20-tree fit) + ncu --set full of the leaf and exact_small kernels
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4_fit20.csv python tools/fit_once.py c4 20 > /dev/null 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:leaf_cta -s 20 -c 1 -f -o gpurun_out/prof_leaf_c4 python tools/fit_once.py c4 20 > /dev/null 2>&1; echo ncu2=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:exact_small -s 20 -c 1 -f -o gpurun_out/prof_exsmall_c4 python tools/fit_once.py c4 20 > /dev/null 2>&1; echo ncu3=$?
for r in prof_leaf_c4 prof_exsmall_c4; do ncu -i gpurun_out/$r.ncu-rep --page source --csv --print-source sass > gpurun_out/${r}_src.csv 2>/dev/null; ncu -i gpurun_out/$r.ncu-rep --page details --csv > gpurun_out/${r}_details.csv 2>/dev/null; done
