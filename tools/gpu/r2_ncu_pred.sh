# ncu --set full of the predict kernel (roofline probe: T=100 predict, fused score, T=1000 predict)
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:predict_kernel -s 4 -c 1 -f -o gpurun_out/prof_pred python tools/roofline_probe.py --families 8 --rows 65536 --trees 1000 --reps 1 > gpurun_out/ncu_pred.log 2>&1; echo ncu=$?
ncu -i gpurun_out/prof_pred.ncu-rep --page raw --csv > gpurun_out/pred_raw.csv 2>/dev/null; echo raw=$?
for i in 0 1 2 3 4; do ncu -i gpurun_out/prof_pred.ncu-rep --page source --csv --print-source sass --launch-skip $i --launch-count 1 > gpurun_out/pred_src_$i.csv 2>/dev/null; done; echo src=$?
ncu -i gpurun_out/prof_pred.ncu-rep --page details --csv > gpurun_out/pred_details.csv 2>/dev/null; echo det=$?
