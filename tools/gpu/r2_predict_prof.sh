set -x
timeout 600 python tools/roofline_probe.py --families 8 --rows 65536 --trees 1000 > gpurun_out/roofline_r2.json
cat gpurun_out/roofline_r2.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:predict_kernel -s 1 -c 5 -o gpurun_out/prof_predict -f python tools/roofline_probe.py --families 8 --rows 65536 --trees 1000 --reps 1 > /dev/null 2> gpurun_out/ncu_predict.err; echo ncu=$?
timeout 900 python tools/engine_timing.py mobilenetv2_sim 10000 1 50 > gpurun_out/engine_timing_mb10k.json; cat gpurun_out/engine_timing_mb10k.json
timeout 900 python tools/engine_timing.py bert_base_sim 6000 1 50 > gpurun_out/engine_timing_bert6k.json; cat gpurun_out/engine_timing_bert6k.json
