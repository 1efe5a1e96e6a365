for tc in 256 128 64; do FAMSEER_PREDICT_TC=$tc timeout 600 python tools/roofline_probe.py --families 8 --rows 65536 --trees 1000 > gpurun_out/rp_$tc.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/rp_$tc.json')); print($tc, {k: (round(v['ms'],4), round(v['gbs'],1)) for k,v in d.items() if isinstance(v, dict) and 'gbs' in v and k!='hist_build' and k!='featurize'})"; done
