"""Per-phase cycle breakdown of the resident trainer (CTA 0) for a bench workload, every device
counter (incl. the FS_RES_HIST_PROBE slots) printed raw: python tools/phase_probe.py c2"""
import sys, json, numpy as np
sys.path.insert(0, '.')
import bench, paper_2201_00194_b200 as fs, torch
W = bench.build_workload(sys.argv[1] if len(sys.argv) > 1 else 'c2', 1000)
dev = fs.Device(0); sp = fs.Spaces(dev, W['spaces']); F = len(W['families'])
x = sp.featurize(W['tr_so'], W['tr_a'], 164)
fo = fs.Forest(dev, F)
fo.fit(x, W['tr_y'], seg=W['tr_seg'], params=fs.GbtParams(W['trees'], 3, 0.1, 2))
dev.counters(reset=True)
torch.cuda.synchronize()
import time
t0 = time.perf_counter()
fo.fit(x, W['tr_y'], seg=W['tr_seg'], params=fs.GbtParams(W['trees'], 3, 0.1, 2))
t1 = time.perf_counter()
print(json.dumps(dev.counters()))
print('fit wall ms', round((t1 - t0) * 1e3, 3))
print(W['families'], np.diff(W['tr_seg']).tolist())
