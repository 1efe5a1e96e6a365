"""Host-side split of bench.py's e2e step (C2): fs_tune_step (host pointers) vs the model export."""
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import bench, paper_2201_00194_b200 as fs
W = bench.build_workload('c2', 1000)
dev = fs.Device(0); sp = fs.Spaces(dev, W['spaces']); F = len(W['families'])
fo = fs.Forest(dev, F); p = fs.GbtParams(100, 3, 0.1, 2)
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
h_so, h_a, h_tso, h_ta, h_y = (pin(W[k]) for k in ('pool_so', 'pool_a', 'tr_so', 'tr_a', 'tr_y'))
fo.fit_records(sp, h_tso, h_ta, bench.PAD, h_y, seg=W['tr_seg'], params=p)
T = {'tune': [], 'export': [], 'total': []}
for it in range(12):
    t0 = time.perf_counter()
    s, pm = fo.tune_step(sp, h_so, h_a, bench.PAD, W['pool_seg'], h_tso, h_ta, h_y, W['tr_seg'], params=p)
    t1 = time.perf_counter()
    for f in range(F):
        e = fo.export(f)
    t2 = time.perf_counter()
    if it >= 2:
        T['tune'].append(t1 - t0); T['export'].append(t2 - t1); T['total'].append(t2 - t0)
print({k: round(1e3 * float(np.median(v)), 3) for k, v in T.items()})
