"""Host cost of exporting every family after a tuning step (C2): first export after the step
(materialises all families) vs a repeat."""
import sys, time, numpy as np, ctypes as C
sys.path.insert(0, '.')
import bench, paper_2201_00194_b200 as fs
from paper_2201_00194_b200 import _capi
W = bench.build_workload('c2', 1000)
dev = fs.Device(0); sp = fs.Spaces(dev, W['spaces']); F = len(W['families'])
fo = fs.Forest(dev, F); p = fs.GbtParams(100, 3, 0.1, 2)
pin = lambda a: np.ascontiguousarray(a)
h_so, h_a, h_tso, h_ta, h_y = (pin(W[k]) for k in ('pool_so', 'pool_a', 'tr_so', 'tr_a', 'tr_y'))
fo.fit_records(sp, h_tso, h_ta, bench.PAD, h_y, seg=W['tr_seg'], params=p)
res = {'py_export': [], 'sizes_only': []}
for it in range(8):
    fo.tune_step(sp, h_so, h_a, bench.PAD, W['pool_seg'], h_tso, h_ta, h_y, W['tr_seg'], params=p)
    t0 = time.perf_counter()
    for f in range(F): fo.export(f)
    t1 = time.perf_counter()
    res['py_export'].append(t1 - t0)
    # second round: already materialised
    t0 = time.perf_counter()
    for f in range(F): fo.export(f)
    t1 = time.perf_counter()
    res['sizes_only'].append(t1 - t0)
print({k: round(1e3 * float(np.median(v[2:])), 3) for k, v in res.items()})
