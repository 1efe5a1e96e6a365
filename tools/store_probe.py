"""Where an incremental retrain's time goes: fs_store (append g records + refit) vs fs_fit_records
on the whole set, per kernel (CUDA events, no graphs) and host wall-clock per call. GPU box only."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2201_00194_b200 as fs  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
W = bench.build_workload(cfg, 1000)
dev = fs.Device(0)
sp = fs.Spaces(dev, W["spaces"])
seg = [int(v) for v in W["tr_seg"]]
F = len(seg) - 1
params = fs.GbtParams(W["trees"], 3, 0.1, 2)
g = 64
gf = [min(g, (seg[f + 1] - seg[f]) // 14) for f in range(F)]
live = [f for f in range(F) if gf[f] > 0]
so, asg, lat = W["tr_so"], W["tr_a"], W["tr_lat"]
st = fs.Store(dev, F, bench.PAD)
start = {f: seg[f + 1] - 12 * gf[f] for f in live}
idx0 = np.concatenate([np.arange(seg[f], start[f]) for f in live])
st.append_records(sp, live, so[idx0], asg[idx0], lat[idx0], seg=np.cumsum([0] + [start[f] - seg[f] for f in live]))
fo = fs.Forest(dev, F)
st.fit(fo, families=live, params=params)
tmp = fs.Store(dev, 1, 0)
tmp.append([0], np.zeros((len(lat), 0)), lat)
y = tmp.read(0)[1]
fo2 = fs.Forest(dev, F)
for k in range(6):
    idx = np.concatenate([np.arange(start[f] + k * gf[f], start[f] + (k + 1) * gf[f]) for f in live])
    sg = np.cumsum([0] + [gf[f] for f in live])
    if k >= 3:
        dev.profile("*")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st.append_records(sp, live, so[idx], asg[idx], lat[idx], seg=sg)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    st.fit(fo, families=live, params=params)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    if k >= 3:
        a = dev.profile_read()
        dev.profile("*")
    idf = np.concatenate([np.arange(seg[f], start[f] + (k + 1) * gf[f]) for f in live])
    sgf = np.cumsum([0] + [start[f] + (k + 1) * gf[f] - seg[f] for f in live])
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    fo2.fit_records(sp, so[idf], asg[idf], bench.PAD, y[idf], seg=list(sgf), params=params)
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    if k >= 3:
        b = dev.profile_read()
        dev.profile(None)
        print(f"step {k}: store append {1e3*(t1-t0):.3f} ms + fit {1e3*(t2-t1):.3f} ms | full fit_records {1e3*(t4-t3):.3f} ms")
        keys = sorted(set(a) | set(b), key=lambda kk: -max(a.get(kk, (0, 0))[1], b.get(kk, (0, 0))[1]))
        for kk in keys[:14]:
            print(f"   {kk:28s} store {a.get(kk, (0, 0))[1]:8.4f}  full {b.get(kk, (0, 0))[1]:8.4f}")
