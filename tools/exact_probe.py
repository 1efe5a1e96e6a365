"""Exact-fold share of a multi-kernel fit (C4/C5 workloads): per-kernel CUDA-event times of one
warm fit with T trees, and the device counters (exact nodes / chains). GPU box only:
    FAMSEER_NO_GRAPH=1 python tools/exact_probe.py c5 50"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2201_00194_b200 as fs  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
trees = int(sys.argv[2]) if len(sys.argv) > 2 else 50
W = bench.build_workload(cfg, 1000)
dev = fs.Device(0)
sp = fs.Spaces(dev, W["spaces"])
N = int(W["tr_seg"][-1])
x = torch.empty((N, bench.PAD), dtype=torch.float64, device="cuda")
so = torch.from_numpy(W["tr_so"]).cuda()
a = torch.from_numpy(W["tr_a"]).cuda()
y = torch.from_numpy(W["tr_y"]).cuda()
sp.featurize_d(so, a, bench.PAD, x)
fo = fs.Forest(dev, len(W["families"]))
p = fs.GbtParams(trees, 3, 0.1, 2)
fo.fit_d(x, y, W["tr_seg"], p)
dev.check()
dev.counters(reset=True)
dev.profile("*")
fo.fit_d(x, y, W["tr_seg"], p)
dev.check()
prof = dev.profile_read()
dev.profile(None)
c = dev.counters(reset=True)
print({k: round(v[1], 2) for k, v in sorted(prof.items(), key=lambda kv: -kv[1][1])[:12]})
print({k: c[k] for k in ("exact_chains", "exact_nodes")}, c.get("exact_reasons"))
