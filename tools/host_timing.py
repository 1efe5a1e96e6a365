"""Host-side stage timing of one fs_fit at a bench workload (FAMSEER_HOST_TIMING diagnostics)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2201_00194_b200 as fs  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
W = bench.build_workload(cfg, 1000)
dev = fs.Device(0)
sp = fs.Spaces(dev, W["spaces"])
N = int(W["tr_seg"][-1])
x = torch.empty((N, bench.PAD), dtype=torch.float64, device="cuda")
so = torch.from_numpy(W["tr_so"]).cuda()
a = torch.from_numpy(W["tr_a"]).cuda()
y = torch.from_numpy(W["tr_y"]).cuda()
torch.cuda.synchronize()
sp.featurize_d(so, a, bench.PAD, x)
fo = fs.Forest(dev, len(W["families"]))
p = fs.GbtParams(W["trees"], 3, 0.1, 2)
for i in range(3):
    if i == 2:
        os.environ["FAMSEER_HOST_TIMING"] = "1"
    fo.fit_d(x, y, W["tr_seg"], p)
    dev.check()
