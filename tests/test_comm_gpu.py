"""fs_comm / fs_topk_allgather (the product's multi-GPU exchange) on the box's one
GPU as a world-size-1 NCCL communicator: the merged per-family top-g records must equal the
first g entries of fs_score's (score, index) permutation of every family, bit for bit, with -1
padding for short pools and absent families."""
import numpy as np
import pytest
import torch

import bench
import paper_2201_00194_b200 as fs
from paper_2201_00194_b200 import sharding

pytestmark = pytest.mark.gpu


def test_topk_allgather_world1_matches_score(dev):
    W = bench.build_workload("c2", seed=1000)
    F = len(W["families"])
    sp = fs.Spaces(dev, W["spaces"])
    fo = fs.Forest(dev, F)
    fo.fit_records(sp, W["tr_so"], W["tr_a"], bench.PAD, W["tr_y"], seg=W["tr_seg"], params=fs.GbtParams(20, 3, 0.1, 2))
    P = int(W["pool_seg"][-1])
    so = torch.from_numpy(W["pool_so"]).cuda()
    a = torch.from_numpy(W["pool_a"]).cuda()
    scores = torch.empty(P, dtype=torch.float64, device="cuda")
    perm = torch.empty(P, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    sp.score_d(fo, so, a, bench.PAD, W["pool_seg"], scores, perm)
    comm = fs.Comm(dev, 1, 0, fs.Comm.new_id())
    g, n_fam = 64, F + 2  # two families no rank owns: all -1
    merged = torch.empty((n_fam, g, 3), dtype=torch.float64, device="cuda")
    comm.topk_allgather(list(range(F)), W["pool_seg"], scores, perm, g, F, n_fam, merged)
    dev.check()
    torch.cuda.synchronize()
    got = merged.cpu().numpy()
    s, p = scores.cpu().numpy(), perm.cpu().numpy()
    exp = sharding.pack_topk(list(range(F)), W["pool_seg"], p, s, g)
    for f in range(F):
        a0, b0 = int(W["pool_seg"][f]), int(W["pool_seg"][f + 1])
        k = min(g, b0 - a0)
        assert np.array_equal(got[f, :k, 0], np.full(k, f))
        assert np.array_equal(got[f, :k, 1], p[a0:a0 + k].astype(np.float64))
        assert np.array_equal(got[f, :k, 2], s[a0 + p[a0:a0 + k]])
        assert (got[f, k:] == -1).all()
    assert (got[F:] == -1).all()
    assert exp.shape[0] == F * g
    comm.close()
    sp.close()
    fo.close()
