"""fs_score_index: candidates as (space id, u64 linear_index) descriptors,
decoded on the device like candidate_from_index (searchspace.cpp:56-66). Scores and the
(score, index) permutation must be bit-identical to fs_score on the equivalent int32[16]
assignments (itself pinned to the oracle) and to the oracle's featurize -> predict -> rank, on
every path: fused (default), unfused featurize -> predict (FAMSEER_SCORE_UNFUSED=1), host and
device pointers."""
import numpy as np
import pytest
import torch

import bench
import paper_2201_00194_b200 as fs

pytestmark = pytest.mark.gpu


def _indices(orc, W, so, a):
    idx = np.zeros(len(so), np.uint64)
    for sid in np.unique(so):
        rows = np.where(so == sid)[0]
        nv = [len(v) for v in W["spaces"][sid]]
        idx[rows] = orc.linear_index(nv, a[rows][:, : len(nv)])
    return idx


@pytest.fixture(scope="module")
def c2(dev, orc):
    W = bench.build_workload("c2", seed=1000)
    sp = fs.Spaces(dev, W["spaces"])
    fo = fs.Forest(dev, len(W["families"]))
    fo.fit_records(sp, W["tr_so"], W["tr_a"], bench.PAD, W["tr_y"], seg=W["tr_seg"], params=fs.GbtParams(40, 3, 0.1, 2))
    idx = _indices(orc, W, W["pool_so"], W["pool_a"])
    yield W, sp, fo, idx
    sp.close()
    fo.close()


def test_index_roundtrip_matches_assignments(c2, orc):
    W, _, _, idx = c2
    so, a = W["pool_so"], W["pool_a"]
    for sid in np.unique(so)[:8]:
        rows = np.where(so == sid)[0]
        nv = [len(v) for v in W["spaces"][sid]]
        assert np.array_equal(orc.candidate_from_index(nv, idx[rows]), a[rows])


@pytest.mark.parametrize("unfused", [False, True])
def test_score_index_equals_score(c2, monkeypatch, unfused):
    W, sp, fo, idx = c2
    if unfused:
        monkeypatch.setenv("FAMSEER_SCORE_UNFUSED", "1")
    s0, p0 = sp.score(fo, W["pool_so"], W["pool_a"], bench.PAD, W["pool_seg"])
    s1, p1 = sp.score_index(fo, W["pool_so"], idx, bench.PAD, W["pool_seg"])
    assert np.array_equal(s0, s1)
    assert np.array_equal(p0, p1)


def test_score_index_device_pointers(c2):
    W, sp, fo, idx = c2
    s0, p0 = sp.score_index(fo, W["pool_so"], idx, bench.PAD, W["pool_seg"])
    so = torch.from_numpy(W["pool_so"]).cuda()
    ix = torch.from_numpy(idx.view(np.int64)).cuda()
    st = torch.empty(len(idx), dtype=torch.float64, device="cuda")
    pt = torch.empty(len(idx), dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    sp.score_index_d(fo, so, ix, bench.PAD, W["pool_seg"], st, pt)
    sp.dev.check()
    assert np.array_equal(st.cpu().numpy(), s0)
    assert np.array_equal(pt.cpu().numpy(), p0)


def test_score_index_matches_oracle(dev, orc):
    knobs = [[1, 2, 4, 7, 8, 14], [1, 2, 4, 8, 16, 32], [1, 2, 4]]
    rng = np.random.default_rng(3)
    a = np.zeros((300, 16), np.int32)
    a[:, :3] = np.stack([rng.integers(0, len(v), 300) for v in knobs], 1)
    x = orc.featurize(knobs, a[:, :3], 164)
    y = np.log(1.0 + x[:, 0] * 0.3 + x[:, 4] ** 2)
    ens = orc.fit(x, y, trees=30)
    sp = fs.Spaces(dev, [knobs])
    fo = fs.Forest(dev, 1)
    fo.upload(0, ens)
    idx = orc.linear_index([len(v) for v in knobs], a[:, :3])
    s, p = sp.score_index(fo, np.zeros(300, np.int32), idx, 164, [0, 300])
    exp = orc.predict(ens, x)
    assert np.array_equal(s, exp)
    assert np.array_equal(p, orc.rank(exp))
    sp.close()
    fo.close()
