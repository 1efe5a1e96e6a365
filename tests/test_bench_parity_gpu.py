"""Parity at the benchmark's own workloads (bench.py configs): every family of the round is fitted
on the GPU in one batched call and must reproduce the oracle's trees bit for bit, and the scored
pool's scores and (score, index) ranking must match. C1-C3 exercise the resident trainer (one CTA
per family), C4 (fewer trees, so the oracle finishes in seconds) the multi-kernel round."""
import numpy as np
import pytest

import bench
import oracle
import paper_2201_00194_b200 as fs

pytestmark = pytest.mark.gpu
FIELDS = ("offsets", "feature", "threshold", "left", "right", "value")


@pytest.mark.parametrize("cfg,trees,path", [("c1", 100, "auto"), ("c2", 100, "auto"), ("c3", 60, "auto"),
                                            ("c2", 30, "multi"), ("c4", 12, "auto")])
def test_bench_round_bit_exact(dev, orc, monkeypatch, cfg, trees, path):
    monkeypatch.setenv("FAMSEER_FIT_PATH", path)
    W = bench.build_workload(cfg, 1000)
    x = bench._featurize_host(W, orc)
    seg, y = W["tr_seg"], W["tr_y"]
    F = len(W["families"])
    fo = fs.Forest(dev, F)
    fo.fit(x, y, seg=list(seg), params=fs.GbtParams(trees, 3, 0.1, 2))
    sp = fs.Spaces(dev, W["spaces"])
    scores, perm = sp.score(fo, W["pool_so"], W["pool_a"], bench.PAD, W["pool_seg"])
    xp = None
    for f in range(F):
        a, b = int(seg[f]), int(seg[f + 1])
        exp = orc.fit(x[a:b], y[a:b], trees=trees)
        got = fo.export(f)
        assert got.base == exp.base, (cfg, f)
        for k in FIELDS:
            assert np.array_equal(getattr(got, k), getattr(exp, k)), (cfg, f, k)
        internal = exp.feature >= 0
        np.testing.assert_allclose(got.gain[internal], exp.gain[internal], rtol=1e-5, atol=0)
        # scoring: featurize + predict + rank of this family's pool
        pa, pb = int(W["pool_seg"][f]), int(W["pool_seg"][f + 1])
        if xp is None:
            xp = _featurize_pool(W, orc)
        s_exp = orc.predict(exp, xp[pa:pb])
        assert np.array_equal(scores[pa:pb], s_exp), (cfg, f)
        assert np.array_equal(perm[pa:pb], orc.rank(s_exp)), (cfg, f)


def _featurize_pool(W, orc):
    P = int(W["pool_seg"][-1])
    x = np.zeros((P, bench.PAD))
    for sid in np.unique(W["pool_so"]):
        rows = np.where(W["pool_so"] == sid)[0]
        kn = W["spaces"][sid]
        x[rows] = orc.featurize(kn, W["pool_a"][rows][:, : len(kn)], bench.PAD)
    return x


@pytest.mark.parametrize("cfg", ["c2", "c3"])
def test_score_fused_equals_featurize_then_predict(dev, orc, monkeypatch, cfg):
    """fs_score's fused descriptor path (no feature matrix) == featurize -> predict -> rank."""
    W = bench.build_workload(cfg, 7)
    x = bench._featurize_host(W, orc)
    F = len(W["families"])
    fo = fs.Forest(dev, F)
    fo.fit(x, W["tr_y"], seg=list(W["tr_seg"]), params=fs.GbtParams(40, 3, 0.1, 2))
    sp = fs.Spaces(dev, W["spaces"])
    s1, p1 = sp.score(fo, W["pool_so"], W["pool_a"], bench.PAD, W["pool_seg"])
    monkeypatch.setenv("FAMSEER_SCORE_UNFUSED", "1")
    s2, p2 = sp.score(fo, W["pool_so"], W["pool_a"], bench.PAD, W["pool_seg"])
    assert np.array_equal(s1, s2) and np.array_equal(p1, p2)
    xp = _featurize_pool(W, orc)
    s3 = fo.predict(xp, seg=list(W["pool_seg"]))
    assert np.array_equal(s1, s3)


def test_fit_records_equals_fit_on_featurized_rows(dev, orc):
    """fs_fit_records (descriptors, device featurize) == fs_fit on the host-featurized rows."""
    W = bench.build_workload("c3", 11)
    sp = fs.Spaces(dev, W["spaces"])
    F = len(W["families"])
    a = fs.Forest(dev, F)
    a.fit_records(sp, W["tr_so"], W["tr_a"], bench.PAD, W["tr_y"], seg=list(W["tr_seg"]),
                  params=fs.GbtParams(30, 3, 0.1, 2))
    b = fs.Forest(dev, F)
    b.fit(bench._featurize_host(W, orc), W["tr_y"], seg=list(W["tr_seg"]), params=fs.GbtParams(30, 3, 0.1, 2))
    for f in range(F):
        ea, eb = a.export(f), b.export(f)
        assert ea.base == eb.base
        for k in FIELDS:
            assert np.array_equal(getattr(ea, k), getattr(eb, k)), (f, k)


@pytest.mark.parametrize("cluster", ["1", "2", "4", "8"])
def test_resident_cluster_sizes_bit_exact(dev, orc, monkeypatch, cluster):
    """The resident trainer's thread-block-cluster shapes (histogram features dealt over 1, 2 or 4
    CTAs, bins exchanged through distributed shared memory) all reproduce the oracle's trees."""
    monkeypatch.setenv("FAMSEER_FIT_PATH", "resident")
    monkeypatch.setenv("FAMSEER_RES_CLUSTER", cluster)
    W = bench.build_workload("c2", 1000)
    x = bench._featurize_host(W, orc)
    seg, y = W["tr_seg"], W["tr_y"]
    F = len(W["families"])
    fo = fs.Forest(dev, F)
    fo.fit(x, y, seg=list(seg), params=fs.GbtParams(40, 3, 0.1, 2))
    for f in range(F):
        a, b = int(seg[f]), int(seg[f + 1])
        exp = orc.fit(x[a:b], y[a:b], trees=40)
        got = fo.export(f)
        assert got.base == exp.base, (cluster, f)
        for k in FIELDS:
            assert np.array_equal(getattr(got, k), getattr(exp, k)), (cluster, f, k)
        np.testing.assert_array_equal(fo.fit_stats(f)[0] + fo.fit_stats(f)[1] > 0, True)
