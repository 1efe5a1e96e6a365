"""fs_tune_step (one tuning round, scheduler.cpp:187-192 + :233-238, with the scoring forked
onto a second stream while the refit runs): scores / permutation must equal fs_score with the
models as they were BEFORE the refit, and the refit models must equal a plain fs_fit /
fs_fit_records on the same rows - bit for bit, host and device variants, over several rounds."""
import numpy as np
import pytest
import torch

import bench
import paper_2201_00194_b200 as fs

pytestmark = pytest.mark.gpu
FIELDS = ("offsets", "feature", "threshold", "left", "right", "value")


@pytest.fixture(scope="module")
def c2(dev):
    W = bench.build_workload("c2", seed=1000)
    sp = fs.Spaces(dev, W["spaces"])
    yield W, sp
    sp.close()


def _same_models(a, b, F):
    for f in range(F):
        ea, eb = a.export(f), b.export(f)
        assert ea.base == eb.base
        for k in FIELDS:
            assert np.array_equal(getattr(ea, k), getattr(eb, k)), (f, k)


def test_tune_step_host_equals_score_then_fit(dev, c2):
    W, sp = c2
    F = len(W["families"])
    p = fs.GbtParams(30, 3, 0.1, 2)
    ref, got = fs.Forest(dev, F), fs.Forest(dev, F)
    rng = np.random.default_rng(5)
    for rnd in range(3):  # the models change every round: round r scores with round r-1's refit
        y = W["tr_y"] + rng.normal(0, 0.01, len(W["tr_y"])) * rnd
        if rnd == 0:
            for fo in (ref, got):
                fo.fit_records(sp, W["tr_so"], W["tr_a"], bench.PAD, W["tr_y"], seg=W["tr_seg"], params=p)
            continue
        s0, p0 = sp.score(ref, W["pool_so"], W["pool_a"], bench.PAD, W["pool_seg"])
        ref.fit_records(sp, W["tr_so"], W["tr_a"], bench.PAD, y, seg=W["tr_seg"], params=p)
        s1, p1 = got.tune_step(sp, W["pool_so"], W["pool_a"], bench.PAD, W["pool_seg"], W["tr_so"], W["tr_a"], y,
                               W["tr_seg"], params=p)
        assert np.array_equal(s0, s1) and np.array_equal(p0, p1), rnd
        _same_models(ref, got, F)
    ref.close()
    got.close()


def test_tune_step_device_equals_score_then_fit(dev, c2):
    W, sp = c2
    F = len(W["families"])
    p = fs.GbtParams(30, 3, 0.1, 2)
    N, P = int(W["tr_seg"][-1]), int(W["pool_seg"][-1])
    so = torch.from_numpy(W["pool_so"]).cuda()
    a = torch.from_numpy(W["pool_a"]).cuda()
    x = torch.from_numpy(sp.featurize(W["tr_so"], W["tr_a"], bench.PAD)).cuda()
    y = torch.from_numpy(W["tr_y"]).cuda()
    y2 = torch.from_numpy(W["tr_y"] * 1.01).cuda()
    torch.cuda.synchronize()
    ref, got = fs.Forest(dev, F), fs.Forest(dev, F)
    for fo in (ref, got):
        fo.fit_d(x, y, W["tr_seg"], p)
    s_ref = torch.empty(P, dtype=torch.float64, device="cuda")
    p_ref = torch.empty(P, dtype=torch.int32, device="cuda")
    s_got, p_got = torch.empty_like(s_ref), torch.empty_like(p_ref)
    torch.cuda.synchronize()
    sp.score_d(ref, so, a, bench.PAD, W["pool_seg"], s_ref, p_ref)
    ref.fit_d(x, y2, W["tr_seg"], p)
    got.tune_step_d(sp, so, a, bench.PAD, W["pool_seg"], s_got, p_got, x, y2, W["tr_seg"], params=p)
    dev.check()
    torch.cuda.synchronize()
    assert torch.equal(s_ref, s_got) and torch.equal(p_ref, p_got)
    _same_models(ref, got, F)
    ref.close()
    got.close()


def test_tune_step_errors_join(dev, c2):
    """A bad pool descriptor raises from the host variant, and the forest stays usable."""
    W, sp = c2
    F = len(W["families"])
    fo = fs.Forest(dev, F)
    p = fs.GbtParams(10, 3, 0.1, 2)
    fo.fit_records(sp, W["tr_so"], W["tr_a"], bench.PAD, W["tr_y"], seg=W["tr_seg"], params=p)
    bad = W["pool_a"].copy()
    bad[3, 0] = 999
    with pytest.raises(fs.InvalidArgument):
        fo.tune_step(sp, W["pool_so"], bad, bench.PAD, W["pool_seg"], W["tr_so"], W["tr_a"], W["tr_y"],
                     W["tr_seg"], params=p)
    s, _ = sp.score(fo, W["pool_so"], W["pool_a"], bench.PAD, W["pool_seg"])
    assert np.isfinite(s).all()
    fo.close()
