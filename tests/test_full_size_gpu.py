"""Full-size checks (BASELINE.json configs C4/C5) through size-independent properties - the
oracle cannot fit these sizes in test time, so the trainer is held to what the reference
guarantees (costmodel_test.cpp:121-202, acceptance_test.cpp:342-356) at scale:
  * bitwise determinism of a refit (costmodel_test.cpp:121-130);
  * bitwise invariance to the order of the training rows (:132-145; the canonical row order);
  * family independence: a family fitted inside a batch == the same family fitted alone;
  * training MSE non-increasing per round (:185-202);
  * predict() on the training rows reproduces the last training MSE (trainer and predict agree
    on every leaf and the tree-order fold)."""
import numpy as np
import pytest

import bench
import paper_2201_00194_b200 as fs

pytestmark = pytest.mark.gpu
FIELDS = ("offsets", "feature", "threshold", "left", "right", "value")


def _fit(dev, sp, W, trees, so, a, y, seg):
    fo = fs.Forest(dev, len(seg) - 1)
    fo.fit_records(sp, so, a, bench.PAD, y, seg=list(seg), params=fs.GbtParams(trees, 3, 0.1, 2))
    return fo


def _same(m1, m2):
    assert m1.base == m2.base
    for k in FIELDS:
        assert np.array_equal(getattr(m1, k), getattr(m2, k)), k


@pytest.mark.parametrize("cfg,trees,check_fams", [("c4", 500, [0, 1, 2]), ("c5", 100, [0, 17, 63])])
def test_full_size_properties(dev, cfg, trees, check_fams):
    W = bench.build_workload(cfg, 1000)
    sp = fs.Spaces(dev, W["spaces"])
    so, a, y, seg = W["tr_so"], W["tr_a"], W["tr_y"], W["tr_seg"]
    fo1 = _fit(dev, sp, W, trees, so, a, y, seg)
    fo2 = _fit(dev, sp, W, trees, so, a, y, seg)
    # rows permuted inside every family
    rng = np.random.default_rng(3)
    perm = np.concatenate([seg[f] + rng.permutation(seg[f + 1] - seg[f]) for f in range(len(seg) - 1)])
    fo3 = _fit(dev, sp, W, trees, so[perm], a[perm], y[perm], seg)
    x = sp.featurize(so, a, bench.PAD)
    pred = fo1.predict(x, seg=list(seg))
    for f in check_fams:
        e1 = fo1.export(f)
        _same(e1, fo2.export(f))
        _same(e1, fo3.export(f))
        lo, hi = int(seg[f]), int(seg[f + 1])
        alone = _fit(dev, sp, W, trees, so[lo:hi], a[lo:hi], y[lo:hi], [0, hi - lo])
        _same(e1, alone.export(0))
        assert np.all(np.diff(e1.mse) <= 1e-12 * np.abs(e1.mse[:-1]))
        err = y[lo:hi] - pred[lo:hi]
        np.testing.assert_allclose(np.mean(err * err), e1.mse[-1], rtol=1e-12)
