"""GPU predict (kernel 2) vs the oracle and the reference's golden scores: scores and leaf
indices bit-exact (costmodel.cpp:135-143, 237-246)."""
import numpy as np
import pytest

import oracle
import paper_2201_00194_b200 as fs
from common import GOLDEN

pytestmark = pytest.mark.gpu
G = np.load(f"{GOLDEN}/golden.npz")
CASES = [str(t) for t in G["fit_cases"]]


def golden_ens(tag):
    return oracle.Ensemble(float(G[f"fit_{tag}_base"][0]), 0.1, G[f"fit_{tag}_offsets"], G[f"fit_{tag}_feature"],
                           G[f"fit_{tag}_threshold"], G[f"fit_{tag}_left"], G[f"fit_{tag}_right"],
                           G[f"fit_{tag}_value"])


def leaf_ids(orc, ens, x):
    return orc.predict(ens, x, leaves=True)[1]


@pytest.mark.parametrize("tag", CASES)
def test_golden_models(dev, orc, tag):
    ens = golden_ens(tag)
    fo = fs.Forest(dev, 1)
    fo.upload(0, ens)
    x = G[f"fit_{tag}_x"]
    s, lo = fo.predict(x, leaves=True)
    assert np.array_equal(s, G[f"fit_{tag}_pred"])
    if ens.n_trees:
        assert np.array_equal(lo[: x.shape[0] * ens.n_trees].reshape(x.shape[0], ens.n_trees), leaf_ids(orc, ens, x))


def test_hand_built_models(dev):
    fo = fs.Forest(dev, 2)
    fo.upload(0, oracle.empty_ensemble())  # costmodel_test.cpp:77-83: fresh model -> 0.0
    one = oracle.Ensemble(0.0, 0.1, np.array([0, 1], np.int32), np.array([-1], np.int32), np.zeros(1),
                          np.array([-1], np.int32), np.array([-1], np.int32), np.array([7.0]))
    fo.upload(1, one)  # :98-105 single leaf -> 0.1*7.0
    s = fo.predict(np.array([[1.0, 2.0, 3.0], [9.0, -4.0, 0.5], [1.0, 0, 0]]), seg=[0, 2, 3])
    assert s[0] == 0.0 and s[1] == 0.0 and s[2] == 0.1 * 7.0
    with pytest.raises(fs.InvalidArgument):  # :238-240
        fo.predict(np.array([[np.nan, 0.0, 0.0]]), seg=[0, 0, 1])
    with pytest.raises(fs.InvalidArgument):
        fo.predict(np.array([[np.inf, 0.0, 0.0]]), seg=[0, 1, 1])


def random_forest(rng, d, trees, depth, n_thr=6, ragged=True):
    off, feat, thr, le, ri, val = [0], [], [], [], [], []
    grid = {f: np.sort(rng.normal(0, 1, n_thr)) for f in range(d)}

    def build(nodes, lvl):
        i = len(nodes)
        nodes.append(None)
        if lvl == depth or (ragged and lvl > 0 and rng.random() < 0.2):
            nodes[i] = (-1, 0.0, -1, -1, float(rng.normal()))
            return i
        f = int(rng.integers(0, d))
        t = float(rng.choice(grid[f]))
        a = build(nodes, lvl + 1)
        b = build(nodes, lvl + 1)
        nodes[i] = (f, t, a, b, 0.0)
        return i

    for _ in range(trees):
        nodes = []
        build(nodes, 0)
        for n in nodes:
            feat.append(n[0]), thr.append(n[1]), le.append(n[2]), ri.append(n[3]), val.append(n[4])
        off.append(len(feat))
    return oracle.Ensemble(float(rng.normal()), 0.1, np.array(off, np.int32), np.array(feat, np.int32),
                           np.array(thr), np.array(le, np.int32), np.array(ri, np.int32), np.array(val))


@pytest.mark.parametrize("depth,trees,n_thr,d,rows", [(3, 200, 6, 40, 700), (1, 10, 3, 40, 700), (5, 50, 8, 40, 700),
                                                      (3, 300, 2000, 2, 700), (10, 5, 4, 40, 700),
                                                      (3, 1200, 40000, 2, 700), (7, 30, 6, 40, 700),
                                                      (8, 20, 6, 40, 700), (4, 64, 6, 41, 700),
                                                      (3, 100, 6, 164, 40000), (3, 33, 6, 41, 40000)])
def test_random_forests_multi_segment(dev, orc, depth, trees, n_thr, d, rows):
    # (3, 300, 2000, 2): >254 distinct thresholds per feature -> 16-bit codes
    # (10, 5, 4, 40): deeper than the heap limit -> generic pre-order kernel
    # (3, 1200, 40000, 2): > 6144 unique thresholds -> threshold tables searched in global memory
    # (7/8, ...): deepest heap trees - pre-order leaf ids above 255 (uint16 leaf ids)
    # (4, 64, 6, 41): levels below the register-held top three; odd row width (no bulk row copies)
    # (3, 100, 6, 164, 40000): 256-candidate tiles, bulk-copied rows with a partial last stage;
    # (3, 33, 6, 41, 40000): the same with coalesced row loads and a partial last tree pass
    rng = np.random.default_rng(depth * 100 + trees)
    ens = [random_forest(rng, d, trees, depth, n_thr) for _ in range(3)]
    fo = fs.Forest(dev, 3)
    for i, e in enumerate(ens):
        fo.upload(i, e)
    seg = [0, rows, rows + 1, rows + 1 + 300]
    # rows hit thresholds exactly sometimes (x == t must go left)
    x = rng.normal(0, 1, size=(seg[-1], d))
    for f in range(d):
        hits = rng.random(seg[-1]) < 0.2
        pool = np.concatenate([e.threshold[e.feature == f] for e in ens] + [np.zeros(1)])
        x[hits, f] = rng.choice(pool, hits.sum())
    s, lo = fo.predict(x, seg=seg, leaves=True)
    off = 0
    for i, e in enumerate(ens):
        rows = x[seg[i]: seg[i + 1]]
        es, el = orc.predict(e, rows, leaves=True)
        assert np.array_equal(s[seg[i]: seg[i + 1]], es)
        n = rows.shape[0] * e.n_trees
        assert np.array_equal(lo[off: off + n].reshape(rows.shape[0], e.n_trees), el)
        off += n


def test_signed_zero_thresholds(dev, orc):
    # x = -0.0 against threshold +0.0 (and vice versa) must go left: -0.0 <= 0.0
    e = oracle.Ensemble(0.0, 0.1, np.array([0, 3, 6], np.int32), np.array([0, -1, -1, 0, -1, -1], np.int32),
                        np.array([0.0, 0, 0, -0.0, 0, 0]), np.array([1, -1, -1, 1, -1, -1], np.int32),
                        np.array([2, -1, -1, 2, -1, -1], np.int32), np.array([0, 1.0, 2.0, 0, 3.0, 4.0]))
    fo = fs.Forest(dev, 1)
    fo.upload(0, e)
    x = np.array([[-0.0], [0.0], [1e-300], [-1e-300]])
    assert np.array_equal(fo.predict(x), orc.predict(e, x))
