"""GPU trainer (kernel 3) vs the reference: trees field-by-field in pre-order, base, predictions and
rankings bit-exact; split gains equal to the reference-order replica (the bar is 1e-5 relative);
train_mse_by_round bit-exact (the reference's sequential fold over canonical rows, costmodel.cpp:215-220)."""
import numpy as np
import pytest

import oracle
import paper_2201_00194_b200 as fs
from common import GOLDEN, families, family_dataset, load_spaces, random_dataset

pytestmark = pytest.mark.gpu
G = np.load(f"{GOLDEN}/golden.npz")
CASES = [str(t) for t in G["fit_cases"]]
TREE_FIELDS = ("offsets", "feature", "threshold", "left", "right", "value")


@pytest.fixture(autouse=True, params=["auto", "multi", "multi_col", "multi_rowmajor"])
def fit_path(request, monkeypatch):
    """Every parity test runs on every trainer shape: the resident one-CTA-per-family kernel (auto
    picks it when the families fit shared memory) and the multi-kernel round with each histogram
    build (limb-atomic default, column layout, row-major)."""
    monkeypatch.setenv("FAMSEER_FIT_PATH", "auto" if request.param == "auto" else "multi")
    if request.param == "multi_col":
        monkeypatch.setenv("FAMSEER_HIST", "col")
    elif request.param == "multi_rowmajor":
        monkeypatch.setenv("FAMSEER_HIST", "rowmajor")
    return request.param


def assert_same_model(got, exp, gains=None):
    assert got.base == exp.base
    for k in TREE_FIELDS:
        a, b = getattr(got, k), getattr(exp, k)
        assert np.array_equal(a, b), (k, a[:20], b[:20])
    if gains is not None:
        internal = exp.feature >= 0
        np.testing.assert_allclose(got.gain[internal], gains[internal], rtol=1e-5, atol=0)
    if len(exp.mse):
        assert np.array_equal(got.mse, exp.mse), np.flatnonzero(got.mse != exp.mse)[:10]


@pytest.mark.parametrize("tag", CASES)
def test_golden_reference_trees(dev, orc, tag):
    x, y = G[f"fit_{tag}_x"], G[f"fit_{tag}_y"]
    trees = int(G[f"fit_{tag}_trees"][0])
    fo = fs.Forest(dev, 1)
    fo.fit(x, y, params=fs.GbtParams(trees, 3, 0.1, 2))
    got = fo.export(0)
    exp = oracle.Ensemble(float(G[f"fit_{tag}_base"][0]), 0.1, G[f"fit_{tag}_offsets"], G[f"fit_{tag}_feature"],
                          G[f"fit_{tag}_threshold"], G[f"fit_{tag}_left"], G[f"fit_{tag}_right"],
                          G[f"fit_{tag}_value"], G[f"fit_{tag}_mse"])
    replica = orc.fit(x, y, trees=trees)
    assert_same_model(got, exp, gains=replica.gain)
    s = fo.predict(x)
    assert np.array_equal(s, G[f"fit_{tag}_pred"])
    assert np.array_equal(dev.rank(s), G[f"fit_{tag}_rank"])


def test_multi_family_batch_with_params(dev, orc):
    doc = load_spaces("resnet50_sim")
    fams = families(doc)
    xs, ys, seg, params = [], [], [0], []
    for i, (f, members) in enumerate(sorted(fams.items())):
        x, lat, _, _ = family_dataset(doc, members, 40, 164, seed=10 + f, orc=orc)
        xs.append(x)
        ys.append(np.log(lat))
        seg.append(seg[-1] + len(x))
        params.append(fs.GbtParams(30 + 10 * i, [3, 2, 4, 1, 3][i % 5], [0.1, 0.3, 0.05, 0.1, 0.2][i % 5],
                                   [2, 2, 5, 2, 10][i % 5]))
    x, y = np.concatenate(xs), np.concatenate(ys)
    fo = fs.Forest(dev, len(params))
    fo.fit(x, y, seg=seg, params=params)
    for f, p in enumerate(params):
        a, b = seg[f], seg[f + 1]
        exp = orc.fit(x[a:b], y[a:b], trees=p.trees, depth=p.depth, lr=p.learning_rate, min_split=p.min_samples_split)
        got = fo.export(f, lr=p.learning_rate)
        assert_same_model(got, exp, gains=exp.gain)
        assert np.array_equal(fo.predict(x, seg=seg)[a:b], orc.predict(exp, x[a:b]))


@pytest.mark.parametrize("kind,n,d,seed", [("c7", 316, 4, 1), ("mse", 232, 3, 2), ("discrete", 2000, 8, 3),
                                         ("c7", 2, 4, 4), ("mse", 3, 3, 5), ("discrete", 5000, 3, 6)])
def test_property_datasets(dev, orc, kind, n, d, seed):
    x, y = random_dataset(seed, n, d, kind)
    fo = fs.Forest(dev, 1)
    fo.fit(x, y, params=fs.GbtParams(50, 3, 0.1, 2))
    exp = orc.fit(x, y, trees=50)
    assert_same_model(fo.export(0), exp, gains=exp.gain)
    got = fo.export(0)
    assert np.all(np.diff(got.mse) <= 1e-12)  # costmodel_test.cpp:185-202


def test_permutation_invariance_bitwise(dev):
    x, y = random_dataset(77, 400, 4, "c7")
    perm = np.random.default_rng(1).permutation(len(y))
    fo = fs.Forest(dev, 2)
    fo.fit(np.concatenate([x, x[perm]]), np.concatenate([y, y[perm]]), seg=[0, 400, 800])
    a, b = fo.export(0), fo.export(1)
    for k in TREE_FIELDS:
        assert np.array_equal(getattr(a, k), getattr(b, k))


def test_degenerate_and_tiny(dev, orc):
    fo = fs.Forest(dev, 4)
    xs = [np.arange(8, dtype=float)[:, None], np.array([[0.0, 1.0], [3.0, 2.0]])[:, :1],
          np.array([[1.0]]), np.zeros((5, 1))]
    ys = [np.full(8, np.log(2.5)), np.log([1.0, 2.0]), np.array([0.3]), np.array([1.0, 2, 3, 4, 5])]
    seg = np.cumsum([0] + [len(v) for v in ys])
    fo.fit(np.concatenate(xs), np.concatenate(ys), seg=seg)
    for f in range(4):
        exp = orc.fit(xs[f], ys[f])
        assert_same_model(fo.export(f), exp)
    # degenerate targets -> constant log(2.5) (costmodel_test.cpp:147-158)
    p = fo.predict(np.array([[-3.0], [42.0], [0], [0], [0], [0]]), seg=[0, 2, 3, 4, 6])
    assert p[0] == p[1] and abs(p[0] - np.log(2.5)) < 1e-12


def test_empty_family_and_errors(dev):
    fo = fs.Forest(dev, 2)
    x, y = random_dataset(1, 50, 3, "mse")
    fo.fit(x, y, seg=[0, 0, 50])
    assert fo.export(0).n_trees == 0 and fo.export(0).base == 0.0
    assert fo.export(1).n_trees == 50
    bad = x.copy()
    bad[7, 1] = np.nan
    with pytest.raises(fs.InvalidArgument):  # costmodel.cpp:178-182
        fo.fit(bad, y)
    with pytest.raises(fs.OutOfRange):
        fo.fit(np.concatenate([x, x]), np.concatenate([y, y]), seg=[0, 50, 100, 100])


def test_signed_zero_features(dev, orc):
    rng = np.random.default_rng(3)
    x = rng.choice([-1.0, -0.0, 0.0, 1.0, 2.0], size=(300, 3))
    y = x[:, 0] * 2 - x[:, 1] + rng.normal(0, 0.1, 300)
    fo = fs.Forest(dev, 1)
    fo.fit(x, y)
    exp = orc.fit(x, y)
    got = fo.export(0)
    for k in TREE_FIELDS:
        assert np.array_equal(getattr(got, k).view(np.int64) if getattr(got, k).dtype == np.float64 else getattr(got, k),
                              getattr(exp, k).view(np.int64) if getattr(exp, k).dtype == np.float64 else getattr(exp, k)), k


@pytest.mark.parametrize("depth,min_split", [(1, 2), (5, 2), (6, 30), (0, 2), (9, 2)])
def test_depth_and_min_split(dev, orc, depth, min_split):
    doc = load_spaces("bert_large_sim")
    members = families(doc)[1]
    x, lat, _, _ = family_dataset(doc, members, 120, 14, seed=depth, orc=orc)
    y = np.log(lat)
    fo = fs.Forest(dev, 1)
    fo.fit(x, y, params=fs.GbtParams(40, depth, 0.1, min_split))
    exp = orc.fit(x, y, trees=40, depth=depth, min_split=min_split)
    assert_same_model(fo.export(0), exp, gains=exp.gain)


def test_fit_stats_reported(dev, orc):
    x, y = G["fit_tune_resnet_f1_x"], G["fit_tune_resnet_f1_y"]
    fo = fs.Forest(dev, 1)
    fo.fit(x, y)
    screened, exact = fo.fit_stats(0)
    assert screened + exact > 0


@pytest.mark.parametrize("tag", CASES[:4])
def test_host_compile_epilogue(dev, orc, monkeypatch, tag):
    """FAMSEER_HOST_COMPILE=1: tree tables read back and compiled on the host (the fallback the
    device epilogue replaces; also what deeper-than-7 trees use) - same trees, same scores."""
    monkeypatch.setenv("FAMSEER_HOST_COMPILE", "1")
    x, y = G[f"fit_{tag}_x"], G[f"fit_{tag}_y"]
    trees = int(G[f"fit_{tag}_trees"][0])
    fo = fs.Forest(dev, 1)
    fo.fit(x, y, params=fs.GbtParams(trees, 3, 0.1, 2))
    assert np.array_equal(fo.export(0).feature, G[f"fit_{tag}_feature"])
    assert np.array_equal(fo.predict(x), G[f"fit_{tag}_pred"])
