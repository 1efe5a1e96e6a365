"""Device-resident training store (fs_store): the reference's
train_cost_model appends each measured batch to the family's training set and refits
(costmodel.cpp:224-235). Every refit from the store must be bit-identical to fs_fit on the same
rows and to the oracle's fit of them (trees, base, train_mse_by_round), through incremental merges, bulk appends, -0.0
families, multi-family batches and subset refits; the maintained canonical order must be the
lexicographic (features..., target) order of costmodel.cpp:161-173."""
import numpy as np
import pytest

import bench
import oracle
import paper_2201_00194_b200 as fs

pytestmark = pytest.mark.gpu
FIELDS = ("offsets", "feature", "threshold", "left", "right", "value")
P = fs.GbtParams(20, 3, 0.1, 2)


def _same(a, b, tag):
    assert a.base == b.base, tag
    for k in FIELDS:
        assert np.array_equal(getattr(a, k), getattr(b, k)), (tag, k)


def _lex_rows(x, y):
    """rows sorted by (features..., target) - np.lexsort's last key is the primary one"""
    keys = [y] + [x[:, j] for j in range(x.shape[1] - 1, -1, -1)]
    return np.lexsort(keys)


def _check_store(dev, st, F, tag):
    """store fit of every family == fs_fit on the store's rows; canonical order is sorted"""
    fa = fs.Forest(dev, F)
    st.fit(fa, params=P)
    xs, ys, seg = [], [], [0]
    for f in range(F):
        x, y, c = st.read(f)
        xs.append(x)
        ys.append(y)
        seg.append(seg[-1] + len(y))
        if c is not None and len(y):
            assert sorted(c.tolist()) == list(range(len(y))), (tag, f)
            o = _lex_rows(x, y)
            # equal keys are identical rows: compare row contents in the two orders
            assert np.array_equal(x[c], x[o]) and np.array_equal(y[c], y[o]), (tag, f)
    fb = fs.Forest(dev, F)
    fb.fit(np.concatenate(xs), np.concatenate(ys), seg=seg, params=P)
    orc = oracle.orc()
    for f in range(F):
        got = fa.export(f)
        _same(got, fb.export(f), (tag, f))
        if len(ys[f]):  # and against the CPU restatement of fit (costmodel.cpp:152-222), not only fs_fit
            exp = orc.fit(xs[f], ys[f], trees=P.trees, depth=P.depth, lr=P.learning_rate,
                          min_split=P.min_samples_split)
            _same(got, exp, (tag, f, "oracle"))
            assert np.array_equal(got.mse, exp.mse), (tag, f, "mse")


def _c3(orc, seed):
    W = bench.build_workload("c3", seed)
    return W, bench._featurize_host(W, orc)


def test_store_incremental_batches_equal_fit(dev, orc):
    W, x = _c3(orc, 3)
    seg, lat = W["tr_seg"], W["tr_lat"]
    F = len(W["families"])
    st = fs.Store(dev, F, x.shape[1])
    cur = [int(seg[f]) for f in range(F)]
    # initial batch: 40 % of each family, then steps of g = 64 rows for every family at once
    fam, sg, rows = [], [0], []
    for f in range(F):
        n0 = max(1, int(0.4 * (seg[f + 1] - seg[f])))
        fam.append(f)
        rows.append(np.arange(cur[f], cur[f] + n0))
        sg.append(sg[-1] + n0)
        cur[f] += n0
    idx = np.concatenate(rows)
    st.append(fam, x[idx], lat[idx], seg=sg)
    _check_store(dev, st, F, "initial")
    for step in range(4):
        fam, sg, rows = [], [0], []
        for f in range(F):
            g = min(64, int(seg[f + 1]) - cur[f])
            if g <= 0:
                continue
            fam.append(f)
            rows.append(np.arange(cur[f], cur[f] + g))
            sg.append(sg[-1] + g)
            cur[f] += g
        idx = np.concatenate(rows)
        st.append(fam, x[idx], lat[idx], seg=sg)
        _check_store(dev, st, F, f"step {step}")


def test_store_bulk_append_then_merges(dev, orc):
    """a batch above the merge limit leaves the order to the next fit, which records it"""
    W, x = _c3(orc, 5)
    a, b = int(W["tr_seg"][0]), int(W["tr_seg"][1])
    xf, lf = x[a:b], W["tr_lat"][a:b]
    reps = np.concatenate([xf, xf, xf])  # 3 copies: > 4096 rows and many exact duplicates (ties)
    lrep = np.concatenate([lf, lf, lf])
    st = fs.Store(dev, 1, x.shape[1])
    st.append([0], reps, lrep)
    assert st.read(0)[2] is None
    _check_store(dev, st, 1, "bulk")
    assert st.read(0)[2] is not None
    for step in range(3):
        sl = slice(64 * step, 64 * step + 64)
        st.append([0], xf[sl], lf[sl] * 1.5)
        _check_store(dev, st, 1, f"after bulk {step}")


def test_store_negative_zero_family(dev, orc):
    W, x = _c3(orc, 7)
    a, b = int(W["tr_seg"][0]), int(W["tr_seg"][1])
    xf, lf = x[a:b].copy(), W["tr_lat"][a:b]
    col = int(np.argmax((xf == 0.0).sum(0)))
    z = np.where(xf[:, col] == 0.0)[0]
    xf[z[::2], col] = -0.0
    st = fs.Store(dev, 1, x.shape[1])
    st.append([0], xf[:700], lf[:700])
    _check_store(dev, st, 1, "negz initial")
    st.append([0], xf[700:764], lf[700:764])
    _check_store(dev, st, 1, "negz step")


def test_store_records_equal_host_rows(dev, orc):
    W, x = _c3(orc, 9)
    F = len(W["families"])
    sp = fs.Spaces(dev, W["spaces"])
    s1 = fs.Store(dev, F, bench.PAD)
    s2 = fs.Store(dev, F, bench.PAD)
    seg = W["tr_seg"]
    fam = list(range(F))
    s1.append_records(sp, fam, W["tr_so"], W["tr_a"], W["tr_lat"], seg=seg)
    s2.append(fam, x, W["tr_lat"], seg=seg)
    for f in range(F):
        a1, b1, _ = s1.read(f)
        a2, b2, _ = s2.read(f)
        assert np.array_equal(a1, a2) and np.array_equal(b1, b2)
    _check_store(dev, s1, F, "records")


def test_store_subset_fit_and_targets(dev, orc):
    W, x = _c3(orc, 11)
    F = len(W["families"])
    seg = W["tr_seg"]
    st = fs.Store(dev, F, x.shape[1])
    st.append(list(range(F)), x, W["tr_lat"], seg=seg)
    for f in range(F):
        _, y, _ = st.read(f)
        np.testing.assert_allclose(y, np.log(W["tr_lat"][seg[f]:seg[f + 1]]), rtol=1e-15, atol=0)
    fo = fs.Forest(dev, F)
    st.fit(fo, families=[2, 0], params=P)
    ref = fs.Forest(dev, F)
    xs = [st.read(f) for f in (2, 0)]
    ref.fit(np.concatenate([xs[0][0], xs[1][0]]), np.concatenate([xs[0][1], xs[1][1]]),
            seg=[0, len(xs[0][1]), len(xs[0][1]) + len(xs[1][1])], params=P)
    _same(fo.export(2), ref.export(0), "subset 2")
    _same(fo.export(0), ref.export(1), "subset 0")
    assert fo.export_n_trees(1) == 0


def test_store_errors(dev, orc):
    W, x = _c3(orc, 13)
    st = fs.Store(dev, 2, x.shape[1])
    with pytest.raises(fs.InvalidArgument):
        st.append([0], x[:0], W["tr_lat"][:0])  # costmodel.cpp:225-227 empty batch
    bad = W["tr_lat"][:10].copy()
    bad[3] = 0.0
    with pytest.raises(fs.InvalidArgument):
        st.append([0], x[:10], bad)  # :229-231 non-positive latency, nothing appended
    assert st.rows(0) == 0
    with pytest.raises(fs.OutOfRange):
        st.append([5], x[:10], W["tr_lat"][:10])
    st.append([1], x[:10], W["tr_lat"][:10])
    assert st.rows(1) == 10 and st.rows(0) == 0
    fo = fs.Forest(dev, 2)
    with pytest.raises(fs.OutOfRange):
        st.fit(fo, families=[3], params=P)
    xn = x[:10].copy()
    xn[2, 1] = np.nan
    st.append([0], xn, W["tr_lat"][:10])
    with pytest.raises(fs.InvalidArgument):
        st.fit(fo, families=[0], params=P)  # costmodel.cpp:178-182 non-finite feature at fit
    st.fit(fo, families=[1], params=P)  # the store stays usable
