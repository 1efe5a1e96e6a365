"""Pin the C restatement (oracle/famtune_oracle.c) before trusting it as the parity checker:
against the golden vectors the reference produced (tests/golden/golden.npz) and, where the
compiled reference is present, differentially on fresh inputs. CPU only."""
import hashlib

import numpy as np
import pytest

import oracle
from common import GOLDEN, load_spaces, random_dataset

G = np.load(f"{GOLDEN}/golden.npz")


def _digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _ens(tag):
    return oracle.Ensemble(float(G[f"fit_{tag}_base"][0]), 0.1, G[f"fit_{tag}_offsets"], G[f"fit_{tag}_feature"],
                           G[f"fit_{tag}_threshold"], G[f"fit_{tag}_left"], G[f"fit_{tag}_right"],
                           G[f"fit_{tag}_value"], G[f"fit_{tag}_mse"])


def test_featurize_exact_layouts(orc):
    # searchspace_test.cpp:59-76
    f = orc.featurize([[8, 16, 32]], [0], 6)[0]
    assert f.tolist() == [3.0, 0.0, 0.0, 0.0, 0.0, 0.0]
    assert np.array_equal(f, G["feat_single"])
    f = orc.featurize([[4, 8], [2, 16]], [0, 0], 5)[0]
    assert f[0] == 2.0 and f[1] == 1.0 and f[4] == 2.0
    assert np.array_equal(f, G["feat_pair"])
    small = orc.featurize([[1, 2, 4, 8], [1, 3, 9], [2, 4]], G["feat_small_assign"], 9)
    assert np.array_equal(small, G["feat_small"])
    assert len({r.tobytes() for r in small}) == 24  # injective (searchspace_test.cpp:91-100)


@pytest.mark.parametrize("name", ["resnet50_sim", "bert_base_sim"])
def test_featurize_model_spaces_digest(orc, name):
    doc = load_spaces(name)
    asg = G[f"feat_{name}_assign"]
    for sid, sg in enumerate(doc["subgraphs"]):
        k = len(sg["knobs"])
        x = orc.featurize(sg["knobs"], asg[sid][:, :k], 164)
        assert _digest(x) == G[f"feat_{name}_digest"][sid]


def test_featurize_rejects_small_pad(orc):
    with pytest.raises(oracle.InvalidArgument):
        orc.featurize([[1, 2], [1, 2]], [0, 0], 4)


@pytest.mark.parametrize("tag", [str(t) for t in G["fit_cases"]])
def test_fit_matches_reference_trees(orc, tag):
    x, y = G[f"fit_{tag}_x"], G[f"fit_{tag}_y"]
    ens = orc.fit(x, y, trees=int(G[f"fit_{tag}_trees"][0]))
    ref = _ens(tag)
    assert ens.base == ref.base
    for k in ("offsets", "feature", "threshold", "left", "right", "value", "mse"):
        assert np.array_equal(getattr(ens, k), getattr(ref, k)), k
    pred = orc.predict(ens, x)
    assert np.array_equal(pred, G[f"fit_{tag}_pred"])
    assert np.array_equal(orc.rank(pred), G[f"fit_{tag}_rank"])


def test_reference_exact_values(orc):
    # costmodel_test.cpp:77-83 fresh model predicts 0; :98-105 single leaf 0.1*7.0
    assert orc.predict(oracle.empty_ensemble(), [1.0, 2.0, 3.0])[0] == 0.0
    e = oracle.Ensemble(0.0, 0.1, np.array([0, 1], np.int32), np.array([-1], np.int32), np.zeros(1),
                        np.array([-1], np.int32), np.array([-1], np.int32), np.array([7.0]))
    assert orc.predict(e, [1.0])[0] == 0.1 * 7.0
    with pytest.raises(oracle.InvalidArgument):
        orc.predict(e, [np.nan])
    # degenerate targets: constant log(2.5) (costmodel_test.cpp:147-158)
    d = orc.fit(G["fit_degenerate_x"], G["fit_degenerate_y"])
    p = orc.predict(d, np.array([[-3.0], [42.0]]))
    assert p[0] == p[1] and abs(p[0] - np.log(2.5)) < 1e-12


def test_mse_monotone_and_permutation_invariant(orc):
    for seed in range(5):
        x, y = random_dataset(100 + seed, 60 + 40 * seed, 3, "mse")
        e = orc.fit(x, y)
        assert np.all(np.diff(e.mse) <= 1e-12)
        perm = np.random.default_rng(seed).permutation(len(y))
        e2 = orc.fit(x[perm], y[perm])
        probe = np.random.default_rng(seed + 7).uniform(0, 8, size=(50, 3))
        assert np.array_equal(orc.predict(e, probe), orc.predict(e2, probe))


def test_rank_matches_std_sort(orc):
    assert np.array_equal(orc.rank(G["rank_scores"]), G["rank_perm"])


def _lemire_select(raw, n_pool, g_eff, epsilon):
    explore = int(g_eff * epsilon)
    by_score = g_eff - explore
    tail = list(range(by_score, n_pool))
    got = list(range(by_score))
    for e in range(explore):
        b = len(tail) - e
        pick = (int(raw[e]) * b) >> 64  # rng.hpp:36-45; rejection has probability b/2^64
        got.append(tail[pick])
        tail[pick], tail[len(tail) - 1 - e] = tail[len(tail) - 1 - e], tail[pick]
    return got


def test_select_replays_reference_stream(orc):
    # scheduler.cpp:194-213 epsilon picks on the mt19937_64 stream mix_seed(42, 0xD4, 0)
    perm = np.arange(1000, dtype=np.int64)
    picks = orc.select(perm, 64, 0.10, orc.mix_seed(42, 0xD4, 0))
    assert list(picks) == _lemire_select(G["rng_raw"], 1000, 64, 0.10)
    assert orc.select(perm[:10], 64, 0.1, 1).tolist() == list(range(10))  # pool <= g: take all


@pytest.mark.skipif(not oracle.ref_available(), reason="compiled reference not present")
def test_fit_differential_vs_reference(orc, ref):
    rng = np.random.default_rng(3)
    for i in range(6):
        kind = ["c7", "mse", "discrete"][i % 3]
        x, y = random_dataset(1000 + i, int(rng.integers(20, 400)), 5, kind)
        a, b = orc.fit(x, y, trees=30), ref.fit(x, y, trees=30)
        for k in ("offsets", "feature", "threshold", "left", "right", "value", "mse"):
            assert np.array_equal(getattr(a, k), getattr(b, k)), (i, k)
        assert a.base == b.base


@pytest.mark.skipif(not oracle.ref_available(), reason="compiled reference not present")
def test_rng_stream_matches_reference(ref):
    assert np.array_equal(ref.rng_draws(42, 0xD4, 0, 64, 1000), G["rng_below"])
    assert np.array_equal(ref.rng_draws(42, 0xD4, 0, 16), G["rng_raw"])


def test_linear_index_pinned(orc):
    """linear_index / candidate_from_index (searchspace.cpp:48-66) against the reference's own
    outputs on every subgraph space of two model files (tests/golden/make_golden_index.py)."""
    L = np.load(f"{GOLDEN}/linear_index.npz")
    names = sorted({k.rsplit("_", 1)[0] for k in L.files})
    assert len(names) == 39
    for name in names:
        model, sid = name.rsplit("_", 1)
        knobs = load_spaces(model)["subgraphs"][int(sid)]["knobs"]
        nv = [len(v) for v in knobs]
        a = L[f"{name}_assign"]
        assert np.array_equal(orc.linear_index(nv, a[:, : len(nv)]), L[f"{name}_index"]), name
        assert np.array_equal(orc.candidate_from_index(nv, L[f"{name}_index"]), L[f"{name}_back"]), name
        assert np.array_equal(L[f"{name}_back"], a), name  # round trip
        assert int(L[f"{name}_index"][0]) == 0 and int(L[f"{name}_index"][-1]) == int(np.prod(nv)) - 1


def test_linear_index_differential_vs_reference(orc, ref):
    rng = np.random.default_rng(11)
    for k in (1, 5, 16):
        knobs = [[1 << i for i in range(int(rng.integers(1, 9)))] for _ in range(k)]
        nv = [len(v) for v in knobs]
        a = np.stack([rng.integers(0, m, 200) for m in nv], 1).astype(np.int32)
        idx = ref.linear_index(knobs, a)
        assert np.array_equal(orc.linear_index(nv, a), idx)
        assert np.array_equal(orc.candidate_from_index(nv, idx)[:, :k], a)
        assert np.array_equal(ref.candidate_from_index(knobs, idx)[:, :k], a)
