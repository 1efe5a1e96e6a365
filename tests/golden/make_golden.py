"""Generate tests/golden/golden.npz from the UNMODIFIED reference (oracle/_ref, compiled from
/root/reference by oracle/Makefile). Run here, in the build container; the .npz is committed and
travels to the GPU box, where /root/reference does not exist.

Contents (every array produced by the reference's own functions):
  feat_*      featurize exact-value cases (searchspace_test.cpp:59-76) + digests of larger ones
  fit_<case>_*  training sets and the reference's fitted trees (fit, costmodel.cpp:152-222),
              its predictions on probe rows (predict :237-246) and their std::sort order
              (scheduler.cpp:187-192)
  rank_*      a score vector with ties and signed zeros and the reference's order
  rng_*       mt19937_64/mix_seed/uniform_below draws (rng.hpp) that pin the epsilon-pick replay

Usage: python tests/golden/make_golden.py
"""
import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle  # noqa: E402
from common import load_spaces, random_dataset  # noqa: E402

REF_MODELS = "/root/reference/proj/models"


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    r = oracle.ref()
    out = {}

    # ---- featurize ---------------------------------------------------------------------------
    out["feat_single"] = r.featurize([[8, 16, 32]], np.array([0], np.int32), 6)
    out["feat_pair"] = r.featurize([[4, 8], [2, 16]], np.array([0, 0], np.int32), 5)
    small = [[1, 2, 4, 8], [1, 3, 9], [2, 4]]
    lin = np.arange(24)
    a = np.stack([lin // 6, (lin // 2) % 3, lin % 2], 1).astype(np.int32)
    out["feat_small_assign"] = a
    out["feat_small"] = r.featurize(small, a, 9)
    # digests over every subgraph space of two model files at pad 164
    rng = np.random.default_rng(5)
    for name in ("resnet50_sim", "bert_base_sim"):
        doc = load_spaces(name)
        asg_all, dig = [], []
        for sg in doc["subgraphs"]:
            kn = sg["knobs"]
            asg = np.stack([rng.integers(0, len(v), 32) for v in kn], 1).astype(np.int32)
            x = r.featurize(kn, asg, 164)
            asg_all.append(np.pad(asg, ((0, 0), (0, 16 - asg.shape[1]))))
            dig.append(digest(x))
        out[f"feat_{name}_assign"] = np.stack(asg_all)
        out[f"feat_{name}_digest"] = np.array(dig)

    # ---- fit / predict / rank ------------------------------------------------------------------
    cases = {}
    # (a) simulator-generated family datasets (experiment.cpp draw_samples style)
    for tag, model, fam, per, pad, trees in (("tiny_f0", "tiny", 0, 40, 9, 50),
                                             ("resnet_f1", "resnet50_sim", 1, 24, 164, 100),
                                             ("bertl_f1", "bert_large_sim", 1, 60, 14, 50)):
        x, lat, sid, asg = r.family_dataset(f"{REF_MODELS}/{model}.json", 0, fam, 7, per, pad)
        cases[tag] = (x, np.log(lat), trees, dict(model=model, sid=sid, asg=asg, lat=lat, pad=pad))
    # (b) training sets accumulated by the reference tuning loop (the inputs fit() really sees)
    for tag, model, budget, fam in (("tune_resnet_f1", "resnet50_sim", 700, 1), ("tune_tiny_f0", "tiny", 60, 0),
                                    ("tune_bertl_f1", "bert_large_sim", 500, 1)):
        _, x, y = r.tune(f"{REF_MODELS}/{model}.json", budget, seed=3, export_family=fam)
        cases[tag] = (x, y, 50, dict(model=model))
    # (c) continuous-feature property-test datasets
    for tag, kind, n in (("c7_a", "c7", 200), ("mse_a", "mse", 150), ("disc_a", "discrete", 300)):
        x, y = random_dataset(11, n, 6, kind)
        cases[tag] = (x, y, 50, {})
    # (d) degenerate / tiny sets (costmodel_test.cpp:113-158)
    cases["degenerate"] = (np.arange(8, dtype=np.float64)[:, None], np.full(8, np.log(2.5)), 50, {})
    cases["two_point"] = (np.array([[0.0, 1.0], [3.0, 2.0]]), np.log(np.array([1.0, 2.0])), 50, {})

    out["fit_cases"] = np.array(sorted(cases))
    for tag, (x, y, trees, meta) in cases.items():
        ens = r.fit(x, y, trees=trees)
        m = r.new_model(0, trees)
        m.load(ens)
        pred = m.predict(x)
        m.free()
        out[f"fit_{tag}_x"] = x
        out[f"fit_{tag}_y"] = y
        out[f"fit_{tag}_trees"] = np.array([trees])
        for k in ("offsets", "feature", "threshold", "left", "right", "value", "mse"):
            out[f"fit_{tag}_{k}"] = getattr(ens, k)
        out[f"fit_{tag}_base"] = np.array([ens.base])
        out[f"fit_{tag}_pred"] = pred
        out[f"fit_{tag}_rank"] = r.rank(pred)
        print(f"{tag:16s} n={x.shape[0]:5d} d={x.shape[1]:3d} trees={ens.n_trees}")

    # ---- rank -----------------------------------------------------------------------------------
    s = np.round(np.random.default_rng(9).normal(0, 1, 5000), 2)
    s[::7] = 0.0
    s[3::11] = -0.0
    out["rank_scores"] = s
    out["rank_perm"] = r.rank(s)

    # ---- rng replay -------------------------------------------------------------------------------
    out["rng_raw"] = r.rng_draws(42, 0xD4, 0, 16)
    out["rng_below"] = r.rng_draws(42, 0xD4, 0, 64, 1000)

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)
    print("wrote", os.path.join(HERE, "golden.npz"), os.path.getsize(os.path.join(HERE, "golden.npz")), "bytes")


if __name__ == "__main__":
    main()
