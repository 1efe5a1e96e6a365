"""Generate tests/golden/full_c4.npz and full_c5.npz: the UNMODIFIED reference's models at the
BASELINE.json full sizes (oracle/_ref, compiled from /root/reference by oracle/Makefile).

  C4: bench.build_workload("c4", 1000) - BERT-base-sim dense / batch_matmul / softmax families,
      16,384 training rows and 16,384 pool candidates each, T = 500, depth 3, lr 0.1.
  C5: bench.build_workload("c5", 1000) - families 0, 17 and 63 of the 64 synthetic families,
      65,536 rows / candidates each, T = 1000.

Only the outputs are committed: the inputs regenerate bit-identically from the seed (numpy
PCG64 streams + the reference's featurize, which the GPU featurize matches bit for bit).
Per family: the reference's fitted trees in pre-order (fit, costmodel.cpp:152-222), its base
prediction and train_mse_by_round (:215-220), sha256 digests of its predictions on the pool
(predict, :237-246) and of their std::sort order (scheduler.cpp:187-192), the top-64 of that
order with their scores, and every 97th score. The oracle restatement's split gains (orc.fit, the
reference-order gain replica the reference never exposes) are stored too, after checking that
the restatement's trees equal the reference's at this size (pins the oracle at full size).

Runs here, in the build container (~30 min on 8 cores). Usage:
    python tests/golden/make_golden_full.py [c4] [c5]
"""
import hashlib
import os
import sys
import threading
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import oracle  # noqa: E402

FULL = {"c4": (None, 500), "c5": ([0, 17, 63], 1000)}


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def featurize(r, W, so, asg, seg, f):
    a, b = int(seg[f]), int(seg[f + 1])
    x = np.zeros((b - a, bench.PAD))
    for sid in np.unique(so[a:b]):
        rows = np.where(so[a:b] == sid)[0]
        kn = W["spaces"][sid]
        x[rows] = r.featurize(kn, asg[a:b][rows][:, : len(kn)], bench.PAD)
    return x


def one_family(r, orc, W, f, trees, out, lock):
    t0 = time.time()
    x = featurize(r, W, W["tr_so"], W["tr_a"], W["tr_seg"], f)
    ta, tb = int(W["tr_seg"][f]), int(W["tr_seg"][f + 1])
    y = W["tr_y"][ta:tb]
    ens = r.fit(x, y, trees=trees)
    t1 = time.time()
    mine = orc.fit(x, y, trees=trees)
    for k in ("offsets", "feature", "threshold", "left", "right", "value"):
        if not np.array_equal(getattr(ens, k), getattr(mine, k)):
            raise SystemExit(f"oracle restatement differs from the reference: family {f} {k}")
    if mine.base != ens.base:
        raise SystemExit(f"oracle base differs: family {f}")
    xp = featurize(r, W, W["pool_so"], W["pool_a"], W["pool_seg"], f)
    m = r.new_model(f, trees)
    m.load(ens)
    pred = m.predict(xp)
    m.free()
    perm = r.rank(pred)
    res = {
        "offsets": ens.offsets, "feature": ens.feature, "threshold": ens.threshold, "left": ens.left,
        "right": ens.right, "value": ens.value, "mse": ens.mse, "base": np.array([ens.base]),
        "gain": mine.gain, "oracle_mse": mine.mse,
        "pred_sha": np.array([digest(pred)]), "rank_sha": np.array([digest(perm.astype(np.int64))]),
        "top_idx": perm[:64].astype(np.int64), "top_score": pred[perm[:64]], "pred_every97": pred[::97],
        "rows": np.array([tb - ta]), "pool": np.array([len(pred)]),
    }
    with lock:
        for k, v in res.items():
            out[f"f{f}_{k}"] = v
        print(f"family {f}: rows={tb - ta} trees={ens.n_trees} nodes={len(ens.feature)} ref fit {t1 - t0:.0f}s "
              f"total {time.time() - t0:.0f}s", flush=True)


def main(cfgs):
    r, orc = oracle.ref(), oracle.orc()
    for cfg in cfgs:
        fams, trees = FULL[cfg]
        W = bench.build_workload(cfg, seed=1000)
        fams = fams if fams is not None else list(range(len(W["families"])))
        out, lock = {"families": np.array(fams), "trees": np.array([trees]), "seed": np.array([1000])}, threading.Lock()
        ts = [threading.Thread(target=one_family, args=(r, orc, W, f, trees, out, lock)) for f in fams]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        if len(out) < 3 + 15 * len(fams):
            raise SystemExit(f"{cfg}: a family failed")
        path = os.path.join(HERE, f"full_{cfg}.npz")
        np.savez_compressed(path, **out)
        print("wrote", path, os.path.getsize(path), "bytes", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["c4", "c5"])
