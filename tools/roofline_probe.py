"""Kernel-level roofline probe at the large configurations (C4/C5 shapes): times featurize,
predict (T-tree model) and the trainer's histogram build with CUDA events and prints algorithmic
GB/s against the measured HBM peak. Meant to be run under ncu as well (see profiles/README.md):

    python tools/roofline_probe.py --families 8 --rows 65536 --trees 1000
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402  (workload generator)
import paper_2201_00194_b200 as fs  # noqa: E402


def random_model(rng, x, trees, depth=3):
    """A depth-`depth` ensemble whose thresholds are actual feature values (as a fit produces)."""
    d = x.shape[1]
    informative = [f for f in range(d) if np.unique(x[:4096, f]).size > 1]
    off, feat, thr, le, ri, val = [0], [], [], [], [], []
    for _ in range(trees):
        nodes = []

        def build(lvl):
            i = len(nodes)
            nodes.append(None)
            if lvl == depth:
                nodes[i] = (-1, 0.0, -1, -1, float(rng.normal(0, 0.1)))
                return i
            f = int(rng.choice(informative))
            t = float(x[int(rng.integers(0, len(x))), f])
            a = build(lvl + 1)
            b = build(lvl + 1)
            nodes[i] = (f, t, a, b, 0.0)
            return i

        build(0)
        for n_ in nodes:
            feat.append(n_[0]), thr.append(n_[1]), le.append(n_[2]), ri.append(n_[3]), val.append(n_[4])
        off.append(len(feat))
    return fs.Ensemble(0.5, 0.1, np.array(off, np.int32), np.array(feat, np.int32), np.array(thr),
                       np.array(le, np.int32), np.array(ri, np.int32), np.array(val))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--families", type=int, default=8)
    ap.add_argument("--rows", type=int, default=65536)
    ap.add_argument("--trees", type=int, default=1000)
    ap.add_argument("--fit-trees", type=int, default=3)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    peak, kind = bench.measured_peak_hbm()
    W = bench.build_workload("c5", 1000)
    F = min(args.families, len(W["families"]))
    seg = W["pool_seg"][: F + 1].copy()
    seg = np.minimum(seg, seg[0] + np.arange(F + 1) * args.rows)
    P = int(seg[-1])
    dev = fs.Device(0)
    stream = torch.cuda.ExternalStream(dev.stream)
    sp = fs.Spaces(dev, W["spaces"])
    so = torch.from_numpy(W["pool_so"][:P].copy()).cuda()
    asg = torch.from_numpy(W["pool_a"][:P].copy()).cuda()
    x = torch.empty((P, bench.PAD), dtype=torch.float64, device="cuda")
    scores = torch.empty(P, dtype=torch.float64, device="cuda")
    out = {"families": F, "rows": P, "peak_gbs": peak, "peak_kind": kind}

    def timeit(fn):
        ts = []
        for _ in range(args.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        return min(ts)

    with torch.cuda.stream(stream):
        sp.featurize_d(so, asg, bench.PAD, x)
        ms = timeit(lambda: sp.featurize_d(so, asg, bench.PAD, x))
        nb = P * (4 * 16 + 4 + 8 * bench.PAD)
        out["featurize"] = {"ms": ms, "bytes": nb, "gbs": nb / ms / 1e6, "frac": nb / ms / 1e6 / peak}
        rng = np.random.default_rng(0)
        xs = x[: min(P, 65536)].cpu().numpy()
        # predict (feature rows from HBM: P*(8*d + 8) bytes) and the fused score
        # (descriptors in, score out: P*(64 + 4 + 8)) at the bench's tree counts; rows (688 MB at
        # 8 x 65,536) exceed L2, so every repetition streams them from HBM
        for T in sorted({100, args.trees}):
            fo = fs.Forest(dev, F)
            for f in range(F):
                fo.upload(f, random_model(rng, xs, T))
            fo.predict_d(x, seg, scores)
            ms = timeit(lambda: fo.predict_d(x, seg, scores))
            nb = P * (8 * bench.PAD + 8)
            key = "predict" if T == args.trees else f"predict_T{T}"
            out[key] = {"ms": ms, "trees": T, "bytes": nb, "gbs": nb / ms / 1e6, "frac": nb / ms / 1e6 / peak,
                        "node_visits_per_s": P * T * 3 / ms * 1e3}
            ms = timeit(lambda: sp.score_d(fo, so, asg, bench.PAD, seg, scores, None))  # perm NULL: no rank
            nb = P * (4 * 16 + 4 + 8)
            out[f"score_fused_T{T}"] = {"ms": ms, "trees": T, "bytes": nb, "gbs": nb / ms / 1e6,
                                        "frac": nb / ms / 1e6 / peak, "node_visits_per_s": P * T * 3 / ms * 1e3,
                                        "note": "featurize -> predict fused (no rank)"}
        fo = fs.Forest(dev, F)
        y = torch.from_numpy(np.resize(W["tr_y"], P)).cuda()
        os.environ["FAMSEER_NO_GRAPH"] = "1"
        dev.profile("fit_hist_build,fit_exact,fit_leaf,fit_screen,fit_partition,fit_rounds")
        dev.counters(reset=True)
        fo.fit_d(x, y, seg, fs.GbtParams(args.fit_trees, 3, 0.1, 2))
        prof = dev.profile_read()
        ctr = dev.counters(reset=True)
        dev.profile(None)
        if "fit_hist_build" in prof:
            n_l, ms = prof["fit_hist_build"]
            out["hist_build"] = {"ms": ms, "launches": n_l, "bytes": ctr["hist_bytes"],
                                 "gbs": ctr["hist_bytes"] / ms / 1e6, "frac": ctr["hist_bytes"] / ms / 1e6 / peak}
        out["fit_kernels_ms"] = {k: v[1] for k, v in prof.items()}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
