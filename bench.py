#!/usr/bin/env python
"""bench.py - FamilySeer per-family cost model (BASELINE.json metric) on B200.

A step = one tuning round of the hot path over every family of the workload: score each
family's candidate pool (featurize -> GBDT predict -> rank, scheduler.cpp:187-192) and refit
each family's model from scratch on its training rows (train_cost_model/fit,
costmodel.cpp:152-235). Default workload = BASELINE.json configs[1] (ResNet-50-sim, all core-op
families, 2048 candidates/family, T=100) at pad_dim 164.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl native|reference]

Prints ONE JSON line (rank 0). value = candidates scored per second over whole rounds (score +
retrain, inputs resident in HBM); e2e = the same through the host-pointer C ABI (fs_score +
fs_fit + model export, copies inside the timed region). Under torchrun every rank tunes its own
family set (weak scaling) and the per-family top-g candidates are all-gathered over NCCL.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "candidates scored/sec & GBDT train rows/sec at 1/2/4/8 B200; % HBM roofline"
PAD = 164
G_TOP = 64  # tune_step batch g (scheduler.cpp:147-148: min(64, B/n))

CONFIGS = {
    # name: (model, family filter, candidates per family, trees, description)
    "c1": ("resnet50_sim", ["conv2d"], 512, 100, "single family (conv2d+ReLU, ResNet-50 subgraphs): 512 candidates x 164 "
           "features, 100-tree GBDT predict + one retrain round"),
    "c2": ("resnet50_sim", None, 2048, 100, "ResNet-50 full tuning round: all subgraph families, 2048 candidates/family, "
           "predict + retrain on 1 B200"),
    "c3": ("mobilenetv2_sim", None, 2048, 100, "MobileNet-V2 family-parallel tuning (depthwise/pointwise families)"),
    "c4": ("bert_base_sim", ["dense", "batch_matmul", "softmax"], 16384, 500,
           "BERT-base subgraph families (dense/batch_matmul/softmax) with 16k-candidate populations and 500-tree models"),
    "c5": ("synthetic64", None, 65536, 1000, "synthetic stress sweep: 64 families x 65k candidates x 164 features, "
           "1000-tree GBDT"),
}


# ------------------------------------------------------------------------------------------
# workload (synthetic: random candidates from the model files' knob spaces, quadratic-bowl
# latencies in the shape of simbackend.cpp:80-102; no datasets or checkpoints exist offline)
# ------------------------------------------------------------------------------------------
def load_spaces(name):
    with open(os.path.join(ROOT, "data", "spaces", name + ".json")) as f:
        return json.load(f)


def synthetic64(seed):
    rng = np.random.default_rng(seed)
    subs = []
    for s in range(64):
        knobs = [[2 ** j for j in range(int(rng.integers(4, 9)))] for _ in range(16)]
        subs.append({"id": s, "core_op": f"syn{s:02d}", "knobs": knobs})
    return {"name": "synthetic64", "subgraphs": subs, "reference_families": {"core-op": list(range(64))}}


def sample_space(rng, knobs, n):
    sizes = [len(v) for v in knobs]
    total = int(np.prod(sizes, dtype=np.float64))
    if n >= total:
        lin = np.arange(total, dtype=np.int64)
    elif total < 4 * n:
        lin = rng.choice(total, size=n, replace=False)
    else:  # large space: draw with replacement then dedup-topup
        lin = np.unique(rng.integers(0, total, size=int(n * 1.2) + 16, dtype=np.int64))
        rng.shuffle(lin)
        lin = lin[:n]
    a = np.zeros((len(lin), 16), np.int32)
    for k in range(len(sizes) - 1, -1, -1):
        a[:, k] = lin % sizes[k]
        lin = lin // sizes[k]
    return a


def latency(rng, knobs, a):
    k = len(knobs)
    z = np.stack([a[:, i] / max(len(knobs[i]) - 1, 1) for i in range(k)], 1)
    opt = rng.uniform(0, 1, k)
    curv = rng.uniform(0.5, 2.0)
    w = rng.uniform(-0.2 / (k * k), 0.2 / (k * k), (k, k))
    w = (w + w.T) / 2
    np.fill_diagonal(w, 0)
    base = math.exp(rng.uniform(math.log(0.1), math.log(10.0)))
    lat = base * (1 + curv * ((z - opt) ** 2).sum(1) + np.einsum("ni,ij,nj->n", z, w, z))
    return lat * np.exp(rng.normal(0, 0.02, len(lat)))


def build_workload(cfg_name, seed):
    model, fam_filter, per_family, trees, desc = CONFIGS[cfg_name]
    doc = synthetic64(seed) if model == "synthetic64" else load_spaces(model)
    subs = doc["subgraphs"]
    fam_of = doc["reference_families"]["core-op"]
    fams = {}
    for sid, f in enumerate(fam_of):
        fams.setdefault(f, []).append(sid)
    rng = np.random.default_rng(seed)
    spaces = [s["knobs"] for s in subs]
    pool_so, pool_a, pool_seg = [], [], [0]
    tr_so, tr_a, tr_lat, tr_seg = [], [], [], [0]
    fam_names = []
    for f in sorted(fams):
        members = fams[f]
        name = subs[members[0]]["core_op"]
        if fam_filter and name not in fam_filter:
            continue
        fam_names.append(name)
        space = sum(int(np.prod([len(v) for v in spaces[s]], dtype=np.float64)) for s in members)
        p = min(per_family, space)
        for dst_so, dst_a, dst_seg, with_lat in ((pool_so, pool_a, pool_seg, False), (tr_so, tr_a, tr_seg, True)):
            share = [p // len(members) + (1 if i < p % len(members) else 0) for i in range(len(members))]
            # respect small subgraph spaces: redistribute leftovers
            caps = [int(np.prod([len(v) for v in spaces[s]], dtype=np.float64)) for s in members]
            share = [min(a, c) for a, c in zip(share, caps)]
            left = p - sum(share)
            for i in range(len(members)):
                if left <= 0:
                    break
                add = min(left, caps[i] - share[i])
                share[i] += add
                left -= add
            cnt = 0
            for sid, n in zip(members, share):
                if n <= 0:
                    continue
                a = sample_space(rng, spaces[sid], n)
                dst_so.append(np.full(len(a), sid, np.int32))
                dst_a.append(a)
                if with_lat:
                    tr_lat.append(latency(rng, spaces[sid], a))
                cnt += len(a)
            dst_seg.append(dst_seg[-1] + cnt)
    W = {
        "config": cfg_name, "desc": desc, "model": model, "trees": trees, "per_family": per_family, "spaces": spaces,
        "families": fam_names,
        "pool_so": np.concatenate(pool_so), "pool_a": np.concatenate(pool_a), "pool_seg": np.array(pool_seg, np.int64),
        "tr_so": np.concatenate(tr_so), "tr_a": np.concatenate(tr_a), "tr_seg": np.array(tr_seg, np.int64),
        "tr_y": np.log(np.concatenate(tr_lat)), "tr_lat": np.concatenate(tr_lat),
    }
    return W


def workload_config(W):
    """The workload the line is quoted on (identical dict in the native and reference arms)."""
    return {"workload": W["desc"], "config": W["config"], "model": W["model"], "families": W["families"],
            "candidates_per_step": int(W["pool_seg"][-1]), "train_rows_per_step": int(W["tr_seg"][-1]),
            "trees": W["trees"], "depth": 3, "learning_rate": 0.1, "pad_dim": PAD, "seed": 1000}


def s8d_fit_bytes(rows, trees, depth=3, d=PAD, s_bin=1):
    """SURVEY.md 8(d) algorithmic bytes of one fit of a family of `rows` rows: one-time binning read
    N*D*8, per level N*D*s_bin codes + 9N (residual + node id), per round 24N (residual,
    prediction, leaf update)."""
    return rows * d * 8 + trees * depth * (rows * d * s_bin + 9 * rows) + trees * 24 * rows


def shard_workload(W, rank, world):
    """This rank's families of a global workload (deterministic LPT on rows*T + pool*T,
    paper_2201_00194_b200/sharding.py); records the global unit counts for whole-job rates."""
    import paper_2201_00194_b200 as fs

    F = len(W["families"])
    ps, ts = W["pool_seg"], W["tr_seg"]
    # the product's partition (fs_shard_families, include/famseer.h); sharding.assign_families is
    # its host-side restatement (tests/test_multigpu_gloo.py checks they agree)
    owner = fs.shard_families(np.diff(ts), np.diff(ps), np.full(F, W["trees"], np.int32), world)
    mine = [f for f in range(F) if owner[f] == rank]
    out = dict(W)
    for key_so, key_a, key_seg in (("pool_so", "pool_a", "pool_seg"), ("tr_so", "tr_a", "tr_seg")):
        seg = W[key_seg]
        idx = np.concatenate([np.arange(seg[f], seg[f + 1]) for f in mine]) if mine else np.zeros(0, np.int64)
        out[key_so], out[key_a] = W[key_so][idx], W[key_a][idx]
        out[key_seg] = np.concatenate([[0], np.cumsum([seg[f + 1] - seg[f] for f in mine])]).astype(np.int64)
        if key_seg == "tr_seg":
            out["tr_y"] = W["tr_y"][idx]
    out["families"] = [W["families"][f] for f in mine]
    out["fam_cap"] = max(owner.count(r) for r in range(world))  # all-gather record slots per rank
    out["family_ids"] = mine
    out["P_global"], out["N_global"] = int(ps[-1]), int(ts[-1])
    return out


# ------------------------------------------------------------------------------------------
# clocks (sampled during the timed region)
# ------------------------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) != 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        busy = [s for s in sm if s > 0.5 * max(mx or [1])] or sm
        return {"sm_mhz": statistics.median(busy) if busy else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peak_hbm():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_traffic(kernel):
    """dram bytes per launch of `kernel` from the committed ncu --set full summary, if any."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f).get(kernel)
    except Exception:
        return None


# ------------------------------------------------------------------------------------------
# native arm
# ------------------------------------------------------------------------------------------
def run_native(args, rank, world, local_rank):
    import torch

    import paper_2201_00194_b200 as fs

    # one process per GPU; FAMSEER_BENCH_SHARE_GPU=1 maps several ranks onto the visible GPUs
    # (multi-rank code-path check on a 1-GPU box; collectives then go through gloo)
    share = os.environ.get("FAMSEER_BENCH_SHARE_GPU") == "1"
    if share:
        local_rank = local_rank % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist

        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    if args.shard == "families":
        # strong scaling: ONE global workload, families LPT-partitioned over ranks
        W_global = build_workload(args.config, seed=1000)
        W = shard_workload(W_global, rank, world)
    else:
        # weak scaling: every rank tunes its own copy of the workload (own seed)
        W = build_workload(args.config, seed=1000 + rank)
        W_global = W
    dev = fs.Device(local_rank)
    stream = torch.cuda.ExternalStream(dev.stream)
    spaces = fs.Spaces(dev, W["spaces"])
    F = len(W["families"])
    forest = fs.Forest(dev, max(F, 1))  # a rank may own no family (--shard families, N > F)
    params = fs.GbtParams(W["trees"], 3, 0.1, 2)
    P = int(W["pool_seg"][-1])
    N = int(W["tr_seg"][-1])
    # whole-job units per step: all ranks' work (the global workload when families are sharded)
    P_job = W.get("P_global", P * world)
    N_job = W.get("N_global", N * world)
    with torch.cuda.stream(stream):
        pool_so = torch.from_numpy(W["pool_so"]).cuda()
        pool_a = torch.from_numpy(W["pool_a"]).cuda()
        tr_so = torch.from_numpy(W["tr_so"]).cuda()
        tr_a = torch.from_numpy(W["tr_a"]).cuda()
        x_tr = torch.empty((N, PAD), dtype=torch.float64, device="cuda")
        y_tr = torch.from_numpy(W["tr_y"]).cuda()
        scores = torch.empty(P, dtype=torch.float64, device="cuda")
        perm = torch.empty(P, dtype=torch.int32, device="cuda")
        flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")  # > 126 MB L2
    stream.synchronize()
    # training rows are MeasurementRecord features (featurized at measurement time, simbackend.cpp:185)
    if F:
        spaces.featurize_d(tr_so, tr_a, PAD, x_tr)
        forest.fit_d(x_tr, y_tr, W["tr_seg"], params)  # model the first round scores with
    dev.check()
    pool_seg, tr_seg = W["pool_seg"], W["tr_seg"]
    fam_base = rank * F if args.shard != "families" else 0
    fam_ids = W.get("family_ids", list(range(F)))

    comm = None
    if dist is not None and not share:
        # the product's exchange (fs_comm over NCCL): rank 0 makes the id, torch.distributed
        # carries its bytes to the other ranks
        cid = [fs.Comm.new_id() if rank == 0 else None]
        dist.broadcast_object_list(cid, src=0)
        comm = fs.Comm(dev, world, rank, cid[0])
        n_fam_all = len(W_global["families"]) * (world if args.shard != "families" else 1)
        merged = torch.empty((n_fam_all, G_TOP, 3), dtype=torch.float64, device="cuda")

    def topk_allgather():
        # per-family top-g records {family, pool index, score}; the only collective
        if comm is not None:  # fs_topk_allgather: pack -> ncclAllGather -> merge, on the device
            comm.topk_allgather([fam_base + f for f in fam_ids], pool_seg, scores, perm, G_TOP,
                                W.get("fam_cap", F), n_fam_all, merged)
            return merged
        idx = []
        for f in range(F):
            a, b = int(pool_seg[f]), int(pool_seg[f + 1])
            k = min(G_TOP, b - a)
            p = perm[a:a + k].long() + a
            rec = torch.stack([torch.full((k,), fam_base + fam_ids[f], dtype=torch.float64, device="cuda"),
                               p.double(), scores[p]], 1)
            if k < G_TOP:
                rec = torch.cat([rec, torch.full((G_TOP - k, 3), -1.0, dtype=torch.float64, device="cuda")])
            idx.append(rec)
        mine = torch.cat(idx) if idx else torch.empty((0, 3), dtype=torch.float64, device="cuda")
        cap = W.get("fam_cap", F) * G_TOP  # every rank contributes the same record count
        if mine.shape[0] < cap:
            mine = torch.cat([mine, torch.full((cap - mine.shape[0], 3), -1.0, dtype=torch.float64, device="cuda")])
        if share:  # gloo path of the shared-GPU check: host tensors
            parts = [torch.empty_like(mine, device="cpu") for _ in range(world)]
            dist.all_gather(parts, mine.cpu())
            return torch.cat(parts)
        out = torch.empty((world * mine.shape[0], 3), dtype=torch.float64, device="cuda")
        dist.all_gather_into_tensor(out, mine)
        return out

    def step(overlap=True):
        # one tuning round: score every pool with the current models + refit every family; by
        # default through fs_tune_step_d (the scoring overlaps the refit on a second stream,
        # identical results), --no-overlap issues fs_score_d then fs_fit_d
        if F and overlap and not args.no_overlap:
            forest.tune_step_d(spaces, pool_so, pool_a, PAD, pool_seg, scores, perm, x_tr, y_tr, tr_seg, params)
        elif F:
            spaces.score_d(forest, pool_so, pool_a, PAD, pool_seg, scores, perm)
            forest.fit_d(x_tr, y_tr, tr_seg, params)
        if dist is not None:
            topk_allgather()

    def timed(fn, k, flush_between=True):
        times = []
        for _ in range(k):
            if flush_between:
                with torch.cuda.stream(stream):
                    flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
        return times

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step()
        dev.check()
        # ---- timed region: device-resident value ----
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()
        clocks = ClockSampler(local_rank)
        clocks.start()
        l0 = dev.launches
        dev.counters(reset=True)
        dev.profile("predict,featurize,score_fused,rank,fit_resident")
        times = timed(step, args.steps)
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        clock_info = clocks.stop()
        launches = dev.launches - l0
        prof = dev.profile_read()
        ctr = dev.counters(reset=True)
        dev.profile(None)
        dev.check()
        total_ms = sum(times)
        if dist is not None:
            t = torch.tensor([total_ms], dtype=torch.float64, device="cpu" if share else "cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            total_ms = float(t.item())
        # ---- per-kernel breakdown: one extra, untimed step with every kernel event-timed. The
        # timed steps replay each boosting round as a CUDA graph (no per-kernel events inside), so
        # this replica runs the same kernels on the same inputs without the graph.
        os.environ["FAMSEER_NO_GRAPH"] = "1"
        dev.profile("*")
        dev.counters(reset=True)
        step(overlap=False)  # kernel times undistorted by the concurrent scoring
        prof_all = dev.profile_read()
        ctr_one = dev.counters(reset=True)
        dev.profile(None)
        del os.environ["FAMSEER_NO_GRAPH"]
        breakdown = {k: round(v[1], 4) for k, v in sorted(prof_all.items(), key=lambda kv: -kv[1][1])}
        score_ms = statistics.median(timed(lambda: F and spaces.score_d(forest, pool_so, pool_a, PAD, pool_seg, scores, perm),
                                           max(3, args.steps)))
        fit_ms = statistics.median(timed(lambda: F and forest.fit_d(x_tr, y_tr, tr_seg, params), max(2, min(args.steps, 5))))
        fit_stats = [forest.fit_stats(f) for f in range(F)]

    # ---- e2e: host buffers through the C ABI, copies inside the timed region ----
    e2e = None
    if not args.no_e2e:
        def pinned(a):  # pinned host staging, as a production caller would hold it
            try:
                return torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
            except Exception:
                return np.ascontiguousarray(a)

        h_so, h_a = pinned(W["pool_so"]), pinned(W["pool_a"])
        # training rows travel as measurement records (candidate descriptor + log latency); their
        # features are computed on the device (fs_fit_records, simbackend.cpp:185)
        h_tso, h_ta, h_y = pinned(W["tr_so"]), pinned(W["tr_a"]), pinned(W["tr_y"])
        d2h = [0]

        def e2e_step():
            if not F:
                d2h[0] = 0
                return
            if args.no_overlap:
                s_h, p_h = spaces.score(forest, h_so, h_a, PAD, pool_seg)
                forest.fit_records(spaces, h_tso, h_ta, PAD, h_y, seg=tr_seg, params=params)
            else:
                s_h, p_h = forest.tune_step(spaces, h_so, h_a, PAD, pool_seg, h_tso, h_ta, h_y, tr_seg, params=params)
            nbytes = s_h.nbytes + p_h.nbytes
            for f in range(F):
                e = forest.export(f)
                nbytes += sum(getattr(e, k).nbytes for k in ("offsets", "feature", "threshold", "left", "right",
                                                              "value", "gain", "mse"))
            d2h[0] = nbytes

        with torch.cuda.stream(stream):
            for _ in range(max(1, args.warmup // 2)):
                e2e_step()
            if dist is not None:
                dist.barrier()
            e_times = timed(e2e_step, args.steps)
        e_total = sum(e_times)
        if dist is not None:
            t = torch.tensor([e_total], dtype=torch.float64, device="cpu" if share else "cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_total = float(t.item())
        h2d = h_so.nbytes + h_a.nbytes + h_tso.nbytes + h_ta.nbytes + h_y.nbytes
        e2e = {"value": P_job * args.steps / (e_total / 1e3), "unit": "candidates/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h[0]),
               "train_rows_per_s": N_job * args.steps / (e_total / 1e3), "ms_per_step": e_total / args.steps,
               "api": ("fs_score + fs_fit_records" if args.no_overlap else "fs_tune_step (score + fit_records, overlapped)")
               + " + fs_forest_export (host pointers)"}

    # ---- incremental retrain (fs_store): the tuning loop's real pattern ----
    incremental = None
    if not args.no_e2e and F:
        with torch.cuda.stream(stream):
            incremental = measure_incremental(dev, spaces, W, params, timed, args.steps)

    # ---- roofline of the dominant kernel (from the per-kernel replica step) ----
    peak, peak_kind = measured_peak_hbm()
    cands = []
    if "fit_hist_build" in prof_all and ctr_one["hist_bytes"]:
        n_l, ms = prof_all["fit_hist_build"]
        cands.append(("fit_hist_build", ms, ctr_one["hist_bytes"], n_l,
                      "rows*(nrep*code_bytes + 8 residual + 4 index), rows counted on device", None))
    fam_rows = [int(W["tr_seg"][f + 1] - W["tr_seg"][f]) for f in range(F)]
    s8d_fit = sum(s8d_fit_bytes(n, W["trees"]) for n in fam_rows)  # one fit of every family of this rank
    if "fit_resident" in prof_all:
        n_l, ms = prof_all["fit_resident"]
        cands.append(("fit_resident", ms, ctr_one["hist_bytes"], n_l,
                      "histogram rows*(nrep + 12) counted on device",
                      "latency-bound: all per-row state lives in shared memory for the whole fit; HBM carries "
                      "only the inputs once, so the HBM fraction is structurally small"))
    for k, formula, per in (("predict", "P*(8*d + 8)", 8 * PAD + 8), ("featurize", "P*(64 + 4 + 8*pad)",
                                                                       4 * 16 + 4 + 8 * PAD),
                            ("score_fused", "P*(64 + 4 + 8): descriptor in, score out", 4 * 16 + 4 + 8)):
        if k in prof_all:
            n_l, ms = prof_all[k]
            cands.append((k, ms, P * per, n_l, formula, None))
    roofline = None
    if cands:
        name, ms, nbytes, n_l, formula, note = max(cands, key=lambda r: r[1])
        ach = nbytes / (ms / 1e3) / 1e9
        # the same kernel against SURVEY.md 8(d)'s per-unit bytes (every row and feature at every
        # level, not only the rows the kernel actually histograms)
        s8d = None
        if name == "fit_resident":
            s8d = {"bytes_per_launch": s8d_fit, "formula": "sum_f N_f*D*8 + T*depth*(N_f*D + 9*N_f) + T*24*N_f, "
                   "D = pad_dim 164, s_bin = 1 (u8 codes), depth 3"}
        elif name == "fit_hist_build":
            per_level = sum(n * (PAD + 9) for n in fam_rows)
            s8d = {"bytes_per_launch": per_level, "formula": "per level: sum_f N_f*D*s_bin + 9*N_f, D = 164, s_bin = 1"}
        if s8d:
            a8 = s8d["bytes_per_launch"] * max(n_l, 1) / (ms / 1e3) / 1e9
            s8d.update({"achieved": round(a8, 2), "frac": round(a8 / peak, 5)})
        roofline = {"bound": "hbm", "kernel": name, "achieved": round(ach, 2), "peak": peak, "unit": "GB/s",
                    "frac": round(ach / peak, 5), "frac_s8d": s8d["frac"] if s8d else None, "s8d": s8d,
                    "peak_kind": peak_kind, "traffic": ncu_traffic(name),
                    "algorithmic_bytes_per_launch": nbytes / max(n_l, 1), "launches": n_l,
                    "avg_launch_ms": ms / max(n_l, 1), "bytes_formula": formula,
                    "measured": "CUDA events on the device stream, one untimed replica step without CUDA graphs",
                    "other_kernels": {r[0]: {"ms": round(r[1], 4), "achieved_gbs": round(r[2] / (r[1] / 1e3) / 1e9, 2)}
                                      for r in cands if r[0] != name}}
        if note:
            roofline["note"] = note
    timed_kernel_ms = {k: round(v[1], 4) for k, v in prof.items()}

    result = {
        "metric": METRIC,
        "value": P_job * args.steps / (total_ms / 1e3),
        "unit": "candidates/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": total_ms / args.steps,
        "higher_is_better": True,
        "scaling": "strong" if args.shard == "families" else "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (random candidates from the model's knob spaces, quadratic-bowl latencies)",
        "config": workload_config(W_global),
        "parallelism": (f"families LPT-sharded over {world} GPU(s) (one global workload)" if args.shard == "families"
                        else f"{world} independent replica(s) of the workload, one per GPU"),
        "l2": "flushed between timed steps (256 MB write)",
        "family_ids": fam_ids,
        "family_model_sha": model_digests(forest, F, fam_ids),
        "train_rows_per_s": N_job * args.steps / (total_ms / 1e3),
        "train_row_rounds_per_s": N_job * W["trees"] * args.steps / (total_ms / 1e3),
        "phases_ms": {"score": score_ms, "fit": fit_ms},
        "scored_per_s_score_only": P * world / (score_ms / 1e3),
        "fit_rows_per_s_fit_only": N_job / (fit_ms / 1e3),
        "fit_nodes": {"screened": int(sum(a for a, _ in fit_stats)), "exact": int(sum(b for _, b in fit_stats))},
        "kernel_ms_one_step": breakdown,
        "kernel_ms_timed_region": timed_kernel_ms,
        "device_counters": ctr,
        "gpu_launches": int(launches),
        "clocks": clock_info,
        "roofline": roofline,
        "e2e": e2e,
        "incremental": incremental,
    }
    if dist is not None:  # every rank's family digests on rank 0
        parts = [None] * world
        dist.all_gather_object(parts, (fam_ids, result["family_model_sha"]))
        result["family_ids"] = sorted(i for ids, _ in parts for i in ids)
        result["family_model_sha"] = {k: v for _, d in parts for k, v in sorted(d.items(), key=lambda kv: int(kv[0]))}
    if rank == 0 and not args.no_cpu:
        result["cpu_baseline"] = cpu_baseline(W, forest, x_tr.cpu().numpy(), min_seconds=args.cpu_seconds)
    if world == 1 and not args.no_secondary and args.config != "c5":
        result["secondary_c5"] = secondary_c5()
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return result


def secondary_c5():
    """BASELINE configs[4] (64 families x 65,536 candidates/rows, T = 1000) at N = 1, where the
    trainer's histogram build - not a latency chain - dominates: its own bench line (a child
    bench.py, 3 warm-up + 2 timed steps, inputs resident, L2 flushed), kept as a block."""
    cmd = [sys.executable, os.path.abspath(__file__), "--config", "c5", "--steps", "2", "--warmup", "3", "--no-e2e",
           "--no-cpu", "--no-secondary"]
    try:
        out = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
        line = [ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1]
        d = json.loads(line)
    except Exception as e:  # pragma: no cover - reported, never fatal for the headline line
        return {"error": f"{type(e).__name__}: {e}"}
    keep = ("value", "unit", "ms_per_step", "steps", "warmup", "config", "train_rows_per_s", "train_row_rounds_per_s",
            "phases_ms", "roofline", "clocks", "gpu_launches", "kernel_ms_one_step", "fit_nodes")
    return {k: d.get(k) for k in keep}


def model_digests(forest, F, fam_ids):
    """sha256 of every fitted family model (pre-order trees, base, train_mse_by_round), keyed by
    global family id: equal digests across --gpus N runs show the per-family results do not depend
    on which GPU computed them."""
    import hashlib

    out = {}
    for f in range(F):
        e = forest.export(f)
        h = hashlib.sha256(np.float64(e.base).tobytes())
        for k in ("offsets", "feature", "threshold", "left", "right", "value", "mse"):
            h.update(np.ascontiguousarray(getattr(e, k)).tobytes())
        out[str(fam_ids[f])] = h.hexdigest()[:16]
    return out


def measure_incremental(dev, spaces, W, params, timed, steps, g=64, warm=2):
    """Retrain as the tuning loop does it (scheduler.cpp:228-235, train_cost_model
    costmodel.cpp:224-235): every step each family receives g new measurement records and is
    refit on everything it holds. Two ways through the public API, both timed with CUDA events
    including the host->device copies: fs_store (the host sends the g new records; the canonical
    order is merged, the refit skips the sort) and fs_fit_records on the family's full record set
    each step (the host resends every record; the fit re-sorts). Families start at their bench
    size minus the held-back batches."""
    import paper_2201_00194_b200 as fs

    seg = [int(v) for v in W["tr_seg"]]
    F = len(seg) - 1
    gf = [min(g, (seg[f + 1] - seg[f]) // (warm + steps + 2)) for f in range(F)]
    live = [f for f in range(F) if gf[f] > 0]
    if not live:
        return None
    so, asg, lat = W["tr_so"], W["tr_a"], W["tr_lat"]
    # targets exactly as the store computes them (std::log on the host, costmodel.cpp:232)
    tmp = fs.Store(dev, 1, 0)
    tmp.append([0], np.zeros((len(lat), 0)), lat)
    y = tmp.read(0)[1]
    tmp.close()
    start = {f: seg[f + 1] - (warm + steps) * gf[f] for f in live}
    store = fs.Store(dev, F, PAD)
    fo_s, fo_f = fs.Forest(dev, F), fs.Forest(dev, F)
    fam0 = live
    idx0 = np.concatenate([np.arange(seg[f], start[f]) for f in fam0])
    sg0 = np.cumsum([0] + [start[f] - seg[f] for f in fam0])
    store.append_records(spaces, fam0, so[idx0], asg[idx0], lat[idx0], seg=sg0)
    store.fit(fo_s, families=live, params=params)
    dev.check()
    step_no = [0]

    def batch(k):
        idx = np.concatenate([np.arange(start[f] + k * gf[f], start[f] + (k + 1) * gf[f]) for f in live])
        sg = np.cumsum([0] + [gf[f] for f in live])
        return idx, sg

    def store_step():
        idx, sg = batch(step_no[0])
        store.append_records(spaces, live, so[idx], asg[idx], lat[idx], seg=sg)
        store.fit(fo_s, families=live, params=params)
        step_no[0] += 1

    full_no = [0]

    def full_step():
        k = full_no[0] + 1
        idx = np.concatenate([np.arange(seg[f], start[f] + k * gf[f]) for f in live])
        sg = np.cumsum([0] + [start[f] + k * gf[f] - seg[f] for f in live])
        fo_f.fit_records(spaces, so[idx], asg[idx], PAD, y[idx], seg=list(sg), params=params)
        full_no[0] += 1

    for _ in range(warm):
        store_step()
        full_step()
    t_store = timed(store_step, steps)
    t_full = timed(full_step, steps)
    # the two paths hold the same rows at the end: identical models
    same = all(np.array_equal(fo_s.export(f).value, fo_f.export(live.index(f)).value) for f in live)
    store.close()
    return {"g_per_family": gf, "families_refit": live, "steps": steps,
            "rows_start": {f: start[f] - seg[f] for f in live},
            "store_ms_per_step": statistics.median(t_store), "full_refit_ms_per_step": statistics.median(t_full),
            "speedup": statistics.median(t_full) / statistics.median(t_store),
            "h2d_bytes_per_step_store": int(sum(gf[f] for f in live) * (4 + 64 + 8)),
            "identical_models": bool(same),
            "api": "fs_store_append_records + fs_store_fit vs fs_fit_records on the whole set"}


# ------------------------------------------------------------------------------------------
# reference CPU arm (oracle/_ref = the unmodified reference core; test/baseline infrastructure)
# ------------------------------------------------------------------------------------------
def _ref_family(W, x_tr, models, f, trees=None):
    """The reference hot path for one family: featurize + predict + std::sort of its pool
    (scheduler.cpp:187-192) and a from-scratch fit on its rows (costmodel.cpp:152-222), on the
    compiled reference (oracle/_ref). Returns (score seconds, fit seconds, trees fitted)."""
    import oracle

    r = oracle.ref()
    pool_so, pool_a, pool_seg = W["pool_so"], W["pool_a"], W["pool_seg"]
    a, b = int(pool_seg[f]), int(pool_seg[f + 1])
    t0 = time.perf_counter()
    x = np.zeros((b - a, PAD))
    for sid in np.unique(pool_so[a:b]):
        rows = np.where(pool_so[a:b] == sid)[0]
        kn = W["spaces"][sid]
        x[rows] = r.featurize(kn, pool_a[a:b][rows][:, : len(kn)], PAD)
    s = models[f].predict(x)
    r.rank(s)
    t1 = time.perf_counter()
    t = trees or W["trees"]
    ta, tb = int(W["tr_seg"][f]), int(W["tr_seg"][f + 1])
    m = r.new_model(f, t)
    m.add_samples(x_tr[ta:tb], W["tr_y"][ta:tb])
    m.fit()
    m.free()
    return t1 - t0, time.perf_counter() - t1, t


def _parallel(fams, threads, fn):
    """Run fn(f) for every family on up to `threads` host threads (ctypes releases the GIL),
    like one std::thread per family. Returns {f: fn(f)}."""
    pending, out, lock = list(fams), {}, threading.Lock()

    def runner():
        while True:
            with lock:
                if not pending:
                    return
                f = pending.pop(0)
            out[f] = fn(f)

    ts = [threading.Thread(target=runner) for _ in range(max(1, min(threads, len(fams))))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    return out


def _ref_round(W, x_tr, models, threads, plan):
    """One (possibly sampled) round on the host cores. plan = (families, tree sample). Full
    rounds time every family with all trees. Sampled rounds (configs too large to run, e.g. C5
    at ~0.3 core-hours per family) time the families in `families` with `tree sample` trees and
    extrapolate linearly in trees and in the family count: per-family time = score + fit * T/t,
    round = ceil(F / threads) waves of the mean family time. Returns (seconds, extrapolated?)."""
    fams, t_s = plan
    F = len(W["families"])
    t0 = time.perf_counter()
    res = _parallel(fams, threads, lambda f: _ref_family(W, x_tr, models, f, t_s))
    wall = time.perf_counter() - t0
    if len(fams) == F and (t_s is None or t_s >= W["trees"]):
        return wall, False
    per = [sc + fi * W["trees"] / t for sc, fi, t in res.values()]
    waves = math.ceil(F / max(1, min(threads, F)))
    return waves * (sum(per) / len(per)), True


def _ref_plan(W, threads):
    """Full rounds when a round is cheap enough; else a bounded sample (~10-20 s of CPU work)."""
    F = len(W["families"])
    rows = [int(W["tr_seg"][f + 1] - W["tr_seg"][f]) for f in range(F)]
    # survey probe P1: ~3.8 us per (row x tree) at d=164 on one core (fit dominates)
    est = max(rows) * W["trees"] * 3.8e-6 * math.ceil(F / max(1, min(threads, F)))
    if est <= 20.0:
        return list(range(F)), None
    big = sorted(range(F), key=lambda f: (-rows[f], f))[: max(1, min(threads, F, 2))]
    t_s = max(1, min(W["trees"], int(10.0 / (max(rows) * 3.8e-6))))
    return big, t_s


def _ref_models(W, forest, x_tr, threads):
    import oracle

    r = oracle.ref()
    models = []
    for f in range(len(W["families"])):
        m = r.new_model(f, W["trees"])
        if forest is not None:
            e = forest.export(f)
            m.load(oracle.Ensemble(e.base, e.lr, e.offsets, e.feature, e.threshold, e.left, e.right, e.value))
        else:
            ta, tb = int(W["tr_seg"][f]), int(W["tr_seg"][f + 1])
            _, t_s = _ref_plan(W, threads)
            m2 = r.new_model(f, min(W["trees"], t_s or W["trees"]))
            m2.add_samples(x_tr[ta:tb], W["tr_y"][ta:tb])
            m2.fit()
            m.load(m2.export())
            m2.free()
        models.append(m)
    return models


def cpu_baseline(W, forest, x_tr, min_seconds=10.0):
    threads = os.cpu_count() or 1
    models = _ref_models(W, forest, x_tr, threads)
    plan = _ref_plan(W, threads)
    P = int(W["pool_seg"][-1])
    rounds, t_sum, extrap, t0 = 0, 0.0, False, time.perf_counter()
    while True:
        sec, extrap = _ref_round(W, x_tr, models, threads, plan)
        t_sum += sec
        rounds += 1
        if time.perf_counter() - t0 >= min_seconds or rounds >= 50:
            break
    fams, t_s = plan
    sample = (f"{rounds} full round(s) of the workload ({P} candidates scored + {int(W['tr_seg'][-1])} rows refit, "
              f"T={W['trees']})" if not extrap else
              f"{rounds} sampled round(s): families {fams} scored in full and fit with {t_s} of {W['trees']} trees, "
              f"EXTRAPOLATED linearly in trees and family count")
    return {"value": P * rounds / t_sum, "unit": "candidates/s", "cores": min(threads, len(W["families"])),
            "kind": "reference", "sample": sample + "; one thread per family; oracle/_ref = unmodified reference "
            "core (-O3, no -march)", "extrapolated": extrap, "seconds": time.perf_counter() - t0,
            "host_cpu": _cpu_model(), "nproc": os.cpu_count()}


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def _featurize_host(W, orc):
    parts = []
    for i in range(len(W["tr_seg"]) - 1):
        a, b = int(W["tr_seg"][i]), int(W["tr_seg"][i + 1])
        x = np.zeros((b - a, PAD))
        for sid in np.unique(W["tr_so"][a:b]):
            rows = np.where(W["tr_so"][a:b] == sid)[0]
            kn = W["spaces"][sid]
            x[rows] = orc.featurize(kn, W["tr_a"][a:b][rows][:, : len(kn)], PAD)
        parts.append(x)
    return np.concatenate(parts)


def run_reference(args, rank, world):
    if rank != 0:
        return None
    import oracle

    try:
        oracle.ref()
    except Exception as e:  # pragma: no cover
        return {"impl": "reference", "unavailable": f"compiled reference missing: {e}"}
    W = build_workload(args.config, seed=1000)
    x_tr = _featurize_host(W, oracle.orc())
    threads = os.cpu_count() or 1
    models = _ref_models(W, None, x_tr, threads)
    plan = _ref_plan(W, threads)
    P, N, F = int(W["pool_seg"][-1]), int(W["tr_seg"][-1]), len(W["families"])
    for _ in range(args.warmup):
        _ref_round(W, x_tr, models, threads, plan)
    times, extrap = [], False
    for _ in range(args.steps):
        sec, extrap = _ref_round(W, x_tr, models, threads, plan)
        times.append(sec)
    total = sum(times)
    v = P * args.steps / total
    cores = min(threads, F)
    return {"metric": METRIC, "impl": "reference", "value": v, "unit": "candidates/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total / args.steps * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (same generator and seed as the native arm's rank 0)",
            "config": workload_config(W),
            "train_rows_per_s": N * args.steps / total,
            "cpu_baseline": {"value": v, "unit": "candidates/s", "cores": cores, "kind": "reference",
                             "sample": ("full rounds" if not extrap else f"sampled rounds {plan}, extrapolated")
                             + " of the workload, one thread per family (oracle/_ref)", "extrapolated": extrap,
                             "host_cpu": _cpu_model(), "nproc": os.cpu_count()},
            "e2e": {"value": v, "unit": "candidates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def self_launch(n):
    """`bench.py --gpus N` without a launcher: re-exec under torchrun, one rank per GPU (NCCL over
    NVLink for the top-k all-gather; NCCL's INFO log, which names the communicator's ranks, goes
    to stderr so stdout keeps the one JSON line)."""
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    env.setdefault("OMP_NUM_THREADS", "1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    sys.stdout.flush()
    os.execvpe(sys.executable, cmd, env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-overlap", action="store_true",
                    help="score then refit as two calls instead of one fs_tune_step (scoring forked onto a second stream)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--shard", default=None, choices=["replicate", "families"],
                    help="families (default for N > 1): one global workload, families LPT-partitioned over "
                         "ranks (strong scaling, SURVEY 8e); replicate: every rank tunes its own workload copy "
                         "(weak scaling)")
    ap.add_argument("--no-secondary", action="store_true", help="skip the secondary C5 block at N = 1")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        self_launch(args.gpus)  # does not return
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.shard is None:
        args.shard = "families" if world > 1 else "replicate"
    if args.impl == "reference":
        res = run_reference(args, rank, world)
    else:
        res = run_native(args, rank, world, local_rank)
    if rank == 0 and res is not None:
        print(json.dumps(res))


if __name__ == "__main__":
    main()
