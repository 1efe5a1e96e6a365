"""paper_2201_00194_b200 - B200-native FamilySeer cost-model hot path.

Python face of libfamseer.so (C ABI in include/famseer.h) used by the tests and bench.py. The
product API mirrors the reference's cost-model interface (famtune, /root/reference/proj/core):

  featurize           searchspace.cpp:90-118      Device.featurize / Spaces
  predict             costmodel.cpp:237-246       Forest.predict
  tune_step ranking   scheduler.cpp:187-192       Device.rank
  fit / train         costmodel.cpp:152-235       Forest.fit / Forest.train
  family grouping     family.cpp:22-140           paper_2201_00194_b200.families

Everything runs on the GPU through the C ABI; there is no CPU fallback. Host numpy arrays go
through the host-pointer entry points (copies inside the call); torch CUDA tensors go through the
``_d`` entry points on the device's stream.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _capi
from ._capi import FS_MAX_KNOBS, GbtParams

__all__ = ["Device", "Spaces", "Forest", "Store", "Comm", "shard_families", "Ensemble", "GbtParams", "FamseerError", "InvalidArgument",
           "DomainError", "OutOfRange", "feature_dim", "FS_MAX_KNOBS"]


class FamseerError(RuntimeError):
    pass


class InvalidArgument(FamseerError, ValueError):
    """std::invalid_argument in the reference."""


class DomainError(FamseerError, ArithmeticError):
    """std::domain_error in the reference."""


class OutOfRange(FamseerError, IndexError):
    """std::out_of_range in the reference."""


_EXC = {_capi.FS_EINVAL: InvalidArgument, _capi.FS_EDOMAIN: DomainError, _capi.FS_ERANGE: OutOfRange}


def _lib():
    return _capi.load()


def _check(rc: int):
    if rc != _capi.FS_OK:
        msg = _lib().fs_last_error().decode()
        raise _EXC.get(rc, FamseerError)(msg)


def _p(a, t):
    return None if a is None else a.ctypes.data_as(t)


def _seg(seg):
    s = np.ascontiguousarray(seg, np.int64)
    return s, s.ctypes.data_as(_capi._i64p)


def feature_dim(k: int) -> int:
    """searchspace.cpp:86-88."""
    return int(_lib().fs_feature_dim(k))


@dataclass
class Ensemble:
    """One family's ensemble in the CostModelState pre-order layout (costmodel.hpp:27-57)."""

    base: float
    lr: float
    offsets: np.ndarray
    feature: np.ndarray
    threshold: np.ndarray
    left: np.ndarray
    right: np.ndarray
    value: np.ndarray
    gain: np.ndarray | None = None
    mse: np.ndarray | None = None

    @property
    def n_trees(self) -> int:
        return len(self.offsets) - 1


class Device:
    """fs_device: one per GPU (stream, scratch, deferred errors)."""

    def __init__(self, ordinal: int = 0):
        h = _capi._vp()
        _check(_lib().fs_device_create(ordinal, C.byref(h)))
        self.h = h
        self.ordinal = ordinal

    def close(self):
        if getattr(self, "h", None):
            _lib().fs_device_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream_ptr: int | None):
        _check(_lib().fs_device_set_stream(self.h, stream_ptr))

    @property
    def stream(self) -> int:
        return _lib().fs_device_stream(self.h) or 0

    def check(self):
        _check(_lib().fs_device_check(self.h))

    @property
    def launches(self) -> int:
        return int(_lib().fs_device_launches(self.h))

    def counters(self, reset: bool = True) -> dict[str, int]:
        """Device work counters: histogram algorithmic bytes/rows, reference-order folds/nodes."""
        out = np.zeros(24, np.int64)
        _check(_lib().fs_device_counters(self.h, _p(out, _capi._i64p), 24, int(reset)))
        d = dict(zip(("hist_bytes", "hist_rows", "exact_chains", "exact_nodes"), (int(v) for v in out[:4])))
        names = ("residual", "plan", "hist", "derive", "screen", "tie_class", "decide", "exact_fold", "split",
                 "partition", "leaves", "mse")
        if out[4:16].any():
            d["resident_phase_cycles_cta0"] = {k: int(v) for k, v in zip(names, out[4:16])}
        if out[16:20].any():
            d["exact_reasons"] = {k: int(v) for k, v in zip(("multi_candidate_feature", "different_partitions",
                                                               "orders_differ", "uncertain_sign"), out[16:20])}
        if out[20:24].any():
            d["probe"] = [int(v) for v in out[20:24]]
        return d

    # -- per-kernel CUDA-event timing ------------------------------------------------------------
    def profile(self, kernels: str | None):
        """Enable event timing for a comma-separated kernel list ("*" = all, None = off)."""
        _check(_lib().fs_device_profile(self.h, kernels.encode() if kernels else None))

    def profile_read(self) -> dict[str, tuple[int, float]]:
        L = _lib()
        need = L.fs_device_profile_names(self.h, None, 0)
        buf = C.create_string_buffer(max(int(need), 1))
        L.fs_device_profile_names(self.h, buf, need)
        out = {}
        for name in filter(None, buf.value.decode().split(",")):
            cnt, ms = C.c_int64(), C.c_double()
            _check(L.fs_device_profile_read(self.h, name.encode(), C.byref(cnt), C.byref(ms)))
            out[name] = (cnt.value, ms.value)
        return out

    # -- ranking (scheduler.cpp:187-192) --------------------------------------------------------
    def rank(self, scores, seg=None):
        s = np.ascontiguousarray(scores, np.float64)
        if seg is None:
            seg = [0, len(s)]
        sg, sp = _seg(seg)
        perm = np.zeros(len(s), np.int32)
        _check(_lib().fs_rank(self.h, len(sg) - 1, sp, _p(s, _capi._dp), _p(perm, _capi._i32p)))
        return perm

    def pairwise_accuracy(self, scores, latency) -> float:
        """costmodel.cpp:248-277 over precomputed scores (pair count on the device)."""
        s = np.ascontiguousarray(scores, np.float64)
        lat = np.ascontiguousarray(latency, np.float64)
        out = C.c_double()
        _check(_lib().fs_pairwise_accuracy(self.h, len(s), _p(s, _capi._dp), _p(lat, _capi._dp), C.byref(out)))
        return out.value

    def pairwise_accuracy_batch(self, scores, latency, seg) -> np.ndarray:
        """Per-segment pairwise accuracy in one launch (the accuracy heatmap's model x
        validation-set grid, experiment.cpp:135-167)."""
        s = np.ascontiguousarray(scores, np.float64)
        lat = np.ascontiguousarray(latency, np.float64)
        sg, sp = _seg(seg)
        out = np.zeros(len(sg) - 1)
        _check(_lib().fs_pairwise_accuracy_batch(self.h, len(sg) - 1, sp, _p(s, _capi._dp), _p(lat, _capi._dp),
                                                  _p(out, _capi._dp)))
        return out

    def rank_d(self, scores_t, seg, perm_t):
        sg, sp = _seg(seg)
        _check(_lib().fs_rank_d(self.h, len(sg) - 1, sp, scores_t.data_ptr(), perm_t.data_ptr()))


class Spaces:
    """fs_spaces: knob-space table; featurize (searchspace.cpp:90-118) over a population."""

    def __init__(self, dev: Device, spaces):
        """spaces: list (one per space) of lists of knob value lists."""
        self.dev = dev
        self.k = [len(s) for s in spaces]
        nk = np.array(self.k, np.int32)
        nv = np.zeros((len(spaces), FS_MAX_KNOBS), np.int32)
        vals = []
        for i, s in enumerate(spaces):
            for j, v in enumerate(s):
                nv[i, j] = len(v)
                vals.extend(int(a) for a in v)
        va = np.array(vals if vals else [1], np.int64)
        h = _capi._vp()
        _check(_lib().fs_spaces_create(dev.h, len(spaces), _p(nk, _capi._i32p), _p(nv, _capi._i32p),
                                       _p(va, _capi._i64p), C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            _lib().fs_spaces_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def max_feature_dim(self) -> int:
        return int(_lib().fs_spaces_max_feature_dim(self.h))

    def featurize(self, space_of, assign, pad_dim: int):
        so = np.ascontiguousarray(space_of, np.int32)
        a = np.zeros((len(so), FS_MAX_KNOBS), np.int32)
        src = np.asarray(assign, np.int32)
        if src.ndim == 1:
            src = src[None]
        a[:, : src.shape[1]] = src
        out = np.zeros((len(so), pad_dim))
        _check(_lib().fs_featurize(self.dev.h, self.h, len(so), _p(so, _capi._i32p), _p(a, _capi._i32p), pad_dim,
                                   _p(out, _capi._dp)))
        return out

    def featurize_d(self, space_of_t, assign_t, pad_dim: int, out_t):
        _check(_lib().fs_featurize_d(self.dev.h, self.h, space_of_t.numel(), space_of_t.data_ptr(),
                                     assign_t.data_ptr(), pad_dim, out_t.data_ptr()))

    def score(self, forest: "Forest", space_of, assign, pad_dim: int, seg):
        """tune_step's scoring block (scheduler.cpp:187-192): featurize -> predict -> rank, host
        buffers in and out. Returns (scores, perm) with perm segment-local."""
        so = np.ascontiguousarray(space_of, np.int32)
        a = np.ascontiguousarray(assign, np.int32)
        sg, sp = _seg(seg)
        scores = np.zeros(len(so))
        perm = np.zeros(len(so), np.int32)
        _check(_lib().fs_score(self.dev.h, self.h, forest.h, len(sg) - 1, sp, _p(so, _capi._i32p),
                               _p(a, _capi._i32p), pad_dim, _p(scores, _capi._dp), _p(perm, _capi._i32p)))
        return scores, perm

    def score_index(self, forest: "Forest", space_of, index, pad_dim: int, seg):
        """fs_score from (space id, linear_index) descriptors (searchspace.cpp:48-66): the device
        decodes each u64 mixed-radix index like candidate_from_index. Returns (scores, perm)."""
        so = np.ascontiguousarray(space_of, np.int32)
        ix = np.ascontiguousarray(index, np.uint64)
        sg, sp = _seg(seg)
        scores = np.empty(len(so), np.float64)
        perm = np.empty(len(so), np.int32)
        _check(_lib().fs_score_index(self.dev.h, self.h, forest.h, len(sg) - 1, sp, _p(so, _capi._i32p),
                                     _p(ix, _capi._u64p), pad_dim, _p(scores, _capi._dp), _p(perm, _capi._i32p)))
        return scores, perm

    def score_index_d(self, forest: "Forest", space_of_t, index_t, pad_dim: int, seg, scores_t, perm_t):
        sg, sp = _seg(seg)
        _check(_lib().fs_score_index_d(self.dev.h, self.h, forest.h, len(sg) - 1, sp, space_of_t.data_ptr(),
                                       index_t.data_ptr(), pad_dim, scores_t.data_ptr(),
                                       None if perm_t is None else perm_t.data_ptr()))

    def score_d(self, forest: "Forest", space_of_t, assign_t, pad_dim: int, seg, scores_t, perm_t):
        sg, sp = _seg(seg)
        _check(_lib().fs_score_d(self.dev.h, self.h, forest.h, len(sg) - 1, sp, space_of_t.data_ptr(),
                                 assign_t.data_ptr(), pad_dim, scores_t.data_ptr(),
                                 None if perm_t is None else perm_t.data_ptr()))


class Forest:
    """fs_forest: one ensemble per family (TuningEngine::models_, scheduler.cpp:123-130)."""

    def __init__(self, dev: Device, n_families: int):
        self.dev = dev
        self.n = n_families
        h = _capi._vp()
        _check(_lib().fs_forest_create(dev.h, n_families, C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            _lib().fs_forest_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def upload(self, family: int, ens):
        off = np.ascontiguousarray(ens.offsets, np.int32)
        feat = np.ascontiguousarray(ens.feature, np.int32)
        thr = np.ascontiguousarray(ens.threshold, np.float64)
        le = np.ascontiguousarray(ens.left, np.int32)
        ri = np.ascontiguousarray(ens.right, np.int32)
        va = np.ascontiguousarray(ens.value, np.float64)
        _check(_lib().fs_forest_upload(self.h, family, float(ens.base), float(ens.lr), len(off) - 1,
                                       _p(off, _capi._i32p), _p(feat, _capi._i32p), _p(thr, _capi._dp),
                                       _p(le, _capi._i32p), _p(ri, _capi._i32p), _p(va, _capi._dp)))

    def export(self, family: int, lr: float = 0.1) -> Ensemble:
        raw = _lib().fs_forest_export_raw
        hdr = np.zeros(4, np.float64)  # base | n_trees, n_nodes (int32 pair in the second word)
        a0 = hdr.ctypes.data
        _check(raw(self.h, family, a0, a0 + 8, a0 + 12, *([None] * 8)))
        t, n = int(hdr[1:2].view(np.int32)[0]), int(hdr[1:2].view(np.int32)[1])
        # one int32 and one float64 buffer, the arrays as views
        ib = np.empty(t + 1 + 3 * n, np.int32)
        db = np.empty(3 * n + max(t, 1), np.float64)
        ia, da = ib.ctypes.data, db.ctypes.data
        _check(raw(self.h, family, a0, None, None, ia, ia + 4 * (t + 1), da, ia + 4 * (t + 1 + n),
                   ia + 4 * (t + 1 + 2 * n), da + 8 * n, da + 16 * n, da + 24 * n))
        off, feat, le, ri = ib[:t + 1], ib[t + 1:t + 1 + n], ib[t + 1 + n:t + 1 + 2 * n], ib[t + 1 + 2 * n:]
        thr, va, gain, mse = db[:n], db[n:2 * n], db[2 * n:3 * n], db[3 * n:3 * n + t]
        return Ensemble(float(hdr[0]), lr, off, feat, thr, le, ri, va, gain, mse)

    def predict(self, x, seg=None, leaves: bool = False):
        x = np.ascontiguousarray(x, np.float64)
        if x.ndim == 1:
            x = x[None]
        if seg is None:
            seg = [0, x.shape[0]]
        sg, sp = _seg(seg)
        out = np.zeros(x.shape[0])
        lo = None
        if leaves:
            total = 0
            for f in range(len(sg) - 1):
                total += int(sg[f + 1] - sg[f]) * self.export_n_trees(f)
            lo = np.zeros(max(total, 1), np.uint16)
        _check(_lib().fs_predict(self.dev.h, self.h, len(sg) - 1, sp, x.shape[1], _p(x, _capi._dp),
                                 _p(out, _capi._dp), _p(lo, _capi._u16p)))
        return (out, lo) if leaves else out

    def predict_d(self, x_t, seg, scores_t, leaves_t=None):
        sg, sp = _seg(seg)
        _check(_lib().fs_predict_d(self.dev.h, self.h, len(sg) - 1, sp, x_t.shape[1], x_t.data_ptr(),
                                   scores_t.data_ptr(), None if leaves_t is None else leaves_t.data_ptr()))

    def export_n_trees(self, family: int) -> int:
        nt = C.c_int32()
        _check(_lib().fs_forest_export(self.h, family, None, C.byref(nt), *([None] * 10)))
        return nt.value

    def fit(self, x, target, seg=None, params=None):
        """Refit each family segment from scratch (costmodel.cpp:152-222)."""
        x = np.ascontiguousarray(x, np.float64)
        y = np.ascontiguousarray(target, np.float64)
        if seg is None:
            seg = [0, x.shape[0]]
        sg, sp = _seg(seg)
        nf = len(sg) - 1
        pa = _params_array(params, nf)
        d = x.shape[1] if x.ndim == 2 else 0
        _check(_lib().fs_fit(self.dev.h, self.h, nf, sp, d, _p(x, _capi._dp), _p(y, _capi._dp), pa))

    def fit_d(self, x_t, target_t, seg, params=None):
        sg, sp = _seg(seg)
        nf = len(sg) - 1
        pa = _params_array(params, nf)
        _check(_lib().fs_fit_d(self.dev.h, self.h, nf, sp, x_t.shape[1], x_t.data_ptr(), target_t.data_ptr(), pa))

    def fit_records(self, spaces: "Spaces", space_of, assign, pad_dim: int, target, seg=None, params=None):
        """Refit from measurement records (candidate descriptors + log latency): features are
        computed on the device (simbackend.cpp:185), the host sends 68 B per record."""
        so = np.ascontiguousarray(space_of, np.int32)
        a = np.ascontiguousarray(assign, np.int32)
        if a.ndim != 2 or a.shape[1] != 16:
            raise InvalidArgument("assign must be [n][16] value indices")
        y = np.ascontiguousarray(target, np.float64)
        if seg is None:
            seg = [0, len(so)]
        sg, sp = _seg(seg)
        nf = len(sg) - 1
        pa = _params_array(params, nf)
        _check(_lib().fs_fit_records(self.dev.h, self.h, spaces.h, nf, sp, _p(so, _capi._i32p), _p(a, _capi._i32p),
                                     pad_dim, _p(y, _capi._dp), pa))

    def fit_records_d(self, spaces: "Spaces", space_of_t, assign_t, pad_dim: int, target_t, seg, params=None):
        sg, sp = _seg(seg)
        nf = len(sg) - 1
        pa = _params_array(params, nf)
        _check(_lib().fs_fit_records_d(self.dev.h, self.h, spaces.h, nf, sp, space_of_t.data_ptr(),
                                       assign_t.data_ptr(), pad_dim, target_t.data_ptr(), pa))

    def tune_step_d(self, spaces: "Spaces", pool_so_t, pool_a_t, pad_dim: int, pool_seg, scores_t, perm_t, x_t,
                    target_t, fit_seg, params=None):
        """One tuning round, overlapped (fs_tune_step_d): score the pools with the CURRENT models
        (scheduler.cpp:187-192) while refitting every fit segment (:233-238); same results as
        Spaces.score_d followed by fit_d."""
        psg, psp = _seg(pool_seg)
        fsg, fsp = _seg(fit_seg)
        pa = _params_array(params, len(fsg) - 1)
        _check(_lib().fs_tune_step_d(self.dev.h, spaces.h, self.h, len(psg) - 1, psp, pool_so_t.data_ptr(),
                                     pool_a_t.data_ptr(), pad_dim, scores_t.data_ptr(),
                                     None if perm_t is None else perm_t.data_ptr(), len(fsg) - 1, fsp,
                                     x_t.data_ptr(), target_t.data_ptr(), pa))

    def tune_step(self, spaces: "Spaces", pool_so, pool_a, pad_dim: int, pool_seg, tr_so, tr_a, tr_target, fit_seg,
                  params=None):
        """fs_tune_step, host buffers: returns (scores, perm) of the pools under the models as
        they were, then the forest holds the refit models (training rows as records)."""
        so = np.ascontiguousarray(pool_so, np.int32)
        a = np.ascontiguousarray(pool_a, np.int32)
        tso = np.ascontiguousarray(tr_so, np.int32)
        ta = np.ascontiguousarray(tr_a, np.int32)
        ty = np.ascontiguousarray(tr_target, np.float64)
        psg = np.ascontiguousarray(pool_seg, np.int64)
        fsg = np.ascontiguousarray(fit_seg, np.int64)
        pa = _params_array(params, len(fsg) - 1)
        scores = np.empty(len(so), np.float64)
        perm = np.empty(len(so), np.int32)
        # raw addresses (the per-step call builds no ctypes pointer objects)
        _check(_lib().fs_tune_step_raw(self.dev.h, spaces.h, self.h, len(psg) - 1, psg.ctypes.data, so.ctypes.data,
                                       a.ctypes.data, pad_dim, scores.ctypes.data, perm.ctypes.data, len(fsg) - 1,
                                       fsg.ctypes.data, tso.ctypes.data, ta.ctypes.data, ty.ctypes.data, pa))
        return scores, perm

    def fit_stats(self, family: int):
        a, b = C.c_int64(), C.c_int64()
        _check(_lib().fs_forest_fit_stats(self.h, family, C.byref(a), C.byref(b)))
        return a.value, b.value


class Store:
    """fs_store: every family's training set kept on the device across retrains (SURVEY.md 8f
    row 2; CostModelState::training_set, costmodel.hpp:48-57). append() is train_cost_model's
    push_back (costmodel.cpp:224-233: target = log(latency)), fit() its refit (:152-222); the
    canonical row order is maintained by merge-insert instead of re-sorted per fit."""

    def __init__(self, dev: Device, n_families: int, d: int):
        self.dev = dev
        self.n = n_families
        self.d = d
        h = _capi._vp()
        _check(_lib().fs_store_create(dev.h, n_families, d, C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            _lib().fs_store_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @staticmethod
    def _segs(family, seg, n):
        fam = np.ascontiguousarray(np.atleast_1d(family), np.int32)
        if seg is None:
            seg = [0, n]
        sg = np.ascontiguousarray(seg, np.int64)
        if len(sg) != len(fam) + 1:
            raise InvalidArgument("seg must have one more entry than family")
        return fam, sg

    def append(self, family, x, latency_ms, seg=None):
        """Rows [seg[k], seg[k+1]) of x / latency_ms go to family[k]."""
        xa = np.ascontiguousarray(x, np.float64).reshape(-1, self.d) if self.d else np.zeros((len(latency_ms), 0))
        lat = np.ascontiguousarray(latency_ms, np.float64)
        fam, sg = self._segs(family, seg, len(lat))
        _check(_lib().fs_store_append(self.h, len(fam), _p(fam, _capi._i32p), _p(sg, _capi._i64p),
                                      _p(xa, _capi._dp), _p(lat, _capi._dp)))

    def append_records(self, spaces: "Spaces", family, space_of, assign, latency_ms, seg=None):
        so = np.ascontiguousarray(space_of, np.int32)
        a = np.ascontiguousarray(assign, np.int32)
        if a.ndim != 2 or a.shape[1] != 16:
            raise InvalidArgument("assign must be [n][16] value indices")
        lat = np.ascontiguousarray(latency_ms, np.float64)
        fam, sg = self._segs(family, seg, len(lat))
        _check(_lib().fs_store_append_records(self.h, spaces.h, len(fam), _p(fam, _capi._i32p),
                                              _p(sg, _capi._i64p), _p(so, _capi._i32p), _p(a, _capi._i32p),
                                              _p(lat, _capi._dp)))

    def rows(self, family: int) -> int:
        r = C.c_int64()
        _check(_lib().fs_store_rows(self.h, family, C.byref(r)))
        return r.value

    def read(self, family: int):
        """(x, target, canonical order or None) of one family, rows in append order."""
        n = self.rows(family)
        x = np.zeros((n, self.d))
        y = np.zeros(n)
        c = np.zeros(n, np.int32)
        ok = C.c_int32()
        _check(_lib().fs_store_read(self.h, family, _p(x, _capi._dp), _p(y, _capi._dp), _p(c, _capi._i32p),
                                    C.byref(ok)))
        return x, y, (c if ok.value else None)

    def fit(self, forest: "Forest", families=None, params=None):
        fam = np.ascontiguousarray(range(self.n) if families is None else families, np.int32)
        pa = _params_array(params, len(fam))
        _check(_lib().fs_store_fit(self.h, forest.h, len(fam), _p(fam, _capi._i32p), pa))


def _params_array(params, n):
    if params is None:
        params = GbtParams(50, 3, 0.1, 2)
    if isinstance(params, GbtParams):
        params = [params] * n
    arr = (GbtParams * n)(*params)
    return arr


# ---- multi-GPU: family-parallel tuning -------------------------------------------
def shard_families(rows, pool, trees, world: int) -> list[int]:
    """fs_shard_families: deterministic LPT owner rank per family (cost rows*T + pool*T)."""
    r = np.ascontiguousarray(rows, np.int64)
    p = np.ascontiguousarray(pool, np.int64)
    t = np.ascontiguousarray(trees, np.int32)
    owner = np.zeros(len(r), np.int32)
    _check(_lib().fs_shard_families(len(r), _p(r, _capi._i64p), _p(p, _capi._i64p), _p(t, _capi._i32p), world,
                                    _p(owner, _capi._i32p)))
    return owner.tolist()


class Comm:
    """fs_comm: the NCCL communicator of one rank (one process per GPU). Rank 0 makes the id
    (Comm.new_id()); the caller broadcasts the bytes to the other ranks."""

    ID_BYTES = 128

    @staticmethod
    def new_id() -> bytes:
        buf = (C.c_uint8 * Comm.ID_BYTES)()
        _check(_lib().fs_comm_id(buf))
        return bytes(buf)

    def __init__(self, dev: Device, world: int, rank: int, comm_id: bytes):
        self.dev = dev
        buf = (C.c_uint8 * Comm.ID_BYTES).from_buffer_copy(comm_id)
        h = C.c_void_p()
        _check(_lib().fs_comm_create(dev.h, world, rank, buf, C.byref(h)))
        self.h = h.value

    def topk_allgather(self, family_ids, seg, scores_t, perm_t, g: int, fam_cap: int, n_families: int, merged_t):
        """Every local family's first g ranked candidates, all-gathered and merged on the device
        into merged_t [n_families][g][3] (family id, pool index, score; -1 where absent)."""
        ids = np.ascontiguousarray(family_ids, np.int32)
        sg = np.ascontiguousarray(seg, np.int64)
        _check(_lib().fs_topk_allgather(self.h, len(ids), _p(ids, _capi._i32p), _p(sg, _capi._i64p),
                                        scores_t.data_ptr(), perm_t.data_ptr(), g, fam_cap, n_families,
                                        merged_t.data_ptr()))

    def close(self):
        if getattr(self, "h", None):
            _lib().fs_comm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
