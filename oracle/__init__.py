"""TEST INFRASTRUCTURE ONLY - ctypes faces of the CPU checkers.

* ``orc``  - the plain-C restatement in ``oracle/famtune_oracle.c`` (liboracle.so).
* ``ref``  - the unmodified reference core compiled from /root/reference into
  ``oracle/_ref/libfamtune_ref.so`` (see oracle/Makefile, oracle/ref_shim.cpp).

Only tests/, ``__graft_entry__.smoke()`` and the cpu_baseline / ``--impl reference`` legs of
bench.py may import this package. The product (``paper_2201_00194_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libfamtune_ref.so")

_dp = C.POINTER(C.c_double)
_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_u64p = C.POINTER(C.c_uint64)
_u8p = C.POINTER(C.c_uint8)
_u16p = C.POINTER(C.c_uint16)


def _p(a, t):
    return a.ctypes.data_as(t) if a is not None else None


def build(with_ref: bool | None = None) -> None:
    """Compile liboracle.so (and oracle/_ref when /root/reference is present)."""
    targets = ["oracle"]
    if with_ref is None:
        with_ref = os.path.isdir("/root/reference/proj/core/src")
    if with_ref:
        # the compiled reference core, and the reference's unchanged tuning engine linked both
        # against it (engine_ref) and against the B200 drop-in (engine_b200) for
        # tests/test_engine_e2e.py - built here, they travel to the GPU box as binaries
        targets += ["ref", "engines"]
    subprocess.run(["make", "-s", "-C", HERE, "-j8", *targets], check=True)


class OracleError(RuntimeError):
    pass


class InvalidArgument(OracleError, ValueError):
    pass


class DomainError(OracleError, ArithmeticError):
    pass


class OutOfRange(OracleError, IndexError):
    pass


_ERRS = {1: InvalidArgument, 2: DomainError, 3: OutOfRange, 4: OracleError}


@dataclass
class Ensemble:
    """Flat pre-order tree ensemble (costmodel.hpp:27-57 laid out as arrays)."""

    base: float
    lr: float
    offsets: np.ndarray  # int32 [T+1]
    feature: np.ndarray  # int32 [nodes]
    threshold: np.ndarray  # f64
    left: np.ndarray  # int32
    right: np.ndarray  # int32
    value: np.ndarray  # f64
    mse: np.ndarray = field(default_factory=lambda: np.zeros(0))  # f64 [T]
    gain: np.ndarray | None = None  # f64 [nodes] (oracle replica only)

    @property
    def n_trees(self) -> int:
        return len(self.offsets) - 1

    def tree(self, t):
        a, b = self.offsets[t], self.offsets[t + 1]
        return (self.feature[a:b], self.threshold[a:b], self.left[a:b], self.right[a:b], self.value[a:b])


def empty_ensemble(base=0.0, lr=0.1) -> Ensemble:
    z32 = np.zeros(0, np.int32)
    return Ensemble(base, lr, np.zeros(1, np.int32), z32, np.zeros(0), z32, z32, np.zeros(0))


class _Orc:
    def __init__(self, path=ORACLE_SO):
        if not os.path.exists(path):
            build(with_ref=False)
        L = C.CDLL(path)
        L.orc_last_error.restype = C.c_char_p
        L.orc_featurize.argtypes = [C.c_int, _i32p, _i64p, _i32p, C.c_int64, C.c_int, C.c_int, _dp]
        L.orc_predict.argtypes = [C.c_double, C.c_double, C.c_int, _i32p, _i32p, _dp, _i32p, _i32p, _dp,
                                  C.c_int64, C.c_int, _dp, _dp, _u16p]
        L.orc_rank.argtypes = [C.c_int64, _dp, _i64p]
        L.orc_fit.argtypes = [C.c_int64, C.c_int, _dp, _dp, C.c_int, C.c_int, C.c_double, C.c_int, _dp,
                              C.POINTER(C.c_int), _i32p, _i32p, _dp, _i32p, _i32p, _dp, _dp, _dp, C.c_int64]
        L.orc_pairwise_accuracy.argtypes = [_dp, _dp, C.c_int64, _dp]
        L.orc_select.argtypes = [C.c_int64, _i64p, C.c_int, C.c_double, C.c_uint64, _i64p]
        L.orc_mix_seed.restype = C.c_uint64
        L.orc_mix_seed.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
        L.orc_linear_index.argtypes = [C.c_int, _i32p, _i32p, C.c_int64, C.c_int, _u64p]
        L.orc_candidate_from_index.argtypes = [C.c_int, _i32p, _u64p, C.c_int64, C.c_int, _i32p]
        self.L = L

    def _chk(self, rc):
        if rc not in (0, None) and rc > 0 and rc in _ERRS:
            raise _ERRS[rc](self.L.orc_last_error().decode())
        return rc

    def featurize(self, values_per_knob, assign, pad_dim):
        nv = np.array([len(v) for v in values_per_knob], np.int32)
        vals = np.ascontiguousarray(np.concatenate([np.asarray(v, np.int64) for v in values_per_knob]))
        a = np.ascontiguousarray(assign, np.int32)
        if a.ndim == 1:
            a = a[None]
        out = np.zeros((a.shape[0], pad_dim))
        self._chk(self.L.orc_featurize(len(values_per_knob), _p(nv, _i32p), _p(vals, _i64p), _p(a, _i32p),
                                       a.shape[0], a.shape[1], pad_dim, _p(out, _dp)))
        return out

    def linear_index(self, nvals, assign):
        """searchspace.cpp:48-54 for every row of assign (int32 [p][>= k])."""
        nv = np.ascontiguousarray(nvals, np.int32)
        a = np.ascontiguousarray(np.atleast_2d(assign), np.int32)
        out = np.zeros(a.shape[0], np.uint64)
        self.L.orc_linear_index(len(nv), _p(nv, _i32p), _p(a, _i32p), a.shape[0], a.shape[1], _p(out, _u64p))
        return out

    def candidate_from_index(self, nvals, index, stride=16):
        """searchspace.cpp:56-66 for every index: int32 [p][stride] (knobs beyond k are 0)."""
        nv = np.ascontiguousarray(nvals, np.int32)
        ix = np.ascontiguousarray(index, np.uint64)
        out = np.zeros((len(ix), stride), np.int32)
        self.L.orc_candidate_from_index(len(nv), _p(nv, _i32p), _p(ix, _u64p), len(ix), stride, _p(out, _i32p))
        return out

    def predict(self, ens: Ensemble, x, leaves=False):
        x = np.ascontiguousarray(x, np.float64)
        if x.ndim == 1:
            x = x[None]
        out = np.zeros(x.shape[0])
        lo = np.zeros((x.shape[0], max(ens.n_trees, 1)), np.uint16) if leaves else None
        self._chk(self.L.orc_predict(ens.base, ens.lr, ens.n_trees, _p(ens.offsets, _i32p),
                                     _p(ens.feature, _i32p), _p(ens.threshold, _dp), _p(ens.left, _i32p),
                                     _p(ens.right, _i32p), _p(ens.value, _dp), x.shape[0], x.shape[1],
                                     _p(x, _dp), _p(out, _dp), _p(lo, _u16p)))
        return (out, lo[:, : ens.n_trees]) if leaves else out

    def rank(self, scores):
        s = np.ascontiguousarray(scores, np.float64)
        perm = np.zeros(len(s), np.int64)
        self._chk(self.L.orc_rank(len(s), _p(s, _dp), _p(perm, _i64p)))
        return perm

    def fit(self, x, target, trees=50, depth=3, lr=0.1, min_split=2) -> Ensemble:
        x = np.ascontiguousarray(x, np.float64)
        y = np.ascontiguousarray(target, np.float64)
        n, d = x.shape
        cap = max(trees, 1) * ((1 << (depth + 1)) - 1)
        base = C.c_double()
        nt = C.c_int()
        off = np.zeros(trees + 1, np.int32)
        feat = np.zeros(cap, np.int32)
        thr = np.zeros(cap)
        left = np.zeros(cap, np.int32)
        right = np.zeros(cap, np.int32)
        val = np.zeros(cap)
        gain = np.zeros(cap)
        mse = np.zeros(max(trees, 1))
        self._chk(self.L.orc_fit(n, d, _p(x, _dp), _p(y, _dp), trees, depth, lr, min_split, C.byref(base),
                                 C.byref(nt), _p(off, _i32p), _p(feat, _i32p), _p(thr, _dp), _p(left, _i32p),
                                 _p(right, _i32p), _p(val, _dp), _p(gain, _dp), _p(mse, _dp), cap))
        t = nt.value
        m = off[t]
        return Ensemble(base.value, lr, off[: t + 1].copy(), feat[:m].copy(), thr[:m].copy(), left[:m].copy(),
                        right[:m].copy(), val[:m].copy(), mse[:t].copy(), gain[:m].copy())

    def pairwise_accuracy(self, scores, latency):
        s = np.ascontiguousarray(scores, np.float64)
        l = np.ascontiguousarray(latency, np.float64)
        out = C.c_double()
        self._chk(self.L.orc_pairwise_accuracy(_p(s, _dp), _p(l, _dp), len(s), C.byref(out)))
        return out.value

    def select(self, perm, g_eff, epsilon, stream_seed):
        perm = np.ascontiguousarray(perm, np.int64)
        picks = np.zeros(max(g_eff, len(perm)), np.int64)
        n = self._chk(self.L.orc_select(len(perm), _p(perm, _i64p), g_eff, epsilon, stream_seed, _p(picks, _i64p)))
        return picks[:n]

    def mix_seed(self, seed, a=0, b=0):
        return self.L.orc_mix_seed(seed, a, b)


class _Ref:
    """The reference's own implementation (oracle/_ref). Raises if it was never built."""

    def __init__(self, path=REF_SO):
        if not os.path.exists(path):
            build(with_ref=True)
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: build it here (needs /root/reference)")
        L = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_featurize.argtypes = [C.c_int, _i32p, _i64p, _i32p, C.c_int64, C.c_int, C.c_int, _dp]
        L.ref_featurize_checked.argtypes = [C.c_int, _i32p, _i64p, _i32p, C.c_int, C.c_int, _dp]
        L.ref_model_new.restype = C.c_void_p
        L.ref_model_new.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_int]
        L.ref_model_free.argtypes = [C.c_void_p]
        L.ref_model_add_samples.argtypes = [C.c_void_p, C.c_int64, C.c_int, _dp, _dp]
        L.ref_model_fit.argtypes = [C.c_void_p]
        L.ref_model_train.argtypes = [C.c_void_p, C.c_int64, C.c_int, _dp, _dp]
        for f in ("ref_model_num_trees", "ref_model_num_nodes", "ref_model_num_samples"):
            getattr(L, f).argtypes = [C.c_void_p]
        L.ref_model_export.argtypes = [C.c_void_p, _dp, _i32p, _i32p, _dp, _i32p, _i32p, _dp, _dp]
        L.ref_model_import.argtypes = [C.c_void_p, C.c_double, C.c_int, _i32p, _i32p, _dp, _i32p, _i32p, _dp]
        L.ref_predict.argtypes = [C.c_void_p, C.c_int64, C.c_int, _dp, _dp]
        L.ref_pairwise_accuracy.argtypes = [C.c_void_p, C.c_int64, C.c_int, _dp, _dp, _dp]
        L.ref_dump_model.restype = C.c_int64
        L.ref_dump_model.argtypes = [C.c_void_p, C.c_char_p, C.c_int64]
        L.ref_rank.argtypes = [C.c_int64, _dp, _i64p]
        L.ref_model_info.argtypes = [C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.ref_cluster.restype = C.c_int64
        L.ref_cluster.argtypes = [C.c_char_p, C.c_int, _i32p, C.c_char_p, C.c_int64]
        L.ref_subgraph_space.argtypes = [C.c_char_p, C.c_int, C.POINTER(C.c_int), _i32p, _i64p]
        L.ref_subgraph_info.restype = C.c_int64
        L.ref_subgraph_info.argtypes = [C.c_char_p, C.c_int, C.c_char_p, C.c_int64]
        L.ref_family_dataset.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_uint64, C.c_int, C.c_int, C.c_int64,
                                         _dp, _dp, _i32p, _i32p, _i64p]
        L.ref_tune.restype = C.c_int64
        L.ref_tune.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int64, C.c_double, C.c_uint64, C.c_int, C.c_int,
                               C.c_double, C.c_int, C.c_int, C.c_int64, _dp, _dp, _i64p, C.POINTER(C.c_int),
                               C.c_char_p, C.c_int64]
        L.ref_rng_draws.restype = C.c_uint64
        L.ref_rng_draws.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_int, C.c_uint64, _u64p]
        L.ref_linear_index.argtypes = [C.c_int, _i32p, _i64p, _i32p, C.c_int64, C.c_int, _u64p]
        L.ref_candidate_from_index.argtypes = [C.c_int, _i32p, _i64p, _u64p, C.c_int64, C.c_int, _i32p]
        self.L = L

    def _chk(self, rc):
        if rc:
            raise _ERRS.get(rc, OracleError)(self.L.ref_last_error().decode())

    # -- featurize -------------------------------------------------------------------------
    def featurize(self, values_per_knob, assign, pad_dim):
        nv = np.array([len(v) for v in values_per_knob], np.int32)
        vals = np.ascontiguousarray(np.concatenate([np.asarray(v, np.int64) for v in values_per_knob]))
        a = np.ascontiguousarray(assign, np.int32)
        if a.ndim == 1:
            out = np.zeros(pad_dim)
            self._chk(self.L.ref_featurize_checked(len(values_per_knob), _p(nv, _i32p), _p(vals, _i64p),
                                                   _p(a, _i32p), len(a), pad_dim, _p(out, _dp)))
            return out
        out = np.zeros((a.shape[0], pad_dim))
        self._chk(self.L.ref_featurize(len(values_per_knob), _p(nv, _i32p), _p(vals, _i64p), _p(a, _i32p),
                                       a.shape[0], a.shape[1], pad_dim, _p(out, _dp)))
        return out

    def linear_index(self, values_per_knob, assign):
        nv = np.array([len(v) for v in values_per_knob], np.int32)
        vals = np.ascontiguousarray(np.concatenate([np.asarray(v, np.int64) for v in values_per_knob]))
        a = np.ascontiguousarray(np.atleast_2d(assign), np.int32)
        out = np.zeros(a.shape[0], np.uint64)
        self._chk(self.L.ref_linear_index(len(nv), _p(nv, _i32p), _p(vals, _i64p), _p(a, _i32p), a.shape[0],
                                          a.shape[1], _p(out, _u64p)))
        return out

    def candidate_from_index(self, values_per_knob, index, stride=16):
        nv = np.array([len(v) for v in values_per_knob], np.int32)
        vals = np.ascontiguousarray(np.concatenate([np.asarray(v, np.int64) for v in values_per_knob]))
        ix = np.ascontiguousarray(index, np.uint64)
        out = np.zeros((len(ix), stride), np.int32)
        self._chk(self.L.ref_candidate_from_index(len(nv), _p(nv, _i32p), _p(vals, _i64p), _p(ix, _u64p), len(ix),
                                                  stride, _p(out, _i32p)))
        return out

    # -- models ----------------------------------------------------------------------------
    def new_model(self, family_id=0, trees=50, depth=3, lr=0.1, min_split=2):
        return RefModel(self, self.L.ref_model_new(family_id, trees, depth, lr, min_split), lr)

    def fit(self, x, target, trees=50, depth=3, lr=0.1, min_split=2) -> Ensemble:
        m = self.new_model(0, trees, depth, lr, min_split)
        try:
            m.add_samples(x, target)
            m.fit()
            return m.export()
        finally:
            m.free()

    def rank(self, scores):
        s = np.ascontiguousarray(scores, np.float64)
        perm = np.zeros(len(s), np.int64)
        self._chk(self.L.ref_rank(len(s), _p(s, _dp), _p(perm, _i64p)))
        return perm

    # -- model files / simulator -------------------------------------------------------------
    def model_info(self, path):
        n, pad = C.c_int(), C.c_int()
        self._chk(self.L.ref_model_info(path.encode(), C.byref(n), C.byref(pad)))
        return n.value, pad.value

    def cluster(self, path, algo=0):
        n, _ = self.model_info(path)
        fam = np.zeros(n, np.int32)
        need = self.L.ref_cluster(path.encode(), algo, _p(fam, _i32p), None, 0)
        if need < 0:
            self._chk(-need)
        buf = C.create_string_buffer(int(need))
        self.L.ref_cluster(path.encode(), algo, _p(fam, _i32p), buf, need)
        return fam, buf.value.decode()

    def subgraph_space(self, path, sid):
        k = C.c_int()
        nv = np.zeros(16, np.int32)
        vals = np.zeros(16 * 4096, np.int64)
        self._chk(self.L.ref_subgraph_space(path.encode(), sid, C.byref(k), _p(nv, _i32p), _p(vals, _i64p)))
        out, off = [], 0
        for i in range(k.value):
            out.append(vals[off: off + nv[i]].tolist())
            off += nv[i]
        return out

    def subgraph_info(self, path, sid):
        need = self.L.ref_subgraph_info(path.encode(), sid, None, 0)
        if need < 0:
            self._chk(-need)
        buf = C.create_string_buffer(int(need))
        self.L.ref_subgraph_info(path.encode(), sid, buf, need)
        seq, full, core, weight = buf.value.decode().split("\t")
        return {"ops": seq.split(","), "serial": full, "core_op": core, "weight": int(weight)}

    def family_dataset(self, path, algo, family, seed, per_subgraph, pad_dim, cap=1 << 20):
        x = np.zeros((cap, pad_dim))
        lat = np.zeros(cap)
        sid = np.zeros(cap, np.int32)
        asg = np.zeros((cap, 16), np.int32)
        n = C.c_int64()
        self._chk(self.L.ref_family_dataset(path.encode(), algo, family, seed, per_subgraph, pad_dim, cap,
                                            _p(x, _dp), _p(lat, _dp), _p(sid, _i32p), _p(asg, _i32p), C.byref(n)))
        k = n.value
        return x[:k].copy(), lat[:k].copy(), sid[:k].copy(), asg[:k].copy()

    def tune(self, path, budget, *, algo=0, foresee=True, p=0.25, seed=1, trees=50, depth=3, lr=0.1,
             min_split=2, export_family=-1, cap=1 << 16):
        _, pad = self.model_info(path)
        x = np.zeros((cap, max(pad, 1)))
        y = np.zeros(cap)
        n = C.c_int64()
        d = C.c_int()
        args = [path.encode(), algo, int(foresee), budget, p, seed, trees, depth, lr, min_split, export_family, cap,
                _p(x, _dp), _p(y, _dp), C.byref(n), C.byref(d)]
        need = self.L.ref_tune(*args, None, 0)
        if need < 0:
            self._chk(-need)
        buf = C.create_string_buffer(int(need))
        self.L.ref_tune(*args, buf, need)
        k, dd = n.value, d.value
        xs = x.reshape(-1)[: k * dd].reshape(k, dd).copy() if dd else np.zeros((0, 0))
        return buf.value.decode(), xs, y[:k].copy()

    def rng_draws(self, seed, a, b, n, bound=0):
        out = np.zeros(n, np.uint64)
        self.L.ref_rng_draws(seed, a, b, n, bound, _p(out, _u64p))
        return out


class RefModel:
    def __init__(self, owner: _Ref, handle, lr):
        self.o, self.h, self.lr = owner, handle, lr

    def free(self):
        if self.h:
            self.o.L.ref_model_free(self.h)
            self.h = None

    def add_samples(self, x, target):
        x = np.ascontiguousarray(x, np.float64)
        y = np.ascontiguousarray(target, np.float64)
        self.o._chk(self.o.L.ref_model_add_samples(self.h, x.shape[0], x.shape[1], _p(x, _dp), _p(y, _dp)))

    def fit(self):
        self.o._chk(self.o.L.ref_model_fit(self.h))

    def train(self, x, latency):
        x = np.ascontiguousarray(x, np.float64)
        if x.ndim == 1:
            x = x[None]
        lat = np.ascontiguousarray(latency, np.float64)
        self.o._chk(self.o.L.ref_model_train(self.h, x.shape[0], x.shape[1] if x.size else 0, _p(x, _dp),
                                             _p(lat, _dp)))

    def export(self) -> Ensemble:
        L = self.o.L
        t = L.ref_model_num_trees(self.h)
        m = L.ref_model_num_nodes(self.h)
        base = C.c_double()
        off = np.zeros(t + 1, np.int32)
        feat = np.zeros(m, np.int32)
        thr = np.zeros(m)
        left = np.zeros(m, np.int32)
        right = np.zeros(m, np.int32)
        val = np.zeros(m)
        mse = np.zeros(max(t, 1))
        self.o._chk(L.ref_model_export(self.h, C.byref(base), _p(off, _i32p), _p(feat, _i32p), _p(thr, _dp),
                                       _p(left, _i32p), _p(right, _i32p), _p(val, _dp), _p(mse, _dp)))
        return Ensemble(base.value, self.lr, off, feat, thr, left, right, val, mse[:t])

    def load(self, ens: Ensemble):
        self.o._chk(self.o.L.ref_model_import(self.h, ens.base, ens.n_trees, _p(ens.offsets, _i32p),
                                              _p(ens.feature, _i32p), _p(ens.threshold, _dp), _p(ens.left, _i32p),
                                              _p(ens.right, _i32p), _p(ens.value, _dp)))

    def predict(self, x):
        x = np.ascontiguousarray(x, np.float64)
        if x.ndim == 1:
            x = x[None]
        out = np.zeros(x.shape[0])
        self.o._chk(self.o.L.ref_predict(self.h, x.shape[0], x.shape[1], _p(x, _dp), _p(out, _dp)))
        return out

    def pairwise_accuracy(self, x, latency):
        x = np.ascontiguousarray(x, np.float64)
        lat = np.ascontiguousarray(latency, np.float64)
        out = C.c_double()
        self.o._chk(self.o.L.ref_pairwise_accuracy(self.h, x.shape[0], x.shape[1] if x.ndim == 2 else 0,
                                                   _p(x, _dp), _p(lat, _dp), C.byref(out)))
        return out.value

    def dump(self):
        need = self.o.L.ref_dump_model(self.h, None, 0)
        buf = C.create_string_buffer(int(need))
        self.o.L.ref_dump_model(self.h, buf, need)
        return buf.value.decode()


_orc = None
_ref = None


def orc() -> _Orc:
    global _orc
    if _orc is None:
        _orc = _Orc()
    return _orc


def ref() -> _Ref:
    global _ref
    if _ref is None:
        _ref = _Ref()
    return _ref


def ref_available() -> bool:
    return os.path.exists(REF_SO)
