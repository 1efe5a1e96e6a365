"""ctypes binding of libfamseer.so (include/famseer.h).

The library is built in-tree (``paper_2201_00194_b200/libfamseer.so``). There is no fallback:
if the shared object is missing or no B200 is visible, every entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# FAMSEER_LIB: an alternative in-tree build of the same library (A/B experiments)
LIB_PATH = os.environ.get("FAMSEER_LIB") or os.path.join(HERE, "libfamseer.so")

FS_OK, FS_EINVAL, FS_EDOMAIN, FS_ERANGE, FS_ECUDA, FS_ENOMEM, FS_ENCCL = range(7)
FS_MAX_KNOBS = 16

_dp = C.POINTER(C.c_double)
_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_u64p = C.POINTER(C.c_uint64)
_u8p = C.POINTER(C.c_uint8)
_u16p = C.POINTER(C.c_uint16)
_vp = C.c_void_p


class GbtParams(C.Structure):
    """fs_gbt_params == famtune::GbtParams (costmodel.hpp:20-25)."""

    _fields_ = [("trees", C.c_int32), ("depth", C.c_int32), ("learning_rate", C.c_double),
                ("min_samples_split", C.c_int32)]


# (name, restype, argtypes) for every symbol include/famseer.h declares.
SIGNATURES = [
    ("fs_last_error", C.c_char_p, []),
    ("fs_version", C.c_char_p, []),
    ("fs_device_create", C.c_int, [C.c_int, C.POINTER(_vp)]),
    ("fs_device_destroy", C.c_int, [_vp]),
    ("fs_device_set_stream", C.c_int, [_vp, _vp]),
    ("fs_device_stream", _vp, [_vp]),
    ("fs_device_check", C.c_int, [_vp]),
    ("fs_device_launches", C.c_int64, [_vp]),
    ("fs_device_counters", C.c_int, [_vp, _i64p, C.c_int32, C.c_int32]),
    ("fs_device_profile", C.c_int, [_vp, C.c_char_p]),
    ("fs_device_profile_read", C.c_int, [_vp, C.c_char_p, _i64p, _dp]),
    ("fs_device_profile_names", C.c_int64, [_vp, C.c_char_p, C.c_int64]),
    ("fs_pairwise_accuracy", C.c_int, [_vp, C.c_int64, _dp, _dp, _dp]),
    ("fs_pairwise_accuracy_batch", C.c_int, [_vp, C.c_int32, _i64p, _dp, _dp, _dp]),
    ("fs_fit_records", C.c_int, [_vp, _vp, _vp, C.c_int32, _i64p, _i32p, _i32p, C.c_int32, _dp,
                                 C.POINTER(GbtParams)]),
    ("fs_fit_records_d", C.c_int, [_vp, _vp, _vp, C.c_int32, _i64p, _vp, _vp, C.c_int32, _vp,
                                   C.POINTER(GbtParams)]),
    ("fs_store_create", C.c_int, [_vp, C.c_int32, C.c_int32, C.POINTER(_vp)]),
    ("fs_store_destroy", C.c_int, [_vp]),
    ("fs_store_append", C.c_int, [_vp, C.c_int32, _i32p, _i64p, _dp, _dp]),
    ("fs_store_append_records", C.c_int, [_vp, _vp, C.c_int32, _i32p, _i64p, _i32p, _i32p, _dp]),
    ("fs_store_rows", C.c_int, [_vp, C.c_int32, _i64p]),
    ("fs_store_read", C.c_int, [_vp, C.c_int32, _dp, _dp, _i32p, _i32p]),
    ("fs_store_fit", C.c_int, [_vp, _vp, C.c_int32, _i32p, C.POINTER(GbtParams)]),
    ("fs_score", C.c_int, [_vp, _vp, _vp, C.c_int32, _i64p, _i32p, _i32p, C.c_int32, _dp, _i32p]),
    ("fs_score_d", C.c_int, [_vp, _vp, _vp, C.c_int32, _i64p, _vp, _vp, C.c_int32, _vp, _vp]),
    ("fs_tune_step_d", C.c_int, [_vp, _vp, _vp, C.c_int32, _i64p, _vp, _vp, C.c_int32, _vp, _vp, C.c_int32, _i64p,
                                  _vp, _vp, _vp]),
    ("fs_tune_step", C.c_int, [_vp, _vp, _vp, C.c_int32, _i64p, _i32p, _i32p, C.c_int32, _dp, _i32p, C.c_int32,
                                _i64p, _i32p, _i32p, _dp, _vp]),
    ("fs_shard_families", C.c_int, [C.c_int32, _i64p, _i64p, _i32p, C.c_int32, _i32p]),
    ("fs_comm_id", C.c_int, [C.POINTER(C.c_uint8)]),
    ("fs_comm_create", C.c_int, [_vp, C.c_int32, C.c_int32, C.POINTER(C.c_uint8), C.POINTER(_vp)]),
    ("fs_comm_destroy", C.c_int, [_vp]),
    ("fs_topk_allgather", C.c_int, [_vp, C.c_int32, _i32p, _i64p, _vp, _vp, C.c_int32, C.c_int32, C.c_int32, _vp]),
    ("fs_score_index", C.c_int, [_vp, _vp, _vp, C.c_int32, _i64p, _i32p, _u64p, C.c_int32, _dp, _i32p]),
    ("fs_score_index_d", C.c_int, [_vp, _vp, _vp, C.c_int32, _i64p, _vp, _vp, C.c_int32, _vp, _vp]),
    ("fs_feature_dim", C.c_int, [C.c_int32]),
    ("fs_spaces_create", C.c_int, [_vp, C.c_int32, _i32p, _i32p, _i64p, C.POINTER(_vp)]),
    ("fs_spaces_destroy", C.c_int, [_vp]),
    ("fs_spaces_max_feature_dim", C.c_int32, [_vp]),
    ("fs_featurize", C.c_int, [_vp, _vp, C.c_int64, _i32p, _i32p, C.c_int32, _dp]),
    ("fs_featurize_d", C.c_int, [_vp, _vp, C.c_int64, _vp, _vp, C.c_int32, _vp]),
    ("fs_forest_create", C.c_int, [_vp, C.c_int32, C.POINTER(_vp)]),
    ("fs_forest_destroy", C.c_int, [_vp]),
    ("fs_forest_upload", C.c_int, [_vp, C.c_int32, C.c_double, C.c_double, C.c_int32, _i32p, _i32p, _dp, _i32p,
                                   _i32p, _dp]),
    ("fs_forest_export", C.c_int, [_vp, C.c_int32, _dp, _i32p, _i32p, _i32p, _i32p, _dp, _i32p, _i32p, _dp, _dp,
                                   _dp]),
    ("fs_predict", C.c_int, [_vp, _vp, C.c_int32, _i64p, C.c_int32, _dp, _dp, _u16p]),
    ("fs_predict_d", C.c_int, [_vp, _vp, C.c_int32, _i64p, C.c_int32, _vp, _vp, _vp]),
    ("fs_rank", C.c_int, [_vp, C.c_int32, _i64p, _dp, _i32p]),
    ("fs_rank_d", C.c_int, [_vp, C.c_int32, _i64p, _vp, _vp]),
    ("fs_fit", C.c_int, [_vp, _vp, C.c_int32, _i64p, C.c_int32, _dp, _dp, C.POINTER(GbtParams)]),
    ("fs_fit_d", C.c_int, [_vp, _vp, C.c_int32, _i64p, C.c_int32, _vp, _vp, C.POINTER(GbtParams)]),
    ("fs_forest_fit_stats", C.c_int, [_vp, C.c_int32, _i64p, _i64p]),
]

_lib = None


def load(path: str = LIB_PATH) -> C.CDLL:
    """Load libfamseer.so and attach signatures. Raises if it was never built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing - run __graft_entry__.build() (no CPU fallback exists)")
    lib = C.CDLL(path)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    # the same export entry with raw addresses (the hot per-family export avoids building a
    # ctypes pointer object per array)
    raw = lib["fs_forest_export"]
    raw.restype = C.c_int
    raw.argtypes = [_vp, C.c_int32] + [C.c_void_p] * 11
    lib.fs_forest_export_raw = raw
    raw = lib["fs_tune_step"]
    raw.restype = C.c_int
    raw.argtypes = [_vp, _vp, _vp, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p,
                    C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, _vp]
    lib.fs_tune_step_raw = raw
    _lib = lib
    return lib
