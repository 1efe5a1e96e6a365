"""Family grouping (family.cpp:22-140) through the drop-in C++ library (libfamtune_b200.so).

Families are the key of the per-family model store; ids must equal the reference's bit for bit.
Host-only (a pure function of subgraph attributes, computed once per tuning run).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "libfamtune_b200.so")
ALGOS = {"core-op": 0, "op-count": 1, "op-sequence": 2}
OP_KINDS = ["conv1d", "conv2d", "conv3d", "depthwise_conv2d", "dense", "batch_matmul", "softmax", "pooling", "relu",
            "gelu", "sigmoid", "tanh", "add", "multiply", "layer_norm", "batch_norm", "embedding", "transpose",
            "reshape", "reduce"]

_lib = None


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            raise ImportError(f"{LIB} missing - run __graft_entry__.build()")
        L = C.CDLL(LIB)
        ip = C.POINTER(C.c_int)
        L.famtune_cluster.restype = C.c_int
        L.famtune_cluster.argtypes = [C.c_int, ip, ip, ip, C.c_int, ip, C.c_char_p, C.c_longlong,
                                      C.POINTER(C.c_longlong)]
        _lib = L
    return _lib


def cluster(subgraphs, algo: str = "core-op"):
    """subgraphs: sequence of dicts with 'core_op' (name) and 'ops' (list of op-kind names), in
    subgraph-id order. Returns (family id per subgraph, registry CSV)."""
    L = _load()
    n = len(subgraphs)
    core = np.array([OP_KINDS.index(s["core_op"]) for s in subgraphs], np.int32)
    off = np.zeros(n + 1, np.int32)
    kinds = []
    for i, s in enumerate(subgraphs):
        kinds.extend(OP_KINDS.index(k) for k in s["ops"])
        off[i + 1] = len(kinds)
    kinds = np.array(kinds or [0], np.int32)
    fam = np.zeros(n, np.int32)
    need = C.c_longlong()
    ip = C.POINTER(C.c_int)
    args = [n, core.ctypes.data_as(ip), off.ctypes.data_as(ip), kinds.ctypes.data_as(ip), ALGOS[algo],
            fam.ctypes.data_as(ip)]
    rc = L.famtune_cluster(*args, None, 0, C.byref(need))
    if rc == 1:
        raise ValueError("clustering requires a non-empty subgraph list")
    if rc:
        raise RuntimeError(f"famtune_cluster failed ({rc})")
    buf = C.create_string_buffer(need.value + 1)
    L.famtune_cluster(*args, buf, need.value + 1, C.byref(need))
    return fam, buf.value.decode()
