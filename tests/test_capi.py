"""CPU checks of the boundary: the C-ABI library loads and exports every symbol include/famseer.h
declares, the Python binding covers all of them, and error codes map to the reference's
exception types. No compute is launched (no GPU here)."""
import ctypes
import os
import re

import pytest

import paper_2201_00194_b200 as fs
from paper_2201_00194_b200 import _capi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "famseer.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(fs_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_capi.LIB_PATH)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_binding_covers_header():
    bound = {n for n, _, _ in _capi.SIGNATURES}
    assert set(declared_symbols()) == bound


def test_pure_host_entry_points():
    lib = _capi.load()
    assert lib.fs_feature_dim(16) == 2 * 16 + 16 * 15 // 2 == 152  # searchspace.cpp:86-88
    assert fs.feature_dim(3) == 9
    assert b"sm_100a" in lib.fs_version()


def test_error_mapping_without_gpu():
    # A NULL device is rejected before any CUDA call, with std::invalid_argument's code.
    with pytest.raises(fs.InvalidArgument):
        fs._check(_capi.load().fs_device_check(None))
    assert issubclass(fs.InvalidArgument, ValueError)
    assert issubclass(fs.OutOfRange, IndexError)
    assert issubclass(fs.DomainError, ArithmeticError)


def test_gbt_params_layout_matches_reference_defaults():
    p = fs.GbtParams(50, 3, 0.1, 2)  # costmodel.hpp:20-25 defaults
    assert (p.trees, p.depth, p.learning_rate, p.min_samples_split) == (50, 3, 0.1, 2)
    assert ctypes.sizeof(fs.GbtParams) == 24
