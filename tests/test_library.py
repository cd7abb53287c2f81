"""The C-ABI library loads and exports every symbol include/pab_b200.h
declares (no compute calls -- this runs without a GPU)."""

import ctypes
import os
import re

from paper_2408_12588_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "pab_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\*?(pab_\w+)\s*\(", hdr, flags=re.M)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    for need in ("pab_attention", "pab_residual_modnorm", "pab_ddim_cfg", "pab_gelu_bf16", "pab_fill_uniform",
                 "pab_softmax_rows"):
        assert need in syms


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    for sym in declared_symbols():
        assert hasattr(lib, sym), sym
        assert sym in _lib.SIGNATURES, sym


def test_status_strings_map_to_reference_kinds():
    lib = _lib.load()
    assert lib.pab_status_string(0) == b"ok"
    assert lib.pab_status_string(1) == b"shape-mismatch"
    assert lib.pab_status_string(2) == b"invalid-config"
    assert lib.pab_status_string(3) == b"policy-error"
    assert b"sm_100a" in lib.pab_version()


def test_argument_validation_without_gpu():
    lib = _lib.load()
    # negative sizes are rejected on the host before any launch
    assert lib.pab_gelu_bf16(None, None, -1, None) == 1
    assert lib.pab_softmax_rows(None, 4, None, 4, -1, 4, 1.0, None) == 1
    assert lib.pab_softmax_rows(None, 4, None, 4, 0, 4, 1.0, None) == 0
    assert lib.pab_ddim_cfg(None, None, None, 0, 3, 10, 1, 4.0, 0.5, 0.6, None) == 1  # guidance needs batch 2
    args = _lib.AttnArgs()
    assert lib.pab_attention(ctypes.byref(args), 0, None) == 1  # null pointers


def test_sm100a_cubin_present():
    data = open(_lib.LIB_PATH, "rb").read()
    assert b"sm_100a" in data or b"sm_100" in data
