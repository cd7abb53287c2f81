"""ctypes binding of libpab_b200.so (the C ABI in include/pab_b200.h).

The library is the product: there is no CPU or eager-PyTorch fallback.  If
the shared object is missing the import of any device entry point raises
``DeviceError`` immediately.
"""

from __future__ import annotations

import ctypes
import os

from .errors import DeviceError, raise_for_status

_HERE = os.path.dirname(os.path.abspath(__file__))
# PAB_LIB_PATH: load a differently-built copy (kernel A/B experiments, scripts/gpu_variants.sh)
LIB_PATH = os.environ.get("PAB_LIB_PATH") or os.path.join(_HERE, "libpab_b200.so")
MAX_PENDING = 8

_lib = None

c_i64 = ctypes.c_int64
c_vp = ctypes.c_void_p


class AttnArgs(ctypes.Structure):
    _fields_ = [
        ("q", c_vp), ("k", c_vp), ("v", c_vp), ("o", c_vp),
        ("q_sa", c_i64), ("q_sb", c_i64), ("q_si", c_i64),
        ("k_sa", c_i64), ("k_sb", c_i64), ("k_si", c_i64),
        ("v_sa", c_i64), ("v_sb", c_i64), ("v_si", c_i64),
        ("o_sa", c_i64), ("o_sb", c_i64), ("o_si", c_i64),
        ("n_a", ctypes.c_int32), ("n_b", ctypes.c_int32), ("n_q", ctypes.c_int32),
        ("n_k", ctypes.c_int32), ("heads", ctypes.c_int32), ("dh", ctypes.c_int32),
        ("scale", ctypes.c_float),
    ]


# exported symbol -> (restype, argtypes); include/pab_b200.h is the source of truth
SIGNATURES = {
    "pab_version": (ctypes.c_char_p, []),
    "pab_status_string": (ctypes.c_char_p, [ctypes.c_int]),
    "pab_last_error": (ctypes.c_char_p, []),
    "pab_residual_modnorm": (
        ctypes.c_int,
        [c_vp, c_vp, ctypes.POINTER(c_vp), ctypes.c_int, c_vp, c_vp, c_vp, c_vp, c_i64, ctypes.c_int,
         ctypes.c_float, ctypes.c_int, c_vp],
    ),
    "pab_residual_modnorm_sp": (
        ctypes.c_int,
        [c_vp, c_vp, ctypes.POINTER(c_vp), ctypes.c_int, c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_i64, c_i64,
         ctypes.c_int, ctypes.c_float, ctypes.c_int, c_vp],
    ),
    "pab_residual_modnorm_tm": (
        ctypes.c_int,
        [c_vp, c_vp, ctypes.POINTER(c_vp), ctypes.c_int, ctypes.c_uint32, c_vp, c_vp, c_vp, c_vp, c_i64, c_i64,
         c_i64, ctypes.c_int, ctypes.c_float, ctypes.c_int, ctypes.c_int, c_vp],
    ),
    "pab_residual_modnorm_ex": (
        ctypes.c_int,
        [c_vp, c_vp, ctypes.POINTER(c_vp), c_vp, ctypes.c_int, c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_i64, c_i64,
         ctypes.c_int, ctypes.c_float, ctypes.c_int, ctypes.c_int, c_vp],
    ),
    "pab_residual_modnorm_peer": (
        ctypes.c_int,
        [c_vp, c_vp, ctypes.POINTER(c_vp), c_vp, ctypes.c_int, ctypes.POINTER(c_vp), c_vp, c_vp, c_vp, c_vp, c_vp,
         ctypes.POINTER(c_vp), c_i64, c_i64, c_i64, c_i64, ctypes.c_int, ctypes.c_int, ctypes.c_float, ctypes.c_int,
         ctypes.c_int, c_vp],
    ),
    "pab_peer_barrier": (ctypes.c_int, [ctypes.POINTER(c_vp), c_vp, ctypes.c_int, ctypes.c_int, c_vp, ctypes.c_double,
                                        c_vp]),
    "pab_ddim_cfg": (
        ctypes.c_int,
        [c_vp, c_vp, ctypes.POINTER(c_vp), ctypes.c_int, ctypes.c_int, c_i64, ctypes.c_int, ctypes.c_double,
         ctypes.c_double, ctypes.c_double, c_vp],
    ),
    "pab_gelu_bf16": (ctypes.c_int, [c_vp, c_vp, c_i64, c_vp]),
    "pab_diff_sums": (ctypes.c_int, [c_vp, c_vp, c_i64, c_vp, c_vp]),
    "pab_add_scaled_f32": (ctypes.c_int, [c_vp, c_vp, c_vp, ctypes.c_float, c_i64, c_vp]),
    "pab_softmax_rows": (ctypes.c_int, [c_vp, c_i64, c_vp, c_i64, c_i64, c_i64, ctypes.c_float, c_vp]),
    "pab_fill_uniform": (
        ctypes.c_int,
        [c_vp, ctypes.c_int, c_i64, c_i64, c_i64, c_i64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_double,
         ctypes.c_double, c_vp],
    ),
    "pab_attention": (ctypes.c_int, [ctypes.POINTER(AttnArgs), ctypes.c_int, c_vp]),
    "pab_gemm_bf16": (ctypes.c_int, [c_vp, c_i64, c_vp, c_i64, c_vp, c_i64, c_i64, c_i64, c_i64, ctypes.c_int, c_vp]),
    "pab_gemm_bf16_residual": (
        ctypes.c_int,
        [c_vp, c_i64, c_vp, c_i64, c_vp, c_i64, c_vp, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64, c_vp],
    ),
    "pab_gemm_bf16_residual_h": (
        ctypes.c_int,
        [c_vp, c_i64, c_vp, c_i64, c_vp, c_i64, c_vp, c_i64, c_vp, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64,
         c_vp],
    ),
    "pab_attention_select": (ctypes.c_int, [ctypes.POINTER(AttnArgs)]),
    "pab_attn_debug_trace": (ctypes.c_int, [c_vp]),
}


def load():
    """Load (once) and return the native library; raises DeviceError if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise DeviceError(
            f"native library {LIB_PATH} is missing; build it with `python -m paper_2408_12588_b200.build`"
        )
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(status: int, what: str) -> None:
    if status:
        lib = load()
        raise_for_status(status, what, lib.pab_last_error().decode())


def ptr_array(ptrs):
    arr = (c_vp * max(1, len(ptrs)))()
    for i, p in enumerate(ptrs):
        arr[i] = p
    return arr
