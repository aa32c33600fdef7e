"""ctypes binding of libanybcq_b200.so -- the C ABI declared in include/anybcq_b200.h.

The library is built in-tree by `__graft_entry__.build()` (nvcc, sm_100a).
There is no fallback: if the shared object is missing or cannot be loaded,
`lib()` raises, so a GPU box without the native code fails loudly instead of
silently computing elsewhere.
"""

from __future__ import annotations

import ctypes as C
import re
from pathlib import Path

from .errors import UsageError

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "libanybcq_b200.so"
HEADER = PKG.parent / "include" / "anybcq_b200.h"

ABCQ_MAX_PLANES = 16
F32, F16 = 0, 1
F16_SILU_GLU = 2  # tiled GEMV x = [g ; u], input f16(silu(g) * u)
LAYOUT_ROWMAJOR, LAYOUT_TILED = 0, 1
E_ARG, E_PRECISION, E_LAYOUT, E_WORKSPACE, E_DEVICE = -1, -2, -3, -4, -5


class AbcqModel(C.Structure):
    """Mirror of `abcq_model_t` (include/anybcq_b200.h)."""

    _fields_ = [
        ("rows", C.c_int32),
        ("cols", C.c_int32),
        ("group_size", C.c_int32),
        ("p_lo", C.c_int32),
        ("p_hi", C.c_int32),
        ("asymmetric", C.c_int32),
        ("layout", C.c_int32),
        ("scale_dtype", C.c_int32),
        ("plane_stride_bytes", C.c_int64),
        ("planes", C.c_void_p),
        ("alpha", C.c_void_p * (ABCQ_MAX_PLANES + 1)),
        ("offset", C.c_void_p * (ABCQ_MAX_PLANES + 1)),
    ]


class AbcqGemvJob(C.Structure):
    """Mirror of `abcq_gemv_job_t` (include/anybcq_b200.h)."""

    _fields_ = [
        ("model", C.POINTER(AbcqModel)),
        ("p", C.c_int32),
        ("x_dtype", C.c_int32),
        ("y_dtype", C.c_int32),
        ("x", C.c_void_p),
        ("y", C.c_void_p),
    ]


_vp, _i32, _i64, _sz = C.c_void_p, C.c_int32, C.c_int64, C.c_size_t
_PM = C.POINTER(AbcqModel)
_PJ = C.POINTER(AbcqGemvJob)

# name -> (restype, argtypes); every symbol declared in the header
SIGNATURES = {
    "abcq_abi_version": (C.c_int, []),
    "abcq_last_error": (C.c_char_p, []),
    "abcq_device_check": (C.c_int, [_i32]),
    "abcq_debug_set_trace": (C.c_int, [_vp]),
    "abcq_set_reserved_sms": (C.c_int, [_i32, C.POINTER(C.c_int32)]),
    "abcq_debug_set_mode": (C.c_int, [_i32]),
    "abcq_debug_gemv_geometry": (C.c_int, [_PM, _i32, C.POINTER(_i32)]),
    "abcq_argmax_workspace_bytes": (C.c_int, [C.POINTER(_sz)]),
    "abcq_argmax_f16": (C.c_int, [_vp, _i32, _vp, _vp, _sz, _vp]),
    "abcq_fit_greedy": (C.c_int, [_vp, _i32, _i32, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _vp]),
    "abcq_fit_ls": (C.c_int, [_vp, _vp, _i32, _i32, _i32, _i32, _i32, _vp, _vp, _vp, _vp]),
    "abcq_fit_bs": (C.c_int, [_vp, _vp, _vp, _i32, _i32, _i32, _i32, _vp, _vp]),
    "abcq_fit_residual_sign": (C.c_int, [_vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _vp, _vp]),
    "abcq_tiled_plane_bytes": (C.c_int, [_i32, _i32, C.POINTER(_i64)]),
    "abcq_tiled_scale_elems": (C.c_int, [_i32, _i32, _i32, C.POINTER(_i64), C.POINTER(_i64)]),
    "abcq_pack_planes": (C.c_int, [_vp, _i32, _i32, _i32, _vp, _vp]),
    "abcq_unpack_planes": (C.c_int, [_vp, _i32, _i32, _i32, _vp, _vp]),
    "abcq_pack_scales": (C.c_int, [_vp, _vp, _i32, _i32, _i32, _i32, _i32, _vp, _vp, _vp]),
    "abcq_lut_build": (C.c_int, [_vp, _i32, _i32, _i32, _vp, _vp]),
    "abcq_gemv_workspace_bytes": (C.c_int, [_PM, C.POINTER(_sz)]),
    "abcq_gemv": (C.c_int, [_PM, _i32, _vp, _i32, _vp, _i32, _vp, _sz, _vp]),
    "abcq_gemv_naive": (C.c_int, [_PM, _i32, _vp, _i32, _vp, _i32, _vp]),
    "abcq_gemv_add_rmsnorm": (C.c_int, [_PM, _i32, _vp, _vp, _vp, C.c_float, _vp, _vp, _i32, _vp, _sz, _vp]),
    "abcq_gemv_rmsnorm_out": (C.c_int, [_PM, _i32, _vp, _i32, _vp, _vp, _vp, C.c_float, _vp, _vp, _sz, _vp]),
    "abcq_peer_state_bytes": (C.c_size_t, []),
    "abcq_gemv_batch_peer": (C.c_int, [_PJ, _i32, _vp, _sz, C.POINTER(_vp), C.POINTER(_vp), _i32, _i32, _vp, _vp, _sz,
                                       _vp]),
    "abcq_peer_wait": (C.c_int, [C.POINTER(_vp), C.POINTER(_vp), _i32, _i32, _vp, _vp, _i64, _vp]),
    "abcq_gemv_batch_max_jobs": (C.c_int, []),
    "abcq_gemv_batch_workspace_bytes": (C.c_int, [_PJ, _i32, C.POINTER(_sz)]),
    "abcq_gemv_batch": (C.c_int, [_PJ, _i32, _vp, _sz, _vp]),
    "abcq_gemm_mixedp_max_batch": (C.c_int, []),
    "abcq_gemm_mixedp_workspace_bytes": (C.c_int, [_PM, _i32, C.POINTER(_sz)]),
    "abcq_gemm_mixedp": (C.c_int, [_PM, _i32, C.POINTER(_i32), _vp, _vp, _i32, _vp, _sz, _vp]),
    "abcq_dequantize": (C.c_int, [_PM, _i32, _vp, _i32, _vp]),
    # decode-step harness ops
    "abcq_add_rmsnorm_f16": (C.c_int, [_vp, _vp, _vp, _vp, _i32, C.c_float, _vp]),
    "abcq_rope_append_f16": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _i32, _vp]),
    "abcq_attn_decode_workspace_bytes": (C.c_int, [_i32, _i32, C.POINTER(_sz)]),
    "abcq_attn_decode_f16": (C.c_int, [_vp, _vp, _vp, _i32, _i32, _i32, _i32, C.c_float, _vp, _vp, _sz, _vp]),
    "abcq_rope_attn_decode_f16": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32, C.c_float,
                                            _vp, _vp, _sz, _vp]),
    "abcq_silu_mul_f16": (C.c_int, [_vp, _vp, _vp, _i32, _vp]),
}

_LIB = None


def header_symbols() -> list[str]:
    """Function names declared in include/anybcq_b200.h."""
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\**\s+\**(abcq_\w+)\s*\(", text, re.M)))


def lib() -> C.CDLL:
    global _LIB
    if _LIB is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH.name} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
                "(nvcc, sm_100a). There is no CPU fallback.")
        handle = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = handle
    return _LIB


def last_error() -> str:
    msg = lib().abcq_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str = "") -> None:
    """Map an ABI return code to the reference's error convention."""
    if rc == 0:
        return
    msg = last_error() or what
    if rc < 0:
        raise UsageError(msg)
    raise RuntimeError(f"CUDA failure in {what or 'libanybcq_b200'}: {msg}")


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None for None)."""
    return None if t is None else t.data_ptr()
