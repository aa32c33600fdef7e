"""ctypes wrapper of the C oracle -- TEST / BASELINE INFRASTRUCTURE ONLY."""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from .build_oracle import OUT, build

_L = None


def _lib():
    global _L
    if _L is None:
        if not OUT.exists():
            build()
        _L = C.CDLL(str(OUT))
        _L.abcq_oracle_lut_gemv.restype = C.c_int
        _L.abcq_oracle_lut_gemv.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p,
                                            C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_int]
        _L.abcq_oracle_lut_build8.restype = None
        _L.abcq_oracle_lut_build8.argtypes = [C.c_void_p, C.c_int, C.c_void_p]
    return _L


def cpu_threads() -> int:
    return os.cpu_count() or 1


def lut_gemv(words, cols, group_size, alpha, offset, p, x, threads=1) -> np.ndarray:
    """GemvEngine.lut restated in C (aligned groups); y f64 (rows,)."""
    words = np.ascontiguousarray(words, dtype=np.uint32)
    alpha = np.ascontiguousarray(alpha, dtype=np.float32)
    off = None if offset is None else np.ascontiguousarray(offset, dtype=np.float32)
    x = np.ascontiguousarray(np.asarray(x, dtype=np.float64).ravel())
    planes, rows, _ = words.shape
    y = np.empty(rows, dtype=np.float64)
    rc = _lib().abcq_oracle_lut_gemv(words.ctypes.data, planes, rows, cols, group_size, alpha.ctypes.data,
                                     None if off is None else off.ctypes.data, p, x.ctypes.data,
                                     y.ctypes.data, int(threads))
    if rc != 0:
        raise ValueError("C oracle needs chunk-aligned groups (group_size % 8 == 0)")
    return y


def lut_build8(x) -> np.ndarray:
    x = np.ascontiguousarray(np.asarray(x, dtype=np.float64).ravel())
    t = np.empty(((len(x) + 7) // 8, 256), dtype=np.float32)
    _lib().abcq_oracle_lut_build8(x.ctypes.data, len(x), t.ctypes.data)
    return t
