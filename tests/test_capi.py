"""The C ABI library loads, exports every symbol include/anybcq_b200.h declares,
and rejects bad arguments with the documented codes (no GPU needed)."""

import ctypes as C

import pytest

from paper_2510_10467_b200 import _lib


def test_library_exports_every_header_symbol():
    lib = _lib.lib()
    declared = _lib.header_symbols()
    assert len(declared) >= 12
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing
    assert set(declared) == set(_lib.SIGNATURES), "ctypes table out of sync with the header"
    assert lib.abcq_abi_version() == 1


def test_struct_layout_matches_header():
    # 8 int32 + int64 + 1 + 2*17 pointers
    assert C.sizeof(_lib.AbcqModel) == 8 * 4 + 8 + 8 * (1 + 2 * 17)


def test_tiled_sizes():
    lib = _lib.lib()
    b = C.c_int64()
    assert lib.abcq_tiled_plane_bytes(4096, 4096, C.byref(b)) == 0
    assert b.value == 4096 * 4096 // 8                     # no padding at aligned shapes
    assert lib.abcq_tiled_plane_bytes(17, 300, C.byref(b)) == 0
    assert b.value == 2 * 2 * 512                          # 2 row tiles x 2 slices x 512 B
    na, no = C.c_int64(), C.c_int64()
    assert lib.abcq_tiled_scale_elems(4096, 4096, 3, C.byref(na), C.byref(no)) == 0
    assert na.value == 3 * 4096 * 32 and no.value == 4096 * 32
    assert lib.abcq_tiled_plane_bytes(0, 5, C.byref(b)) == _lib.E_ARG


def test_argument_errors_without_device():
    lib = _lib.lib()
    assert lib.abcq_gemv(None, 2, None, 0, None, 0, None, 0, None) == _lib.E_ARG
    m = _lib.AbcqModel()
    m.rows, m.cols, m.group_size, m.p_lo, m.p_hi = 16, 256, 128, 2, 4
    m.layout, m.scale_dtype, m.planes = _lib.LAYOUT_TILED, _lib.F32, 0x1000
    assert lib.abcq_gemv(C.byref(m), 5, 0x2000, 0, 0x3000, 0, None, 0, None) == _lib.E_PRECISION
    assert "precision 5 outside [2, 4]" in _lib.last_error()
    m.group_size = 64
    assert lib.abcq_gemv(C.byref(m), 2, 0x2000, 0, 0x3000, 0, None, 0, None) == _lib.E_LAYOUT
    with pytest.raises(Exception):
        _lib.check(_lib.E_PRECISION)
    assert lib.abcq_lut_build(0x10, 0, 8, 9, 0x20, None) == _lib.E_ARG


def test_silu_glu_dtype_validation_without_device():
    lib = _lib.lib()
    m = _lib.AbcqModel()
    m.rows, m.cols, m.group_size, m.p_lo, m.p_hi = 16, 256, 64, 2, 4
    m.layout, m.scale_dtype, m.planes = _lib.LAYOUT_ROWMAJOR, _lib.F32, 0x1000
    m.alpha[2] = 0x4000
    # the gated input exists only for the tiled kernel, and never for the naive path
    assert lib.abcq_gemv(C.byref(m), 2, 0x2000, _lib.F16_SILU_GLU, 0x3000, 0, None, 0, None) == _lib.E_LAYOUT
    assert "SiLU-gated" in _lib.last_error()
    assert lib.abcq_gemv_naive(C.byref(m), 2, 0x2000, _lib.F16_SILU_GLU, 0x3000, 0, None) == _lib.E_ARG
    assert lib.abcq_gemv(C.byref(m), 2, 0x2000, 3, 0x3000, 0, None, 0, None) == _lib.E_ARG
    assert lib.abcq_gemv(C.byref(m), 2, 0x2000, 0, 0x3000, _lib.F16_SILU_GLU, None, 0, None) == _lib.E_ARG
