"""Generate golden fixtures from the REAL reference package (build container only).

Run here (not on the GPU box -- /root/reference does not exist there):

    python tests/golden/make_golden.py

The reference (/root/reference/pkg/src/anybcq) is copied to a scratch dir
first so numba's JIT cache never writes into /root/reference. Outputs are
small .npz files next to this script; tests/test_oracle.py checks the oracle
restatement against them and the GPU parity tests use the same models.
"""

from __future__ import annotations

import os
import shutil
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF_SRC = Path("/root/reference/pkg/src")


def _import_reference():
    scratch = Path(tempfile.mkdtemp(prefix="anybcq_ref_"))
    shutil.copytree(REF_SRC / "anybcq", scratch / "anybcq")
    os.environ.setdefault("NUMBA_CACHE_DIR", str(scratch / "numba_cache"))
    sys.dont_write_bytecode = True
    sys.path.insert(0, str(scratch))
    import anybcq  # noqa: E402

    return anybcq


def _dump_model(model):
    out = {
        "words": np.ascontiguousarray(model.bitplanes.words, dtype=np.uint32),
        "cols": np.int64(model.bitplanes.cols),
        "group_size": np.int64(model.config.group_size),
        "p_lo": np.int64(model.p_lo),
        "p_hi": np.int64(model.p_hi),
        "asymmetric": np.int64(1 if model.config.asymmetric else 0),
    }
    for p, st in model.scale_sets.items():
        out[f"alpha_{p}"] = np.ascontiguousarray(st.alpha, dtype=np.float32)
        if st.offset is not None:
            out[f"offset_{p}"] = np.ascontiguousarray(st.offset, dtype=np.float32)
    return out


def _case(ab, name, model, xs, chunk_widths=(8,)):
    data = _dump_model(model)
    for p in model.precisions:
        for si, x in enumerate(xs):
            x = np.asarray(x, dtype=np.float32).ravel()
            data[f"x_{si}"] = x
            for mu in chunk_widths:
                eng = ab.GemvEngine(model, chunk_width=mu)
                y, st = eng.lut(p, x)
                data[f"lut{mu}_p{p}_x{si}"] = y
                data[f"stats_p{p}"] = np.array(
                    [st.plane_bytes_fetched, st.scale_bytes_fetched, st.lut_build_count],
                    dtype=np.int64)
            yn, _ = ab.GemvEngine(model).naive(p, x)
            data[f"naive_p{p}_x{si}"] = yn
            data[f"oracle_p{p}_x{si}"] = ab.dequant_oracle(model, p, x)
    np.savez_compressed(HERE / f"{name}.npz", **data)
    print(f"wrote {name}.npz  shape={model.shape} p={model.p_lo}:{model.p_hi} "
          f"g={model.config.group_size} mode={model.config.mode}")


def main():
    ab = _import_reference()
    rg = ab.random_gaussian
    QC = ab.QuantConfig
    bm = ab.build_multiprecision

    # tests/test_gemv.py:25-28 fixture
    m = bm(rg(32, 128, seed=14), 2, 4, QC(group_size=32, cycles=2))
    _case(ab, "g32_32x128", m, [rg(1, 128, seed=s) for s in range(5)] + [np.zeros(128)],
          chunk_widths=(4, 8))
    # tests/test_gemv.py:31-36 (ragged g=40, asymmetric)
    m = bm(rg(16, 80, seed=15), 2, 3, QC(group_size=40, mode="asymmetric", cycles=2))
    _case(ab, "asym_g40_16x80", m, [rg(1, 80, seed=s) for s in (2, 3)], chunk_widths=(4, 8))
    # tests/test_gemv.py:142-151
    m = bm(rg(64, 256, seed=23), 2, 3, QC(group_size=128, cycles=2))
    _case(ab, "g128_64x256", m, [rg(1, 256, seed=40 + s) for s in range(3)])
    # tests/test_gemv.py:94-101 single active column
    m = bm(np.array([[3.0, 1.0, -1.0, -3.0]], dtype=np.float32), 1, 2, QC(group_size=4, cycles=2))
    _case(ab, "single_col_1x4", m, [np.array([1.0, 0.0, 0.0, 0.0])])
    # tests/test_acceptance.py:235-252 small asymmetric g=25 model
    m = bm(rg(16, 100, seed=901), 2, 3, QC(group_size=25, mode="asymmetric", cycles=1))
    _case(ab, "asym_g25_16x100", m, [rg(1, 100, seed=902)])
    # g=128 shapes the fast kernel takes: ragged K, ragged N, asymmetric
    m = bm(rg(37, 200, seed=31), 1, 3, QC(group_size=128, cycles=1))
    _case(ab, "g128_ragged_37x200", m, [rg(1, 200, seed=32 + s) for s in range(2)])
    m = bm(rg(128, 1024, seed=41), 2, 4, QC(group_size=128, mode="asymmetric", cycles=1))
    _case(ab, "asym_g128_128x1024", m, [rg(1, 1024, seed=42 + s) for s in range(2)])
    # tests/test_acceptance.py:203-232 (criterion 6 model, 512x4096, p 2:4)
    m = bm(rg(512, 4096, seed=700), 2, 4, QC(group_size=128, cycles=2))
    _case(ab, "g128_512x4096", m, [rg(1, 4096, seed=800 + 101 * 2 + t) for t in range(2)])

    # LookupTable goldens (gemv.py:67-81)
    lut = {}
    x = rg(1, 1024, seed=1).ravel()
    lut["x8"] = x
    lut["t8"] = ab.LookupTable.build(x, 8).tables
    x4 = rg(1, 40, seed=6).ravel()
    lut["x4"] = x4
    lut["t4"] = ab.LookupTable.build(x4, 4).tables
    x13 = rg(1, 13, seed=9).ravel()
    lut["x13"] = x13
    lut["t13_8"] = ab.LookupTable.build(x13, 8).tables
    np.savez_compressed(HERE / "lut_tables.npz", **lut)
    # PRNG goldens (tensor_io.py:105-128)
    np.savez_compressed(
        HERE / "prng.npz",
        g_3x5_s42=rg(3, 5, seed=42), g_1x7_s0=rg(1, 7, seed=0),
        g_4x4_s7=rg(4, 4, seed=7), g_2x3_big=rg(2, 3, seed=2**63 + 12345))
    # packing goldens (packing.py:22-37)
    rng = np.random.default_rng(5)
    codes = np.where(rng.random((3, 5, 100)) < 0.5, -1, 1).astype(np.int8)
    np.savez_compressed(HERE / "packing.npz", codes=codes, words=ab.pack_signs(codes))
    print("done")


def containers():
    """ABCQ container + FMAT goldens written by the reference's own writers
    (model_format.py:46-79, tensor_io.py:53-57): byte-level fixtures for the
    container reader/writer (paper_2510_10467_b200/container.py)."""
    ab = _import_reference()
    from anybcq.model_format import serialize
    from anybcq.tensor_io import save_matrix
    rg = ab.random_gaussian
    QC = ab.QuantConfig
    m = ab.build_multiprecision(rg(64, 256, seed=23), 2, 3, QC(group_size=128, cycles=2))
    serialize(m, HERE / "container_g128_64x256_w4.abcq", scale_width=4)
    m = ab.build_multiprecision(rg(128, 1024, seed=41), 2, 4, QC(group_size=128, mode="asymmetric", cycles=1))
    serialize(m, HERE / "container_asym_128x1024_w2.abcq", scale_width=2)
    m = ab.build_multiprecision(rg(16, 80, seed=15), 2, 3, QC(group_size=40, mode="asymmetric", cycles=2))
    serialize(m, HERE / "container_asym_g40_16x80_w4.abcq", scale_width=4)
    save_matrix(rg(3, 256, seed=5), HERE / "x_3x256.fmat")
    print("containers done")


if __name__ == "__main__":
    if "--containers" in sys.argv:
        containers()
    else:
        main()
