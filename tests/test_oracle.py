"""The CPU oracle (oracle/anybcq_oracle.py) pinned against the reference's own
golden vectors (restated from /root/reference/pkg/tests) and against outputs of
the real reference package (tests/golden/*.npz, made by make_golden.py)."""

import numpy as np
import pytest

from conftest import GOLDEN_CASES, load_case
from oracle import anybcq_oracle as O


# --- reference golden vectors, restated ------------------------------------

def test_lut_two_bit_enumeration():
    # tests/test_gemv.py:43-46
    t = O.lut_build(np.array([0.5, 2.0], dtype=np.float32), 2)
    assert t.shape == (1, 4)
    assert np.array_equal(t[0], np.float32([-2.5, -1.5, 1.5, 2.5]))


def test_lut_all_ones_entry_is_chunk_sum():
    # tests/test_gemv.py:49-54
    x = O.random_gaussian(1, 64, seed=3).ravel()
    t = O.lut_build(x, 8)
    assert np.allclose(t[:, 255], x.reshape(8, 8).sum(axis=1, dtype=np.float32), atol=1e-6)


def test_lut_complement_symmetry():
    # tests/test_gemv.py:57-62
    x = O.random_gaussian(1, 40, seed=6).ravel()
    t = O.lut_build(x, 4)
    assert np.max(np.abs(t + t[:, ::-1])) <= 1e-6 * np.abs(x).sum()


def test_lut_ragged_tail():
    # tests/test_gemv.py:65-68
    t = O.lut_build(np.ones(13, dtype=np.float32), 4)
    assert t.shape[0] == 4 and t[3, 0b0001] == pytest.approx(1.0)


def test_bit_addressing():
    # tests/test_packing.py:16-26
    codes = -np.ones((1, 70), dtype=np.int8)
    codes[0, [0, 33, 69]] = 1
    w = O.pack_signs(codes)
    assert w[0, 0] == 1 and w[0, 1] == 1 << 1 and w[0, 2] == 1 << 5


def test_padding_bits_zero():
    # tests/test_packing.py:29-33
    w = O.pack_signs(np.ones((2, 40), dtype=np.int8))
    assert w.shape == (2, 2) and np.all(w[:, 1] == np.uint32(0xFF))


@pytest.mark.parametrize("cols", [1, 7, 32, 33, 64, 100])
def test_pack_unpack_identity(cols):
    # tests/test_packing.py:7-13
    rng = np.random.default_rng(cols)
    codes = np.where(rng.random((3, cols)) < 0.5, -1, 1).astype(np.int8)
    assert np.array_equal(O.unpack_signs(O.pack_signs(codes), cols), codes)


def test_gaussian_reference_values():
    # tests/test_tensor_io.py:117-133 (documented splitmix64 + Box-Muller)
    ctr = np.arange(1, 5, dtype=np.uint64)
    z = O.splitmix64(np.uint64(42) + ctr * np.uint64(O.GOLDEN))
    top = (z >> np.uint64(11)).astype(np.float64)
    u1 = (top[0::2] + 1.0) * 2.0 ** -53
    u2 = top[1::2] * 2.0 ** -53
    r = np.sqrt(-2.0 * np.log(u1))
    want = np.array([r[0] * np.cos(2 * np.pi * u2[0]), r[0] * np.sin(2 * np.pi * u2[0]),
                     r[1] * np.cos(2 * np.pi * u2[1]), r[1] * np.sin(2 * np.pi * u2[1])],
                    dtype=np.float32)
    assert np.array_equal(O.random_gaussian(2, 2, seed=42).ravel(), want)


def test_gaussian_prefix_stability():
    # tests/test_tensor_io.py:99-103
    big = O.random_gaussian(8, 8, seed=3).ravel()
    assert np.array_equal(big[:16], O.random_gaussian(2, 8, seed=3).ravel())


def test_counters_formula():
    # tests/test_gemv.py:154-174, tests/test_acceptance.py:235-252 (traffic law)
    s = O.gemv_stats(3, 32, 128, 32, False)
    assert s["plane_bytes_fetched"] == 3 * 32 * 4 * 4 and s["scale_bytes_fetched"] == 3 * 32 * 4 * 4
    s2, s3 = O.gemv_stats(2, 16, 80, 40, True), O.gemv_stats(3, 16, 80, 40, True)
    assert s3["scale_bytes_fetched"] - s2["scale_bytes_fetched"] == 16 * 2 * 4
    assert O.gemv_stats(4, 16, 100, 25, True)["plane_bytes_fetched"] == 4 * 16 * 4 * 4


def test_row_chunks_cover_range():
    # tests/test_parallel.py:15-20
    for rows in (1, 5, 17):
        for workers in (1, 2, 4, 40):
            flat = [i for lo, hi in O.row_chunks(rows, workers) for i in range(lo, hi)]
            assert flat == list(range(rows))


# --- against outputs of the real reference (tests/golden) --------------------

def test_prng_matches_reference():
    with np.load("tests/golden/prng.npz") as z:
        assert np.array_equal(O.random_gaussian(3, 5, 42), z["g_3x5_s42"])
        assert np.array_equal(O.random_gaussian(1, 7, 0), z["g_1x7_s0"])
        assert np.array_equal(O.random_gaussian(4, 4, 7), z["g_4x4_s7"])
        assert np.array_equal(O.random_gaussian(2, 3, 2**63 + 12345), z["g_2x3_big"])


def test_packing_matches_reference():
    with np.load("tests/golden/packing.npz") as z:
        assert np.array_equal(O.pack_signs(z["codes"]), z["words"])
        assert np.array_equal(O.unpack_signs(z["words"], 100), z["codes"])


def test_lut_tables_bit_exact_vs_reference():
    with np.load("tests/golden/lut_tables.npz") as z:
        assert np.array_equal(O.lut_build(z["x8"], 8), z["t8"])
        assert np.array_equal(O.lut_build(z["x4"], 4), z["t4"])
        assert np.array_equal(O.lut_build(z["x13"], 8), z["t13_8"])


def _model(c):
    words, cols, g = c["words"], int(c["cols"]), int(c["group_size"])
    return words, cols, g


@pytest.mark.parametrize("name", GOLDEN_CASES)
def test_oracle_matches_reference_outputs(name):
    c = load_case(name)
    words, cols, g = _model(c)
    p_lo, p_hi = int(c["p_lo"]), int(c["p_hi"])
    nx = len([k for k in c if k.startswith("x_")])
    for p in range(p_lo, p_hi + 1):
        a, off = c[f"alpha_{p}"], c.get(f"offset_{p}")
        for si in range(nx):
            x = c[f"x_{si}"]
            for mu in (4, 8):
                key = f"lut{mu}_p{p}_x{si}"
                if key in c:
                    y = O.gemv_lut(words, cols, g, a, off, p, x, mu)
                    assert O.rel_dev(y, c[key]) <= 1e-12, (key, O.rel_dev(y, c[key]))
            yn = O.gemv_naive(words, cols, g, a, off, p, x)
            assert O.rel_dev(yn, c[f"naive_p{p}_x{si}"]) <= 1e-12
            yo = O.dequant_oracle(words, cols, g, a, off, p, x)
            assert O.rel_dev(yo, c[f"oracle_p{p}_x{si}"]) <= 1e-12
        st = O.gemv_stats(p, words.shape[1], cols, g, off is not None)
        assert [st["plane_bytes_fetched"], st["scale_bytes_fetched"], 1] == list(c[f"stats_p{p}"])


def test_single_active_column_known_answer():
    # tests/test_gemv.py:94-101: y=3 at p=2, y=2 at p=1
    c = load_case("single_col_1x4")
    words, cols, g = _model(c)
    x = np.array([1.0, 0, 0, 0])
    assert O.gemv_naive(words, cols, g, c["alpha_2"], None, 2, x)[0] == pytest.approx(3.0, abs=1e-6)
    assert O.gemv_naive(words, cols, g, c["alpha_1"], None, 1, x)[0] == pytest.approx(2.0, abs=1e-6)


# --- the C restatement (bench cpu_baseline / --impl reference arm) ----------

def test_c_oracle_table_bit_exact():
    from oracle import c_oracle
    with np.load("tests/golden/lut_tables.npz") as z:
        assert np.array_equal(c_oracle.lut_build8(z["x8"]), z["t8"])
        assert np.array_equal(c_oracle.lut_build8(z["x13"]), z["t13_8"])


@pytest.mark.parametrize("name", ["g32_32x128", "g128_64x256", "g128_ragged_37x200",
                                  "asym_g128_128x1024", "g128_512x4096"])
@pytest.mark.parametrize("threads", [1, 3])
def test_c_oracle_matches_reference(name, threads):
    from oracle import c_oracle
    c = load_case(name)
    words, cols, g = _model(c)
    for p in range(int(c["p_lo"]), int(c["p_hi"]) + 1):
        y = c_oracle.lut_gemv(words, cols, g, c[f"alpha_{p}"], c.get(f"offset_{p}"), p, c["x_0"], threads)
        assert O.rel_dev(y, c[f"lut8_p{p}_x0"]) <= 1e-12
