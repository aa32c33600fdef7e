"""ABCQ container + FMAT files + CLI/service surface, CPU side: byte-level
parity with files the reference itself wrote (tests/golden/container_*.abcq,
x_3x256.fmat -- tests/golden/make_golden.py --containers), the reference's
validation order and error classes (model_format.py:82-154,
tests/test_model_format.py), and CLI exit codes before any device work
(cli.py:1-8)."""

import shutil
import struct
import zlib

import numpy as np
import pytest

from conftest import GOLDEN, load_case
from oracle import anybcq_oracle as O

import paper_2510_10467_b200 as P
from paper_2510_10467_b200 import container as C
from paper_2510_10467_b200 import tensor_io as T

CONTAINERS = {
    # file: (golden npz case with the same model, cycles, scale width)
    "container_g128_64x256_w4.abcq": ("g128_64x256", 2, 4),
    "container_asym_128x1024_w2.abcq": ("asym_g128_128x1024", 1, 2),
    "container_asym_g40_16x80_w4.abcq": ("asym_g40_16x80", 2, 4),
}


def model_from_case(name, cycles):
    c = load_case(name)
    words, cols, g = c["words"], int(c["cols"]), int(c["group_size"])
    p_lo, p_hi = int(c["p_lo"]), int(c["p_hi"])
    sets = {p: P.ScaleTensor(c[f"alpha_{p}"], c.get(f"offset_{p}"), g) for p in range(p_lo, p_hi + 1)}
    mode = "asymmetric" if int(c["asymmetric"]) else "symmetric"
    return P.MultiPrecisionModel(P.BitPlaneSet(p_hi, words.shape[1], cols, words), sets, p_lo, p_hi,
                                 P.QuantConfig(g, mode, cycles))


@pytest.mark.parametrize("fname", sorted(CONTAINERS))
def test_writer_is_byte_identical_to_reference(tmp_path, fname):
    case, cycles, width = CONTAINERS[fname]
    out = tmp_path / "m.abcq"
    C.serialize(model_from_case(case, cycles), out, scale_width=width)
    assert out.read_bytes() == (GOLDEN / fname).read_bytes()


@pytest.mark.parametrize("fname", sorted(CONTAINERS))
def test_reader_matches_reference_model(tmp_path, fname):
    case, cycles, width = CONTAINERS[fname]
    m = C.deserialize(GOLDEN / fname)
    ref = model_from_case(case, cycles)
    assert m.shape == ref.shape and (m.p_lo, m.p_hi) == (ref.p_lo, ref.p_hi)
    assert m.config == ref.config
    assert np.array_equal(m.bitplanes.words, ref.bitplanes.words)
    for p in ref.precisions:
        want = ref.scale_sets[p].alpha
        if width == 2:
            want = want.astype(np.float16).astype(np.float32)   # model_format.py:43-52
        assert np.array_equal(m.scale_sets[p].alpha, want)
        if ref.config.asymmetric:
            wz = ref.scale_sets[p].offset
            if width == 2:
                wz = wz.astype(np.float16).astype(np.float32)
            assert np.array_equal(m.scale_sets[p].offset, wz)
    # read -> write round trip is byte-identical (tests/test_model_format.py)
    C.serialize(m, tmp_path / "rt.abcq", scale_width=width)
    assert (tmp_path / "rt.abcq").read_bytes() == (GOLDEN / fname).read_bytes()


def test_layout_offsets_and_size_law():
    raw = (GOLDEN / "container_asym_128x1024_w2.abcq").read_bytes()
    lay = C.read_layout(raw)
    assert (lay.rows, lay.cols, lay.p_lo, lay.p_hi, lay.scale_width, lay.asymmetric) == (128, 1024, 2, 4, 2, True)
    # file-size law (tests/test_model_format.py:99-106)
    G = 1024 // 128
    want = lay.header_end + 4 * 128 * 32 * 4 + (2 + 3 + 4) * 128 * G * 2 + 3 * 128 * G * 2 + 4
    assert lay.total_bytes == len(raw) == want
    assert lay.set_offset(3) == lay.set_offset(2) + 2 * 128 * G * 2


def _mutate(tmp_path, fn):
    raw = bytearray((GOLDEN / "container_g128_64x256_w4.abcq").read_bytes())
    raw = fn(raw)
    path = tmp_path / "bad.abcq"
    path.write_bytes(bytes(raw))
    return path


def _recrc(raw):
    raw[-4:] = struct.pack("<I", zlib.crc32(bytes(raw[:-4])))
    return raw


@pytest.mark.parametrize("mutation,err", [
    (lambda r: b"XBCQ" + r[4:], P.BadMagicError),
    (lambda r: r[:4] + struct.pack("<I", 2) + r[8:], P.BadVersionError),
    (lambda r: r[:6], P.TruncatedError),
    (lambda r: r[:-10], P.TruncatedError),
    (lambda r: r + b"\0", P.FileFormatError),
    (lambda r: r[:200] + bytes([r[200] ^ 1]) + r[201:], P.ChecksumError),
    (lambda r: r[:12] + b"[" + r[13:], P.FileFormatError),
    (lambda r: r[:12] + r[12:].replace(b'"scale_width":4', b'"scale_width":3', 1), P.FileFormatError),
])
def test_reader_errors_in_reference_order(tmp_path, mutation, err):
    path = _mutate(tmp_path, mutation)
    with pytest.raises(err):
        C.deserialize(path)


def test_checksum_covers_payload(tmp_path):
    path = _mutate(tmp_path, lambda r: _recrc(r[:300] + bytes([r[300] ^ 0x80]) + r[301:]))
    m = C.deserialize(path)   # re-CRC'd: valid file, one flipped plane bit
    ref = C.deserialize(GOLDEN / "container_g128_64x256_w4.abcq")
    assert not np.array_equal(m.bitplanes.words, ref.bitplanes.words)


def test_fmat_matches_reference_file(tmp_path):
    x = T.load_matrix(GOLDEN / "x_3x256.fmat")
    assert np.array_equal(x, T.random_gaussian(3, 256, 5))
    T.save_matrix(x, tmp_path / "x.fmat")
    assert (tmp_path / "x.fmat").read_bytes() == (GOLDEN / "x_3x256.fmat").read_bytes()
    raw = (GOLDEN / "x_3x256.fmat").read_bytes()
    for bad, err in ((b"QMAT" + raw[4:], P.BadMagicError), (raw[:4] + b"\2" + raw[5:], P.BadVersionError),
                     (raw[:8] + b"\1" + raw[9:], P.UnsupportedDtypeError), (raw[:-4], P.TruncatedError),
                     (raw[:20], P.TruncatedError)):
        (tmp_path / "b.fmat").write_bytes(bad)
        with pytest.raises(err):
            T.load_matrix(tmp_path / "b.fmat")
    with pytest.raises(P.NonFiniteError):
        T.save_matrix(np.array([[np.nan]]), tmp_path / "n.fmat")


def test_random_gaussian_equals_reference_stream():
    with np.load(GOLDEN / "prng.npz") as z:
        assert np.array_equal(T.random_gaussian(3, 5, 42), z["g_3x5_s42"])
        assert np.array_equal(T.random_gaussian(1, 7, 0), z["g_1x7_s0"])
        assert np.array_equal(T.random_gaussian(2, 3, 2**63 + 12345), z["g_2x3_big"])
    assert np.array_equal(T.random_gaussian(17, 33, 9), O.random_gaussian(17, 33, 9))
    with pytest.raises(P.UsageError):
        T.random_gaussian(0, 3, 1)


# --- CLI: validation and I/O errors surface before any device work ------------

def run_cli(*argv):
    from paper_2510_10467_b200.cli import main
    return main(list(argv))


def test_cli_exit_codes(tmp_path, capsys):
    model = GOLDEN / "container_g128_64x256_w4.abcq"
    assert run_cli("gemv", "--model", str(model)) == 2                         # missing flags
    assert run_cli("gemv", "--model", str(model), "--bits", "2", "--x", str(tmp_path / "none.fmat"),
                   "--out", str(tmp_path / "y.fmat")) == 3                     # missing input file
    assert run_cli("bench") == 2                                               # no --model
    assert run_cli("bench", "--model", str(tmp_path / "none.abcq")) == 3
    assert run_cli("bench", "--model", str(model), "--bits", "two") == 2
    assert run_cli("bench", "--model", str(model), "--repeats", "0") == 2
    bad = tmp_path / "bad.abcq"
    bad.write_bytes(b"XBCQ" + model.read_bytes()[4:])
    assert run_cli("bench", "--model", str(bad)) == 3
    err = capsys.readouterr().err
    assert "bad magic" in err


# --- service: routing, model registry and error mapping (no device work) ------

def test_service_registry(tmp_path):
    from fastapi.testclient import TestClient

    from paper_2510_10467_b200.service import create_app
    shutil.copy(GOLDEN / "container_g128_64x256_w4.abcq", tmp_path / "small.abcq")
    (tmp_path / "broken.abcq").write_bytes(b"ABCQ")
    client = TestClient(create_app(tmp_path))
    assert client.get("/health").json()["status"] == "ok"
    info = client.get("/models/small").json()
    assert info == {"name": "small", "rows": 64, "cols": 256, "bits_lo": 2, "bits_hi": 3,
                    "group_size": 128, "mode": "symmetric"}
    assert client.get("/models/nope").status_code == 404
    assert client.get("/models/broken").status_code == 500   # FileFormatError, as upstream (server.py:114-117)
    assert client.post("/models/nope/gemv", json={"precision": 2, "x": [0.0]}).status_code == 404
    assert client.post("/models/small/gemv", json={"precision": 99, "x": [0.0]}).status_code == 422
    assert client.post("/models/small/gemv",
                       json={"precision": 2, "x": [0.0], "path": "fast"}).status_code == 422
