"""GPU quantizer vs the REAL reference's fitting outputs
(tests/golden/quant_*.npz, written by tests/golden/make_golden_quant.py from
bcq.py / progressive.py), plus the reference's own invariants: frozen planes
byte-identical under expansion, error non-increasing in p and along the
alternating trace, the reference's error classes."""

from pathlib import Path

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

GOLDEN = Path(__file__).resolve().parent / "golden"


def _case(name):
    with np.load(GOLDEN / f"quant_{name}.npz") as z:
        return {k: z[k] for k in z.files}


def _cfg(P, c):
    return P.QuantConfig(group_size=int(c["group_size"]), mode="asymmetric" if int(c["asym"]) else "symmetric",
                         cycles=int(c["cycles"]))


def _close(a, b, tol):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30)) <= tol


@pytest.fixture(scope="module")
def P():
    import paper_2510_10467_b200 as P
    return P


@pytest.mark.parametrize("name", ["greedy_sym", "greedy_asym_g40"])
def test_greedy_ls_bs_match_reference(P, name):
    c = _case(name)
    cfg = _cfg(P, c)
    qm = P.greedy_init(c["w"], int(c["q"]), cfg)
    assert np.array_equal(qm.bitplanes.words, c["words"])
    assert _close(qm.scales.alpha, c["alpha"], 1e-6)
    if "offset" in c:
        assert _close(qm.scales.offset, c["offset"], 1e-6)
    st = P.ls_update_scales(c["w"], qm)
    assert _close(st.alpha, c["ls_alpha"], 1e-6)
    if "ls_offset" in c:
        assert _close(st.offset, c["ls_offset"], 1e-6)
    bp = P.bs_recalibrate_codes(c["w"], st)
    assert np.array_equal(bp.words, c["bs_words"])


@pytest.mark.parametrize("name", ["alt_sym", "alt_asym_g64"])
def test_alternate_fit_matches_reference(P, name):
    c = _case(name)
    trace = []
    qm = P.alternate_fit(c["w"], int(c["q"]), _cfg(P, c), trace=trace)
    assert np.array_equal(qm.bitplanes.words, c["words"])
    assert _close(qm.scales.alpha, c["alpha"], 1e-6)
    if "offset" in c:
        assert _close(qm.scales.offset, c["offset"], 1e-6)
    assert _close(trace, c["trace"], 1e-9)
    assert all(b <= a * (1 + 1e-12) for a, b in zip(trace, trace[1:]))   # non-increasing (bcq.py:346-348)


@pytest.mark.parametrize("name", ["multi_sym", "multi_asym_g32", "multi_sym_c0"])
def test_build_multiprecision_matches_reference(P, name):
    c = _case(name)
    m = P.build_multiprecision(c["w"], int(c["p_lo"]), int(c["p_hi"]), _cfg(P, c))
    assert np.array_equal(m.bitplanes.words, c["words"])
    for p in m.precisions:
        assert _close(m.scale_sets[p].alpha, c[f"alpha_{p}"], 1e-6), p
        if f"offset_{p}" in c:
            assert _close(m.scale_sets[p].offset, c[f"offset_{p}"], 1e-6), p
    errs = P.precision_errors(c["w"], m)
    if int(c["cycles"]):
        assert all(errs[p + 1] <= errs[p] + 1e-12 for p in range(m.p_lo, m.p_hi))
    # the fitted model serves through the GEMV engine like any other
    eng = P.GemvEngine(m)
    x = np.random.default_rng(0).standard_normal(m.shape[1])
    for p in m.precisions:
        y, _ = eng.lut(p, x)
        wq = P.quantize.dequantize(P.QuantizedMatrix(m.bitplanes.prefix(p), m.scale_sets[p], m.config), p)
        ref = wq.astype(np.float64) @ x
        assert np.max(np.abs(y - ref)) / np.max(np.abs(ref)) <= 1e-4


def test_expand_step_keeps_frozen_planes(P):
    c = _case("multi_sym")
    cfg = _cfg(P, c)
    base = P.build_multiprecision(c["w"], 2, 2, cfg)
    m3 = P.expand_step(c["w"], base, 3)
    assert m3.bitplanes.words[:2].tobytes() == base.bitplanes.words.tobytes()
    assert m3.scale_sets[2] is base.scale_sets[2]
    with pytest.raises(P.UsageError):
        P.expand_step(c["w"], base, 4)     # next precision is 3


def test_quantizer_errors(P):
    w = np.random.default_rng(1).standard_normal((8, 64)).astype(np.float32)
    cfg = P.QuantConfig(group_size=32, cycles=1)
    with pytest.raises(P.UsageError):
        P.greedy_init(w, 0, cfg)
    with pytest.raises(P.UsageError):
        P.build_multiprecision(w, 3, 2, cfg)
    bad = w.copy()
    bad[0, 0] = np.nan
    with pytest.raises(P.NonFiniteError):
        P.alternate_fit(bad, 2, cfg)
    with pytest.raises(P.UsageError):
        P.greedy_init(w[0], 2, cfg)        # 1-D


def test_live_reference_larger_model(P, tmp_path):
    """When the unmodified reference is installed (baseline/_ref), fit a larger
    matrix both ways and compare (its fitting is numpy; no GPU involved)."""
    import os
    import subprocess
    import sys
    ref = Path(__file__).resolve().parents[1] / "baseline" / "_ref"
    if not (ref / "anybcq").exists():
        pytest.skip("reference not installed")
    rows, cols = 256, 1024
    w = np.random.default_rng(7).standard_normal((rows, cols)).astype(np.float32)
    np.save(tmp_path / "w.npy", w)
    code = ("import sys, numpy as np\n"
            "from anybcq import QuantConfig\n"
            "from anybcq.progressive import build_multiprecision\n"
            "w = np.load(sys.argv[1])\n"
            "m = build_multiprecision(w, 2, 4, QuantConfig(group_size=128, mode='asymmetric', cycles=2))\n"
            "np.savez(sys.argv[2], words=m.bitplanes.words, **{f'a{p}': m.scale_sets[p].alpha for p in (2,3,4)},"
            " **{f'o{p}': m.scale_sets[p].offset for p in (2,3,4)})\n")
    env = dict(os.environ, PYTHONPATH=str(ref), NUMBA_CACHE_DIR=str(tmp_path / "nb"))
    subprocess.run([sys.executable, "-c", code, str(tmp_path / "w.npy"), str(tmp_path / "ref.npz")], env=env,
                   check=True, timeout=600)
    r = dict(np.load(tmp_path / "ref.npz"))
    m = P.build_multiprecision(w, 2, 4, P.QuantConfig(group_size=128, mode="asymmetric", cycles=2))
    same = np.mean(np.unpackbits(~(m.bitplanes.words ^ r["words"]).view(np.uint8)))
    assert same >= 0.9999, same             # codes: bit-identical up to f64 rounding ties
    for p in (2, 3, 4):
        assert _close(m.scale_sets[p].alpha, r[f"a{p}"], 1e-5)
        assert _close(m.scale_sets[p].offset, r[f"o{p}"], 1e-5)


def test_cli_quantize_and_bench_shapes(P, tmp_path, capsys):
    """`quantize` writes a container the engine serves; `bench --shapes` fits
    the synthetic suite on the GPU (cli.py:75-93, 135-158)."""
    from paper_2510_10467_b200.cli import main
    from paper_2510_10467_b200.container import deserialize
    out = tmp_path / "m.abcq"
    assert main(["quantize", "--random", "64x512", "--bits", "2:3", "--cycles", "2", "--mode", "sym",
                 "--scale-width", "2", "--out", str(out), "--format", "csv"]) == 0
    lines = capsys.readouterr().out.strip().splitlines()
    assert lines[0] == "p,relative_sq_error" and len(lines) == 3
    errs = [float(v.split(",")[1]) for v in lines[1:]]
    assert errs[1] <= errs[0]
    m = deserialize(out)
    assert m.shape == (64, 512) and (m.p_lo, m.p_hi) == (2, 3)
    assert main(["bench", "--shapes", "128x256", "--repeats", "3", "--format", "csv", "--dense"]) == 0
    rows = capsys.readouterr().out.strip().splitlines()
    assert rows[0] == "shape,path,p,median_us,plane_bytes,scale_bytes"
    assert {tuple(r.split(",")[1:3]) for r in rows[1:]} >= {("lut", "2"), ("lut", "4"), ("naive", "3"), ("dense", "32")}
    assert main(["bench", "--shapes", "128x256", "--model", str(out)]) == 2   # exactly one source
