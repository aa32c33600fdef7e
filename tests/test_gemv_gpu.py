"""GPU parity tests: the CUDA path (through the C ABI) against the oracle and the
reference's golden outputs. Tolerance: rel_dev (tests/test_gemv.py:20-22)
<= 1e-3 per north_star; the fp32-scale drop-in is held to the reference's own
1e-4 bound (tests/test_gemv.py:112-120)."""

import numpy as np
import pytest

from conftest import GOLDEN_CASES, load_case
from layout_spec import tiled_offsets, tiled_planes, tiled_scales
from oracle import anybcq_oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

NORTH_STAR_TOL = 1e-3   # north_star: within 1e-3 relative (fp32 accumulate)
REF_TOL = 1e-4          # the reference's own path-equivalence bound


@pytest.fixture(scope="module")
def P():
    import paper_2510_10467_b200 as P
    return P


def make_model(P, case):
    words, cols, g = case["words"], int(case["cols"]), int(case["group_size"])
    p_lo, p_hi = int(case["p_lo"]), int(case["p_hi"])
    sets = {p: P.ScaleTensor(case[f"alpha_{p}"], case.get(f"offset_{p}"), g) for p in range(p_lo, p_hi + 1)}
    mode = "asymmetric" if int(case["asymmetric"]) else "symmetric"
    return P.MultiPrecisionModel(P.BitPlaneSet(p_hi, words.shape[1], cols, words), sets, p_lo, p_hi,
                                 P.QuantConfig(g, mode, 0))


def synth_model(P, rows, cols, p_lo, p_hi, asym=False, seed=0):
    words = O.random_words(p_hi, rows, cols, seed=seed)
    rng = np.random.default_rng(seed)
    G = -(-cols // 128)
    sets = {}
    for p in range(p_lo, p_hi + 1):
        a = (0.01 + 0.1 * np.abs(rng.standard_normal((p, rows, G)))).astype(np.float32)
        z = (0.1 * rng.standard_normal((rows, G))).astype(np.float32) if asym else None
        sets[p] = P.ScaleTensor(a, z, 128)
    mode = "asymmetric" if asym else "symmetric"
    return P.MultiPrecisionModel(P.BitPlaneSet(p_hi, rows, cols, words), sets, p_lo, p_hi,
                                 P.QuantConfig(128, mode, 0))


# --- layout: bit-exact packing ------------------------------------------------

@pytest.mark.parametrize("rows,cols", [(1, 1), (15, 7), (16, 128), (17, 100), (37, 200), (5, 256),
                                       (33, 300), (64, 1024), (100, 4096), (48, 14336)])
def test_pack_unpack_bit_exact(P, rows, cols):
    from paper_2510_10467_b200.device_model import DeviceModel
    words = O.random_words(3, rows, cols, seed=rows * 1000 + cols)
    dm = DeviceModel(rows, cols, 128, 1, 3)
    dm.load_planes(words)
    got = dm.planes.cpu().numpy().reshape(3, -1)
    want = tiled_planes(words, rows, cols).reshape(3, -1)
    assert np.array_equal(got, want), "tiled layout differs from the layout spec"
    back = dm.unpack_words().cpu().numpy().view(np.uint32)
    assert np.array_equal(back, words), "unpack(pack(words)) != words"


def test_scale_tiling_exact(P):
    from paper_2510_10467_b200.device_model import DeviceModel
    rows, cols = 37, 300
    m = synth_model(P, rows, cols, 2, 3, asym=True, seed=4)
    dm = DeviceModel.from_model(m)
    for p in (2, 3):
        a = dm.alpha[p].cpu().numpy().reshape(-1)
        assert np.array_equal(a, tiled_scales(m.scale_sets[p].alpha, rows, cols).reshape(-1))
        z = dm.offset[p].cpu().numpy().reshape(-1)
        assert np.array_equal(z, tiled_offsets(m.scale_sets[p].offset, rows, cols).reshape(-1))
    dm16 = DeviceModel.from_model(m, scale_dtype="f16")
    a16 = dm16.alpha[3].cpu().numpy().reshape(-1)
    want16 = tiled_scales(m.scale_sets[3].alpha, rows, cols).astype(np.float16).reshape(-1)
    assert np.array_equal(a16.view(np.uint16), want16.view(np.uint16))


# --- lookup table: bit-exact vs the reference ---------------------------------

def test_lut_build_bit_exact(P):
    with np.load("tests/golden/lut_tables.npz") as z:
        assert np.array_equal(P.LookupTable.build(z["x8"], 8).tables, z["t8"])
        assert np.array_equal(P.LookupTable.build(z["x4"], 4).tables, z["t4"])
        assert np.array_equal(P.LookupTable.build(z["x13"], 8).tables, z["t13_8"])
    t = P.LookupTable.build(np.array([0.5, 2.0], dtype=np.float32), 2).tables
    assert np.array_equal(t[0], np.float32([-2.5, -1.5, 1.5, 2.5]))      # test_gemv.py:43-46
    with pytest.raises(P.UsageError):
        P.LookupTable.build(np.ones(4), 9)


# --- golden cases from the real reference ---------------------------------------

@pytest.mark.parametrize("name", GOLDEN_CASES)
def test_engine_matches_reference_outputs(P, name):
    c = load_case(name)
    model = make_model(P, c)
    nx = len([k for k in c if k.startswith("x_")])
    for mu in (4, 8):
        eng = P.GemvEngine(model, chunk_width=mu)
        for p in model.precisions:
            for si in range(nx):
                x = c[f"x_{si}"]
                y, st = eng.lut(p, x)
                want = c.get(f"lut{mu}_p{p}_x{si}", c[f"lut8_p{p}_x{si}"])
                assert O.rel_dev(y, want) <= REF_TOL
                assert O.rel_dev(y, c[f"oracle_p{p}_x{si}"]) <= REF_TOL
                assert st.lut_build_count == 1
                assert [st.plane_bytes_fetched, st.scale_bytes_fetched] == list(c[f"stats_p{p}"][:2])
                yn, stn = eng.naive(p, x)
                assert O.rel_dev(yn, c[f"naive_p{p}_x{si}"]) <= REF_TOL
                assert stn.lut_build_count == 0
                if not np.any(x):
                    assert np.all(y == 0.0) and np.all(yn == 0.0)   # test_gemv.py:104-109


@pytest.mark.parametrize("name", ["g128_64x256", "asym_g40_16x80", "g128_ragged_37x200"])
def test_module_level_gemv_lut_and_naive(P, name):
    """gemv_lut / gemv_naive (gemv.py:253-258): a fresh engine per call, the
    reference's outputs, counters and chunk-width validation."""
    c = load_case(name)
    model = make_model(P, c)
    x = c["x_0"]
    for p in model.precisions:
        for mu in (4, 8):
            y, st = P.gemv_lut(model, p, x, chunk_width=mu)
            assert O.rel_dev(y, c.get(f"lut{mu}_p{p}_x0", c[f"lut8_p{p}_x0"])) <= REF_TOL
            assert st.lut_build_count == 1
        yn, stn = P.gemv_naive(model, p, x)
        assert O.rel_dev(yn, c[f"naive_p{p}_x0"]) <= REF_TOL
        assert stn.lut_build_count == 0 and stn.plane_bytes_fetched == st.plane_bytes_fetched
    with pytest.raises(P.UsageError):
        P.gemv_lut(model, model.p_lo, x, chunk_width=5)
    with pytest.raises(P.UsageError):
        P.gemv_naive(model, model.p_hi + 1, x)


def test_misaligned_x_rejected(P):
    """A contiguous but misaligned x view (storage offset) is a usage error
    before any launch -- not a misaligned-address fault."""
    m = synth_model(P, 64, 256, 2, 3, seed=4)
    dm = P.DeviceModel.from_model(m, scale_dtype="f16")
    buf = torch.randn(257, device="cuda").half()
    with pytest.raises(P.UsageError):
        dm.gemv(2, buf[1:])
    y = dm.gemv(2, buf[1:].clone())     # an aligned copy works
    assert torch.isfinite(y).all()


def test_single_active_column(P):
    c = load_case("single_col_1x4")                                    # test_gemv.py:94-101
    eng = P.GemvEngine(make_model(P, c))
    x = np.array([1.0, 0.0, 0.0, 0.0])
    assert eng.naive(2, x)[0][0] == pytest.approx(3.0, abs=1e-6)
    assert eng.naive(1, x)[0][0] == pytest.approx(2.0, abs=1e-6)
    assert eng.lut(2, x)[0][0] == pytest.approx(3.0, abs=1e-6)


def test_validation_errors_before_work(P):
    c = load_case("g32_32x128")
    eng = P.GemvEngine(make_model(P, c))
    x = c["x_0"]
    with pytest.raises(P.UsageError):
        eng.naive(1, x)                                                # below p_lo
    with pytest.raises(P.UsageError):
        eng.lut(5, x)                                                  # above p_hi
    with pytest.raises(P.UsageError):
        eng.lut(2, x[:100])                                            # wrong length
    with pytest.raises(P.UsageError):
        P.GemvEngine(make_model(P, c), chunk_width=5)


def test_model_read_only_across_calls(P):
    c = load_case("g128_64x256")
    model = make_model(P, c)
    eng = P.GemvEngine(model)
    before = eng.device_model.planes.clone()
    for p in (3, 2, 3):
        eng.lut(p, c["x_0"])
        eng.naive(p, c["x_1"])
    assert torch.equal(before, eng.device_model.planes)
    assert np.array_equal(eng.device_model.unpack_words().cpu().numpy().view(np.uint32), c["words"])


def test_dequant_oracle_on_gpu(P):
    c = load_case("asym_g128_128x1024")
    model = make_model(P, c)
    for p in (2, 4):
        got = P.dequant_oracle(model, p, c["x_0"])
        assert O.rel_dev(got, c[f"oracle_p{p}_x0"]) <= 1e-10


# --- fp16 deployment widths ---------------------------------------------------

def test_f16_scales_and_io(P):
    c = load_case("asym_g128_128x1024")
    model = make_model(P, c)
    dm = P.DeviceModel.from_model(model, scale_dtype="f16")
    x = c["x_0"].astype(np.float32)
    for p in (2, 3, 4):
        a16 = c[f"alpha_{p}"].astype(np.float16).astype(np.float32)
        z16 = c[f"offset_{p}"].astype(np.float16).astype(np.float32)
        exact = O.gemv_lut(c["words"], 1024, 128, a16, z16, p, x)     # same (f16-rounded) scales
        xd = torch.from_numpy(x).cuda()
        y = dm.gemv(p, xd).cpu().numpy()
        assert O.rel_dev(y, exact) <= REF_TOL
        assert O.rel_dev(y, c[f"lut8_p{p}_x0"]) <= NORTH_STAR_TOL     # vs the f32-scale reference
        yh = dm.gemv(p, xd.half(), out_dtype=torch.float16).float().cpu().numpy()
        xh = x.astype(np.float16).astype(np.float32)
        assert O.rel_dev(yh, O.gemv_lut(c["words"], 1024, 128, a16, z16, p, xh)) <= NORTH_STAR_TOL


# --- full-size shapes (Llama-3-8B / 70B layers) ----------------------------------

SHAPES = [(4096, 4096), (1024, 4096), (14336, 4096), (4096, 14336), (8192, 8192), (28672, 8192),
          (1024, 8192), (8192, 28672)]


@pytest.mark.parametrize("asym", [False, True])
@pytest.mark.parametrize("rows,cols", SHAPES)
def test_full_size_vs_c_oracle(P, rows, cols, asym):
    """Llama-3-8B and -70B layer shapes (incl. 70B k/v 1024x8192 and down
    8192x28672), symmetric and asymmetric, p = 2..4, vs the C oracle."""
    from oracle import c_oracle
    if asym and (rows, cols) not in ((4096, 4096), (1024, 8192), (8192, 28672), (28672, 8192)):
        pytest.skip("asymmetric mode on the 70B shapes and one 8B shape")
    m = synth_model(P, rows, cols, 2, 4, asym=asym, seed=rows + cols)
    dm = P.DeviceModel.from_model(m, scale_dtype="f16")
    x = O.random_gaussian(1, cols, seed=5).ravel().astype(np.float16).astype(np.float32)
    xd = torch.from_numpy(x).cuda()
    for p in (2, 3, 4):
        a16 = m.scale_sets[p].alpha.astype(np.float16).astype(np.float32)
        z16 = m.scale_sets[p].offset.astype(np.float16).astype(np.float32) if asym else None
        want = c_oracle.lut_gemv(m.bitplanes.words, cols, 128, a16, z16, p, x, threads=c_oracle.cpu_threads())
        y = dm.gemv(p, xd).cpu().numpy()
        assert O.rel_dev(y, want) <= NORTH_STAR_TOL
        assert O.rel_dev(y, want) <= 1e-5    # fp32 accumulate: far inside the bound


def test_full_size_properties(P):
    """Size-independent properties at 14336x4096: determinism, zero input,
    linearity in x, and plane-prefix consistency across precisions."""
    rows, cols = 14336, 4096
    m = synth_model(P, rows, cols, 2, 4, asym=True, seed=9)
    dm = P.DeviceModel.from_model(m, scale_dtype="f16")
    x1 = torch.from_numpy(O.random_gaussian(1, cols, seed=1).ravel()).cuda()
    x2 = torch.from_numpy(O.random_gaussian(1, cols, seed=2).ravel()).cuda()
    for p in (2, 3, 4):
        y1 = dm.gemv(p, x1)
        assert torch.equal(y1, dm.gemv(p, x1)), "not deterministic"
        assert torch.count_nonzero(dm.gemv(p, torch.zeros_like(x1))) == 0
        y12 = dm.gemv(p, 0.5 * x1 + 2.0 * x2)
        lin = 0.5 * y1.double() + 2.0 * dm.gemv(p, x2).double()
        assert O.rel_dev(y12.cpu().numpy(), lin.cpu().numpy()) <= 1e-5
        # dense reconstruction on the GPU agrees with the packed path
        w = dm.dequantize(p).double()
        assert O.rel_dev(y1.cpu().numpy(), (w @ x1.double()).cpu().numpy()) <= 1e-5


def test_workspace_per_stream(P):
    rows, cols = 4096, 4096
    m = synth_model(P, rows, cols, 2, 3, seed=11)
    dm = P.DeviceModel.from_model(m, scale_dtype="f16")
    x = torch.from_numpy(O.random_gaussian(1, cols, seed=3).ravel()).cuda()
    ref = {p: dm.gemv(p, x).clone() for p in (2, 3)}
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    outs = []
    for _ in range(20):
        with torch.cuda.stream(s1):
            outs.append((2, dm.gemv(2, x, stream=s1)))
        with torch.cuda.stream(s2):
            outs.append((3, dm.gemv(3, x, stream=s2)))
    torch.cuda.synchronize()
    for p, y in outs:
        assert torch.equal(y, ref[p])


def test_latency_scales_with_precision(P):
    # tests/test_gemv.py:239-246: p=2 is not slower than p=4
    m = synth_model(P, 14336, 4096, 2, 4, seed=12)
    rows = P.bench(m, [2, 4], O.random_gaussian(1, 4096, seed=31).ravel(), repeats=32, paths=("lut",))
    med = {r.precision: r.median_us for r in rows}
    assert med[2] <= med[4]


def test_bench_counters_and_render(P):
    c = load_case("g32_32x128")
    rows = P.bench(make_model(P, c), [2, 4], c["x_0"], repeats=3, include_dense=True)
    by = {(r.path, r.precision): r for r in rows}
    assert by[("lut", 2)].plane_bytes * 2 == by[("lut", 4)].plane_bytes
    assert by[("dense", 32)].plane_bytes == 32 * 128 * 4     # the reference's dense row (gemv.py:344)
    assert ("dense_f16", 16) not in by
    rows16 = P.bench(make_model(P, c), [2], c["x_0"], repeats=2, include_dense_f16=True)
    assert {(r.path, r.precision): r for r in rows16}[("dense_f16", 16)].plane_bytes == 32 * 128 * 2
    csv = P.render_bench_csv(rows)
    assert csv.splitlines()[0] == "shape,path,p,median_us,plane_bytes,scale_bytes"
    assert len(csv.splitlines()) == len(rows) + 1
    with pytest.raises(P.UsageError):
        P.bench(make_model(P, c), [2], c["x_0"], repeats=0)


@pytest.mark.parametrize("asym", [False, True])
def test_gemv_batch_32_random_jobs_vs_oracle(P, asym):
    """The full batch width (32 jobs): random shapes (ragged rows/cols, one-slice
    and many-slice jobs), random per-job precision, shared and distinct x --
    exercises the cost-balanced CTA ranges, single-piece rounds with builder
    warp groups, and the per-job arrival counters; every output vs the oracle,
    twice (counters self-reset), and bitwise equal to single calls."""
    from paper_2510_10467_b200.device_model import gemv_batch
    rng = np.random.default_rng(7)
    shapes = [(int(rng.integers(1, 600)), int(rng.choice([100, 256, 300, 1024, 2000, 4096]))) for _ in range(12)]
    models = [(P.DeviceModel.from_model(synth_model(P, r, c, 1, 4, asym=asym, seed=i), scale_dtype="f16"),
               synth_model(P, r, c, 1, 4, asym=asym, seed=i)) for i, (r, c) in enumerate(shapes)]
    xs = {}
    jobs, want = [], []
    for n in range(32):
        dm, host = models[n % len(models)]
        p = int(rng.integers(1, 5))
        if dm.cols not in xs or n % 5 == 0:
            xs[dm.cols] = O.random_gaussian(1, dm.cols, seed=100 + n).ravel().astype(np.float16)
        x = xs[dm.cols]
        xd = torch.from_numpy(x).cuda()
        out = torch.empty(dm.rows, device="cuda", dtype=torch.float32)
        jobs.append((dm, p, xd, out))
        st = host.scale_sets[p]
        a16 = st.alpha.astype(np.float16).astype(np.float32)
        z16 = st.offset.astype(np.float16).astype(np.float32) if asym else None
        want.append(O.gemv_lut(host.bitplanes.words, dm.cols, 128, a16, z16, p, x.astype(np.float32)))
    for _ in range(2):
        gemv_batch(jobs)
        torch.cuda.synchronize()
        for (dm, p, _, out), w in zip(jobs, want):
            assert O.rel_dev(out.cpu().numpy(), w) <= REF_TOL, (dm.rows, dm.cols, p)
    for dm, p, xd, out in jobs[:6]:  # single calls take the cluster kernel: same values to f32 rounding
        assert _rel(dm.gemv(p, xd), out) <= 1e-5


def _rel(a, b):
    a, b = a.double(), b.double()
    return float((a - b).norm() / max(float(b.norm()), 1e-30))


# cluster GEMV geometries forced through abcq_debug_set_mode(5000 + 100*slots
# + 10*C + tiles/warp; C digit 6 = 16): every cluster size, one and two CTAs
# per SM, one and two tiles per warp -- incl. clusters wider than the slices
CLUSTER_FORCE = [5000, 5112, 5122, 5142, 5182, 5162, 5262, 5281, 5221, 5141]


@pytest.mark.parametrize("rows,cols,asym,sd", [(4096, 4096, False, "f16"), (1000, 2000, True, "f32"),
                                               (37, 200, False, "f16"), (300, 14336, True, "f16"),
                                               (6144, 4096, False, "f32")])
def test_cluster_gemv_geometries_vs_oracle(P, rows, cols, asym, sd):
    from paper_2510_10467_b200 import _lib
    L = _lib.lib()
    m = synth_model(P, rows, cols, 1, 5, asym=asym, seed=rows * 3 + cols)
    dm = P.DeviceModel.from_model(m, scale_dtype=sd)
    x = O.random_gaussian(1, cols, seed=7).ravel().astype(np.float16)
    xd = torch.from_numpy(x).cuda()
    xf = x.astype(np.float32)
    want = {}
    for p in range(1, 6):
        st = m.scale_sets[p]
        a = st.alpha.astype(np.float16).astype(np.float32) if sd == "f16" else st.alpha
        z = None
        if asym:
            z = st.offset.astype(np.float16).astype(np.float32) if sd == "f16" else st.offset
        want[p] = O.gemv_lut(m.bitplanes.words, cols, 128, a, z, p, xf)
    try:
        L.abcq_debug_set_mode(27)  # every shape through the cluster kernel
        for force, warps in [(f, 6000) for f in CLUSTER_FORCE] + [(5162, 6008), (5142, 6008), (5112, 6008)]:
            L.abcq_debug_set_mode(warps)     # consumer warps: automatic, or 8 with one CTA per SM
            L.abcq_debug_set_mode(force)
            for p in (1, 2, 4, 5):
                y = dm.gemv(p, xd)
                torch.cuda.synchronize()
                assert O.rel_dev(y.cpu().numpy(), want[p]) <= 1e-5, (force, p)
                assert torch.equal(y, dm.gemv(p, xd)), (force, p)   # bitwise repeatable
    finally:
        L.abcq_debug_set_mode(5000)
        L.abcq_debug_set_mode(6000)
        L.abcq_debug_set_mode(0)


def test_gemv_batch_matches_single_calls(P):
    """One persistent launch over mixed shapes / precisions (incl. the same model
    at several p, as per-request precision does) == separate calls. Single
    calls of small layers take the cluster kernel (DSMEM split-K, another fixed
    summation order): equal to f32 rounding, and each path bitwise repeatable."""
    from paper_2510_10467_b200.device_model import gemv_batch
    shapes = [(4096, 4096), (1024, 4096), (14336, 4096), (4096, 14336), (37, 200), (16, 256)]
    models = [P.DeviceModel.from_model(synth_model(P, r, c, 2, 4, seed=r + c), scale_dtype="f16") for r, c in shapes]
    xs = {c: torch.from_numpy(O.random_gaussian(1, c, seed=c).ravel()).cuda().half() for _, c in shapes}
    jobs, want = [], []
    for k, dm in enumerate(models):
        for p in ((2, 4) if k == 0 else (2 + k % 3,)):
            jobs.append((dm, p, xs[dm.cols], torch.empty(dm.rows, device="cuda", dtype=torch.float16)))
            want.append(dm.gemv(p, xs[dm.cols], out_dtype=torch.float16).clone())
    gemv_batch(jobs)
    torch.cuda.synchronize()
    first = [o.clone() for *_, o in jobs]
    for (dm, p, _, out), w in zip(jobs, want):
        assert _rel(out, w) <= 2e-3, (dm.rows, dm.cols, p)  # fp16 y: one rounding apart at most
    for (dm, p, x, _), w in zip(jobs, want):
        assert torch.equal(dm.gemv(p, x, out_dtype=torch.float16), w)  # single calls repeat bitwise
    gemv_batch(jobs)  # a second run (reused workspace) is identical
    torch.cuda.synchronize()
    for (_, _, _, out), w in zip(jobs, first):
        assert torch.equal(out, w)


def test_gemv_batch_plan_repeated_launches(P):
    """GemvBatchPlan (validated once, one C-ABI call per launch) == gemv_batch,
    bitwise, over repeated launches on two streams (per-stream workspaces),
    with the inputs changed in place between launches."""
    from paper_2510_10467_b200.device_model import gemv_batch
    shapes = [(4096, 4096), (1024, 4096), (14336, 4096)]
    models = [P.DeviceModel.from_model(synth_model(P, r, c, 2, 4, seed=r), scale_dtype="f16") for r, c in shapes]
    x = torch.from_numpy(O.random_gaussian(1, 4096, seed=5).ravel()).cuda().half()
    jobs = [(dm, p, x, torch.empty(dm.rows, device="cuda", dtype=torch.float16)) for dm in models for p in (2, 3, 4)]
    plan = P.GemvBatchPlan(jobs)
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    for it in range(4):
        x.copy_(torch.from_numpy(O.random_gaussian(1, 4096, seed=10 + it).ravel()).half())
        torch.cuda.synchronize()
        want = [o.clone() for o in gemv_batch([(dm, p, x, torch.empty_like(out)) for dm, p, _, out in jobs])]
        with torch.cuda.stream(streams[it & 1]):
            plan.launch(streams[it & 1])
        torch.cuda.synchronize()
        for (_, _, _, out), w in zip(jobs, want):
            assert torch.equal(out, w)
    with pytest.raises(P.UsageError):
        P.GemvBatchPlan([(models[0], 5, x, jobs[0][3])])  # precision outside [p_lo, p_hi]


def test_gemv_batch_more_jobs_than_one_launch(P):
    """40 jobs (> abcq_gemv_batch_max_jobs) split over two launches == single calls, bitwise."""
    from paper_2510_10467_b200 import _lib
    from paper_2510_10467_b200.device_model import gemv_batch
    assert _lib.lib().abcq_gemv_batch_max_jobs() < 40
    dms = [P.DeviceModel.from_model(synth_model(P, r, 512, 2, 4, seed=r), scale_dtype="f16") for r in (64, 200, 1000)]
    x = torch.from_numpy(O.random_gaussian(1, 512, seed=9).ravel()).cuda().half()
    jobs = [(dms[k % 3], 2 + k % 3, x, torch.empty(dms[k % 3].rows, device="cuda", dtype=torch.float16))
            for k in range(40)]
    gemv_batch(jobs)
    torch.cuda.synchronize()
    for dm, p, _, out in jobs:
        assert _rel(out, dm.gemv(p, x, out_dtype=torch.float16)) <= 2e-3


def test_split_k_completion_paths_agree(P):
    """Trailing-CTA completion (one launch) and the standalone PDL-chained
    reduce kernel (debug mode 22) give bitwise-identical y (fixed chain order)."""
    from paper_2510_10467_b200 import _lib
    from paper_2510_10467_b200.device_model import gemv_batch
    dms = [P.DeviceModel.from_model(synth_model(P, r, c, 2, 4, seed=r + c), scale_dtype="f16")
           for r, c in ((4096, 4096), (1024, 14336), (300, 1000))]
    x = {c: torch.from_numpy(O.random_gaussian(1, c, seed=c).ravel()).cuda().half() for c in (4096, 14336, 1000)}
    jobs = [(dm, p, x[dm.cols], torch.empty(dm.rows, device="cuda", dtype=torch.float16)) for dm in dms for p in (2, 4)]
    gemv_batch(jobs)
    torch.cuda.synchronize()
    fused = [o.clone() for *_, o in jobs]
    _lib.lib().abcq_debug_set_mode(22)
    try:
        gemv_batch(jobs)
        torch.cuda.synchronize()
    finally:
        _lib.lib().abcq_debug_set_mode(0)
    for (*_, o), f in zip(jobs, fused):
        assert torch.equal(o, f)


@pytest.mark.parametrize("asym,sd", [(False, "f16"), (True, "f16"), (True, "f32")])
def test_batch_schedule_variants_bitwise_equal(P, asym, sd):
    """The schedule only decides which warp / CTA / completion block does an
    item, never the arithmetic: the slot-sized chunk split of multi-round CTAs
    vs the round-1 cost split (debug mode 32), the completion blocks of >16-slice
    jobs first vs job order (29), the schedule reversed over the CTAs (33) --
    bitwise equal y, over a batch of many short pieces (k/v-sized jobs at
    several precisions, a 56-slice job)."""
    from paper_2510_10467_b200 import _lib
    from paper_2510_10467_b200.device_model import gemv_batch
    shapes = [(1024, 4096), (4096, 4096), (512, 14336), (2000, 1000), (16, 4096)]
    dms = [P.DeviceModel.from_model(synth_model(P, r, c, 1, 4, asym=asym, seed=r + c), scale_dtype=sd)
           for r, c in shapes]
    x = {c: torch.from_numpy(O.random_gaussian(1, c, seed=c).ravel()).cuda().half() for _, c in shapes}
    jobs = [(dm, p, x[dm.cols], torch.empty(dm.rows, device="cuda", dtype=torch.float16))
            for p in (1, 2, 3, 4) for dm in dms]  # (f32 asymmetric scales: 4-item slots)
    gemv_batch(jobs)
    torch.cuda.synchronize()
    base = [o.clone() for *_, o in jobs]
    for mode in (32, 29, 33):
        _lib.lib().abcq_debug_set_mode(mode)
        try:
            for o in (j[3] for j in jobs):
                o.fill_(0)
            gemv_batch(jobs)
            torch.cuda.synchronize()
        finally:
            _lib.lib().abcq_debug_set_mode(0)
        for (dm, p, _, o), b in zip(jobs, base):
            assert torch.equal(o, b), (mode, dm.rows, dm.cols, p)


def test_reserved_sms_same_results(P):
    """abcq_set_reserved_sms: a smaller persistent grid (SMs left to a kernel
    running beside it) changes only the schedule -- bitwise equal y; the
    bound check is a usage error."""
    from paper_2510_10467_b200.device_model import gemv_batch, set_reserved_sms
    dms = [P.DeviceModel.from_model(synth_model(P, r, c, 2, 4, seed=r + c), scale_dtype="f16")
           for r, c in ((4096, 4096), (1024, 14336))]
    x = {c: torch.from_numpy(O.random_gaussian(1, c, seed=c).ravel()).cuda().half() for c in (4096, 14336)}
    jobs = [(dm, p, x[dm.cols], torch.empty(dm.rows, device="cuda", dtype=torch.float16)) for dm in dms for p in (2, 4)]
    gemv_batch(jobs)
    torch.cuda.synchronize()
    base = [o.clone() for *_, o in jobs]
    try:
        assert set_reserved_sms(20) == 0
        gemv_batch(jobs)
        torch.cuda.synchronize()
        with pytest.raises(P.UsageError):
            set_reserved_sms(100000)
    finally:
        assert set_reserved_sms(0) == 20
    for (*_, o), b in zip(jobs, base):
        assert torch.equal(o, b)


def test_gemv_batch_asymmetric(P):
    from paper_2510_10467_b200.device_model import gemv_batch
    ms = [P.DeviceModel.from_model(synth_model(P, r, 1024, 2, 3, asym=True, seed=r)) for r in (128, 300)]
    x = torch.from_numpy(O.random_gaussian(1, 1024, seed=3).ravel()).cuda()
    jobs = [(m, p, x, torch.empty(m.rows, device="cuda")) for m in ms for p in (2, 3)]
    gemv_batch(jobs)
    for m, p, _, out in jobs:
        assert _rel(out, m.gemv(p, x)) <= 1e-5


@pytest.mark.parametrize("asym", [False, True])
@pytest.mark.parametrize("rows,cols", [(64, 256), (37, 200), (4096, 4096), (1024, 14336)])
def test_gemm_mixedp_matches_per_request_oracle(P, rows, cols, asym):
    """B <= 16 requests with mixed precision in one tensor-core pass == the
    reference's per-request loop (cli.py:122-126) on the oracle."""
    m = synth_model(P, rows, cols, 2, 4, asym=asym, seed=rows * 7 + cols)
    dm = P.DeviceModel.from_model(m, scale_dtype="f16")
    for B in (1, 5, 16):
        ps = [2 + (b * 7 + B) % 3 for b in range(B)]
        X = np.stack([O.random_gaussian(1, cols, seed=100 + b).ravel() for b in range(B)])
        Xh = X.astype(np.float16).astype(np.float32)  # the kernel computes on fp16 x
        Y = dm.gemm_mixedp(ps, torch.from_numpy(Xh).cuda()).cpu().numpy()
        for b, p in enumerate(ps):
            a16 = m.scale_sets[p].alpha.astype(np.float16).astype(np.float32)
            z = m.scale_sets[p].offset
            z16 = None if z is None else z.astype(np.float16).astype(np.float32)
            want = O.gemv_lut(m.bitplanes.words, cols, 128, a16, z16, p, Xh[b])
            assert O.rel_dev(Y[b], want) <= 1e-4, (B, b, p, O.rel_dev(Y[b], want))


@pytest.mark.parametrize("asym", [False, True])
def test_gemm_mixedp_mlp_shape_b16_vs_c_oracle(P, asym):
    """The Llama-3-8B gate/up shape (14336x4096) at B = 16 mixed precisions
    (BASELINE config 3) vs the C oracle, per request."""
    from oracle import c_oracle
    rows, cols = 14336, 4096
    m = synth_model(P, rows, cols, 2, 4, asym=asym, seed=77)
    dm = P.DeviceModel.from_model(m, scale_dtype="f16")
    ps = [2 + b % 3 for b in range(16)]
    X = np.stack([O.random_gaussian(1, cols, seed=300 + b).ravel() for b in range(16)])
    Xh = X.astype(np.float16).astype(np.float32)
    Y = dm.gemm_mixedp(ps, torch.from_numpy(Xh).cuda()).cpu().numpy()
    for b, p in enumerate(ps):
        a16 = m.scale_sets[p].alpha.astype(np.float16).astype(np.float32)
        z16 = m.scale_sets[p].offset.astype(np.float16).astype(np.float32) if asym else None
        want = c_oracle.lut_gemv(m.bitplanes.words, cols, 128, a16, z16, p, Xh[b], threads=c_oracle.cpu_threads())
        assert O.rel_dev(Y[b], want) <= 1e-4, (b, p, O.rel_dev(Y[b], want))


@pytest.mark.parametrize("asym", [False, True])
@pytest.mark.parametrize("scale_dtype", ["f16", "f32"])
def test_gemm_mixedp_tcgen05_variant(P, asym, scale_dtype):
    """The tcgen05 GEMM (A = expanded sign planes in tensor memory, B = X in
    shared memory, D in tensor memory; opt-in debug mode 40) against the
    per-request oracle, ragged rows/cols, B in {1, 7, 16}, p up to 6."""
    from paper_2510_10467_b200 import _lib
    rows, cols = 300, 1000
    m = synth_model(P, rows, cols, 2, 6, asym=asym, seed=11)
    dm = P.DeviceModel.from_model(m, scale_dtype=scale_dtype)
    _lib.lib().abcq_debug_set_mode(40)
    try:
        for B in (1, 7, 16):
            ps = [(2, 4, 6, 3)[b % 4] for b in range(B)]
            X = np.stack([O.random_gaussian(1, cols, seed=300 + b).ravel() for b in range(B)])
            Xh = X.astype(np.float16).astype(np.float32)
            Y = dm.gemm_mixedp(ps, torch.from_numpy(Xh).cuda()).cpu().numpy()
            for b, p in enumerate(ps):
                a = m.scale_sets[p].alpha
                z = m.scale_sets[p].offset
                if scale_dtype == "f16":
                    a = a.astype(np.float16).astype(np.float32)
                    z = None if z is None else z.astype(np.float16).astype(np.float32)
                want = O.gemv_lut(m.bitplanes.words, cols, 128, a, z, p, Xh[b])
                assert O.rel_dev(Y[b], want) <= 1e-4, (B, b, p, O.rel_dev(Y[b], want))
    finally:
        _lib.lib().abcq_debug_set_mode(0)


@pytest.mark.parametrize("scale_dtype", ["f16", "f32"])
def test_gemm_mixedp_deep_precisions(P, scale_dtype):
    """p_max > 4 (planes staged in two rounds), more than kMaxSets distinct
    precisions in one batch (global scale loads), f32 scale sets, and a cols
    value that is not a multiple of 8 (scalar X staging)."""
    rows, cols = 200, 1000
    m = synth_model(P, rows, cols, 1, 7, asym=False, seed=5)
    dm = P.DeviceModel.from_model(m, scale_dtype=scale_dtype)
    ps = [1 + b % 7 for b in range(16)]
    X = np.stack([O.random_gaussian(1, cols, seed=200 + b).ravel() for b in range(16)])
    Xh = X.astype(np.float16).astype(np.float32)
    Y = dm.gemm_mixedp(ps, torch.from_numpy(Xh).cuda()).cpu().numpy()
    for b, p in enumerate(ps):
        a = m.scale_sets[p].alpha
        if scale_dtype == "f16":
            a = a.astype(np.float16).astype(np.float32)
        want = O.gemv_lut(m.bitplanes.words, cols, 128, a, None, p, Xh[b])
        assert O.rel_dev(Y[b], want) <= 1e-4, (b, p, O.rel_dev(Y[b], want))


# --- torch.ops.anybcq_b200 (SURVEY §8b device operator) -------------------------

def test_torch_ops_match_device_model(P):
    from paper_2510_10467_b200 import ops
    m = synth_model(P, 1024, 4096, 2, 4, seed=11)
    dm = P.DeviceModel.from_model(m, scale_dtype="f16")
    h = ops.register(dm)
    try:
        x = torch.from_numpy(O.random_gaussian(1, 4096, seed=3).ravel()).cuda().half()
        for p in (2, 3, 4):
            y = torch.ops.anybcq_b200.gemv(h, x, p)
            assert y.dtype == torch.float16 and y.shape == (1024,)
            assert torch.equal(y, dm.gemv(p, x, out_dtype=torch.float16))   # same launch, bitwise
        X = torch.randn(3, 4096, device="cuda")
        Y = torch.ops.anybcq_b200.gemm_mixedp(h, X, [2, 4, 3])
        assert torch.equal(Y, dm.gemm_mixedp([2, 4, 3], X))
        W = torch.ops.anybcq_b200.dequantize(h, 3, X)
        assert torch.equal(W, dm.dequantize(3))
        torch.library.opcheck(torch.ops.anybcq_b200.gemv.default, (h, x, 3),
                              test_utils=("test_schema", "test_faketensor"))
        # the op captures into a CUDA graph (the decode harness path)
        xs = x.clone()
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            torch.ops.anybcq_b200.gemv(h, xs, 3)     # workspace for this stream, outside capture
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            yg = torch.ops.anybcq_b200.gemv(h, xs, 3)
        xs.copy_(x.flip(0))
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(yg, dm.gemv(3, x.flip(0).contiguous(), out_dtype=torch.float16))
    finally:
        ops.unregister(h)


# --- SiLU-gated input (ABCQ_F16_SILU_GLU): silu(g)*u formed in the table build ----

@pytest.mark.parametrize("rows,cols,asym", [(4096, 14336, False), (256, 1024, True), (37, 200, False),
                                            (48, 1000, True), (37, 1001, False), (20, 333, True)])
def test_silu_glu_input_matches_separate_silu_mul(P, rows, cols, asym):
    from paper_2510_10467_b200.decode import silu_mul
    m = synth_model(P, rows, cols, 2, 4, asym=asym, seed=rows ^ cols)
    dm = P.DeviceModel.from_model(m, scale_dtype="f16")
    g = torch.Generator(device="cuda").manual_seed(cols)
    gu = (2 * torch.randn(2 * cols, device="cuda", generator=g)).half()
    act = torch.empty(cols, device="cuda", dtype=torch.float16)
    silu_mul(gu[:cols], gu[cols:], act)
    for p in (2, 3, 4):
        for yd in (torch.float16, torch.float32):
            fused = dm.gemv(p, gu, out_dtype=yd, silu_glu=True)
            sep = dm.gemv(p, act, out_dtype=yd)
            assert torch.equal(fused, sep)      # same f16 input bits -> same launch result
    # and the separate path itself against the oracle on that input
    a16 = m.scale_sets[3].alpha.astype(np.float16).astype(np.float32)
    z16 = m.scale_sets[3].offset.astype(np.float16).astype(np.float32) if asym else None
    want = O.gemv_lut(m.bitplanes.words, cols, 128, a16, z16, 3, act.float().cpu().numpy())
    assert O.rel_dev(dm.gemv(3, gu, silu_glu=True).cpu().numpy(), want) <= NORTH_STAR_TOL
    with pytest.raises(P.UsageError):
        dm.gemv(3, gu.float(), silu_glu=True)
    with pytest.raises(P.UsageError):
        dm.gemv(3, gu[:cols], silu_glu=True)


def test_silu_glu_mixed_with_plain_jobs_in_one_batch(P):
    """C-ABI batch: a SiLU-gated job next to plain f16 jobs (the gate is per job)."""
    import ctypes as C
    from paper_2510_10467_b200 import _lib
    from paper_2510_10467_b200.decode import silu_mul
    L = _lib.lib()
    dms = [P.DeviceModel.from_model(synth_model(P, r, c, 2, 4, seed=r + c), scale_dtype="f16")
           for r, c in ((512, 1024), (256, 2048), (48, 1000))]
    g = torch.Generator(device="cuda").manual_seed(5)
    xs = [torch.randn(dms[0].cols, device="cuda", generator=g).half(),
          (2 * torch.randn(2 * dms[1].cols, device="cuda", generator=g)).half(),   # [gate ; up]
          torch.randn(dms[2].cols, device="cuda", generator=g).half()]
    glu = [False, True, False]
    ps = [3, 4, 2]
    ys = [torch.empty(dm.rows, device="cuda", dtype=torch.float16) for dm in dms]
    arr = (_lib.AbcqGemvJob * 3)()
    for k, dm in enumerate(dms):
        arr[k].model = C.pointer(dm._struct)
        arr[k].p = ps[k]
        arr[k].x_dtype = _lib.F16_SILU_GLU if glu[k] else _lib.F16
        arr[k].y_dtype = _lib.F16
        arr[k].x = xs[k].data_ptr()
        arr[k].y = ys[k].data_ptr()
    need = C.c_size_t()
    _lib.check(L.abcq_gemv_batch_workspace_bytes(arr, 3, C.byref(need)))
    ws = torch.zeros(max(int(need.value), 16), dtype=torch.uint8, device="cuda")
    _lib.check(L.abcq_gemv_batch(arr, 3, ws.data_ptr(), ws.numel(), torch.cuda.current_stream().cuda_stream))
    act = torch.empty(dms[1].cols, device="cuda", dtype=torch.float16)
    silu_mul(xs[1][:dms[1].cols], xs[1][dms[1].cols:], act)
    want = P.gemv_batch([(dms[0], 3, xs[0], torch.empty_like(ys[0])), (dms[1], 4, act, torch.empty_like(ys[1])),
                         (dms[2], 2, xs[2], torch.empty_like(ys[2]))])
    for k in range(3):
        assert torch.equal(ys[k], want[k]), k
    # an f32 job next to a gated one is rejected before any work
    arr[0].x_dtype = _lib.F32
    assert L.abcq_gemv_batch(arr, 3, ws.data_ptr(), ws.numel(), None) == _lib.E_ARG


def test_row_sharded_gemv_nccl_world1(P):
    """RowShardedGemv on the CUDA engine through a world-size-1 NCCL group:
    the plan-launched shard GEMV lands in the gather buffer, y vs the oracle."""
    import os
    import socket

    import torch.distributed as dist
    from paper_2510_10467_b200.parallel import RowShardedGemv
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        m = synth_model(P, 1000, 2048, 2, 4, seed=21)
        eng = RowShardedGemv(m, scale_dtype="f16", device="cuda")
        x = O.random_gaussian(1, 2048, seed=4).ravel().astype(np.float16)
        xd = torch.from_numpy(x).cuda()
        for p in (2, 3, 4):
            y = eng.gemv(p, xd)
            torch.cuda.synchronize()
            a16 = m.scale_sets[p].alpha.astype(np.float16).astype(np.float32)
            want = O.gemv_lut(m.bitplanes.words, 2048, 128, a16, None, p, x.astype(np.float32))
            assert y.shape == (1000,) and O.rel_dev(y.float().cpu().numpy(), want) <= 1e-3
        eng.gather()
        torch.cuda.synchronize()
    finally:
        dist.destroy_process_group()


def test_fused_peer_allgather_world1(P):
    """The fused all-gather (abcq_gemv_batch_peer through torch symmetric
    memory) at world size 1: the rows land in the gathered buffer bitwise as
    a plain batch launch writes them, the epoch advances once per launch and
    is published in the signal slot, the consumer wait passes (no timeout),
    and the host checks reject outputs outside the buffer / one-slice jobs."""
    import os
    import socket

    import torch.distributed as dist
    from paper_2510_10467_b200.device_model import gemv_batch
    from paper_2510_10467_b200.parallel import PeerGather
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        shapes = [(4096, 4096), (1000, 2048), (512, 14336)]
        dms = [P.DeviceModel.from_model(synth_model(P, r, c, 2, 4, seed=r + c), scale_dtype="f16") for r, c in shapes]
        x = {c: torch.from_numpy(O.random_gaussian(1, c, seed=c).ravel()).cuda().half() for _, c in shapes}
        specs = [(dm, p) for p in (2, 4) for dm in dms]
        R = sum(dm.rows for dm, _ in specs)
        g = PeerGather(R)
        views, off = [], 0
        for dm, _ in specs:
            views.append(g.local[off:off + dm.rows])
            off += dm.rows
        plan = g.plan([(dm, p, x[dm.cols], v) for (dm, p), v in zip(specs, views)])
        want = gemv_batch([(dm, p, x[dm.cols], torch.empty(dm.rows, device="cuda", dtype=torch.float16))
                           for dm, p in specs])
        for it in (1, 2, 3):
            g.local.fill_(0)
            plan.launch()
            g.wait()
            torch.cuda.synchronize()
            assert int(g.err.item()) == 0
            assert int(g.state[0].item()) == it
            for v, w in zip(views, want):
                assert torch.equal(v, w)
        with pytest.raises(P.UsageError):  # an output outside the gathered rows
            g.plan([(dms[0], 2, x[4096], torch.empty(4096, device="cuda", dtype=torch.float16))])
    finally:
        dist.destroy_process_group()


def test_fused_peer_stores_two_buffers_one_gpu(P):
    """The peer-store data path on one GPU: a 2-'rank' launch whose 'peer'
    buffer is a second local buffer -- rank 0's rows land in both buffers at
    the same offsets (bitwise), the wait publishes the epoch in both signal
    arrays and times out (err, no hang) on the 'rank' that never runs, and the
    C-ABI argument checks hold (peer_bases[rank] must be local)."""
    import ctypes as C

    from paper_2510_10467_b200 import _lib
    from paper_2510_10467_b200.device_model import GemvBatchPlan, gemv_batch
    L = _lib.lib()
    dms = [P.DeviceModel.from_model(synth_model(P, r, 4096, 2, 4, seed=r), scale_dtype="f16") for r in (4096, 1024)]
    x = torch.from_numpy(O.random_gaussian(1, 4096, seed=3).ravel()).cuda().half()
    R = sum(dm.rows for dm in dms)
    buf = [torch.zeros(2 * R, dtype=torch.float16, device="cuda") for _ in range(2)]  # 2 'ranks' x R rows
    sig = [torch.zeros(8, dtype=torch.int32, device="cuda") for _ in range(2)]
    state = torch.zeros(int(L.abcq_peer_state_bytes()) // 4, dtype=torch.int32, device="cuda")
    views, off = [], 0
    for dm in dms:
        views.append(buf[0][off:off + dm.rows])  # rank 0's slice of its own buffer
        off += dm.rows
    plan = GemvBatchPlan([(dm, 3, x, v) for dm, v in zip(dms, views)])
    ws = torch.zeros(plan.need, dtype=torch.uint8, device="cuda")
    bases = (C.c_void_p * 2)(buf[0].data_ptr(), buf[1].data_ptr())
    sigs = (C.c_void_p * 2)(sig[0].data_ptr(), sig[1].data_ptr())
    sh = torch.cuda.current_stream().cuda_stream
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    for it in (1, 2):
        _lib.check(L.abcq_gemv_batch_peer(plan.arr, plan.n, buf[0].data_ptr(), buf[0].numel() * 2, bases, sigs, 2, 0,
                                          state.data_ptr(), ws.data_ptr(), ws.numel(), sh), "abcq_gemv_batch_peer")
        torch.cuda.synchronize()
        want = gemv_batch([(dm, 3, x, torch.empty(dm.rows, device="cuda", dtype=torch.float16)) for dm in dms])
        assert torch.equal(buf[0][:R], torch.cat(want)) and torch.equal(buf[1][:R], buf[0][:R])
        assert int(state[0]) == it - 1  # this launch is still pending: published by the next one / the wait
        # the wait publishes it to both signal arrays, then times out on 'rank 1' (nobody runs it): err = 1 + 1
        err.zero_()
        _lib.check(L.abcq_peer_wait(bases, sigs, 2, 0, state.data_ptr(), err.data_ptr(), 2_000_000, sh), "abcq_peer_wait")
        torch.cuda.synchronize()
        assert int(state[0]) == it and int(sig[0][0]) == it and int(sig[1][0]) == it and int(err) == 2
    assert not buf[1][R:].any()  # rank 1's rows: nobody wrote them
    swapped = (C.c_void_p * 2)(buf[1].data_ptr(), buf[0].data_ptr())
    with pytest.raises(P.UsageError):
        _lib.check(L.abcq_gemv_batch_peer(plan.arr, plan.n, buf[0].data_ptr(), buf[0].numel() * 2, swapped, sigs, 2, 0,
                                          state.data_ptr(), ws.data_ptr(), ws.numel(), sh), "abcq_gemv_batch_peer")


def test_stream_workspace_shared_and_grown(P):
    """One split-K workspace per (device, stream) serves every model and batch
    launched in order on it (counters at offset 0 of every layout): models of
    different sizes interleaved on one stream -- the workspace growing under
    them, the replaced buffer kept alive for whoever cached it -- give
    bitwise the results of the same calls each on a fresh stream."""
    from paper_2510_10467_b200 import device_model as DMm
    st = torch.cuda.Stream()
    small = P.DeviceModel.from_model(synth_model(P, 512, 4096, 2, 4, seed=1), scale_dtype="f16")
    big = P.DeviceModel.from_model(synth_model(P, 8192, 8192, 2, 4, seed=2), scale_dtype="f16")
    xs = {c: torch.from_numpy(O.random_gaussian(1, c, seed=c).ravel()).cuda().half() for c in (4096, 8192)}
    calls = [(small, 2), (big, 3), (small, 4), (big, 2), (small, 3)]
    want = []
    for dm, p in calls:  # each on its own fresh stream (its own workspace)
        s2 = torch.cuda.Stream()
        with torch.cuda.stream(s2):
            want.append(DMm.gemv_batch([(dm, p, xs[dm.cols], torch.empty(dm.rows, device="cuda",
                                                                            dtype=torch.float16))], s2)[0])
        torch.cuda.synchronize()
    n_old = len(DMm._STREAM_WS_OLD)
    got = []
    with torch.cuda.stream(st):
        for dm, p in calls:
            got.append(DMm.gemv_batch([(dm, p, xs[dm.cols], torch.empty(dm.rows, device="cuda",
                                                                           dtype=torch.float16))], st)[0])
    torch.cuda.synchronize()
    assert len(DMm._STREAM_WS_OLD) >= n_old + 1  # it grew under the small model's first call
    for g, w in zip(got, want):
        assert torch.equal(g, w)
