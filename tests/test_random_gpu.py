"""Seeded random parity cases (a bounded slice of tools/fuzz_gemv.py): random
ragged shapes, group sizes, precisions, symmetric / asymmetric models and
f16 / f32 scale sets through single GEMVs (every dispatch: automatic, the
cluster kernel for every size, the persistent kernel), gemv_batch job lists
under each schedule variant (bitwise equal across them) and gemm_mixedp,
each output against the C oracle."""

import numpy as np
import pytest

from oracle import anybcq_oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-5


@pytest.fixture(scope="module")
def P():
    import paper_2510_10467_b200 as P
    return P


@pytest.fixture
def L():
    from paper_2510_10467_b200 import _lib
    lib = _lib.lib()
    yield lib
    lib.abcq_debug_set_mode(0)


def make(P, rows, cols, gs, p_hi, asym, seed):
    words = O.random_words(p_hi, rows, cols, seed=seed)
    r = np.random.default_rng(seed)
    G = -(-cols // gs)
    sets = {}
    for p in range(1, p_hi + 1):
        al = (0.01 + 0.1 * np.abs(r.standard_normal((p, rows, G)))).astype(np.float32)
        z = (0.1 * r.standard_normal((rows, G))).astype(np.float32) if asym else None
        sets[p] = P.ScaleTensor(al, z, gs)
    return P.MultiPrecisionModel(P.BitPlaneSet(p_hi, rows, cols, words), sets, 1, p_hi,
                                 P.QuantConfig(gs, "asymmetric" if asym else "symmetric", 0))


def want(m, sd, p, x):
    """C oracle on the scales the device holds (f16-rounded for f16 sets), and
    each row's magnitude sum (the f32 rounding scale of a cancelling row)."""
    from oracle import c_oracle
    st = m.scale_sets[p]
    q = (lambda v: v.astype(np.float16).astype(np.float32)) if sd == "f16" else (lambda v: v)
    z = None if st.offset is None else q(st.offset)
    gs = m.config.group_size
    w = c_oracle.lut_gemv(m.bitplanes.words, m.bitplanes.cols, gs, q(st.alpha), z, p, x.astype(np.float32),
                          threads=c_oracle.cpu_threads())
    xa = np.abs(x.astype(np.float64))
    X = np.add.reduceat(xa, np.arange(0, xa.size, gs))
    mag = np.abs(q(st.alpha)[:p]).astype(np.float64).sum(0) @ X
    if z is not None:
        mag += np.abs(z).astype(np.float64) @ X
    return w, mag


def close(y, wm, tol=TOL, mtol=1e-6):
    w, mag = wm
    return O.rel_dev(y, w) <= tol or bool(np.all(np.abs(y - w) <= mtol * np.maximum(mag, 1e-30)))


def dim(rng, lo, hi):
    return int(np.exp(rng.uniform(np.log(lo), np.log(hi))))


@pytest.mark.parametrize("seed", range(6))
def test_random_single_gemv_every_dispatch(P, L, seed):
    rng = np.random.default_rng(1000 + seed)
    for case in range(4):
        rows, cols = dim(rng, 1, 20000), dim(rng, 1, 20000)
        while rows * cols > 24 << 20:
            rows, cols = dim(rng, 1, 20000), dim(rng, 1, 20000)
        gs = 128 if case < 3 else int(rng.choice([32, 64, 256]))
        p_hi, asym = int(rng.integers(1, 9)), bool(rng.random() < 0.4)
        sd = "f16" if rng.random() < 0.7 else "f32"
        m = make(P, rows, cols, gs, p_hi, asym, seed=seed * 10 + case)
        dm = P.DeviceModel.from_model(m, scale_dtype=sd)
        x = O.random_gaussian(1, cols, seed=seed * 10 + case).ravel().astype(np.float16)
        xd = torch.from_numpy(x).cuda()
        ps = sorted({int(v) for v in rng.integers(1, p_hi + 1, size=2)})
        wants = {p: want(m, sd, p, x) for p in ps}
        for mode in (0, 27, 23):  # automatic; cluster kernel for every size; never the cluster kernel
            L.abcq_debug_set_mode(0)
            L.abcq_debug_set_mode(mode)
            for p in ps:
                y = dm.gemv(p, xd).cpu().numpy()
                assert close(y, wants[p]), (rows, cols, gs, p, asym, sd, mode, O.rel_dev(y, wants[p][0]))


@pytest.mark.parametrize("seed", range(4))
def test_random_batches_every_schedule(P, L, seed):
    from paper_2510_10467_b200.device_model import gemv_batch
    rng = np.random.default_rng(2000 + seed)
    asym, sd = bool(seed & 1), ("f16", "f32")[seed >> 1 & 1]
    models = []
    for i in range(int(rng.integers(2, 6))):
        rows, cols = dim(rng, 1, 12000), dim(rng, 1, 12000)
        m = make(P, rows, cols, 128, int(rng.integers(1, 9)), asym, seed=seed * 10 + i)
        models.append((m, P.DeviceModel.from_model(m, scale_dtype=sd)))
    xs, jobs, wants = {}, [], []
    for j in range(int(rng.integers(8, 33))):
        m, dm = models[int(rng.integers(0, len(models)))]
        p = int(rng.integers(1, m.p_hi + 1))
        if dm.cols not in xs or rng.random() < 0.3:
            xs[dm.cols] = O.random_gaussian(1, dm.cols, seed=seed * 100 + j).ravel().astype(np.float16)
        x = xs[dm.cols]
        jobs.append((dm, p, torch.from_numpy(x).cuda(), torch.empty(dm.rows, device="cuda")))
        wants.append(want(m, sd, p, x))
    ref = None
    for mode in (0, 29, 32, 33, 22):  # schedules; separate completion kernel
        L.abcq_debug_set_mode(0)
        L.abcq_debug_set_mode(mode)
        for o in jobs:
            o[3].fill_(float("nan"))
        gemv_batch(jobs)
        torch.cuda.synchronize()
        outs = [o[3].clone() for o in jobs]
        for (dm, p, _, _), y, w in zip(jobs, outs, wants):
            assert close(y.cpu().numpy(), w), (dm.rows, dm.cols, p, mode)
        if ref is None:
            ref = outs
        else:
            assert all(torch.equal(u, v) for u, v in zip(ref, outs)), mode


@pytest.mark.parametrize("seed", range(3))
def test_random_gemm_mixedp(P, L, seed):
    rng = np.random.default_rng(3000 + seed)
    for case in range(2):
        rows, cols = dim(rng, 1, 12000), dim(rng, 1, 12000)
        p_hi, asym = int(rng.integers(1, 9)), bool(rng.random() < 0.4)
        sd = "f16" if rng.random() < 0.7 else "f32"
        m = make(P, rows, cols, 128, p_hi, asym, seed=seed * 10 + case)
        dm = P.DeviceModel.from_model(m, scale_dtype=sd)
        B = int(rng.integers(1, 17))
        ps = [int(v) for v in rng.integers(1, p_hi + 1, size=B)]
        X = np.stack([O.random_gaussian(1, cols, seed=seed * 100 + b).ravel() for b in range(B)]).astype(np.float16)
        wants = [want(m, sd, p, X[b]) for b, p in enumerate(ps)]
        for mode in (0, 40):  # mma.sync kernel; tcgen05 variant
            L.abcq_debug_set_mode(0)
            L.abcq_debug_set_mode(mode)
            Y = dm.gemm_mixedp(ps, torch.from_numpy(X).cuda()).cpu().numpy()
            for b, p in enumerate(ps):
                assert close(Y[b], wants[b], tol=1e-4, mtol=1e-5), (rows, cols, B, b, p, asym, sd, mode)


@pytest.mark.parametrize("seed", range(3))
def test_random_single_gemv_io_dtypes(P, L, seed):
    """f32 x and/or f16 y on random shapes: the table build from f32 x and the
    f16 output rounding (held to north_star's 1e-3)."""
    rng = np.random.default_rng(4000 + seed)
    for case in range(4):
        rows, cols = dim(rng, 1, 16000), dim(rng, 1, 16000)
        while rows * cols > 16 << 20:
            rows, cols = dim(rng, 1, 16000), dim(rng, 1, 16000)
        p_hi, asym = int(rng.integers(1, 9)), bool(rng.random() < 0.4)
        sd = "f16" if rng.random() < 0.7 else "f32"
        m = make(P, rows, cols, 128, p_hi, asym, seed=seed * 10 + case)
        dm = P.DeviceModel.from_model(m, scale_dtype=sd)
        x32 = O.random_gaussian(1, cols, seed=seed * 10 + case).ravel().astype(np.float32)
        p = int(rng.integers(1, p_hi + 1))
        w = want(m, sd, p, x32)
        for mode in (0, 27, 23):
            L.abcq_debug_set_mode(0)
            L.abcq_debug_set_mode(mode)
            y32 = dm.gemv(p, torch.from_numpy(x32).cuda()).cpu().numpy()
            assert close(y32, w), (rows, cols, p, asym, sd, mode, "f32 x")
            y16 = dm.gemv(p, torch.from_numpy(x32).cuda(), out_dtype=torch.float16).float().cpu().numpy()
            assert close(y16, w, tol=1e-3, mtol=1e-3), (rows, cols, p, asym, sd, mode, "f16 y")
