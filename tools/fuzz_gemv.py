"""Randomised parity sweep of the GEMV entry points vs the C oracle (a GPU
tool, not part of the suite): random shapes (1..32768 rows/cols, log-uniform,
ragged), group sizes (128 tiled; 32/64/256 row-major), precisions, symmetric /
asymmetric, f16 / f32 scales, single calls under the dispatch modes (automatic,
27 = cluster kernel for every single GEMV, 28 = cluster kernel for any size
<= 32 slices) random gemv_batch job lists (schedule modes 0/29/32/33) and gemm_mixedp
calls (automatic / tcgen05 mode 40).
Every output vs the C oracle at 1e-5 relative deviation (few-row outputs:
each element within 1e-6 of its magnitude sum, see ok()), batch outputs also
bitwise equal across schedule modes.
    python tools/fuzz_gemv.py --seconds 300 --seed 1 > gpurun_out/fuzz.json"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2510_10467_b200 as P  # noqa: E402
from paper_2510_10467_b200 import _lib  # noqa: E402
from paper_2510_10467_b200.device_model import gemv_batch  # noqa: E402
from oracle import anybcq_oracle as O, c_oracle  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--seconds", type=float, default=300)
ap.add_argument("--seed", type=int, default=1)
a = ap.parse_args()
rng = np.random.default_rng(a.seed)
L = _lib.lib()
TOL = 1e-5
T = c_oracle.cpu_threads()


def dim(lo, hi):
    return int(np.exp(rng.uniform(np.log(lo), np.log(hi))))


def make(rows, cols, gs, p_hi, asym, seed):
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


def want(m, sd, asym, p, x):
    st = m.scale_sets[p]
    q = (lambda v: v.astype(np.float16).astype(np.float32)) if sd == "f16" else (lambda v: v)
    z = q(st.offset) if asym else None
    w = c_oracle.lut_gemv(m.bitplanes.words, m.bitplanes.cols, m.config.group_size, q(st.alpha), z, p,
                          x.astype(np.float32), threads=T)
    # per-row magnitude sum_k sum_g |alpha| sum_{c in g} |x_c| (+ |z| ...): the
    # scale of f32 rounding for a row whose dot product cancels
    gs = m.config.group_size
    xa = np.abs(x.astype(np.float64))
    X = np.add.reduceat(xa, np.arange(0, xa.size, gs))
    mag = np.abs(q(st.alpha)[:p]).astype(np.float64).sum(0) @ X
    if z is not None:
        mag += np.abs(z).astype(np.float64) @ X
    return w, mag


def ok(y, wm, tol=TOL, mtol=1e-6):
    """1e-5 relative deviation, or -- for the few-row outputs where one
    cancelling dot product dominates the norm -- every element within 1e-6
    of its magnitude sum (f32 accumulation over <= 32768 terms)."""
    w, mag = wm
    d = O.rel_dev(y, w)
    return d <= tol or bool(np.all(np.abs(y - w) <= mtol * np.maximum(mag, 1e-30))), float(d)


fails, n_single, n_batch, n_jobs, n_gemm = [], 0, 0, 0, 0
t0 = time.time()
case = 0
while time.time() - t0 < a.seconds:
    case += 1
    u = rng.random()
    kind = "batch" if u < 0.35 else "gemm" if u < 0.5 else "single"
    if kind == "gemm":
        # gemm_mixedp (B <= 16 requests, mixed precisions, one pass over the
        # planes): automatic kernel and the tcgen05 variant (mode 40); the
        # suite's bound for it is 1e-4
        rows, cols = dim(1, 16384), dim(1, 16384)
        p_hi, asym = int(rng.integers(1, 9)), bool(rng.random() < 0.4)
        sd = "f16" if rng.random() < 0.7 else "f32"
        m = make(rows, cols, 128, p_hi, asym, seed=case)
        dm = P.DeviceModel.from_model(m, scale_dtype=sd)
        B = int(rng.integers(1, 17))
        ps = [int(v) for v in rng.integers(1, p_hi + 1, size=B)]
        X = np.stack([O.random_gaussian(1, cols, seed=case * 100 + b).ravel() for b in range(B)]).astype(np.float16)
        wants = {}
        for mode in (0, 40):
            L.abcq_debug_set_mode(0)
            L.abcq_debug_set_mode(mode)
            Y = dm.gemm_mixedp(ps, torch.from_numpy(X).cuda()).cpu().numpy()
            for b, p in enumerate(ps):
                if (b, p) not in wants:
                    wants[(b, p)] = want(m, sd, asym, p, X[b])
                good, d = ok(Y[b], wants[(b, p)], tol=1e-4, mtol=1e-5)
                if not good:
                    fails.append(dict(kind=kind, rows=rows, cols=cols, B=B, b=b, p=p, asym=asym, sd=sd, mode=mode,
                                      dev=d))
        L.abcq_debug_set_mode(0)
        n_gemm += 1
    elif kind == "single":
        rows, cols = dim(1, 32768), dim(1, 32768)
        while rows * cols > 64 << 20:          # keep the oracle at seconds per case
            rows, cols = dim(1, 32768), dim(1, 32768)
        gs = 128 if rng.random() < 0.75 else int(rng.choice([32, 64, 256]))
        p_hi, asym = int(rng.integers(1, 9)), bool(rng.random() < 0.4)
        sd = "f16" if rng.random() < 0.7 else "f32"
        m = make(rows, cols, gs, p_hi, asym, seed=case)
        dm = P.DeviceModel.from_model(m, scale_dtype=sd)
        x = O.random_gaussian(1, cols, seed=case).ravel().astype(np.float16)
        xd = torch.from_numpy(x).cuda()
        for mode in (0, 27, 28):
            L.abcq_debug_set_mode(0)
            L.abcq_debug_set_mode(mode)
            for p in sorted(set(int(v) for v in rng.integers(1, p_hi + 1, size=2))):
                y = dm.gemv(p, xd).cpu().numpy()
                good, d = ok(y, want(m, sd, asym, p, x))
                n_single += 1
                if not good:
                    fails.append(dict(kind=kind, rows=rows, cols=cols, gs=gs, p=p, asym=asym, sd=sd, mode=mode,
                                      dev=float(d)))
        L.abcq_debug_set_mode(0)
    else:
        nm = int(rng.integers(1, 7))
        asym = bool(rng.random() < 0.4)
        sd = "f16" if rng.random() < 0.7 else "f32"
        models = []
        for i in range(nm):
            rows, cols = dim(1, 16384), dim(1, 16384)
            p_hi = int(rng.integers(1, 9))
            m = make(rows, cols, 128, p_hi, asym, seed=case * 10 + i)
            models.append((m, P.DeviceModel.from_model(m, scale_dtype=sd)))
        nj = int(rng.integers(1, 33))
        xs, jobs, wants = {}, [], []
        for j in range(nj):
            m, dm = models[int(rng.integers(0, nm))]
            p = int(rng.integers(1, m.p_hi + 1))
            if dm.cols not in xs or rng.random() < 0.3:
                xs[dm.cols] = O.random_gaussian(1, dm.cols, seed=case * 100 + j).ravel().astype(np.float16)
            x = xs[dm.cols]
            jobs.append((dm, p, torch.from_numpy(x).cuda(), torch.empty(dm.rows, device="cuda")))
            wants.append(want(m, sd, asym, p, x))
        ref = None
        for mode in (0, 29, 32, 33):
            L.abcq_debug_set_mode(0)
            L.abcq_debug_set_mode(mode)
            for o in jobs:
                o[3].fill_(float("nan"))
            gemv_batch(jobs)
            torch.cuda.synchronize()
            outs = [o[3].clone() for o in jobs]
            for (dm, p, _, _), y, w in zip(jobs, outs, wants):
                good, d = ok(y.cpu().numpy(), w)
                if not good:
                    fails.append(dict(kind=kind, rows=dm.rows, cols=dm.cols, p=p, asym=asym, sd=sd, mode=mode,
                                      jobs=nj, dev=float(d)))
            if ref is None:
                ref = outs
            elif not all(torch.equal(u, v) for u, v in zip(ref, outs)):
                fails.append(dict(kind="batch-bitwise", mode=mode, jobs=nj, shapes=[(j[0].rows, j[0].cols) for j in jobs]))
        L.abcq_debug_set_mode(0)
        n_batch += 1
        n_jobs += nj
    if len(fails) > 20:
        break
print(json.dumps(dict(seed=a.seed, cases=case, single_calls=n_single, batches=n_batch, batch_jobs=n_jobs, gemm_calls=n_gemm,
                      seconds=round(time.time() - t0, 1), failures=fails)))
sys.exit(1 if fails else 0)
