"""Replica of the batch kernel's host partition (abcq_gemv_lut.cu, g_partition 0)
and a least-squares fit of the measured per-CTA stream time
(gpurun_out/lp_cta_durs.json from tools/layer_probe.py --mixed) on the
per-CTA work features -- to calibrate the schedule's cost model.
    python tools/sched_fit.py [--piece 150] [--json gpurun_out/lp_cta_durs.json]"""
import argparse
import json

import numpy as np

LAYERS = [("q", 4096, 4096), ("k", 1024, 4096), ("v", 1024, 4096), ("o", 4096, 4096),
          ("gate", 14336, 4096), ("up", 14336, 4096), ("down", 4096, 14336)]


def jobs_of(ps=(2, 3, 4)):
    return [(n, r, c, p) for p in ps for n, r, c in LAYERS]


def partition(jobs, grid=148, piece=150, per_item=None, per_piece=None):
    """CTA ranges of the greedy fill; per_item(j) / per_piece(j) override the cost
    (defaults = the library's: p*64 per item, piece*64 per piece)."""
    per_item = per_item or (lambda j: jobs[j][3] * 64)
    per_piece = per_piece or (lambda j: piece * 64)
    NRT = [-(-r // 16) for _, r, _, _ in jobs]
    NS = [-(-c // 256) for _, _, c, _ in jobs]
    items_j = [a * b for a, b in zip(NRT, NS)]
    ibase = np.concatenate([[0], np.cumsum(items_j)]).astype(int)
    items = int(ibase[-1])

    def fill(T, write):
        j = g = 0
        cta = []
        for b in range(grid):
            cta.append(g)
            cost = 0
            while g < items:
                while g >= ibase[j + 1]:
                    j += 1
                loc = g - ibase[j]
                s = loc // NRT[j]
                pend = ibase[j] + (s + 1) * NRT[j]
                start, per = per_piece(j), per_item(j)
                if cost > 0 and cost + start + per > T:
                    break
                cost += start
                take = max(1, (T - cost) // per)
                take = min(take, pend - g)
                cost += take * per
                g += take
                if cost >= T:
                    break
        cta.append(g)
        return g >= items, cta

    lo, hi = 1, 1 << 40
    while lo < hi:
        mid = (lo + hi) // 2
        if fill(mid, False)[0]:
            hi = mid
        else:
            lo = mid + 1
    cta = fill(lo, True)[1]
    cta[-1] = items
    return cta, ibase, NRT


def features(jobs, cta, ibase, NRT):
    F = []
    for b in range(len(cta) - 1):
        g, hi = cta[b], cta[b + 1]
        f = dict(blocks=0, items=0, pieces=0, byp={2: 0, 3: 0, 4: 0}, tiles_small=0)
        while g < hi:
            j = int(np.searchsorted(ibase, g, side="right") - 1)
            s = (g - ibase[j]) // NRT[j]
            e = min(ibase[j] + (s + 1) * NRT[j], hi)
            p = jobs[j][3]
            f["blocks"] += (e - g) * p
            f["items"] += e - g
            f["pieces"] += 1
            f["byp"][p] += e - g
            g = e
        F.append(f)
    return F


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--piece", type=int, default=150)
    ap.add_argument("--json", default="gpurun_out/lp_cta_durs.json")
    a = ap.parse_args()
    jobs = jobs_of()
    cta, ibase, NRT = partition(jobs, piece=a.piece)
    F = features(jobs, cta, ibase, NRT)
    d = json.load(open(a.json))
    dur = np.array(d["durs"]).mean(0)
    keep = np.arange(147)  # CTA 147 = remainder
    X = np.array([[f["byp"][2], f["byp"][3], f["byp"][4], f["pieces"], 1.0] for f in F])[keep]
    y = dur[keep]
    coef, *_ = np.linalg.lstsq(X, y, rcond=None)
    res = y - X @ coef
    print("fit us = %.4f*items_p2 + %.4f*items_p3 + %.4f*items_p4 + %.3f*pieces + %.2f ; resid rms %.2f (raw std %.2f)"
          % (*coef, res.std(), y.std()))
    print("per-item us: p2 %.4f p3 %.4f p4 %.4f -> per block %.4f %.4f %.4f; piece = %.0f p2-blocks"
          % (coef[0], coef[1], coef[2], coef[0] / 2, coef[1] / 3, coef[2] / 4, coef[3] / (coef[0] / 2)))
    X2 = np.array([[f["blocks"], f["items"], f["pieces"], 1.0] for f in F])[keep]
    c2, *_ = np.linalg.lstsq(X2, y, rcond=None)
    r2 = y - X2 @ c2
    print("fit us = %.5f*blocks + %.5f*items + %.3f*pieces + %.2f ; resid rms %.2f" % (*c2, r2.std()))
    print("  => item = %.2f blocks, piece = %.0f blocks" % (c2[1] / c2[0], c2[2] / c2[0]))
    worst = np.argsort(-np.abs(r2))[:8]
    for b in worst:
        print("   CTA %3d: dur %.1f pred %.1f  items %d blocks %d pieces %d" % (
            b, y[b], (X2 @ c2)[b], F[b]["items"], F[b]["blocks"], F[b]["pieces"]))


def piece_list(jobs, cta, ibase, NRT, b):
    g, hi = cta[b], cta[b + 1]
    out = []
    while g < hi:
        j = int(np.searchsorted(ibase, g, side="right") - 1)
        s = (g - ibase[j]) // NRT[j]
        e = min(ibase[j] + (s + 1) * NRT[j], hi)
        out.append((j, e - g, jobs[j][3]))
        g = e
    return out


def explore(jobs, cta, ibase, NRT, y):
    PL = [piece_list(jobs, cta, ibase, NRT, b) for b in range(147)]
    for K in (16, 32, 48, 64, 96, 128):
        X = np.array([[sum(n * p for _, n, p in pl), len(pl), sum(max(0, K - n) for _, n, _ in pl), 1.0] for pl in PL])
        c, *_ = np.linalg.lstsq(X, y, rcond=None)
        print(f"K={K}: blocks {c[0]:.5f} piece {c[1]:.3f} short {c[2]:.4f} const {c[3]:.2f} resid {np.std(y - X @ c):.2f}")
    # per-job-type items
    names = sorted({n for n, *_ in jobs})
    X = np.array([[sum(n * p for j, n, p in pl if jobs[j][0] == nm) for nm in names] + [len(pl), 1.0] for pl in PL])
    c, *_ = np.linalg.lstsq(X, y, rcond=None)
    print("per-layer block cost (us/1000 blocks):", {nm: round(v * 1000, 2) for nm, v in zip(names, c)},
          "piece %.3f const %.2f resid %.2f" % (c[-2], c[-1], np.std(y - X @ c)))


if __name__ == "__main__":
    explore(jobs, cta, ibase, NRT, y)


def explore2(jobs, cta, ibase, NRT, y):
    PL = [piece_list(jobs, cta, ibase, NRT, b) for b in range(147)]
    rows = {j: jobs[j][1] for j in range(len(jobs))}
    def fit(cols, names):
        X = np.array(cols).T
        c, *_ = np.linalg.lstsq(X, y, rcond=None)
        print(" ", " ".join(f"{n}={v:.5f}" for n, v in zip(names, c)), f"resid {np.std(y - X @ c):.2f} max {np.abs(y - X @ c).max():.2f}")
        return c
    blocks = [sum(n * p for _, n, p in pl) for pl in PL]
    items = [sum(n for _, n, _ in pl) for pl in PL]
    pieces = [len(pl) for pl in PL]
    big = [sum(n * p for j, n, p in pl if rows[j] > 8192) for pl in PL]
    small = [sum(n * p for j, n, p in pl if rows[j] < 2048) for pl in PL]
    fit([blocks, items, pieces], ["blk", "item", "piece"])
    fit([blocks, pieces], ["blk", "piece"])
    fit([blocks, big, small, pieces], ["blk", "blk_bigrows", "blk_smallrows", "piece"])
    fit([blocks, big, small, pieces, [1.0] * len(y)], ["blk", "blk_bigrows", "blk_smallrows", "piece", "const"])


if __name__ == "__main__":
    explore2(jobs, cta, ibase, NRT, y)


def explore3(jobs, cta, ibase, NRT, y):
    PL = [piece_list(jobs, cta, ibase, NRT, b) for b in range(147)]
    def fit(cols, names):
        X = np.array(cols, dtype=float).T
        c, *_ = np.linalg.lstsq(X, y, rcond=None)
        print(" ", " ".join(f"{n}={v:.5f}" for n, v in zip(names, c)), f"resid {np.std(y - X @ c):.2f} max {np.abs(y - X @ c).max():.2f}")
    bp = [[sum(n * p for _, n, p in pl if p == q) for pl in PL] for q in (2, 3, 4)]
    pieces = [len(pl) for pl in PL]
    fit(bp + [pieces], ["b2", "b3", "b4", "piece"])
    # piece cost by job rows class
    cls = lambda j: 0 if jobs[j][1] < 2048 else (2 if jobs[j][1] > 8192 else 1)
    pc = [[sum(1 for j, n, p in pl if cls(j) == k) for pl in PL] for k in range(3)]
    blocks = [sum(n * p for _, n, p in pl) for pl in PL]
    fit([blocks] + pc, ["blk", "piece_small", "piece_mid", "piece_big"])
    fit(bp + pc, ["b2", "b3", "b4", "piece_small", "piece_mid", "piece_big"])


if __name__ == "__main__":
    explore3(jobs, cta, ibase, NRT, y)
