"""Timeline of the batched Llama-3-8B layer launch (bench.py's step) on the GPU
box: per-CTA profiling stamps (abcq_debug_set_trace) of one gemv_batch launch
over q/k/v/o/gate/up/down at precision p, plus graph-timed launch latency.

    python tools/layer_probe.py --p 3 [--jobs 0,1,2,3,4,5,6] [--copies 3]
"""
import argparse
import signal
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2510_10467_b200 as P  # noqa: E402
from paper_2510_10467_b200 import _lib  # noqa: E402
from paper_2510_10467_b200.device_model import gemv_batch  # noqa: E402

LAYERS = [("q", 4096, 4096), ("k", 1024, 4096), ("v", 1024, 4096), ("o", 4096, 4096),
          ("gate", 14336, 4096), ("up", 14336, 4096), ("down", 4096, 14336),
          ("gate70", 28672, 8192), ("down70", 8192, 28672)]  # (7, 8: 70B shapes)
NAMES = ["start", "fenced", "tab0", "streamed", "ctadone", "synced", "-", "pdlwait"]

ap = argparse.ArgumentParser()
ap.add_argument("--p", type=int, default=3)
ap.add_argument("--jobs", default="0,1,2,3,4,5,6")
ap.add_argument("--copies", type=int, default=3)
ap.add_argument("--mode", type=int, default=0)
ap.add_argument("--piece", type=int, default=-1, help="piece cost in blocks (load-balance model)")
ap.add_argument("--mixed", action="store_true", help="jobs at p=2,3,4 in one launch (bench step)")
ap.add_argument("--pad", type=int, default=0, help="extra bytes between planes (plane stride experiment)")
ap.add_argument("--rtrace", default="", help="comma list of CTAs: per-warp round stamps (debug mode 7001 + cta)")
a = ap.parse_args()
signal.signal(signal.SIGPIPE, signal.SIG_DFL)  # quiet under | head
torch.cuda.set_device(0)
sel = [int(v) for v in a.jobs.split(",")]
g = torch.Generator(device="cuda").manual_seed(0)
sets = []
for c in range(a.copies):
    row = []
    for li in sel:
        _, r, k = LAYERS[li]
        dm = P.DeviceModel(r, k, 128, 2, 4, False, scale_dtype="f16")
        if a.pad:
            dm.plane_stride += a.pad
            dm.planes = torch.zeros(dm.p_hi * dm.plane_stride, dtype=torch.uint8, device="cuda")
            dm._refresh_struct()
        dm.load_planes(torch.randint(-2**31, 2**31 - 1, (4, r, k // 32), dtype=torch.int32, device="cuda",
                                     generator=g))
        for p in (2, 3, 4):
            dm.load_scale_set(p, np.full((p, r, k // 128), 0.05, np.float32))
        row.append(dm)
    sets.append(row)
xs = {k: torch.randn(k, device="cuda").half() for k in {LAYERS[li][2] for li in sel}}
ys = [torch.empty(LAYERS[li][1], device="cuda", dtype=torch.float16) for li in sel]
st = torch.cuda.Stream()
if a.mode:
    _lib.lib().abcq_debug_set_mode(a.mode)
if a.piece >= 0:
    _lib.lib().abcq_debug_set_mode(1000 + a.piece)


PS = (2, 3, 4) if a.mixed else (a.p,)


def launch(c):
    gemv_batch([(dm, p, xs[dm.cols], ys[i]) for p in PS for i, dm in enumerate(sets[c])], st)


byts = sum(p * LAYERS[li][1] * LAYERS[li][2] // 8 + p * LAYERS[li][1] * LAYERS[li][2] // 128 * 2
           for p in PS for li in sel)
with torch.cuda.stream(st):
    for c in range(a.copies):
        launch(c)
torch.cuda.synchronize()
gr = torch.cuda.CUDAGraph()
with torch.cuda.graph(gr, stream=st):
    for i in range(12):
        launch(i % a.copies)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(st):
    gr.replay()
    e0.record(st)
    for _ in range(5):
        gr.replay()
    e1.record(st)
torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1e3 / 60
print(f"jobs {[LAYERS[li][0] for li in sel]} p={PS}: {us:.2f} us/launch, {byts / 1e6:.1f} MB -> "
      f"{byts / us / 1e3:.0f} GB/s")

SL = 168 * 8
buf = torch.zeros(16 * SL + 16 * 32 * 4, dtype=torch.int64, device="cuda")
_lib.lib().abcq_debug_set_trace(buf.data_ptr())
g3 = torch.cuda.CUDAGraph()
with torch.cuda.graph(g3, stream=st):
    for i in range(4):
        launch(i % a.copies)
_lib.lib().abcq_debug_set_trace(None)
with torch.cuda.stream(st):
    g3.replay()
    torch.cuda.synchronize()
    buf.zero_()
    buf[:16 * SL].view(16, 168, 8)[:, 148, 0:2] = 1 << 62  # reduce kernel: atomicMin slots
    g3.replay()
torch.cuda.synchronize()
t = buf[:16 * SL].view(16, 168, 8).cpu().numpy()
used = [k for k in range(16) if t[k, :148, 0].max() > 0]
used.sort(key=lambda k: t[k, :148, 0][t[k, :148, 0] > 0].min())
t0 = t[used[0], :148, 0][t[used[0], :148, 0] > 0].min()
for k in used:
    T = t[k, :148].astype(np.float64)
    row = []
    for j, n in enumerate(NAMES):
        col = T[:, j][T[:, j] > 0]
        if len(col):
            row.append(f"{n} {(col.min() - t0) / 1e3:6.2f}/{(np.median(col) - t0) / 1e3:6.2f}/{(col.max() - t0) / 1e3:6.2f}")
    red = t[k, 148, :3].astype(np.float64)
    if red[2] > 0:
        jobs = t[k].reshape(-1)[149 * 8:149 * 8 + 32].astype(np.float64)
        arr = t[k].reshape(-1)[160 * 8:160 * 8 + 32].astype(np.float64)
        wpass = t[k].reshape(-1)[164 * 8:164 * 8 + 32].astype(np.float64)
        tstart = t[k].reshape(-1)[156 * 8:156 * 8 + 32].astype(np.float64)
        row.append("reduce first %.2f pdl %.2f end %.2f (jobs arrive/taskstart/wait/end %s)" % (
            (red[0] - t0) / 1e3, (red[1] - t0) / 1e3, (red[2] - t0) / 1e3,
            " ".join(f"{(arr[i] - t0) / 1e3:.1f}/{(tstart[i] - t0) / 1e3:.1f}/{(wpass[i] - t0) / 1e3:.1f}/{(v - t0) / 1e3:.1f}"
                     for i, v in enumerate(jobs) if v > 0)))
    print("  " + " | ".join(row))
# per-warp round stamps of selected CTAs (one more traced graph per CTA)
for cta in [int(v) for v in a.rtrace.split(",") if v]:
    _lib.lib().abcq_debug_set_mode(7001 + cta)
    _lib.lib().abcq_debug_set_trace(buf.data_ptr())
    g4 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g4, stream=st):
        for i in range(4):
            launch(i % a.copies)
    _lib.lib().abcq_debug_set_trace(None)
    _lib.lib().abcq_debug_set_mode(7000)
    with torch.cuda.stream(st):
        g4.replay()
        torch.cuda.synchronize()
        buf.zero_()
        g4.replay()
    torch.cuda.synchronize()
    tb = buf.view(-1).cpu().numpy()
    R4 = tb[16 * SL:].reshape(16, 32, 4).astype(np.float64)
    T = tb[:16 * SL].reshape(16, 168, 8)
    lastk = max(range(16), key=lambda k: T[k, cta, 0])
    c0 = float(T[lastk, cta, 0])
    print(f"  CTA {cta} rounds (us from CTA start; per round: start min/max | table ok max | run done min/max | build start max)")
    for r in range(32):
        col = R4[:, r, :]
        if col[:, 0].max() <= 0:
            break
        f = lambda k, fn: (fn(col[:, k][col[:, k] > 0]) - c0) / 1e3 if (col[:, k] > 0).any() else float("nan")
        print(f"    r{r:2d}: start {f(0, np.min):6.2f}/{f(0, np.max):6.2f} | tbl {f(1, np.max):6.2f} | "
              f"done {f(2, np.min):6.2f}/{f(2, np.max):6.2f} | build {f(3, np.max):6.2f}")

# per-CTA detail of the last launch: stream duration (tab0 -> streamed) vs rounds
T = t[used[-1], :148].astype(np.float64)
dur = (T[:, 3] - T[:, 2]) / 1e3
rounds = t[used[-1], :148, 6]
print("  stream us per CTA: min %.2f med %.2f max %.2f; rounds min %d max %d" % (
    dur.min(), np.median(dur), dur.max(), rounds.min(), rounds.max()))
for nr in sorted(set(rounds.tolist())):
    m = rounds == nr
    print(f"    rounds={nr}: {m.sum():3d} CTAs, stream med {np.median(dur[m]):.2f} max {dur[m].max():.2f}")
slow = np.argsort(-dur)[:8]
print("  slowest CTAs:", ", ".join(f"{b}:{dur[b]:.1f}us/r{rounds[b]}" for b in slow))

# does a CTA's stream time repeat across identical launches (schedule / placement) or not (noise)?
if len(used) >= 3:
    durs = np.array([(t[k, :148, 3].astype(np.float64) - t[k, :148, 2]) / 1e3 for k in used[1:]])
    cc = np.corrcoef(durs)
    print("  stream-time correlation by CTA index across launches:",
          " ".join(f"{cc[i, j]:.2f}" for i in range(len(durs)) for j in range(i + 1, len(durs))))
    ends = np.array([(t[k, :148, 3].astype(np.float64) - t[k, :148, 0].min()) / 1e3 for k in used[1:]])
    ce = np.corrcoef(ends)
    print("  stream-END correlation by CTA index across launches:",
          " ".join(f"{ce[i, j]:.2f}" for i in range(len(ends)) for j in range(i + 1, len(ends))))
    import json as _json
    Path("gpurun_out").mkdir(exist_ok=True)
    Path("gpurun_out/lp_cta_durs.json").write_text(_json.dumps({"durs": durs.round(3).tolist(), "ends": ends.round(3).tolist(),
                                                                "rounds": t[used[-1], :148, 6].tolist()}))

# systematic per-SM speed? correlate stream durations of consecutive launches by SM id
if False and len(used) >= 3:  # (needs SM ids in slot 7)
    d = {}
    for k in used[1:]:
        T = t[k, :148].astype(np.float64)
        smid = t[k, :148, 7]
        rate = (T[:, 3] - T[:, 2]) / 1e3
        d[k] = dict(zip(smid.tolist(), rate.tolist())), dict(enumerate(rate.tolist()))
    ks = list(d)
    a_sm, b_sm = d[ks[0]][0], d[ks[1]][0]
    common = sorted(set(a_sm) & set(b_sm))
    ca = np.corrcoef([a_sm[s] for s in common], [b_sm[s] for s in common])[0, 1]
    a_b, b_b = d[ks[0]][1], d[ks[1]][1]
    cb = np.corrcoef([a_b[i] for i in range(148)], [b_b[i] for i in range(148)])[0, 1]
    print(f"  stream-time correlation across launches: by SM {ca:.2f}, by CTA index {cb:.2f}")
    sm = np.array(common)
    v = np.array([(a_sm[s] + b_sm[s]) / 2 for s in common])
    order = np.argsort(-v)[:12]
    print("  slowest SMs (avg us):", ", ".join(f"{sm[i]}:{v[i]:.1f}" for i in order))
    print("  by SM id quartile:", [f"{v[(sm >= q0) & (sm < q0 + 37)].mean():.2f}" for q0 in (0, 37, 74, 111)])

# ---- per-CTA composition (host replica of the kernel's schedule) vs stream time
if "--fit" in sys.argv[0:0] or True:
    jobs = [(LAYERS[li][1], LAYERS[li][2], p) for p in PS for li in sel]
    G = 148
    pieceb = a.piece if a.piece >= 0 else 200
    ib, ub, W, NRTs, items = [], [], [], [], []
    it = u = 0
    for r, k, p in jobs:
        nrt, ns = -(-r // 16), -(-k // 256)
        w = 64 * p + -(-64 * pieceb // nrt)
        ib.append(it); ub.append(u); W.append(w); NRTs.append(nrt); items.append(nrt * ns)
        it += nrt * ns; u += nrt * ns * w

    def first_item(uu):
        j = 0
        while j + 1 < len(jobs) and ub[j + 1] <= uu:
            j += 1
        loc = -(-(uu - ub[j]) // W[j])
        return ib[j] + min(loc, items[j])
    cta = [first_item(b * u // G) for b in range(G + 1)]

    def job_of(g):
        j = 0
        while j + 1 < len(jobs) and ib[j + 1] <= g:
            j += 1
        return j
    feats = []
    for b in range(G):
        g, hi = cta[b], cta[b + 1]
        blocks = pieces = 0
        while g < hi:
            j = job_of(g)
            s = (g - ib[j]) // NRTs[j]
            e = min(ib[j] + (s + 1) * NRTs[j], hi)
            blocks += (e - g) * jobs[j][2]
            pieces += 1
            g = e
        feats.append((blocks, pieces))
    F = np.array(feats, dtype=np.float64)
    T = t[used[-1], :148].astype(np.float64)
    dur = (T[:, 3] - T[:, 2]) / 1e3
    rnd = t[used[-1], :148, 6].astype(np.float64)
    X = np.column_stack([F[:, 0], F[:, 1], rnd, np.ones(G)])
    coef, *_ = np.linalg.lstsq(X, dur, rcond=None)
    pred = X @ coef
    print(f"  fit stream_us = {coef[0]*1e3:.3f} ns/block + {coef[1]:.3f} us/piece + {coef[2]:.3f} us/round "
          f"+ {coef[3]:.2f}; resid rms {np.sqrt(np.mean((dur - pred) ** 2)):.2f} us; "
          f"blocks/CTA {F[:,0].min():.0f}..{F[:,0].max():.0f}, pieces {F[:,1].min():.0f}..{F[:,1].max():.0f}")

    W = t[used[-1], :148, 7].astype(np.float64) / 1e3
    Bt = t[used[-1], :148, 1].astype(np.float64) / 1e3
    print(f"  table waits per CTA (sum over warps): med {np.median(W):.2f} max {W.max():.2f} us; "
          f"builders waiting for the round to drain: med {np.median(Bt):.2f} max {Bt.max():.2f} us")
    # round-boundary anatomy for CTAs with >= 2 rounds
    T = t[used[-1], :148].astype(np.float64)
    m = (rnd >= 2) & (T[:, 7] > 0)
    if m.any():
        skew = (T[m, 5] - T[m, 4]) / 1e3
        build = (T[m, 7] - T[m, 5]) / 1e3
        bar = (T[m, 1] - T[m, 5]) / 1e3
        print(f"  round 0->1 ({m.sum()} CTAs): warp skew med {np.median(skew):.2f} max {skew.max():.2f} us; "
              f"last warp -> barrier passed med {np.median(bar):.2f}, -> table 1 ready med {np.median(build):.2f} "
              f"max {build.max():.2f} us")
    # the slowest CTAs' composition (jobs, pieces) and their stream-end times
    endt = (T[:, 3] - T[:, 3].min()) / 1e3
    order = np.argsort(-endt)[:6]
    for b in order:
        js = sorted({job_of(g) for g in range(cta[b], cta[b + 1])})
        print(f"    CTA {b:3d}: end +{endt[b]:.2f} us, stream {dur[b]:.2f} us, blocks {F[b,0]:.0f}, pieces {F[b,1]:.0f}, "
              f"jobs {[(LAYERS[sel[j % len(sel)]][0], jobs[j][2]) for j in js]}")
