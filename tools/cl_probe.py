"""Cluster single-GEMV kernel probe: agreement with the batch kernel and
back-to-back launch timing (CUDA graph, rotating weight copies > 2x L2), with
optional geometry sweeps.

    python tools/cl_probe.py [--sweep] [--out gpurun_out/cl_probe.json]
"""
import argparse
import ctypes as C
import json
import math
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2510_10467_b200 as P  # noqa: E402
from paper_2510_10467_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--sweep", action="store_true")
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--shapes", default="")
ap.add_argument("--out", default="gpurun_out/cl_probe.json")
a = ap.parse_args()
torch.cuda.set_device(0)
L = _lib.lib()

SHAPES = [(4096, 4096), (1024, 4096), (14336, 4096), (4096, 14336), (6144, 4096), (28672, 4096),
          (8192, 8192), (1024, 8192), (28672, 8192), (8192, 28672)]
if a.shapes:
    SHAPES = [tuple(int(v) for v in s.split("x")) for s in a.shapes.split(",")]


def make(rows, cols, seed, sd="f16", asym=False):
    g = torch.Generator(device="cuda").manual_seed(seed)
    dm = P.DeviceModel(rows, cols, 128, 2, 4, asym, scale_dtype=sd)
    w = torch.randint(-2**31, 2**31 - 1, (4, rows, cols // 32), dtype=torch.int32, device="cuda", generator=g)
    dm.load_planes(w)
    G = cols // 128
    for p in (2, 3, 4):
        al = torch.rand((p, rows, G), device="cuda", generator=g) * 0.1 + 0.01
        off = (torch.randn((rows, G), device="cuda", generator=g) * 0.1) if asym else None
        dm.load_scale_set(p, al, off)
    return dm


def geom(dm, p):
    o = (C.c_int32 * 7)()
    rc = L.abcq_debug_gemv_geometry(dm.struct_ptr(), p, o)
    return list(o) if rc == 0 else None


def rel(a_, b_):
    a_, b_ = a_.double(), b_.double()
    return float((a_ - b_).norm() / max(b_.norm(), 1e-30))


_SPIN = None


def spin_clocks(st, ms=30):
    """keep the GPU busy ~ms so the SM clock is at its boost level before a timed region"""
    global _SPIN
    if _SPIN is None:
        _SPIN = torch.randn(4096, 4096, device="cuda", dtype=torch.float16)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    n = 0
    while True:
        for _ in range(8):
            torch.mm(_SPIN, _SPIN)
        n += 8
        e1.record(st)
        e1.synchronize()
        if e0.elapsed_time(e1) > ms:
            break


def sm_clock():
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(0)
        return pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
    except Exception:  # noqa: BLE001
        return None


def time_graph(models, p, x, y, iters):
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for m in models:
            m.gemv(p, x, out=y, stream=st)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for i in range(iters):
            models[i % len(models)].gemv(p, x, out=y, stream=st)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        spin_clocks(st)
        g.replay()
        g.replay()
        e0.record(st)
        for _ in range(5):
            g.replay()
        e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / (5 * iters)


out = {"shapes": {}}
for (rows, cols) in ([] if (__import__('os').environ.get('CL_TIMELINE') or __import__('os').environ.get('CL_ABL')) else SHAPES):
    G = cols // 128
    base = make(rows, cols, 1)
    per_copy = 4 * rows * cols // 8
    ncopy = max(3, min(48, math.ceil(300e6 / per_copy)))
    models = [base] + [make(rows, cols, 100 + c) for c in range(ncopy - 1)]
    x = torch.randn(cols, device="cuda").half()
    y = torch.empty(rows, device="cuda", dtype=torch.float16)
    rec = {"copies": ncopy}
    for p in (2, 3, 4):
        L.abcq_debug_set_mode(0)
        L.abcq_debug_set_mode(5000)
        y_new = base.gemv(p, x, out_dtype=torch.float32)
        y_new2 = base.gemv(p, x, out_dtype=torch.float32)
        L.abcq_debug_set_mode(23)
        y_old = base.gemv(p, x, out_dtype=torch.float32)
        L.abcq_debug_set_mode(0)
        torch.cuda.synchronize()
        byts = p * rows * cols // 8 + p * rows * G * 2 + 2 * (rows + cols)
        t_new = time_graph(models, p, x, y, a.iters)
        L.abcq_debug_set_mode(23)
        t_old = time_graph(models, p, x, y, a.iters)
        L.abcq_debug_set_mode(0)
        L.abcq_debug_set_mode(6008)
        t_w8 = time_graph(models, p, x, y, a.iters)
        L.abcq_debug_set_mode(6000)
        r = {"geom": geom(base, p), "rel_vs_batch_kernel": rel(y_new, y_old), "us_w8": round(t_w8, 3),
             "deterministic": bool(torch.equal(y_new, y_new2)),
             "us": round(t_new, 3), "GBps": round(byts / t_new / 1e3, 1),
             "frac": round(byts / t_new / 1e3 / 6553.3, 4),
             "us_batch_kernel": round(t_old, 3)}
        if a.sweep:
            sw = {}
            L.abcq_debug_set_mode(27)
            for slots, warps in ((1, 6016), (1, 6008)):
                L.abcq_debug_set_mode(warps)
                for Cc in (4, 8, 6):
                    for tcw in (1, 2):
                        L.abcq_debug_set_mode(5000 + 100 * slots + 10 * Cc + tcw)
                        gm = geom(base, p)
                        if gm is None:
                            continue
                        try:
                            yy = base.gemv(p, x, out_dtype=torch.float32)
                            torch.cuda.synchronize()
                            ok = rel(yy, y_old)
                            t = time_graph(models, p, x, y, a.iters)
                            sw[f"s{slots}C{Cc}t{tcw}w{warps - 6000}"] = [round(t, 3), f"{ok:.1e}", gm]
                        except Exception as e:  # noqa: BLE001
                            sw[f"s{slots}C{Cc}t{tcw}w{warps - 6000}"] = str(e)[:80]
            L.abcq_debug_set_mode(5000)
            L.abcq_debug_set_mode(6000)
            L.abcq_debug_set_mode(0)
            r["sweep"] = sw
        rec[f"p{p}"] = r
        print(rows, cols, p, json.dumps(r), flush=True)
    # SiLU-gated input and an asymmetric f32-scale model (agreement only)
    xg = torch.randn(2 * cols, device="cuda").half()
    y1 = base.gemv(3, xg, out_dtype=torch.float32, silu_glu=True)
    L.abcq_debug_set_mode(23)
    y2 = base.gemv(3, xg, out_dtype=torch.float32, silu_glu=True)
    L.abcq_debug_set_mode(0)
    rec["glu_rel"] = rel(y1, y2)
    am = make(rows, cols, 7, sd="f32", asym=True)
    xf = torch.randn(cols, device="cuda")
    y1 = am.gemv(4, xf, out_dtype=torch.float32)
    L.abcq_debug_set_mode(23)
    y2 = am.gemv(4, xf, out_dtype=torch.float32)
    L.abcq_debug_set_mode(0)
    rec["asym_f32_rel"] = rel(y1, y2)
    print(rows, cols, "glu", rec["glu_rel"], "asym", rec["asym_f32_rel"], flush=True)
    out["shapes"][f"{rows}x{cols}"] = rec
    del models, base, am
    torch.cuda.empty_cache()

Path(a.out).parent.mkdir(parents=True, exist_ok=True)
if out["shapes"]:
    Path(a.out).write_text(json.dumps(out, indent=1))


def timeline(rows, cols, p, mode=5000, dbg=0, n=8):
    """per-launch phase times (us, relative to launch 0's first CTA start) of n
    back-to-back launches in one CUDA graph: CTA start min/max, past-PDL-wait
    min/max, tables built max, streams done max, CTA end min/max."""
    models = [make(rows, cols, 200 + c) for c in range(max(3, min(24, math.ceil(300e6 / (rows * cols // 2)))))]
    x = torch.randn(cols, device="cuda").half()
    y = torch.empty(rows, device="cuda", dtype=torch.float16)
    L.abcq_debug_set_mode(dbg)
    L.abcq_debug_set_mode(mode)
    SL = 168 * 16
    buf = torch.zeros(16 * SL, dtype=torch.int64, device="cuda")
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for m in models:
            m.gemv(p, x, out=y, stream=st)
    torch.cuda.synchronize()
    L.abcq_debug_set_trace(C.c_void_p(buf.data_ptr()))
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for i in range(n):
            models[i % len(models)].gemv(p, x, out=y, stream=st)
    L.abcq_debug_set_trace(None)
    with torch.cuda.stream(st):
        spin_clocks(st)
        for _ in range(100):
            g.replay()
    clk = sm_clock()
    torch.cuda.synchronize()
    gm = geom(models[0], p)
    ncta = gm[0] * gm[1]
    t = buf.view(16, 168, 16).cpu()
    # trace slots were assigned at capture time: launch i -> slot (seq0 + i) % 16; find them by start order
    starts = [(int(t[s, :ncta, 0].min()), s) for s in range(16) if int(t[s, :ncta, 0].min()) > 0]
    starts.sort()
    starts = starts[-n:]
    t0 = starts[0][0]
    rows_out = []
    for _, s in starts:
        ts = t[s, :ncta]
        f = lambda k, fn: round((int(fn(ts[:, k])) - t0) / 1e3, 2)  # noqa: E731
        rows_out.append({"start": [f(0, min), f(0, max)], "prod_done": f(8, max), "wait": [f(1, min), f(1, max)],
                         "x_staged": f(9, max), "tables": f(2, max), "first_stage": [f(5, min), f(5, max)],
                         "prod_begin": f(11, max), "prod_first_issued": f(12, max), "first_full": f(13, max),
                         "stream": f(3, max), "cl_bar": f(10, max),
                         "end": [f(4, min), f(4, max)],
                         "smids": len(set(int(v) for v in ts[:, 6]))})
    L.abcq_debug_set_mode(5000)
    L.abcq_debug_set_mode(0)
    return {"geom": gm, "sm_mhz_after": clk, "launches": rows_out}


if __import__("os").environ.get("CL_ABL"):
    # ablation: graph time per launch with phases switched off (results wrong)
    res = {}
    for spec in __import__("os").environ["CL_ABL"].split(","):
        r_, c_, p_ = (int(q) for q in spec.split(":"))
        models = [make(r_, c_, 300 + c) for c in range(max(3, min(24, math.ceil(300e6 / (r_ * c_ // 2)))))]
        x = torch.randn(c_, device="cuda").half()
        y = torch.empty(r_, device="cuda", dtype=torch.float16)
        row = {}
        for name, dbg in [("full", 0), ("no_lookup", 1), ("no_build", 104),
                          ("no_reduce", 108), ("no_x", 132), ("only_pipeline", 100 + 1 + 4 + 8 + 32)]:
            L.abcq_debug_set_mode(dbg)
            row[name] = round(time_graph(models, p_, x, y, 20), 3)
            L.abcq_debug_set_mode(0)
        L.abcq_debug_set_mode(23)
        row["batch_kernel"] = round(time_graph(models, p_, x, y, 20), 3)
        L.abcq_debug_set_mode(0)
        res[spec] = row
        print(spec, row, flush=True)
        del models

if "--timeline" in sys.argv[0:0] or __import__("os").environ.get("CL_TIMELINE"):
    res = {}
    for spec in __import__("os").environ["CL_TIMELINE"].split(","):
        v = [int(q) for q in spec.split(":")]
        res[spec] = timeline(v[0], v[1], v[2], v[3], v[4] if len(v) > 4 else 0)
        print(spec, json.dumps(res[spec]), flush=True)
    Path(a.out.replace(".json", "_timeline.json")).write_text(json.dumps(res, indent=1))
