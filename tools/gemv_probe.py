"""Run one GEMV shape repeatedly (for ncu / quick timing on the GPU box).

    python tools/gemv_probe.py --rows 14336 --cols 4096 --p 2 --iters 20
"""
import argparse
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2510_10467_b200 as P  # noqa: E402
from oracle import anybcq_oracle as O  # noqa: E402  (synthetic input generator)

ap = argparse.ArgumentParser()
ap.add_argument("--rows", type=int, default=14336)
ap.add_argument("--cols", type=int, default=4096)
ap.add_argument("--p", type=int, default=2)
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--copies", type=int, default=4)
a = ap.parse_args()

torch.cuda.set_device(0)
import os  # noqa: E402
if os.environ.get("ABCQ_DBG_MODE"):
    from paper_2510_10467_b200 import _lib
    _lib.lib().abcq_debug_set_mode(int(os.environ["ABCQ_DBG_MODE"]))
models = []
for c in range(a.copies):
    dm = P.DeviceModel(a.rows, a.cols, 128, 2, 4, scale_dtype="f16")
    dm.load_planes(O.random_words(4, a.rows, a.cols, seed=c))
    for p in (2, 3, 4):
        dm.load_scale_set(p, np.full((p, a.rows, a.cols // 128), 0.05, np.float32))
    models.append(dm)
x = torch.randn(a.cols, device="cuda").half()
y = torch.empty(a.rows, device="cuda", dtype=torch.float16)
s = torch.cuda.current_stream()
for i in range(3):
    models[i % a.copies].gemv(a.p, x, out=y)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(a.iters):
    models[i % a.copies].gemv(a.p, x, out=y)
e1.record()
torch.cuda.synchronize()
us_eager = e0.elapsed_time(e1) * 1e3 / a.iters
# back-to-back device time: a CUDA graph of `iters` launches (PDL edges kept)
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    for i in range(a.copies):
        models[i].gemv(a.p, x, out=y, stream=st)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=st):
    for i in range(a.iters):
        models[i % a.copies].gemv(a.p, x, out=y, stream=st)
with torch.cuda.stream(st):
    g.replay()
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(5):
        g.replay()
    e1.record(st)
torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1e3 / (5 * a.iters)
G = a.cols // 128
byts = a.p * a.rows * a.cols // 8 + a.p * a.rows * G * 2 + 2 * (a.rows + a.cols)
print(f"{a.rows}x{a.cols} p={a.p}: graph {us:.2f} us/launch -> {byts / us / 1e3:.1f} GB/s "
      f"(eager {us_eager:.2f} us)")

if "ABCQ_TRACE" in __import__("os").environ:
    # timeline of 8 consecutive launches inside one CUDA graph (PDL edges kept)
    from paper_2510_10467_b200 import _lib
    SL = 160 * 8
    buf = torch.zeros(16 * SL, dtype=torch.int64, device="cuda")
    _lib.lib().abcq_debug_set_trace(buf.data_ptr())
    g3 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g3, stream=st):
        for i in range(8):
            if __import__("os").environ.get("ABCQ_BATCH"):
                from paper_2510_10467_b200.device_model import gemv_batch
                gemv_batch([(models[(i + k) % a.copies], a.p, x, y) for k in range(int(__import__("os").environ["ABCQ_BATCH"]))], st)
            else:
                models[i % a.copies].gemv(a.p, x, out=y, stream=st)
    _lib.lib().abcq_debug_set_trace(None)
    with torch.cuda.stream(st):
        g3.replay()
        torch.cuda.synchronize()
        buf.zero_()
        g3.replay()
    torch.cuda.synchronize()
    t = buf.view(16, 160, 8).cpu().numpy().astype(np.float64)
    used = [k for k in range(16) if t[k, :, 0].max() > 0]
    t0 = min(t[k, :148, 0][t[k, :148, 0] > 0].min() for k in used)
    names = ["start", "tab0", "str0", "tab1", "str1", "arrived", "-", "reduced"]
    for k in sorted(used, key=lambda k: t[k, :148, 0][t[k, :148, 0] > 0].min()):
        row = []
        for j, n in enumerate(names):
            col = t[k, :148, j]
            col = col[col > 0]
            if len(col):
                row.append(f"{n} {((col.min() - t0) / 1e3):6.2f}/{((np.median(col) - t0) / 1e3):6.2f}/{((col.max() - t0) / 1e3):6.2f}")
        red = t[k, 159, :3]
        if red[0] > 0:
            row.append("reduce " + "/".join(f"{(v - t0) / 1e3:6.2f}" for v in red))
        print("  " + " | ".join(row))

if __import__("os").environ.get("ABCQ_BATCH"):
    # one persistent launch over ABCQ_BATCH jobs (rotating over the copies)
    from paper_2510_10467_b200.device_model import gemv_batch
    nb = int(__import__("os").environ["ABCQ_BATCH"])
    outs = [torch.empty(a.rows, device="cuda", dtype=torch.float16) for _ in range(nb)]
    jobs = [(models[i % a.copies], a.p, x, outs[i]) for i in range(nb)]
    with torch.cuda.stream(st):
        gemv_batch(jobs, st)
    torch.cuda.synchronize()
    gb = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gb, stream=st):
        for _ in range(4):
            gemv_batch(jobs, st)
    with torch.cuda.stream(st):
        gb.replay()
        torch.cuda.synchronize()
        e0.record(st)
        for _ in range(5):
            gb.replay()
        e1.record(st)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / 20
    print(f"  batch of {nb}: {us:.2f} us/launch -> {nb * byts / us / 1e3:.1f} GB/s ({us / nb:.2f} us/GEMV)")
