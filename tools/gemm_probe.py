"""Mixed-precision small-batch GEMM timing on the Llama-3-8B MLP block
(gate/up 14336x4096, down 4096x14336), B in {1,2,4,8,16}, p pattern 2,3,4,...:
tensor-core GEMM (one pass over the planes) vs B batched LUT GEMV jobs.

    python tools/gemm_probe.py
"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2510_10467_b200 as P  # noqa: E402
from paper_2510_10467_b200.device_model import gemv_batch  # noqa: E402
from oracle import anybcq_oracle as O  # noqa: E402  (synthetic input generator)

torch.cuda.set_device(0)
SHAPES = [("gate", 14336, 4096), ("up", 14336, 4096), ("down", 4096, 14336)]
COPIES = 2
models = {}
for name, r, c in SHAPES:
    models[name] = []
    for k in range(COPIES):
        dm = P.DeviceModel(r, c, 128, 2, 4, scale_dtype="f16")
        dm.load_planes(O.random_words(4, r, c, seed=k * 10 + r))
        for p in (2, 3, 4):
            dm.load_scale_set(p, np.full((p, r, c // 128), 0.05, np.float32))
        models[name].append(dm)
st = torch.cuda.Stream()


def timeit(fn, reps=10):
    with torch.cuda.stream(st):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        fn()
    with torch.cuda.stream(st):
        g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(reps):
            g.replay()
        b.record(st)
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / reps


for B in (1, 2, 4, 8, 16):
    ps = [2 + b % 3 for b in range(B)]
    pmax = max(ps)
    X = {c: torch.randn(B, c, device="cuda").half() for _, _, c in SHAPES}
    outs = {n: torch.empty(B, r, device="cuda", dtype=torch.float16) for n, r, _ in SHAPES}

    def gemm():
        for k in range(COPIES):
            for n, r, c in SHAPES:
                models[n][k].gemm_mixedp(ps, X[c], out_dtype=torch.float16, stream=st)

    def lut_jobs():
        for k in range(COPIES):
            for n, r, c in SHAPES:
                gemv_batch([(models[n][k], ps[b], X[c][b], outs[n][b]) for b in range(B)], st)

    t_g = timeit(gemm) / COPIES
    t_l = timeit(lut_jobs) / COPIES
    plane_bytes = sum(pmax * r * c // 8 for _, r, c in SHAPES)
    print(f"B={B:2d} p={ps}: tensor-core GEMM {t_g:7.1f} us/MLP block ({plane_bytes / t_g / 1e3:6.0f} GB/s of planes, "
          f"{B * 1e6 / t_g:8.0f} req-blocks/s) | {B} LUT jobs {t_l:7.1f} us")
