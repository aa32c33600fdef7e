"""Time (and, under ncu, capture) the mixed-precision tensor-core GEMM on one
Llama-3-8B MLP matrix: python tools/gemm_probe.py [--rows 14336] [--cols 4096] [--B 16] [--iters 50]"""
import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2510_10467_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--rows", type=int, default=14336)
ap.add_argument("--cols", type=int, default=4096)
ap.add_argument("--B", type=int, default=16)
ap.add_argument("--iters", type=int, default=50)
ap.add_argument("--mode", type=int, default=0, help="abcq_debug_set_mode (40: the tcgen05 variant)")
a = ap.parse_args()
dev = torch.device("cuda", 0)
from paper_2510_10467_b200 import _lib  # noqa: E402
_lib.lib().abcq_debug_set_mode(a.mode)
gen = torch.Generator(device="cuda").manual_seed(0)
dm = P.DeviceModel(a.rows, a.cols, 128, 2, 4, False, scale_dtype="f16")
dm.load_planes(torch.randint(-2**31, 2**31 - 1, (4, a.rows, a.cols // 32), dtype=torch.int32, device=dev, generator=gen))
for p in (2, 3, 4):
    dm.load_scale_set(p, 0.01 + 0.1 * torch.randn(p, a.rows, a.cols // 128, device=dev, generator=gen).abs())
ps = [(2, 3, 4)[b % 3] for b in range(a.B)]
X = torch.randn(a.B, a.cols, device=dev).half()
for _ in range(3):
    dm.gemm_mixedp(ps, X)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.iters):
    dm.gemm_mixedp(ps, X)
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1e3 / a.iters
bits = max(ps) * a.rows * a.cols
print(f"gemm {a.rows}x{a.cols} B={a.B} pmax={max(ps)}: {us:.2f} us/call, {bits / 8 / us / 1e3:.1f} GB/s of planes")
