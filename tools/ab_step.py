"""A/B the bench step (bench.py's 21-GEMV batched launch, same inputs) under
kernel debug modes (abcq_debug_set_mode), device-timed through a CUDA graph.

    python tools/ab_step.py 0 5 0 5
"""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2510_10467_b200 as P  # noqa: E402
from paper_2510_10467_b200 import _lib  # noqa: E402
from paper_2510_10467_b200.device_model import gemv_batch  # noqa: E402

modes = [int(v) for v in sys.argv[1:]] or [0]
torch.cuda.set_device(0)
models, _ = bench.make_layer_models(P, 1, len(bench.PRECISIONS))
xs = {k: torch.randn(k, device="cuda").half() for k in {c for _, _, c in bench.LAYERS}}
ys = [[torch.empty(m.rows, dtype=torch.float16, device="cuda") for m in row] for row in models]
st = torch.cuda.Stream()
jobs = [(models[pi][li], p, xs[models[pi][li].cols], ys[pi][li])
        for pi, p in enumerate(bench.PRECISIONS) for li in range(len(bench.LAYERS))]
ref = None
for mode in modes:
    _lib.lib().abcq_debug_set_mode(mode)
    with torch.cuda.stream(st):
        for _ in range(3):
            gemv_batch(jobs, st)
    torch.cuda.synchronize()
    out = torch.cat([y for row in ys for y in row]).float().clone()
    if ref is None:
        ref = out
    same = bool(torch.equal(out, ref))
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for _ in range(10):
            gemv_batch(jobs, st)
    with torch.cuda.stream(st):
        g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(5):
            g.replay()
        b.record(st)
    torch.cuda.synchronize()
    us = a.elapsed_time(b) * 1e3 / 50
    print(f"mode {mode}: {us:.2f} us/step  {bench.step_bytes() / us / 1e3:.0f} GB/s  bitwise-equal-to-first {same}")
_lib.lib().abcq_debug_set_mode(0)
