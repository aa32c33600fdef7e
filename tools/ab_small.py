"""A/B single GEMVs and decoder-grouped launches (the latency-bound cases)
under kernel debug modes (abcq_debug_set_mode), weights rotating over copies
> 2x L2; outputs are checked bitwise against the first mode's.

    python tools/ab_small.py 0 22      # e.g. default vs the standalone reduce kernel
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
p = 2
torch.cuda.set_device(0)
pool = bench.make_layer_models(P, 1, 5, seed0=500, p_lo=2, p_hi=4)
xs = {k: torch.randn(k, device="cuda").half() for k in {c for _, _, c in bench.LAYERS}}
ys = [[torch.empty(m.rows, dtype=torch.float16, device="cuda") for m in row] for row in pool]
st = torch.cuda.Stream()


def timed(fn, n=5, reps=10):
    with torch.cuda.stream(st):
        for c in range(n):
            fn(c)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for c in range(n):
            fn(c)
    with torch.cuda.stream(st):
        g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(reps):
            g.replay()
        b.record(st)
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / (reps * n)


ref = {}
for mode in modes:
    _lib.lib().abcq_debug_set_mode(mode)
    row = {}
    for pp in (2, 3, 4):
        for li, (name, r, k) in enumerate(bench.LAYERS):
            row[f"{name}_p{pp}"] = timed(lambda c: pool[c][li].gemv(pp, xs[k], out=ys[c][li], stream=st))
        row[f"grouped_p{pp}"] = timed(lambda c: [gemv_batch([(pool[c][li], pp, xs[pool[c][li].cols], ys[c][li])
                                                             for li in g], st) for g in bench.DECODER_GROUPS])
        out = torch.cat([y for y in ys[0]]).float().clone()
        same = "" if pp not in ref else ("bitwise-equal" if torch.equal(out, ref[pp]) else "DIFFERENT")
        ref.setdefault(pp, out)
        row[f"check_p{pp}"] = same
    print(f"mode {mode}: " + "  ".join(f"{k} {v:.2f}" if isinstance(v, float) else f"{k} {v}" for k, v in row.items()),
          flush=True)
_lib.lib().abcq_debug_set_mode(0)
