"""A/B bench.py's per_shape section (single launches back to back, > 2x L2
of weight copies) under library debug modes, alternating:
    python tools/per_shape_ab.py 0 32 [--rounds 2]"""
import argparse
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2510_10467_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("modes", nargs="+", type=int)
ap.add_argument("--rounds", type=int, default=2)
a = ap.parse_args()
torch.cuda.set_device(0)
ctx = bench.Ctx(torch.device("cuda:0"), torch.cuda.Stream(), 0, 1)
xs = {k: torch.randn(k, device="cuda").half() for k in {c for _, _, c in bench.LAYERS}}
for r in range(a.rounds):
    for m in a.modes:
        _lib.lib().abcq_debug_set_mode(0)
        _lib.lib().abcq_debug_set_mode(m)
        res = bench.per_shape(ctx, xs)
        print(json.dumps({"mode": m, **{k: v["us"] for k, v in res.items() if isinstance(v, dict)}}), flush=True)
_lib.lib().abcq_debug_set_mode(0)
