"""A/B of the decode step (BASELINE config 4) under library debug modes:
    python tools/decode_ab.py --modes 0,23 [--layers 32]
mode 23 routes single GEMVs through the batch kernel instead of the cluster kernel."""
import argparse
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2510_10467_b200 import _lib  # noqa: E402
from paper_2510_10467_b200.decode import LlamaConfig, QuantizedLlamaStep, time_step  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--modes", default="0,23")
ap.add_argument("--layers", type=int, default=32)
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--cluster-qkv-o", action="store_true", help="also time q/k/v and o through abcq_gemv (cluster kernel)")
a = ap.parse_args()
torch.cuda.set_device(0)
qm = QuantizedLlamaStep(LlamaConfig(layers=a.layers), p=3, ctx=1024)
out = {}
for spec in a.modes.split(","):
    _lib.lib().abcq_debug_set_mode(0)
    _lib.lib().abcq_debug_set_mode(5000)
    for m in spec.split("+"):
        _lib.lib().abcq_debug_set_mode(int(m))
    mode = spec
    for p in (2, 3, 4):
        qm.p = p
        out[f"mode{mode}_p{p}_ms"] = round(time_step(qm, a.iters), 4)
    print(json.dumps(out), flush=True)
_lib.lib().abcq_debug_set_mode(0)
if a.cluster_qkv_o:
    import paper_2510_10467_b200.decode as D
    for flag in (False, True, False, True):
        D.PERSISTENT_QKV_O = flag
        for p in (2, 3, 4):
            qm.p = p
            out[f"{'persistent' if flag else 'cluster'}_qkv_o_p{p}_ms"] = round(time_step(qm, a.iters), 4)
        print(json.dumps(out), flush=True)
    D.PERSISTENT_QKV_O = True
