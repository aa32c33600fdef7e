"""A/B of the decode step with the add+RMSNorm as the o / down GEMVs'
epilogue (fuse_norm_out, default) vs separate launches:
    python tools/decode_norm_out_ab.py [--rounds 2]"""
import argparse
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2510_10467_b200.decode import LlamaConfig, QuantizedLlamaStep, time_step  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--rounds", type=int, default=2)
a = ap.parse_args()
torch.cuda.set_device(0)
qm = QuantizedLlamaStep(LlamaConfig(), p=3, ctx=1024)
for r in range(a.rounds):
    for fo in (True, False):
        qm.fuse_norm_out = fo
        out = {"fuse_norm_out": fo}
        for p in (2, 3, 4):
            qm.p = p
            out[f"p{p}_ms"] = round(time_step(qm, 20), 4)
        print(json.dumps(out), flush=True)
