"""A/B of the decode step's GEMV routing, alternated and repeated (medians):
q/k/v + o through the persistent batch kernel (default) or the cluster
kernel (abcq_gemv), gate/up through the cluster kernel whenever it has <= 32
slices (debug mode 28) or by size (default).
    python tools/decode_paths_ab.py [--rounds 4] [--iters 40]"""
import argparse
import json
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2510_10467_b200.decode as D  # noqa: E402
from paper_2510_10467_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--rounds", type=int, default=4)
ap.add_argument("--iters", type=int, default=40)
a = ap.parse_args()
torch.cuda.set_device(0)
qm = D.QuantizedLlamaStep(D.LlamaConfig(), p=3, ctx=1024)
configs = {"persistent_qkvo": (True, 0), "cluster_qkvo": (False, 0), "persistent_qkvo+gu_cluster": (True, 28),
           "cluster_qkvo+gu_cluster": (False, 28)}
res = {k: {p: [] for p in (2, 3, 4)} for k in configs}
for _ in range(a.rounds):
    for name, (pers, mode) in configs.items():
        D.PERSISTENT_QKV_O = pers
        _lib.lib().abcq_debug_set_mode(mode)
        for p in (2, 3, 4):
            qm.p = p
            res[name][p].append(D.time_step(qm, a.iters))
        _lib.lib().abcq_debug_set_mode(0)
D.PERSISTENT_QKV_O = True
print(json.dumps({k: {f"p{p}": round(statistics.median(v), 4) for p, v in d.items()} for k, d in res.items()}))
