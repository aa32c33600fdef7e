"""Decode step (p=3) with one linear kind skipped at a time: each GEMV kind's marginal cost in the chain."""
import sys, json
sys.path.insert(0, "/root/repo")
import torch
import paper_2510_10467_b200.decode as D
from paper_2510_10467_b200.decode import LlamaConfig, QuantizedLlamaStep, time_step
torch.cuda.set_device(0)
qm = QuantizedLlamaStep(LlamaConfig(layers=32), p=3, ctx=1024)
out = {"full": round(time_step(qm, 20), 4)}
real = {}
for name in ("qkv", "o", "gu", "down"):
    for mats in qm.layers:
        dm = mats[name]
        real[id(dm)] = dm.gemv
    class Skip:
        def __init__(s, dm): s.dm = dm
        def gemv(s, p, x, out=None, **k): return out
    saved = [mats[name] for mats in qm.layers]
    for mats in qm.layers:
        mats[name] = Skip(mats[name])
    out["skip_" + name] = round(time_step(qm, 20), 4)
    for mats, dm in zip(qm.layers, saved):
        mats[name] = dm
# the harness ops: attention (RoPE + KV append + split-L attention + combine) and add+RMSNorm
attn = qm.attn
qm.attn = lambda li, q, k, v: attn.out
out["skip_attention"] = round(time_step(qm, 20), 4)
qm.attn = attn
norm = D.add_rmsnorm
D.add_rmsnorm = lambda *a, **k: None
out["skip_add_rmsnorm"] = round(time_step(qm, 20), 4)
D.add_rmsnorm = norm
lm = qm.lm_head
qm.lm_head = lm[:16].contiguous()
qm.logits = qm.logits[:16]
out["skip_lm_head"] = round(time_step(qm, 20), 4)
qm.lm_head = lm
out["full2"] = round(time_step(qm, 20), 4)
print(json.dumps(out))
