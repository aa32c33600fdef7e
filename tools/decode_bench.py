"""Llama-3-8B batch-1 decode step, AnyBCQ linears at p vs dense fp16 (BASELINE
config 4; paper Table 5): tokens/s from CUDA-graph replays of one full step
(32 layers + fp16 lm_head), random weights. Prints one JSON line.

    python tools/decode_bench.py [--p 3] [--ctx 1024] [--layers 32] [--iters 20]
"""
import argparse
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2510_10467_b200.decode import Fp16LlamaStep, LlamaConfig, QuantizedLlamaStep, time_step  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--p", type=int, nargs="+", default=[2, 3, 4])
ap.add_argument("--ctx", type=int, default=1024)
ap.add_argument("--layers", type=int, default=32)
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--no-fp16", action="store_true")
ap.add_argument("--ab-stack", action="store_true", help="also time separate q/k/v and gate/up models (batched)")
ap.add_argument("--ab-glu", action="store_true", help="also time the step with a separate silu_mul launch")
ap.add_argument("--breakdown", action="store_true", help="also time the step without its linears")
a = ap.parse_args()
torch.cuda.set_device(0)
cfg = LlamaConfig(layers=a.layers)
out = {"metric": "Llama-3-8B decode tokens/s (batch 1)", "ctx": a.ctx, "layers": a.layers,
       "data": "random weights (device RNG planes, fp16 scales), random KV cache",
       "timing": "CUDA graph of one decode step, CUDA events", "anybcq": {}}
qm = QuantizedLlamaStep(cfg, p=a.p[0], ctx=a.ctx)
for p in a.p:
    qm.p = p
    ms = time_step(qm, a.iters)
    gb = qm.linear_bytes() + cfg.vocab * cfg.hidden * 2
    out["anybcq"][f"p{p}"] = {"ms_per_token": round(ms, 4), "tokens_per_s": round(1e3 / ms, 1),
                              "weight_GB_per_token": round(gb / 1e9, 3),
                              "weight_GBps": round(gb / (ms * 1e-3) / 1e9, 1)}
    if a.ab_glu:
        qm.fuse_glu = False
        out["anybcq"][f"p{p}"]["ms_per_token_separate_silu_mul"] = round(time_step(qm, a.iters), 4)
        qm.fuse_glu = True
if a.ab_stack:  # the same step with q/k/v and gate/up as separate models in one batched launch each
    sm = QuantizedLlamaStep(cfg, p=a.p[0], ctx=a.ctx, stack_rows=False)
    for p in a.p:
        sm.p = p
        out["anybcq"][f"p{p}"]["ms_per_token_unstacked"] = round(time_step(sm, a.iters), 4)
    del sm
    torch.cuda.empty_cache()
if a.breakdown:  # the same step with the linears skipped: attention, norms, lm_head, ...
    import paper_2510_10467_b200.decode as D
    real_batch = D.gemv_batch
    D.gemv_batch = lambda jobs, stream=None: None
    for mats in qm.layers:
        for dm in mats.values():
            dm._real_gemv, dm.gemv = dm.gemv, (lambda p, x, out=None, **k: out)
    out["non_linear_ms_per_token"] = round(time_step(qm, a.iters), 4)
    D.gemv_batch = real_batch
    for mats in qm.layers:
        for dm in mats.values():
            dm.gemv = dm._real_gemv
del qm
torch.cuda.empty_cache()
if not a.no_fp16:
    fm = Fp16LlamaStep(cfg, ctx=a.ctx)
    ms = time_step(fm, a.iters)
    gb = fm.linear_bytes() + cfg.vocab * cfg.hidden * 2
    out["fp16"] = {"ms_per_token": round(ms, 4), "tokens_per_s": round(1e3 / ms, 1),
                   "weight_GB_per_token": round(gb / 1e9, 3), "weight_GBps": round(gb / (ms * 1e-3) / 1e9, 1)}
    for k, v in out["anybcq"].items():
        v["speedup_vs_fp16"] = round(out["fp16"]["ms_per_token"] / v["ms_per_token"], 2)
print(json.dumps(out))
