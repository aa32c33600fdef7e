"""Per-op device time of the decode harness's non-GEMV ops (Llama-3-8B shapes,
ctx 1024): each op replayed back to back in a CUDA graph, CUDA events."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2510_10467_b200.decode import LlamaConfig, _Attention, add_rmsnorm, silu_mul  # noqa: E402


def t(fn, n=200):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(n):
            fn()
    with torch.cuda.stream(s):
        g.replay()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        g.replay()
        b.record(s)
    torch.cuda.synchronize()
    return round(a.elapsed_time(b) * 1e3 / n, 2)


torch.cuda.set_device(0)
cfg = LlamaConfig(layers=2)
gen = torch.Generator(device="cuda").manual_seed(0)
f16 = dict(device="cuda", dtype=torch.float16)
x, r, w, y = (torch.randn(4096, **f16, generator=gen) for _ in range(4))
att = _Attention(cfg, 1024, torch.device("cuda"), gen)
q, k, v = torch.randn(4096, **f16), torch.randn(1024, **f16), torch.randn(1024, **f16)
gu, act = torch.randn(2 * 14336, **f16), torch.empty(14336, **f16)
lm = torch.randn(cfg.vocab, 4096, **f16) * 0.02
tok = torch.empty((), device="cuda", dtype=torch.int64)
out = {"us_per_launch_back_to_back": {
    "add_rmsnorm": t(lambda: add_rmsnorm(x, r, w, y, 1e-5)),
    "silu_mul": t(lambda: silu_mul(gu[:14336], gu[14336:], act)),
}}
att.fused = True
out["us_per_launch_back_to_back"]["rope_attn_fused"] = t(lambda: att(1, q, k, v))
att.fused = False
out["us_per_launch_back_to_back"]["rope_append+attn_partial+combine"] = t(lambda: att(1, q, k, v))
out["us_per_launch_back_to_back"]["lm_head_mv+argmax"] = t(lambda: torch.argmax(torch.mv(lm, x), out=tok), 20)
print(json.dumps(out))
