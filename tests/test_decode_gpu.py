"""Decode-step harness: the fused non-GEMV ops against
plain PyTorch fp32 references of the same op, and one tiny quantized step."""

import math

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def test_add_rmsnorm_and_silu_mul():
    from paper_2510_10467_b200.decode import add_rmsnorm, silu_mul
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn(4096, device="cuda", generator=g).half()
    r = torch.randn(4096, device="cuda", generator=g).half()
    w = torch.randn(4096, device="cuda", generator=g).half()
    y = torch.empty_like(x)
    x0 = x.clone()
    add_rmsnorm(x, r, w, y, 1e-5)
    xs = (x0.float() + r.float()).half().float()
    assert torch.equal(x, xs.half())
    want = xs * torch.rsqrt(xs.pow(2).mean() + 1e-5) * w.float()
    assert torch.allclose(y.float(), want, rtol=2e-3, atol=2e-3)
    a = torch.empty_like(x)
    silu_mul(x0, r, a)
    assert torch.allclose(a.float(), torch.nn.functional.silu(x0.float()) * r.float(), rtol=2e-3, atol=2e-3)


def test_rope_append_and_attention_decode():
    from paper_2510_10467_b200.decode import LlamaConfig, _Attention
    cfg = LlamaConfig(layers=2)
    g = torch.Generator(device="cuda").manual_seed(1)
    ctx = 300
    att = _Attention(cfg, ctx, torch.device("cuda"), g)
    q = torch.randn(cfg.hidden, device="cuda", generator=g).half()
    k = torch.randn(1024, device="cuda", generator=g).half()
    v = torch.randn(1024, device="cuda", generator=g).half()
    q0, k0 = q.clone(), k.clone()
    out = att(1, q, k, v).clone()
    d = cfg.head_dim

    def rope(t, heads):
        t = t.float().view(heads, d)
        c, s = att.cos, att.sin
        return torch.cat([t[:, :d // 2] * c - t[:, d // 2:] * s, t[:, d // 2:] * c + t[:, :d // 2] * s], -1)
    qr, kr = rope(q0, cfg.heads), rope(k0, cfg.kv_heads)
    assert torch.allclose(q.float().view(cfg.heads, d), qr, rtol=2e-3, atol=2e-3)
    assert torch.equal(att.k_cache[1, :, ctx].float(), kr.half().float())
    assert torch.equal(att.v_cache[1, :, ctx], v.view(cfg.kv_heads, d))
    K = att.k_cache[1].float()                       # (kv, L, d)
    V = att.v_cache[1].float()
    qg = q.float().view(cfg.kv_heads, cfg.heads // cfg.kv_heads, d)
    p = torch.softmax(qg @ K.transpose(1, 2) / math.sqrt(d), -1)
    want = (p @ V).reshape(cfg.hidden)
    assert torch.allclose(out.float(), want, rtol=5e-3, atol=5e-3)


def test_quantized_step_runs_and_is_deterministic():
    from paper_2510_10467_b200.decode import LlamaConfig, QuantizedLlamaStep, time_step
    cfg = LlamaConfig(layers=2, vocab=1000)
    m = QuantizedLlamaStep(cfg, p=3, ctx=64)
    x0 = m.x.clone()
    t1 = m.step().item()
    m.x.copy_(x0)
    t2 = m.step().item()
    assert t1 == t2 and 0 <= t1 < 1000
    assert time_step(m, iters=2, warmup=1) > 0
