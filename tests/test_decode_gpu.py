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
    att.fused = False   # the separate launches (rotate q/k in place); the fused kernel is checked against them
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


def test_quantized_step_fused_glu_equals_separate_silu_mul():
    from paper_2510_10467_b200.decode import LlamaConfig, QuantizedLlamaStep
    cfg = LlamaConfig(layers=2, vocab=1000)
    m = QuantizedLlamaStep(cfg, p=3, ctx=64, fuse_glu=True)
    x0 = m.x.clone()
    k0, v0 = m.attn.k_cache.clone(), m.attn.v_cache.clone()
    t1 = m.step().item()
    x1, d1 = m.x.clone(), m.d.clone()
    m.x.copy_(x0)
    m.attn.k_cache.copy_(k0)
    m.attn.v_cache.copy_(v0)
    m.fuse_glu = False
    t2 = m.step().item()
    assert t1 == t2
    assert torch.equal(m.d, d1) and torch.equal(m.x, x1)   # bitwise: same f16 input to the down GEMV


@pytest.mark.parametrize("ctx", [1024, 63, 64, 300, 0])
def test_fused_rope_attention_equals_separate_launches(ctx):
    """rope_append + attn_decode (+ combine) vs the one-launch fused kernel: bitwise,
    including the new cache row; repeated launches exercise the counter self-reset."""
    from paper_2510_10467_b200.decode import LlamaConfig, _Attention
    cfg = LlamaConfig(layers=2)
    g = torch.Generator(device="cuda").manual_seed(ctx + 7)
    att = _Attention(cfg, ctx, torch.device("cuda"), g)
    q = torch.randn(cfg.hidden, device="cuda", generator=g).half()
    k = torch.randn(1024, device="cuda", generator=g).half()
    v = torch.randn(1024, device="cuda", generator=g).half()
    kc0, vc0 = att.k_cache.clone(), att.v_cache.clone()
    att.fused = False
    want = att(1, q.clone(), k.clone(), v.clone()).clone()
    kc1, vc1 = att.k_cache.clone(), att.v_cache.clone()
    att.fused = True
    for _ in range(3):
        att.k_cache.copy_(kc0)
        att.v_cache.copy_(vc0)
        qq, kk = q.clone(), k.clone()
        got = att(1, qq, kk, v).clone()
        assert torch.equal(got, want)
        assert torch.equal(att.k_cache, kc1) and torch.equal(att.v_cache, vc1)
        assert torch.equal(qq, q) and torch.equal(kk, k)   # inputs left unrotated


def test_quantized_step_separate_qkv_gateup_models():
    from paper_2510_10467_b200.decode import LlamaConfig, QuantizedLlamaStep
    cfg = LlamaConfig(layers=2, vocab=1000)
    m = QuantizedLlamaStep(cfg, p=2, ctx=64, stack_rows=False)
    assert set(m.layers[0]) == {"q", "k", "v", "o", "gate", "up", "down"}
    x0 = m.x.clone()
    t1 = m.step().item()
    m.x.copy_(x0)
    assert m.step().item() == t1 and 0 <= t1 < 1000


def test_fused_attention_workspace_reused_across_positions():
    """One workspace (sized once for the largest context) serves the fused
    RoPE + attention kernel at decreasing and increasing positions: the
    per-head counters sit at a fixed offset, so every call
    completes and matches the separate launches bitwise."""
    import ctypes as C
    from paper_2510_10467_b200 import _lib
    from paper_2510_10467_b200.decode import LlamaConfig, _rope_tables
    cfg = LlamaConfig(layers=1)
    L = _lib.lib()
    lmax = 1025
    g = torch.Generator(device="cuda").manual_seed(11)
    shape = (cfg.kv_heads, lmax, cfg.head_dim)
    kc0 = torch.randn(shape, device="cuda", dtype=torch.float16, generator=g)
    vc0 = torch.randn(shape, device="cuda", dtype=torch.float16, generator=g)
    n = C.c_size_t()
    _lib.check(L.abcq_attn_decode_workspace_bytes(cfg.heads, lmax, C.byref(n)))
    ws = torch.zeros(int(n.value), dtype=torch.uint8, device="cuda")      # shared by every fused call
    ws_sep = torch.zeros(int(n.value), dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    scale = 1.0 / math.sqrt(cfg.head_dim)
    for pos in (1024, 300, 63, 64, 0, 700, 5):
        q = torch.randn(cfg.hidden, device="cuda", generator=g).half()
        k = torch.randn(1024, device="cuda", generator=g).half()
        v = torch.randn(1024, device="cuda", generator=g).half()
        cos, sin = _rope_tables(cfg, pos, "cuda")
        kc, vc = kc0.clone(), vc0.clone()
        out = torch.empty(cfg.hidden, device="cuda", dtype=torch.float16)
        _lib.check(L.abcq_rope_attn_decode_f16(q.data_ptr(), k.data_ptr(), v.data_ptr(), cos.data_ptr(),
                                               sin.data_ptr(), kc.data_ptr(), vc.data_ptr(), cfg.heads, cfg.kv_heads,
                                               lmax, pos, scale, out.data_ptr(), ws.data_ptr(), ws.numel(), st))
        kc2, vc2, q2, k2 = kc0.clone(), vc0.clone(), q.clone(), k.clone()
        want = torch.empty_like(out)
        _lib.check(L.abcq_rope_append_f16(q2.data_ptr(), k2.data_ptr(), v.data_ptr(), cos.data_ptr(), sin.data_ptr(),
                                          kc2.data_ptr(), vc2.data_ptr(), cfg.heads, cfg.kv_heads, cfg.head_dim,
                                          lmax, pos, st))
        _lib.check(L.abcq_attn_decode_f16(q2.data_ptr(), kc2.data_ptr(), vc2.data_ptr(), cfg.heads, cfg.kv_heads,
                                          lmax, pos + 1, scale, want.data_ptr(), ws_sep.data_ptr(), ws_sep.numel(),
                                          st))
        torch.cuda.synchronize()
        assert torch.equal(out, want), pos
        assert torch.equal(kc, kc2) and torch.equal(vc, vc2), pos


class _DenseGemv:
    """A linear with the dense weights abcq_dequantize reconstructs (bcq.py:372-378),
    applied in fp32 by torch -- the reference for one AnyBCQ GEMV of the step."""

    def __init__(self, dm, p):
        self.w = dm.dequantize(p)            # (rows, cols) f32 on the device
        self.cols = dm.cols

    def gemv(self, p, x, out=None, silu_glu=False):
        if silu_glu:
            g, u = x[:self.cols].float(), x[self.cols:].float()
            x = (torch.nn.functional.silu(g) * u).half()   # the f16 input the fused GEMV forms
        y = self.w @ x.float()
        out.copy_(y.to(out.dtype))
        return out


@pytest.mark.parametrize("p", [2, 3, 4])
def test_quantized_step_matches_dense_dequantized_step(p):
    """A 2-layer Llama-3-8B-shaped decode step with every linear an AnyBCQ GEMV
    vs the same step with the dense weights abcq_dequantize reconstructs (fp32
    torch matmuls, the same f16 rounding points): residual stream and final
    hidden state agree to f16 rounding."""
    from paper_2510_10467_b200.decode import LlamaConfig, QuantizedLlamaStep
    cfg = LlamaConfig(layers=2, vocab=1000)
    m = QuantizedLlamaStep(cfg, p=p, ctx=64)
    x0 = m.x.clone()
    k0, v0 = m.attn.k_cache.clone(), m.attn.v_cache.clone()
    m.step()
    x_q, h_q = m.x.float().clone(), m.h.float().clone()
    dense = [{name: _DenseGemv(dm, p) for name, dm in mats.items()} for mats in m.layers]
    m.layers = dense
    m.x.copy_(x0)
    m.attn.k_cache.copy_(k0)
    m.attn.v_cache.copy_(v0)
    m.step()
    x_d, h_d = m.x.float(), m.h.float()
    rel = lambda a, b: float((a - b).norm() / b.norm())  # noqa: E731
    assert rel(x_q, x_d) <= 1e-2, rel(x_q, x_d)
    assert rel(h_q, h_d) <= 1e-2, rel(h_q, h_d)


@pytest.mark.parametrize("n", [1, 1000, 128256, 40000])
def test_argmax_matches_torch(n):
    from paper_2510_10467_b200.decode import _Argmax
    am = _Argmax(torch.device("cuda"))
    g = torch.Generator(device="cuda").manual_seed(n)
    out = torch.empty((), device="cuda", dtype=torch.int64)
    for trial in range(3):
        x = torch.randn(n, device="cuda", generator=g).half()
        if trial == 2 and n > 10:   # ties: the first occurrence wins
            x[n // 3] = x[n - 2] = x.max() + 1
        am(x, out)
        assert int(out) == int(torch.argmax(x)), (n, trial)


def test_quantized_step_fused_norm_equals_separate_add_rmsnorm(monkeypatch):
    """add + RMSNorm inside the q/k/v and gate/up GEMVs (abcq_gemv_add_rmsnorm)
    == the separate add_rmsnorm launch: bitwise equal step state and token
    (the separate path's GEMVs on the same persistent kernel)."""
    import paper_2510_10467_b200.decode as D
    from paper_2510_10467_b200.decode import LlamaConfig, QuantizedLlamaStep
    monkeypatch.setattr(D, "PERSISTENT_QKV_O", True)
    cfg = LlamaConfig(layers=3, vocab=1000)
    m = QuantizedLlamaStep(cfg, p=3, ctx=64, fuse_norm=True)
    x0 = m.x.clone()
    k0, v0 = m.attn.k_cache.clone(), m.attn.v_cache.clone()
    t1 = m.step().item()
    x1, gu1, qkv1 = m.x.clone(), m.gu.clone(), m.qkv.clone()
    m.x.copy_(x0)
    m.attn.k_cache.copy_(k0)
    m.attn.v_cache.copy_(v0)
    m.fuse_norm = False
    t2 = m.step().item()
    assert t1 == t2
    assert torch.equal(m.x, x1) and torch.equal(m.gu, gu1) and torch.equal(m.qkv, qkv1)


def test_gemv_add_rmsnorm_matches_separate_ops():
    """One model, the fused input vs add_rmsnorm + gemv (both bitwise), incl.
    no residual, and the C-ABI alias check."""
    import paper_2510_10467_b200 as P
    from paper_2510_10467_b200.decode import add_rmsnorm
    dm = P.DeviceModel(6144, 4096, 128, 2, 4, scale_dtype="f16")
    g = torch.Generator(device="cuda").manual_seed(5)
    dm.load_planes(torch.randint(-2**31, 2**31 - 1, (4, 6144, 128), dtype=torch.int32, device="cuda", generator=g))
    for q in (2, 3, 4):
        dm.load_scale_set(q, 0.01 + 0.01 * torch.rand((q, 6144, 32), device="cuda", generator=g))
    x = torch.randn(4096, device="cuda", generator=g).half()
    r = torch.randn(4096, device="cuda", generator=g).half()
    w = (1 + 0.1 * torch.randn(4096, device="cuda", generator=g)).half()
    for res in (r, None):
        xo = torch.empty_like(x)
        y = torch.empty(6144, device="cuda", dtype=torch.float16)
        dm.gemv_add_rmsnorm(3, x, res, w, 1e-5, out=y, x_out=xo)
        xs, h = x.clone(), torch.empty_like(x)
        add_rmsnorm(xs, res, w, h, 1e-5)
        want = torch.empty_like(y)
        P.gemv_batch([(dm, 3, h, want)])
        torch.cuda.synchronize()
        assert torch.equal(y, want)
        assert torch.equal(xo, xs)
    with pytest.raises(P.UsageError):
        dm.gemv_add_rmsnorm(3, x, r, w, 1e-5, out=y, x_out=x)   # x_out aliases x


def test_quantized_step_norm_out_equals_separate_add_rmsnorm(monkeypatch):
    """add + RMSNorm as the o / down GEMVs' epilogue (abcq_gemv_rmsnorm_out,
    fuse_norm_out=True) == the separate launches: bitwise equal step state and
    token (the separate path's GEMVs on the same persistent kernel)."""
    import paper_2510_10467_b200.decode as D
    from paper_2510_10467_b200.decode import LlamaConfig, QuantizedLlamaStep
    monkeypatch.setattr(D, "PERSISTENT_QKV_O", True)
    cfg = LlamaConfig(layers=3, vocab=1000)
    m = QuantizedLlamaStep(cfg, p=3, ctx=64, fuse_norm_out=True)
    assert m.fuse_norm_out
    x0 = m.x.clone()
    k0, v0 = m.attn.k_cache.clone(), m.attn.v_cache.clone()
    t1 = m.step().item()
    x1, h1, gu1, qkv1, lg1 = m.x.clone(), m.h.clone(), m.gu.clone(), m.qkv.clone(), m.logits.clone()
    m.x.copy_(x0)
    m.attn.k_cache.copy_(k0)
    m.attn.v_cache.copy_(v0)
    m.fuse_norm_out = False
    t2 = m.step().item()
    assert t1 == t2
    for a, b in ((m.x, x1), (m.h, h1), (m.gu, gu1), (m.qkv, qkv1), (m.logits, lg1)):
        assert torch.equal(a, b)


@pytest.mark.parametrize("rows,cols,glu,asym,sd", [(4096, 4096, False, False, "f16"), (4096, 14336, True, False, "f16"),
                                                  (8192, 1024, False, False, "f16"), (1000, 1000, False, True, "f32"),
                                                  (37, 300, True, True, "f16")])
def test_gemv_rmsnorm_out_matches_separate_ops(rows, cols, glu, asym, sd):
    """The norm epilogue vs the persistent GEMV + add_rmsnorm launch (both
    bitwise): y, the updated residual stream and h; plus the usage checks."""
    import paper_2510_10467_b200 as P
    from paper_2510_10467_b200.decode import add_rmsnorm
    dm = P.DeviceModel(rows, cols, 128, 2, 4, asym, scale_dtype=sd)
    g = torch.Generator(device="cuda").manual_seed(rows + cols)
    wpr, G = -(-cols // 32), -(-cols // 128)
    dm.load_planes(torch.randint(-2**31, 2**31 - 1, (4, rows, wpr), dtype=torch.int32, device="cuda", generator=g))
    for q in (2, 3, 4):
        z = 0.01 * torch.randn((rows, G), device="cuda", generator=g) if asym else None
        dm.load_scale_set(q, (0.01 + 0.01 * torch.rand((q, rows, G), device="cuda", generator=g)) / 4, z)
    x = torch.randn(2 * cols if glu else cols, device="cuda", generator=g).half()
    s0 = torch.randn(rows, device="cuda", generator=g).half()
    w = (1 + 0.1 * torch.randn(rows, device="cuda", generator=g)).half()
    for p in (2, 4):
        y, st, h = torch.empty_like(s0), s0.clone(), torch.empty_like(s0)
        for _ in range(2):  # twice: the self-resetting counters
            st.copy_(s0)
            dm.gemv_rmsnorm_out(p, x, y, st, w, 1e-5, h, silu_glu=glu)
        ref_y = torch.empty_like(y)
        _batch_one(dm, p, x, ref_y, glu)
        st_ref, h_ref = s0.clone(), torch.empty_like(s0)
        add_rmsnorm(st_ref, ref_y, w, h_ref, 1e-5)
        torch.cuda.synchronize()
        assert torch.equal(y, ref_y), p
        assert torch.equal(st, st_ref) and torch.equal(h, h_ref), p
    with pytest.raises(P.UsageError):
        dm.gemv_rmsnorm_out(2, x, y, y, w, 1e-5, h, silu_glu=glu)  # stream aliases y


def _batch_one(dm, p, x, y, glu):
    """y = W_p x through the persistent batch kernel (a batch of one job)."""
    import ctypes as C
    from paper_2510_10467_b200 import _lib
    from paper_2510_10467_b200.device_model import dtype_code
    job = _lib.AbcqGemvJob()
    job.model = C.pointer(dm._struct)
    job.p = p
    job.x_dtype = _lib.F16_SILU_GLU if glu else dtype_code(x.dtype)
    job.y_dtype = dtype_code(y.dtype)
    job.x = x.data_ptr()
    job.y = y.data_ptr()
    ws = dm.workspace(None)
    _lib.check(_lib.lib().abcq_gemv_batch(C.byref(job), 1, ws.data_ptr(), ws.numel(),
                                           torch.cuda.current_stream().cuda_stream), "abcq_gemv_batch")
