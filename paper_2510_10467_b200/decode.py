"""Llama-3-8B decode-step harness (BASELINE config 4).

One decode step of a Llama-3 architecture at batch 1: every linear layer
(q/k/v/o/gate/up/down of every decoder layer) is an AnyBCQ multi-precision
model served at a chosen precision p through the B200 bit-plane kernels;
embeddings are skipped (the step starts from a hidden state); attention,
RMSNorm, RoPE and SiLU run as fused kernels (abcq_decode_ops.cu) and the fp16
lm_head through cuBLAS. The comparator runs the same step with dense fp16
weights (q/k/v and gate/up fused into one matmul each, as fp16 serving
stacks do).

Weights are random (no checkpoints offline): bit-planes from the device RNG,
scales 0.01 + 0.1|N(0,1)| in fp16, so the step moves exactly the bytes a real
model would. The KV cache holds `ctx` positions of random keys/values and the
step attends over all of them and writes position `ctx` (static shapes, so
the whole step is captured in one CUDA graph).

Per layer the quantized step issues 4 GEMV launches: q/k/v and gate/up are
row-stacked models (BCQ scales are per row and group, so stacking is exact;
`stack_rows=False` keeps them separate, one abcq_gemv_batch launch each),
then [o] and [down], plus the fused
harness ops of abcq_decode_ops.cu (add+RMSNorm x2, and RoPE + KV append +
split-L decode attention + combine as ONE launch) -- the fp16 comparator uses
the same fused ops. SiLU(gate)*up
is formed inside the down GEMV's table build (x dtype ABCQ_F16_SILU_GLU over the
[gate ; up] buffer, bitwise equal to the separate silu_mul launch, which the
fp16 comparator and `fuse_glu=False` still issue).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import ctypes as C

import torch

from . import _lib
from .device_model import DeviceModel, gemv_batch


@dataclass(frozen=True)
class LlamaConfig:
    hidden: int = 4096
    layers: int = 32
    heads: int = 32
    kv_heads: int = 8
    intermediate: int = 14336
    vocab: int = 128256
    rope_theta: float = 500000.0
    eps: float = 1e-5

    @property
    def head_dim(self) -> int:
        return self.hidden // self.heads

    def linear_shapes(self):
        """(name, rows, cols) of one decoder layer's linears."""
        h, kv = self.hidden, self.kv_heads * self.head_dim
        return [("q", h, h), ("k", kv, h), ("v", kv, h), ("o", h, h),
                ("gate", self.intermediate, h), ("up", self.intermediate, h), ("down", h, self.intermediate)]


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def add_rmsnorm(x, residual, w, y, eps):
    """x += residual (if given); y = rmsnorm(x) * w -- one fused kernel (f16)."""
    _lib.check(_lib.lib().abcq_add_rmsnorm_f16(x.data_ptr(), residual.data_ptr() if residual is not None else None,
                                               w.data_ptr(), y.data_ptr(), x.numel(), eps, _stream()),
               "abcq_add_rmsnorm_f16")


def silu_mul(g, u, a):
    _lib.check(_lib.lib().abcq_silu_mul_f16(g.data_ptr(), u.data_ptr(), a.data_ptr(), g.numel(), _stream()),
               "abcq_silu_mul_f16")


class _Argmax:
    """Greedy token: abcq_argmax_f16 over the logits (one PDL launch; torch.argmax
    took ~40 us on 128K logits) into a preallocated int64 scalar."""

    def __init__(self, device):
        n = C.c_size_t()
        _lib.check(_lib.lib().abcq_argmax_workspace_bytes(C.byref(n)))
        self.ws = torch.zeros(int(n.value), dtype=torch.uint8, device=device)

    def __call__(self, logits, out):
        _lib.check(_lib.lib().abcq_argmax_f16(logits.data_ptr(), logits.numel(), out.data_ptr(), self.ws.data_ptr(),
                                              self.ws.numel(), _stream()), "abcq_argmax_f16")
        return out


def _rope_tables(cfg: LlamaConfig, pos: int, device):
    d = cfg.head_dim
    inv = 1.0 / (cfg.rope_theta ** (torch.arange(0, d, 2, device=device, dtype=torch.float64) / d))
    ang = pos * inv
    return torch.cos(ang).float(), torch.sin(ang).float()


class _Attention:
    """KV cache (layers, kv_heads, ctx + 1, d) + the fused RoPE/append and
    split-L GQA decode kernels; the new token sits at position `ctx`."""

    def __init__(self, cfg: LlamaConfig, ctx: int, device, gen):
        self.cfg, self.ctx, self.lmax = cfg, ctx, ctx + 1
        shape = (cfg.layers, cfg.kv_heads, self.lmax, cfg.head_dim)
        self.k_cache = torch.randn(shape, device=device, dtype=torch.float16, generator=gen)
        self.v_cache = torch.randn(shape, device=device, dtype=torch.float16, generator=gen)
        self.cos, self.sin = _rope_tables(cfg, ctx, device)
        self.scale = 1.0 / math.sqrt(cfg.head_dim)
        n = C.c_size_t()
        _lib.check(_lib.lib().abcq_attn_decode_workspace_bytes(cfg.heads, self.lmax, C.byref(n)))
        self.ws = torch.zeros(int(n.value), dtype=torch.uint8, device=device)  # (fused: self-resetting counters)
        self.fused = True  # rope + append + attention + combine in one launch
        self.out = torch.empty(cfg.hidden, dtype=torch.float16, device=device)

    def __call__(self, layer: int, q, k, v):
        cfg, L = self.cfg, _lib.lib()
        kc, vc = self.k_cache[layer], self.v_cache[layer]
        if self.fused:
            _lib.check(L.abcq_rope_attn_decode_f16(
                q.data_ptr(), k.data_ptr(), v.data_ptr(), self.cos.data_ptr(), self.sin.data_ptr(), kc.data_ptr(),
                vc.data_ptr(), cfg.heads, cfg.kv_heads, self.lmax, self.ctx, self.scale, self.out.data_ptr(),
                self.ws.data_ptr(), self.ws.numel(), _stream()), "abcq_rope_attn_decode_f16")
            return self.out
        _lib.check(L.abcq_rope_append_f16(q.data_ptr(), k.data_ptr(), v.data_ptr(), self.cos.data_ptr(),
                                          self.sin.data_ptr(), kc.data_ptr(), vc.data_ptr(), cfg.heads,
                                          cfg.kv_heads, cfg.head_dim, self.lmax, self.ctx, _stream()),
                   "abcq_rope_append_f16")
        _lib.check(L.abcq_attn_decode_f16(q.data_ptr(), kc.data_ptr(), vc.data_ptr(), cfg.heads, cfg.kv_heads,
                                          self.lmax, self.lmax, self.scale, self.out.data_ptr(), self.ws.data_ptr(),
                                          self.ws.numel(), _stream()), "abcq_attn_decode_f16")
        return self.out


# q/k/v and o: the cluster kernel (abcq_gemv) -- after round 2's changes to
# the persistent kernel it measured faster for them inside the step at every
# p (tools/decode_paths_ab.py: p2/p3/p4 2.069/2.304/2.420 vs 2.104/2.326/2.479
# ms/token); True routes them through the persistent batch kernel
PERSISTENT_QKV_O = False


def _persistent(m, p, x, out):
    """One GEMV through the persistent batch kernel (a batch of one); other
    linear objects (e.g. a dense test reference) through their own gemv()."""
    if isinstance(m, DeviceModel) and PERSISTENT_QKV_O:
        gemv_batch([(m, p, x, out)])
    else:
        m.gemv(p, x, out=out)


class QuantizedLlamaStep:
    """Decode step with AnyBCQ linears at precision p (p_lo..p_hi resident)."""

    def __init__(self, cfg: LlamaConfig = LlamaConfig(), p: int = 3, p_lo: int = 2, p_hi: int = 4,
                 ctx: int = 1024, device=None, seed: int = 0, fuse_glu: bool = True, stack_rows: bool = True,
                 fuse_norm: bool | None = None, fuse_norm_out: bool = False):
        self.cfg, self.p, self.fuse_glu, self.stack_rows = cfg, p, fuse_glu, stack_rows
        # fuse_norm_out: the add + RMSNorm after the o and down projections runs
        # as those GEMVs' epilogue (abcq_gemv_rmsnorm_out: the block that
        # completes the split-K sums last does stream += y; h = rmsnorm(stream)
        # * w, bitwise equal to the separate launch) -- two launches fewer per
        # layer, but measured slower: p3 2.37 vs 2.25 ms/token (the one-CTA
        # epilogue serialises at the grid's tail, where the separate 1-block
        # launch ran while the next GEMV's CTAs were already prefetching;
        # tools/decode_norm_out_ab.py), so off by default
        if fuse_norm and fuse_norm_out:
            raise ValueError("fuse_norm (GEMV input side) and fuse_norm_out (output side) are exclusive")
        self.fuse_norm_out = fuse_norm_out and fuse_glu and stack_rows
        # fuse_norm: add + RMSNorm formed inside the q/k/v and gate/up GEMVs'
        # table builds (abcq_gemv_add_rmsnorm on the persistent kernel, bitwise
        # equal to the separate launch + that GEMV). On by default (unless
        # fuse_norm_out): with round 2's persistent-kernel schedule it measures
        # p2/p3/p4 1.991/2.147/2.300 vs 1.994/2.337/2.434 ms/token for the
        # separate launch (tools/decode_norm_ab.py, medians of 3 alternated
        # rounds; early in round 2 it measured 2.14 vs 2.11 at p=3, the other way)
        self.fuse_norm = (not fuse_norm_out) if fuse_norm is None else fuse_norm
        self.device = torch.device(device or f"cuda:{torch.cuda.current_device()}")
        gen = torch.Generator(device=self.device).manual_seed(seed)
        self.layers = []
        for _ in range(cfg.layers):
            mats = {}
            shapes = cfg.linear_shapes()
            if stack_rows:  # q/k/v and gate/up as one row-stacked model each (BCQ is per row: exact)
                sh = {n: (r, c) for n, r, c in shapes}
                shapes = [("qkv", sh["q"][0] + sh["k"][0] + sh["v"][0], cfg.hidden), ("o",) + sh["o"],
                          ("gu", 2 * cfg.intermediate, cfg.hidden), ("down",) + sh["down"]]
            for name, r, c in shapes:
                dm = DeviceModel(r, c, 128, p_lo, p_hi, False, scale_dtype="f16", device=self.device)
                dm.load_planes(torch.randint(-2**31, 2**31 - 1, (p_hi, r, c // 32), dtype=torch.int32,
                                             device=self.device, generator=gen))
                for q in range(p_lo, p_hi + 1):
                    a = 0.01 + 0.1 * torch.randn(q, r, c // 128, device=self.device, generator=gen).abs()
                    dm.load_scale_set(q, a * (0.5 / math.sqrt(c)))  # keep activations O(1) across layers
                mats[name] = dm
            self.layers.append(mats)
        self.norm_w = [(torch.ones(cfg.hidden, device=self.device, dtype=torch.float16),
                        torch.ones(cfg.hidden, device=self.device, dtype=torch.float16)) for _ in range(cfg.layers)]
        self.final_norm = torch.ones(cfg.hidden, device=self.device, dtype=torch.float16)
        self.lm_head = (torch.randn(cfg.vocab, cfg.hidden, device=self.device, dtype=torch.float16,
                                    generator=gen) * 0.02)
        self.attn = _Attention(cfg, ctx, self.device, gen)
        hd, kvd, inter = cfg.hidden, cfg.kv_heads * cfg.head_dim, cfg.intermediate
        f16 = dict(device=self.device, dtype=torch.float16)
        self.x = torch.randn(hd, **f16, generator=gen)
        self.x_alt = torch.empty(hd, **f16)  # the fused norms write x + residual here (ping-pong)
        self.qkv = torch.empty(hd + 2 * kvd, **f16)
        self.q, self.k, self.v = self.qkv[:hd], self.qkv[hd:hd + kvd], self.qkv[hd + kvd:]
        self.o = torch.empty(hd, **f16)
        self.gu = torch.empty(2 * inter, **f16)   # [gate ; up]: the down GEMV's SiLU-gated input
        self.g, self.u = self.gu[:inter], self.gu[inter:]
        self.d = torch.empty(hd, **f16)
        self.h, self.act = torch.empty(hd, **f16), torch.empty(inter, **f16)
        self.token = torch.empty((), device=self.device, dtype=torch.int64)
        self.logits = torch.empty(cfg.vocab, **f16)
        self.argmax = _Argmax(self.device)

    def linear_bytes(self) -> int:
        """Algorithmic bytes the quantized linears read per step (planes + set p)."""
        p = self.p
        return sum(p * r * c // 8 + p * r * (c // 128) * 2 for _, r, c in self.cfg.linear_shapes()) * self.cfg.layers

    def _norm_linear(self, mats, name, cur, nxt, resid, w, out):
        """out = W rmsnorm(cur + resid) * w; returns the residual stream buffer
        after the add (nxt when the norm is fused into the GEMV, else cur)."""
        cfg, p = self.cfg, self.p
        dm = mats.get(name)
        if self.fuse_norm and self.stack_rows and isinstance(dm, DeviceModel):
            dm.gemv_add_rmsnorm(p, cur, resid, w, cfg.eps, out=out, x_out=nxt)
            return nxt
        add_rmsnorm(cur, resid, w, self.h, cfg.eps)
        if self.stack_rows:
            _persistent(dm, p, self.h, out) if name == "qkv" else dm.gemv(p, self.h, out=out)
        elif name == "qkv":
            gemv_batch([(mats["q"], p, self.h, self.q), (mats["k"], p, self.h, self.k),
                        (mats["v"], p, self.h, self.v)])
        else:
            gemv_batch([(mats["gate"], p, self.h, self.g), (mats["up"], p, self.h, self.u)])
        return cur

    def step(self):
        if self.fuse_norm_out:
            return self._step_norm_out()
        cfg, p = self.cfg, self.p
        resid = None
        cur, nxt = self.x, self.x_alt  # an even number of fused norms per step: it ends in self.x
        for li, mats in enumerate(self.layers):
            # q/k/v and o: see PERSISTENT_QKV_O
            new = self._norm_linear(mats, "qkv", cur, nxt, resid, self.norm_w[li][0], self.qkv)
            cur, nxt = (new, cur) if new is not cur else (cur, nxt)
            a = self.attn(li, self.q, self.k, self.v)
            _persistent(mats["o"], p, a, self.o)
            # y = [gate ; up]: exactly the down GEMV's SiLU-gated input layout
            new = self._norm_linear(mats, "gu", cur, nxt, self.o, self.norm_w[li][1], self.gu)
            cur, nxt = (new, cur) if new is not cur else (cur, nxt)
            if self.fuse_glu:  # silu(gate)*up formed inside the down GEMV's table build
                mats["down"].gemv(p, self.gu, out=self.d, silu_glu=True)
            else:
                silu_mul(self.g, self.u, self.act)
                mats["down"].gemv(p, self.act, out=self.d)
            resid = self.d
        assert cur is self.x
        add_rmsnorm(self.x, resid, self.final_norm, self.h, cfg.eps)
        torch.mv(self.lm_head, self.h, out=self.logits)
        return self.argmax(self.logits, self.token)

    def _step_norm_out(self):
        """The step with every add+RMSNorm but the first fused into the GEMV
        before it: o -> (x += o; h = norm2(x)), down -> (x += d; h = norm1 of
        the next layer, or the final norm). Same arithmetic as step()."""
        cfg, p = self.cfg, self.p
        n = len(self.layers)
        add_rmsnorm(self.x, None, self.norm_w[0][0], self.h, cfg.eps)
        for li, mats in enumerate(self.layers):
            _persistent(mats["qkv"], p, self.h, self.qkv)
            a = self.attn(li, self.q, self.k, self.v)
            _norm_out(mats["o"], p, a, self.o, self.x, self.norm_w[li][1], cfg.eps, self.h)
            mats["gu"].gemv(p, self.h, out=self.gu)
            w_next = self.norm_w[li + 1][0] if li + 1 < n else self.final_norm
            _norm_out(mats["down"], p, self.gu, self.d, self.x, w_next, cfg.eps, self.h, silu_glu=True)
        torch.mv(self.lm_head, self.h, out=self.logits)
        return self.argmax(self.logits, self.token)


def _norm_out(m, p, x, out, stream, w, eps, h, silu_glu=False):
    """out = W x, then stream += out; h = rmsnorm(stream) * w -- one launch for a
    DeviceModel (its norm epilogue), else the GEMV and the separate launch."""
    if isinstance(m, DeviceModel):
        m.gemv_rmsnorm_out(p, x, out, stream, w, eps, h, silu_glu=silu_glu)
    else:
        m.gemv(p, x, out=out, silu_glu=silu_glu) if silu_glu else m.gemv(p, x, out=out)
        add_rmsnorm(stream, out, w, h, eps)


class Fp16LlamaStep:
    """The same step with dense fp16 weights (cuBLAS), q/k/v and gate/up fused."""

    def __init__(self, cfg: LlamaConfig = LlamaConfig(), ctx: int = 1024, device=None, seed: int = 1):
        self.cfg = cfg
        self.device = torch.device(device or f"cuda:{torch.cuda.current_device()}")
        gen = torch.Generator(device=self.device).manual_seed(seed)
        f16 = dict(device=self.device, dtype=torch.float16)
        hd, kvd, inter = cfg.hidden, cfg.kv_heads * cfg.head_dim, cfg.intermediate
        s = 1.0 / math.sqrt(hd)
        self.layers = []
        for _ in range(cfg.layers):
            self.layers.append({
                "qkv": torch.randn(hd + 2 * kvd, hd, **f16, generator=gen) * s,
                "o": torch.randn(hd, hd, **f16, generator=gen) * s,
                "gu": torch.randn(2 * inter, hd, **f16, generator=gen) * s,
                "down": torch.randn(hd, inter, **f16, generator=gen) * (1.0 / math.sqrt(inter)),
            })
        self.norm_w = torch.ones(hd, **f16)
        self.lm_head = torch.randn(cfg.vocab, hd, **f16, generator=gen) * 0.02
        self.attn = _Attention(cfg, ctx, self.device, gen)
        self.x = torch.randn(hd, **f16, generator=gen)
        self.h, self.o, self.d = torch.empty(hd, **f16), torch.empty(hd, **f16), torch.empty(hd, **f16)
        self.qkv, self.gu = torch.empty(hd + 2 * kvd, **f16), torch.empty(2 * inter, **f16)
        self.act = torch.empty(inter, **f16)
        self.token = torch.empty((), device=self.device, dtype=torch.int64)
        self.logits = torch.empty(cfg.vocab, **f16)
        self.argmax = _Argmax(self.device)

    def linear_bytes(self) -> int:
        return sum(r * c * 2 for _, r, c in self.cfg.linear_shapes()) * self.cfg.layers

    def step(self):
        cfg = self.cfg
        hd, kvd, inter = cfg.hidden, cfg.kv_heads * cfg.head_dim, cfg.intermediate
        resid = None
        for li, w in enumerate(self.layers):
            add_rmsnorm(self.x, resid, self.norm_w, self.h, cfg.eps)
            torch.mv(w["qkv"], self.h, out=self.qkv)
            a = self.attn(li, self.qkv[:hd], self.qkv[hd:hd + kvd], self.qkv[hd + kvd:])
            torch.mv(w["o"], a, out=self.o)
            add_rmsnorm(self.x, self.o, self.norm_w, self.h, cfg.eps)
            torch.mv(w["gu"], self.h, out=self.gu)
            silu_mul(self.gu[:inter], self.gu[inter:], self.act)
            torch.mv(w["down"], self.act, out=self.d)
            resid = self.d
        add_rmsnorm(self.x, resid, self.norm_w, self.h, cfg.eps)
        torch.mv(self.lm_head, self.h, out=self.logits)
        return self.argmax(self.logits, self.token)


def time_step(model, iters: int = 20, warmup: int = 3) -> float:
    """ms per decode step: the whole step captured as one CUDA graph, replayed
    back to back, CUDA events on the replay stream."""
    st = torch.cuda.Stream(device=model.device)
    with torch.cuda.stream(st):
        for _ in range(warmup):
            model.step()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        model.step()
    with torch.cuda.stream(st):
        for _ in range(warmup):
            g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(iters):
            g.replay()
        b.record(st)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters
