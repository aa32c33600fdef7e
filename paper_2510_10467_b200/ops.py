"""Torch operators over the C ABI: `torch.ops.anybcq_b200.*` (SURVEY §8b,
"the device path is exposed as a TORCH_LIBRARY op ... for the decode harness").

The reference has no device operator; its innermost boundary is the numba
`_lut_kernel` driven by `GemvEngine.lut` (`/root/reference/pkg/src/anybcq/gemv.py:84-95,188-222`),
which returns host f64. These ops are the device-resident form of the same
computation, for callers that stay on the GPU (a decoder, a CUDA graph, a
torch program): inputs and outputs are CUDA tensors, the launch is
asynchronous on torch's current stream, and every op is a thin wrapper over
one C-ABI entry point of libanybcq_b200.so (include/anybcq_b200.h) — no
torch types cross the ABI.

A `DeviceModel` is const device memory shared by all calls (gemv.py:99-103);
ops name it by an integer handle from `register()`, so the schema stays
plain (`int`, `Tensor`, `int[]`) and the ops work under CUDA-graph capture
and FakeTensor tracing (the fake kernels read only the model's shape).

    h = ops.register(dm)
    y = torch.ops.anybcq_b200.gemv(h, x, 3)                  # y = W_3 x
    Y = torch.ops.anybcq_b200.gemm_mixedp(h, X, [2, 4, 3])   # per-request p
"""

from __future__ import annotations

import itertools
import threading

import torch

from .errors import UsageError

_LOCK = threading.Lock()
_MODELS: dict[int, object] = {}
_NEXT = itertools.count(1)


def register(model) -> int:
    """Make `model` (a DeviceModel) addressable by the ops; returns its handle."""
    for attr in ("rows", "cols"):
        if not hasattr(model, attr):
            raise UsageError(f"register() needs a DeviceModel, got {type(model).__name__}")
    with _LOCK:
        h = next(_NEXT)
        _MODELS[h] = model
    return h


def unregister(handle: int) -> None:
    with _LOCK:
        _MODELS.pop(int(handle), None)


def model(handle: int):
    try:
        return _MODELS[int(handle)]
    except KeyError:
        raise UsageError(f"unknown model handle {handle}") from None


def _out_dtype(t: torch.Tensor) -> torch.dtype:
    # y in the activation's width (f16 decode / f32 parity); the kernels write f16 or f32
    return t.dtype if t.dtype in (torch.float16, torch.float32) else torch.float32


@torch.library.custom_op("anybcq_b200::gemv", mutates_args=())
def gemv(handle: int, x: torch.Tensor, p: int) -> torch.Tensor:
    """y = Σ_{i<p} α^(p)_i ⊙ (B_i x), batch 1 (abcq_gemv). x: (cols,) f16/f32 CUDA."""
    m = model(handle)
    if x.dtype not in (torch.float16, torch.float32):
        x = x.float()
    return m.gemv(p, x.reshape(-1), out_dtype=_out_dtype(x))


@gemv.register_fake
def _gemv_fake(handle: int, x: torch.Tensor, p: int) -> torch.Tensor:
    m = model(handle)
    if x.numel() != m.cols:
        raise UsageError(f"input length {x.numel()} != cols {m.cols}")
    return x.new_empty((m.rows,), dtype=_out_dtype(x))


@torch.library.custom_op("anybcq_b200::gemm_mixedp", mutates_args=())
def gemm_mixedp(handle: int, X: torch.Tensor, ps: list[int]) -> torch.Tensor:
    """Y[b] = W_{ps[b]} X[b] for B <= 16 requests in one pass over the planes
    (abcq_gemm_mixedp). X: (B, cols) CUDA; Y: (B, rows) in X's width."""
    return model(handle).gemm_mixedp(list(ps), X, out_dtype=_out_dtype(X))


@gemm_mixedp.register_fake
def _gemm_mixedp_fake(handle: int, X: torch.Tensor, ps: list[int]) -> torch.Tensor:
    m = model(handle)
    if X.dim() != 2 or X.shape[0] != len(ps) or X.shape[1] != m.cols:
        raise UsageError(f"X must be ({len(ps)}, {m.cols}), got {tuple(X.shape)}")
    return X.new_empty((len(ps), m.rows), dtype=_out_dtype(X))


@torch.library.custom_op("anybcq_b200::dequantize", mutates_args=())
def dequantize(handle: int, p: int, like: torch.Tensor) -> torch.Tensor:
    """Dense Ŵ_p (rows, cols) in `like`'s dtype/device (bcq.py:372-378; abcq_dequantize)."""
    return model(handle).dequantize(p, dtype=_out_dtype(like))


@dequantize.register_fake
def _dequantize_fake(handle: int, p: int, like: torch.Tensor) -> torch.Tensor:
    m = model(handle)
    return like.new_empty((m.rows, m.cols), dtype=_out_dtype(like))
