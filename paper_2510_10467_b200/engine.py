"""Drop-in GEMV engine -- mirrors the reference module anybcq.gemv
(/root/reference/pkg/src/anybcq/gemv.py) on the B200.

Same names, signatures, return types and error behaviour:

  * GemvEngine(model, chunk_width=8)            gemv.py:98-128
      .lut(p, x)   -> (y float64 [N], GemvStats)  gemv.py:188-222
      .naive(p, x) -> (y float64 [N], GemvStats)  gemv.py:170-186
  * gemv_lut / gemv_naive                       gemv.py:253-258
  * LookupTable.build                           gemv.py:55-81
  * dequant_oracle, dense_gemv_reference        gemv.py:261-277
  * GemvStats, BenchRow, bench, render_*        gemv.py:47-52, 284-367

UsageError is raised for a precision outside [p_lo, p_hi], a wrong input
length or a bad chunk width, before any device work (gemv.py:106-108,148-156).
All arithmetic runs in libanybcq_b200.so on the GPU; the host only moves x in
and y out. `chunk_width` is validated and recorded for API compatibility: the
device kernels always use the mu=8 table (mu=4 gives the same function).
Extra device-side API: GemvEngine.gemv(p, x_tensor) returns a device tensor
without synchronising (the decode / serving path).
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .device_model import DeviceModel, require_cuda
from .errors import UsageError
from .model import group_bounds, group_count

CHUNK_WIDTHS = (4, 8)


@dataclass
class GemvStats:
    """Exact traffic counters of one call (gemv.py:47-52, 158-168)."""

    plane_bytes_fetched: int
    scale_bytes_fetched: int
    lut_build_count: int
    elapsed_s: float


@dataclass(frozen=True, eq=False)
class LookupTable:
    """Signed partial sums of every chunk of x, built on the GPU
    (abcq_lut_build), bit-identical to gemv.py:67-81."""

    chunk_width: int
    tables: np.ndarray  # (chunks, 2^chunk_width) float32

    @classmethod
    def build(cls, x, chunk_width: int, device=None) -> "LookupTable":
        if not 1 <= chunk_width <= 8:
            raise UsageError(f"chunk width must be in [1, 8], got {chunk_width}")
        dev = require_cuda(device)
        xd = torch.as_tensor(np.asarray(x, dtype=np.float32).ravel()).to(dev)
        chunks = (xd.numel() + chunk_width - 1) // chunk_width
        out = torch.empty(chunks, 1 << chunk_width, dtype=torch.float32, device=dev)
        with torch.cuda.device(dev):
            _lib.check(_lib.lib().abcq_lut_build(xd.data_ptr(), _lib.F32, xd.numel(), chunk_width,
                                                 out.data_ptr(), torch.cuda.current_stream().cuda_stream),
                       "abcq_lut_build")
        return cls(chunk_width, out.cpu().numpy())


class GemvEngine:
    """Executes GEMV against one immutable model at any servable precision.

    The model's planes and every scale set are uploaded once at construction
    (DeviceModel); calls at different precisions share them and never modify
    them (gemv.py:99-103).
    """

    def __init__(self, model, chunk_width: int = 8, *, scale_dtype: str = "f32", device=None):
        if chunk_width not in CHUNK_WIDTHS:
            raise UsageError(f"chunk width must be one of {CHUNK_WIDTHS}")
        self.model = model
        self.chunk_width = chunk_width
        self.rows, self.cols = model.shape
        self.group_size = model.config.group_size
        self.groups = group_count(self.cols, self.group_size)
        self.chunks = (self.cols + chunk_width - 1) // chunk_width
        self.aligned = self.group_size % chunk_width == 0 or self.groups == 1
        self.device_model = (model if isinstance(model, DeviceModel)
                             else DeviceModel.from_model(model, scale_dtype=scale_dtype, device=device))
        self.device = self.device_model.device

    # ---- reference-compatible host API ----------------------------------------
    def _validate(self, p: int, x) -> np.ndarray:
        if p not in self.model.precisions:
            raise UsageError(f"precision {p} outside [{self.model.p_lo}, {self.model.p_hi}]")
        x = np.asarray(x, dtype=np.float64).ravel()
        if len(x) != self.cols:
            raise UsageError(f"input length {len(x)} != cols {self.cols}")
        return x

    def _stats(self, p: int, lut_builds: int, elapsed: float) -> GemvStats:
        wpr = (self.cols + 31) // 32
        scale_bytes = p * self.rows * self.groups * 4
        if self.model.config.asymmetric:
            scale_bytes += self.rows * self.groups * 4
        return GemvStats(p * self.rows * wpr * 4, scale_bytes, lut_builds, elapsed)

    def _run(self, fn, p, x):
        x = self._validate(p, x)
        t0 = time.perf_counter()
        with torch.cuda.device(self.device):
            xd = torch.from_numpy(x.astype(np.float32)).to(self.device, non_blocking=True)
            y = fn(p, xd)
            out = y.to("cpu").numpy().astype(np.float64)
        return out, time.perf_counter() - t0

    def lut(self, p: int, x) -> tuple[np.ndarray, GemvStats]:
        """Table path on the sm_100a kernel: one table build per call."""
        y, dt = self._run(self.device_model.gemv, p, x)
        return y, self._stats(p, 1, dt)

    def naive(self, p: int, x) -> tuple[np.ndarray, GemvStats]:
        """Column-decode path (generic kernel, f64 accumulation)."""
        y, dt = self._run(self.device_model.gemv_naive, p, x)
        return y, self._stats(p, 0, dt)

    # ---- device API -----------------------------------------------------------
    def gemv(self, p: int, x: torch.Tensor, out=None, out_dtype=torch.float32, stream=None) -> torch.Tensor:
        """Asynchronous device GEMV: x (cols,) f32/f16 CUDA tensor -> y (rows,)."""
        if p not in self.model.precisions:
            raise UsageError(f"precision {p} outside [{self.model.p_lo}, {self.model.p_hi}]")
        return self.device_model.gemv(p, x, out=out, out_dtype=out_dtype, stream=stream)


def gemv_naive(model, p: int, x):
    return GemvEngine(model).naive(p, x)


def gemv_lut(model, p: int, x, chunk_width: int = 8):
    return GemvEngine(model, chunk_width).lut(p, x)


def dense_gemv_reference(w, x, group_size: int = 128, device=None) -> np.ndarray:
    """Dense f32 GEMV baseline (gemv.py:261-269), as a cuBLAS matvec on the GPU."""
    dev = require_cuda(device)
    wd = torch.as_tensor(np.asarray(w, dtype=np.float32)).to(dev)
    xd = torch.as_tensor(np.asarray(x, dtype=np.float32).ravel()).to(dev)
    return (wd @ xd).cpu().numpy()


def dequant_oracle(model, p: int, x) -> np.ndarray:
    """Dense-reconstruction product (gemv.py:272-277): W_p reconstructed on the
    GPU (abcq_dequantize, f64 sum -> f32), then an f64 matvec."""
    dm = model if isinstance(model, DeviceModel) else DeviceModel.from_model(model)
    w = dm.dequantize(p).to(torch.float64)
    xd = torch.as_tensor(np.asarray(x, dtype=np.float64).ravel()).to(dm.device)
    return (w @ xd).cpu().numpy()


# ---------------------------------------------------------------------------
# benchmarking (gemv.py:284-367), timed on the device with CUDA events
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class BenchRow:
    rows: int
    cols: int
    path: str
    precision: int
    median_us: float
    min_us: float
    plane_bytes: int
    scale_bytes: int


def _time_device(fn, repeats: int, warmup: int = 1, inner: int = 32) -> tuple[float, float]:
    """Median/min device microseconds per call; each sample times `inner`
    back-to-back launches between CUDA events so host enqueue gaps do not
    count (the reference times single calls with perf_counter, gemv.py:296-305)."""
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(max(warmup, 1)):  # also allocates the stream's workspace
            fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()  # the `inner` launches replay without host gaps
    with torch.cuda.graph(g, stream=s):
        for _ in range(inner):
            fn()
    times = []
    with torch.cuda.stream(s):
        g.replay()
        for _ in range(repeats):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            g.replay()
            b.record(s)
            b.synchronize()
            times.append(a.elapsed_time(b) * 1e3 / inner)
    arr = np.asarray(times)
    return float(np.median(arr)), float(arr.min())


def bench(model, precisions, x, repeats: int = 32, paths=("naive", "lut"),
          include_dense: bool = False, dense_weights=None, include_dense_f16: bool = False) -> list[BenchRow]:
    """Median/min device latency per (path, precision) with exact counters.

    include_dense: the reference's dense row ("dense", 32, rows*cols*4) --
    the f32 GEMV of the p_hi weights (dequantized, or `dense_weights`), here a
    cuBLAS f32 matvec (gemv.py:335-344). include_dense_f16: an extra
    ("dense_f16", 16, rows*cols*2) row, the cuBLAS half-precision GEMV the
    north star compares against."""
    if repeats < 1:
        raise UsageError("repeats must be >= 1")
    for path in paths:
        if path not in ("naive", "lut"):
            raise UsageError(f"unknown path {path!r}")
    engine = GemvEngine(model)
    dm = engine.device_model
    xd = torch.as_tensor(np.asarray(x, dtype=np.float32).ravel()).to(dm.device)
    rows, cols = model.shape
    out = []
    with torch.cuda.device(dm.device):
        for path in paths:
            runner = dm.gemv if path == "lut" else dm.gemv_naive
            for p in precisions:
                engine._validate(p, np.zeros(cols))
                med, lo = _time_device(lambda: runner(p, xd), repeats)
                st = engine._stats(p, 0, 0.0)
                out.append(BenchRow(rows, cols, path, p, med, lo, st.plane_bytes_fetched,
                                    st.scale_bytes_fetched))
        if include_dense or include_dense_f16:
            if dense_weights is None:
                wf = dm.dequantize(model.p_hi, torch.float32)
            else:
                wf = torch.as_tensor(np.asarray(dense_weights, dtype=np.float32)).to(dm.device)
        if include_dense:
            med, lo = _time_device(lambda: torch.mv(wf, xd), repeats)
            out.append(BenchRow(rows, cols, "dense", 32, med, lo, rows * cols * 4, 0))
        if include_dense_f16:
            wh, xh = wf.half(), xd.half()
            med, lo = _time_device(lambda: torch.mv(wh, xh), repeats)
            out.append(BenchRow(rows, cols, "dense_f16", 16, med, lo, rows * cols * 2, 0))
    return out


def render_bench_text(rows: list[BenchRow]) -> str:
    header = (f"{'shape':<14}{'path':<8}{'p':>3}{'median_us':>12}"
              f"{'plane_bytes':>14}{'scale_bytes':>13}{'GB/s':>10}")
    lines = [header]
    for r in rows:
        gbs = (r.plane_bytes + r.scale_bytes) / (r.median_us * 1e-6) / 1e9 if r.median_us else 0.0
        lines.append(f"{str(r.rows) + 'x' + str(r.cols):<14}{r.path:<8}{r.precision:>3}"
                     f"{r.median_us:>12.2f}{r.plane_bytes:>14}{r.scale_bytes:>13}{gbs:>10.1f}")
    return "\n".join(lines)


def render_bench_csv(rows: list[BenchRow]) -> str:
    lines = ["shape,path,p,median_us,plane_bytes,scale_bytes"]
    for r in rows:
        lines.append(f"{r.rows}x{r.cols},{r.path},{r.precision},"
                     f"{r.median_us:.2f},{r.plane_bytes},{r.scale_bytes}")
    return "\n".join(lines)


__all__ = ["BenchRow", "GemvEngine", "GemvStats", "LookupTable", "bench", "dense_gemv_reference",
           "dequant_oracle", "gemv_lut", "gemv_naive", "render_bench_csv", "render_bench_text",
           "group_bounds"]
