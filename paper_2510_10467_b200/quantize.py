"""BCQ fitting on the GPU: the producer of the planes and scale sets the GEMV
path serves. Same names, arguments, return types and
errors as the reference's fitting API (/root/reference/pkg/src/anybcq/
bcq.py:298-391, progressive.py:82-175); the f64 fitting internals run as CUDA
kernels (csrc/abcq_quantize.cu, C ABI abcq_fit_*):

    greedy_init           bcq.py:298-306   (_greedy64, bcq.py:160-180)
    ls_update_scales      bcq.py:309-324   (_ls64 / _solve_psd_batch, bcq.py:183-230)
    bs_recalibrate_codes  bcq.py:327-339   (_bs_codes64, bcq.py:269-295)
    alternate_fit         bcq.py:342-369
    expand_step           progressive.py:105-145
    build_multiprecision  progressive.py:148-168
    precision_errors      progressive.py:171-175

Codes live on the device as int8 (q, rows, cols) of -1/+1 between the steps;
only the results (packed words, f32 scales) come back to the host.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .device_model import _stream_handle, require_cuda
from .errors import NonFiniteError, UsageError
from .model import BitPlaneSet, MultiPrecisionModel, QuantConfig, ScaleTensor, group_count, words_per_row

MAX_PLANES = _lib.ABCQ_MAX_PLANES
MAX_GROUP = 1024


@dataclass(frozen=True, eq=False)
class QuantizedMatrix:
    """Planes + one scale set (bcq.py:99-123)."""

    bitplanes: BitPlaneSet
    scales: ScaleTensor
    config: QuantConfig

    def __post_init__(self):
        if self.bitplanes.planes != self.scales.planes:
            raise UsageError(f"{self.bitplanes.planes} planes but {self.scales.planes} scale planes")
        if self.scales.rows != self.bitplanes.rows:
            raise UsageError("scale rows do not match plane rows")
        if self.scales.groups != group_count(self.bitplanes.cols, self.scales.group_size):
            raise UsageError("scale groups do not match cols/group_size")

    @property
    def planes(self) -> int:
        return self.bitplanes.planes

    @property
    def shape(self) -> tuple[int, int]:
        return self.bitplanes.rows, self.bitplanes.cols


def _validate(w, name="weights") -> np.ndarray:
    """tensor_io.validate_matrix (tensor_io.py:40-49): 2-D, non-empty, finite, f32."""
    w = np.ascontiguousarray(w, dtype=np.float32)
    if w.ndim != 2:
        raise UsageError(f"{name} must be 2-D, got shape {w.shape}")
    if w.shape[0] < 1 or w.shape[1] < 1:
        raise UsageError(f"{name} dimensions must be >= 1, got {w.shape}")
    if not np.isfinite(w).all():
        raise NonFiniteError(f"{name} contains NaN or Inf")
    return w


class _Fit:
    """Device state of one fit: w (f64), codes (int8), alpha / offset (f64)."""

    def __init__(self, w: np.ndarray, group_size: int, asym: bool, device=None):
        if group_size > MAX_GROUP:
            raise UsageError(f"group_size {group_size} > {MAX_GROUP} (device fitting)")
        self.dev = require_cuda(device)
        self.rows, self.cols = w.shape
        self.g, self.asym = int(group_size), bool(asym)
        self.G = group_count(self.cols, self.g)
        self.w = torch.from_numpy(w.astype(np.float64)).to(self.dev)
        self.L = _lib.lib()

    def st(self):
        return _stream_handle(None)

    def greedy(self, q: int):
        codes = torch.empty((q, self.rows, self.cols), dtype=torch.int8, device=self.dev)
        alpha = torch.zeros((q, self.rows, self.G), dtype=torch.float64, device=self.dev)
        offset = torch.empty((self.rows, self.G), dtype=torch.float64, device=self.dev) if self.asym else None
        scratch = torch.empty((self.rows, self.cols), dtype=torch.float64, device=self.dev)
        _lib.check(self.L.abcq_fit_greedy(self.w.data_ptr(), self.rows, self.cols, self.g, q, int(self.asym),
                                          codes.data_ptr(), alpha.data_ptr(), _lib.ptr(offset), scratch.data_ptr(),
                                          self.st()), "abcq_fit_greedy")
        return codes, alpha, offset

    def ls(self, codes):
        q = codes.shape[0]
        alpha = torch.empty((q, self.rows, self.G), dtype=torch.float64, device=self.dev)
        offset = torch.empty((self.rows, self.G), dtype=torch.float64, device=self.dev) if self.asym else None
        ridged = torch.zeros(1, dtype=torch.int32, device=self.dev)
        _lib.check(self.L.abcq_fit_ls(self.w.data_ptr(), codes.data_ptr(), q, self.rows, self.cols, self.g,
                                      int(self.asym), alpha.data_ptr(), _lib.ptr(offset), ridged.data_ptr(),
                                      self.st()), "abcq_fit_ls")
        return alpha, offset, ridged

    def bs(self, alpha, offset, out=None):
        q = alpha.shape[0]
        codes = out if out is not None else torch.empty((q, self.rows, self.cols), dtype=torch.int8,
                                                        device=self.dev)
        _lib.check(self.L.abcq_fit_bs(self.w.data_ptr(), alpha.data_ptr(), _lib.ptr(offset), q, self.rows,
                                      self.cols, self.g, codes.data_ptr(), self.st()), "abcq_fit_bs")
        return codes

    def residual_sign(self, codes, alpha, offset):
        q = codes.shape[0]
        plane = torch.empty((self.rows, self.cols), dtype=torch.int8, device=self.dev)
        _lib.check(self.L.abcq_fit_residual_sign(self.w.data_ptr(), codes.data_ptr(), alpha.data_ptr(),
                                                 _lib.ptr(offset), q, self.rows, self.cols, self.g,
                                                 plane.data_ptr(), self.st()), "abcq_fit_residual_sign")
        return plane

    def dequant(self, codes, alpha, offset):
        return _dequant64(codes, alpha, offset, self.g)

    def sq_error(self, codes, alpha, offset) -> float:
        d = self.w - self.dequant(codes, alpha, offset)
        return float((d * d).sum())


def _dequant64(codes, alpha, offset, g: int) -> torch.Tensor:
    """_dequant64 (bcq.py:137-152) on the device: planes ascending, offset last."""
    q, rows, cols = codes.shape
    idx = torch.arange(cols, device=codes.device) // g
    rec = torch.zeros((rows, cols), dtype=torch.float64, device=codes.device)
    for i in range(q):
        rec += codes[i].to(torch.float64) * alpha[i][:, idx]
    if offset is not None:
        rec += offset[:, idx]
    return rec


def _pack(codes: torch.Tensor) -> BitPlaneSet:
    """int8 codes (q, rows, cols) on the device -> packed words (packing.py:22-30)."""
    q, rows, cols = codes.shape
    wpr = words_per_row(cols)
    bits = torch.zeros((q, rows, wpr * 32), dtype=torch.int64, device=codes.device)
    bits[..., :cols] = (codes > 0).to(torch.int64)
    shifts = torch.arange(32, device=codes.device, dtype=torch.int64)
    words = (bits.view(q, rows, wpr, 32) << shifts).sum(-1)
    return BitPlaneSet(q, rows, cols, words.cpu().numpy().astype(np.uint32))


def _scales(alpha, offset, cfg) -> ScaleTensor:
    return ScaleTensor(alpha=alpha.cpu().numpy().astype(np.float32),
                       offset=None if offset is None else offset.cpu().numpy().astype(np.float32),
                       group_size=cfg.group_size)


def _freeze(codes, alpha, offset, cfg) -> QuantizedMatrix:
    return QuantizedMatrix(_pack(codes), _scales(alpha, offset, cfg), cfg)


def _codes_dev(bitplanes, dev) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(bitplanes.codes())).to(dev)


def _check_q(q):
    if not 1 <= q <= MAX_PLANES:
        raise UsageError(f"plane count must be in [1, {MAX_PLANES}], got {q}")


# ---------------------------------------------------------------------------
# public operations (bcq.py:298-391)
# ---------------------------------------------------------------------------

def greedy_init(w, q: int, cfg: QuantConfig) -> QuantizedMatrix:
    """Residual-sign initialization: plane i+1 signs the running residual,
    its scale is the group mean absolute residual."""
    w = _validate(w)
    _check_q(q)
    f = _Fit(w, cfg.group_size, cfg.asymmetric)
    return _freeze(*f.greedy(q), cfg)


def ls_update_scales(w, qm: QuantizedMatrix) -> ScaleTensor:
    """Refit all scales (and offset) by per-group ordinary least squares with
    the planes fixed; degenerate groups fall back to a small ridge."""
    w = _validate(w)
    if w.shape != qm.shape:
        raise UsageError(f"weights {w.shape} do not match model {qm.shape}")
    f = _Fit(w, qm.config.group_size, qm.config.asymmetric)
    alpha, offset, _ = f.ls(_codes_dev(qm.bitplanes, f.dev))
    return _scales(alpha, offset, qm.config)


def bs_recalibrate_codes(w, scales: ScaleTensor) -> BitPlaneSet:
    """Reassign every code to the nearest representable level given fixed
    scales (the optimum over all 2^q sign patterns per weight)."""
    w = _validate(w)
    if w.shape[0] != scales.rows:
        raise UsageError(f"weights rows {w.shape[0]} != scale rows {scales.rows}")
    if group_count(w.shape[1], scales.group_size) != scales.groups:
        raise UsageError("weights cols do not match scale groups")
    if scales.planes > MAX_PLANES:
        raise UsageError(f"recalibration limited to {MAX_PLANES} planes, got {scales.planes}")
    f = _Fit(w, scales.group_size, scales.offset is not None)
    alpha = torch.from_numpy(scales.alpha.astype(np.float64)).to(f.dev)
    offset = None if scales.offset is None else torch.from_numpy(scales.offset.astype(np.float64)).to(f.dev)
    return _pack(f.bs(alpha, offset))


def alternate_fit(w, q: int, cfg: QuantConfig, trace: list | None = None) -> QuantizedMatrix:
    """Greedy initialization plus cfg.cycles alternating refinement cycles
    (scale least squares, then code recalibration); `trace` receives the
    total squared error after the init and after every half-step."""
    w = _validate(w)
    _check_q(q)
    f = _Fit(w, cfg.group_size, cfg.asymmetric)
    codes, alpha, offset = f.greedy(q)
    if trace is not None:
        trace.append(f.sq_error(codes, alpha, offset))
    for _ in range(cfg.cycles):
        alpha, offset, _ = f.ls(codes)
        if trace is not None:
            trace.append(f.sq_error(codes, alpha, offset))
        f.bs(alpha, offset, out=codes)
        if trace is not None:
            trace.append(f.sq_error(codes, alpha, offset))
    return _freeze(codes, alpha, offset, cfg)


def dequantize(qm: QuantizedMatrix, p: int) -> np.ndarray:
    """Dense f32 reconstruction from the first p planes and their scales (bcq.py:372-378)."""
    if not 1 <= p <= qm.planes:
        raise UsageError(f"precision {p} out of range [1, {qm.planes}]")
    dev = require_cuda()
    codes = _codes_dev(qm.bitplanes.prefix(p), dev)
    alpha = torch.from_numpy(qm.scales.alpha[:p].astype(np.float64)).to(dev)
    off = qm.scales.offset
    offset = None if off is None else torch.from_numpy(off.astype(np.float64)).to(dev)
    return _dequant64(codes, alpha, offset, qm.config.group_size).to(torch.float32).cpu().numpy()


def relative_reconstruction_error(w, qm: QuantizedMatrix, p: int | None = None) -> float:
    """||w - dequantize(qm, p)||^2 / ||w||^2 (bcq.py:381-400)."""
    w = _validate(w)
    p = qm.planes if p is None else p
    denom = float(np.dot(w.ravel().astype(np.float64), w.ravel().astype(np.float64)))
    if denom == 0.0:
        return 0.0
    d = w.astype(np.float64) - dequantize(qm, p).astype(np.float64)
    return float(np.dot(d.ravel(), d.ravel())) / denom


# ---------------------------------------------------------------------------
# progressive precision (progressive.py:105-175)
# ---------------------------------------------------------------------------

def _expand(f: _Fit, codes, alpha_prev, offset_prev, cycles: int):
    """One precision up: `cycles` rounds of sign(residual of the frozen planes
    under the current set) -> the new plane, then a least-squares refit of all
    p scales (+ offset). Returns (new plane, alpha, offset)."""
    q = codes.shape[0]
    alpha = torch.cat([alpha_prev, torch.zeros((1,) + tuple(alpha_prev.shape[1:]), dtype=torch.float64,
                                               device=f.dev)])
    offset = offset_prev
    plane = torch.ones((f.rows, f.cols), dtype=torch.int8, device=f.dev)  # sign(0) convention
    for _ in range(cycles):
        plane = f.residual_sign(codes, alpha[:q], offset)
        stacked = torch.cat([codes, plane[None]])
        alpha, offset, _ = f.ls(stacked)
    return plane, alpha, offset


def expand_step(w, model: MultiPrecisionModel, p: int) -> MultiPrecisionModel:
    """Add precision p = model.p_hi + 1: existing planes and scale sets are
    reused unchanged (the planes below p stay byte-identical)."""
    w = _validate(w)
    if w.shape != model.shape:
        raise UsageError(f"weights {w.shape} do not match model {model.shape}")
    if p != model.p_hi + 1:
        raise UsageError(f"next precision is {model.p_hi + 1}, got {p}")
    if p > MAX_PLANES:
        raise UsageError(f"precision {p} exceeds the {MAX_PLANES}-plane limit")
    cfg = model.config
    f = _Fit(w, cfg.group_size, cfg.asymmetric)
    prev = model.scale_sets[model.p_hi]
    codes = _codes_dev(model.bitplanes, f.dev)
    alpha_prev = torch.from_numpy(prev.alpha.astype(np.float64)).to(f.dev)
    offset_prev = None if prev.offset is None else torch.from_numpy(prev.offset.astype(np.float64)).to(f.dev)
    plane, alpha, offset = _expand(f, codes, alpha_prev, offset_prev, cfg.cycles)
    new = _pack(plane[None])
    words = np.concatenate([model.bitplanes.words, new.words], axis=0)
    planes = BitPlaneSet(p, model.bitplanes.rows, model.bitplanes.cols, words)
    assert planes.words[: p - 1].tobytes() == model.bitplanes.words.tobytes(), "frozen planes were modified"
    sets = dict(model.scale_sets)
    sets[p] = _scales(alpha, offset, cfg)
    return MultiPrecisionModel(planes, sets, model.p_lo, p, cfg)


def build_multiprecision(w, p_lo: int, p_hi: int, cfg: QuantConfig) -> MultiPrecisionModel:
    """Fit the base precision (alternate_fit), then expand one bit at a time
    up to p_hi -- one device-resident fit, no host round trip between steps."""
    w = _validate(w)
    if not 1 <= p_lo <= p_hi <= MAX_PLANES:
        raise UsageError(f"invalid precision range [{p_lo}, {p_hi}]")
    f = _Fit(w, cfg.group_size, cfg.asymmetric)
    codes, alpha, offset = f.greedy(p_lo)
    for _ in range(cfg.cycles):
        alpha, offset, _ = f.ls(codes)
        f.bs(alpha, offset, out=codes)
    sets = {p_lo: (alpha, offset)}
    for p in range(p_lo + 1, p_hi + 1):
        # expand from the STORED (f32) previous set, as expand_step does (progressive.py:121-124)
        alpha = alpha.to(torch.float32).to(torch.float64)
        offset = None if offset is None else offset.to(torch.float32).to(torch.float64)
        plane, alpha, offset = _expand(f, codes, alpha, offset, cfg.cycles)
        codes = torch.cat([codes, plane[None]])
        sets[p] = (alpha, offset)
    planes = _pack(codes)
    return MultiPrecisionModel(planes, {p: _scales(a, o, cfg) for p, (a, o) in sets.items()}, p_lo, p_hi, cfg)


def precision_errors(w, model: MultiPrecisionModel) -> dict[int, float]:
    """Relative squared reconstruction error at every servable precision."""
    w = _validate(w)
    out = {}
    for p in model.precisions:
        qm = QuantizedMatrix(model.bitplanes.prefix(p), model.scale_sets[p], model.config)
        out[p] = relative_reconstruction_error(w, qm)
    return out


__all__ = ["QuantizedMatrix", "alternate_fit", "bs_recalibrate_codes", "build_multiprecision", "dequantize",
           "expand_step", "greedy_init", "ls_update_scales", "precision_errors", "relative_reconstruction_error"]
