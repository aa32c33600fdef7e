"""Multi-GPU row sharding of the bit-plane GEMV.

Groups lie along K inside a row (bcq.py:128-130), so output rows shard with
no split of any group or scale set: rank r owns rows [lo_r, hi_r) of every
plane and every scale set, runs the batch-1 kernel on its shard, and the y
slices are all-gathered over NCCL (NVLink / NVSwitch) -- the one exchange
step of the path. The reference's only parallelism is host row threads
(parallel.py:14-30, gemv.py:196-214); this is its multi-device counterpart.

One process per GPU (`torch.distributed`, backend "nccl"); the host-side
logic is exercised on CPU with backend "gloo" by tests/test_parallel.py.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from .errors import UsageError
from .model import BitPlaneSet, MultiPrecisionModel, ScaleTensor

ROW_ALIGN = 16  # keep shards on 16-row tile boundaries


def row_shard_bounds(rows: int, world: int, rank: int, align: int = ROW_ALIGN) -> tuple[int, int]:
    """Contiguous row range of `rank`: equal shares rounded to `align` rows,
    the last rank takes the remainder."""
    if world < 1 or not 0 <= rank < world:
        raise UsageError(f"bad rank {rank} of {world}")
    per = -(-rows // world)
    per = -(-per // align) * align
    lo = min(rows, rank * per)
    hi = min(rows, lo + per)
    return lo, hi


def shard_model(model, lo: int, hi: int) -> MultiPrecisionModel:
    """Rows [lo, hi) of a MultiPrecisionModel (reference or ours): planes and
    every scale set / offset set sliced along rows (host arrays, views)."""
    if not 0 <= lo < hi <= model.shape[0]:
        raise UsageError(f"empty or out-of-range shard [{lo}, {hi})")
    bp = model.bitplanes
    planes = BitPlaneSet(bp.planes, hi - lo, bp.cols, np.ascontiguousarray(bp.words[:, lo:hi]))
    sets = {}
    for p in model.precisions:
        st = model.scale_sets[p]
        off = None if st.offset is None else np.ascontiguousarray(st.offset[lo:hi])
        sets[p] = ScaleTensor(np.ascontiguousarray(st.alpha[:, lo:hi]), off, st.group_size)
    return MultiPrecisionModel(planes, sets, model.p_lo, model.p_hi, model.config)


class RowShardedGemv:
    """y = W_p x with W's rows sharded over the ranks of `group`.

    Every rank passes the same full model (or only its shard via
    `shard=`), calls `gemv(p, x)` with the same x, and receives the full y.
    `local_gemv(p, x_tensor) -> y_slice` defaults to the CUDA engine
    (DeviceModel.gemv); tests inject a CPU oracle to cover the host logic.
    """

    def __init__(self, model, group=None, *, scale_dtype="f16", device=None, local_gemv=None):
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.rows, self.cols = model.shape
        self.lo, self.hi = row_shard_bounds(self.rows, self.world, self.rank)
        self.shard_rows = max(0, self.hi - self.lo)
        self.pad_rows = row_shard_bounds(self.rows, self.world, 0)[1]  # max shard size
        self.shard = shard_model(model, self.lo, self.hi) if self.shard_rows else None
        self.p_lo, self.p_hi = model.p_lo, model.p_hi
        if local_gemv is None and self.shard is not None:
            from .device_model import DeviceModel

            dm = DeviceModel.from_model(self.shard, scale_dtype=scale_dtype, device=device)
            self.device = dm.device
            local_gemv = lambda p, x: dm.gemv(p, x, out_dtype=x.dtype)  # noqa: E731
        else:
            self.device = torch.device(device) if device is not None else torch.device("cpu")
        self._local = local_gemv

    def gemv(self, p: int, x: torch.Tensor) -> torch.Tensor:
        if not self.p_lo <= p <= self.p_hi:
            raise UsageError(f"precision {p} outside [{self.p_lo}, {self.p_hi}]")
        if x.numel() != self.cols:
            raise UsageError(f"input length {x.numel()} != cols {self.cols}")
        out = torch.zeros(self.pad_rows, dtype=x.dtype, device=x.device)
        if self.shard_rows:
            out[: self.shard_rows] = self._local(p, x)
        if self.world == 1:
            return out[: self.rows]
        full = torch.empty(self.pad_rows * self.world, dtype=x.dtype, device=x.device)
        dist.all_gather_into_tensor(full, out, group=self.group)
        pieces = [full[r * self.pad_rows: r * self.pad_rows + (b[1] - b[0])]
                  for r, b in enumerate(row_shard_bounds(self.rows, self.world, r)
                                        for r in range(self.world))]
        return torch.cat(pieces)
