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

    Every rank passes the same full model (or only its shard, `shard=` with
    `rows=` the full row count), calls `gemv(p, x)` with the same x, and
    receives the full y. All buffers are allocated once: the rank's slice is
    written by one abcq_gemv launch (the cluster kernel for a small shard, the
    persistent kernel for a large one) straight into the all-gather send
    buffer, and y is a view of the gather's receive buffer --
    shards sit on 16-row tile boundaries with every rank but the last holding
    exactly `pad_rows` rows, so the gathered buffer's first `rows` elements
    ARE y in order (no per-call allocation, copy or concatenation).
    `local_gemv(p, x_tensor) -> y_slice` replaces the CUDA engine (tests
    inject a CPU oracle to cover the host logic with gloo).
    """

    def __init__(self, model=None, group=None, *, scale_dtype="f16", device=None, local_gemv=None,
                 dtype=torch.float16, shard=None, rows: int | None = None):
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        if shard is not None:  # this rank's DeviceModel (or host model) only
            if rows is None:
                raise UsageError("shard= needs rows= (the full row count)")
            self.rows, self.cols = int(rows), shard.cols if hasattr(shard, "cols") else shard.shape[1]
        else:
            self.rows, self.cols = model.shape
        self.lo, self.hi = row_shard_bounds(self.rows, self.world, self.rank)
        self.shard_rows = max(0, self.hi - self.lo)
        self.pad_rows = row_shard_bounds(self.rows, self.world, 0)[1]  # max shard size
        src = shard if shard is not None else model
        self.p_lo, self.p_hi = src.p_lo, src.p_hi
        self.dtype = dtype
        self.dm = None
        # this rank's rows of the model (host types; a DeviceModel when passed as shard=)
        self.shard = shard if shard is not None else (shard_model(model, self.lo, self.hi) if self.shard_rows else None)
        if local_gemv is None and self.shard_rows:
            from .device_model import DeviceModel

            if isinstance(self.shard, DeviceModel):
                self.dm = self.shard
            else:
                self.dm = DeviceModel.from_model(self.shard, scale_dtype=scale_dtype, device=device)
            if self.dm.rows != self.shard_rows:
                raise UsageError(f"shard has {self.dm.rows} rows, rank {self.rank} owns {self.shard_rows}")
            self.device = self.dm.device
        else:
            self.device = torch.device(device) if device is not None else torch.device("cpu")
        self._local = local_gemv
        self._send = torch.zeros(self.pad_rows, dtype=dtype, device=self.device)
        self._recv = torch.empty(self.pad_rows * self.world, dtype=dtype, device=self.device)
        self._x = torch.empty(self.cols, dtype=dtype, device=self.device)  # the fixed input buffer

    def local(self, p: int, x: torch.Tensor, stream=None) -> None:
        """This rank's slice of y into the send buffer (no communication)."""
        if not self.p_lo <= p <= self.p_hi:
            raise UsageError(f"precision {p} outside [{self.p_lo}, {self.p_hi}]")
        if x.numel() != self.cols:
            raise UsageError(f"input length {x.numel()} != cols {self.cols}")
        if not self.shard_rows:
            return
        if self._local is not None:
            self._send[: self.shard_rows] = self._local(p, x)
            return
        if x.data_ptr() != self._x.data_ptr():
            self._x.copy_(x.reshape(-1))
        self.dm.gemv(p, self._x, out=self._send[: self.shard_rows], stream=stream)

    def gather(self, async_op: bool = False):
        """All-gather the slices; y = self.y (a view of the receive buffer)."""
        if self.world == 1:
            return None
        return dist.all_gather_into_tensor(self._recv, self._send, group=self.group, async_op=async_op)

    @property
    def y(self) -> torch.Tensor:
        return (self._send if self.world == 1 else self._recv)[: self.rows]

    @property
    def x_buffer(self) -> torch.Tensor:
        """Write x here to skip the input copy of gemv()."""
        return self._x

    def gemv(self, p: int, x: torch.Tensor) -> torch.Tensor:
        self.local(p, x)
        self.gather()
        return self.y
