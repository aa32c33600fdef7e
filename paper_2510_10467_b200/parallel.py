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


class PeerGather:
    """The fused all-gather's buffer: a gathered output
    of `world * rows_per_rank` elements in torch symmetric memory -- every
    rank's copy and signal pad mapped on every GPU (NVLink peer memory) -- so
    that a GEMV launch stores its rows straight into all ranks' copies
    (abcq_gemv_batch_peer) instead of a separate NCCL all-gather. Rank r's
    rows are `local` = buffer[r*R:(r+1)*R]; `plan(jobs)` builds the launch
    (jobs' outputs must be views of `local`); `wait()` enqueues the consumer
    wait (every rank's rows of the latest launch have landed)."""

    def __init__(self, rows_per_rank: int, group=None, dtype=torch.float16, device=None):
        import ctypes as C

        import torch.distributed._symmetric_memory as symm_mem

        from . import _lib
        self.group = group if group is not None else dist.group.WORLD
        self.world = dist.get_world_size(self.group)
        self.rank = dist.get_rank(self.group)
        if self.world > 8:
            raise UsageError("the fused all-gather supports up to 8 ranks (one NVLink domain node)")
        self.rows = int(rows_per_rank)
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.buffer = symm_mem.empty(self.world * self.rows, dtype=dtype, device=dev)
        self.handle = symm_mem.rendezvous(self.buffer, self.group.group_name)
        self.local = self.buffer[self.rank * self.rows:(self.rank + 1) * self.rows]
        self._bases = (C.c_void_p * self.world)(*[int(v) for v in self.handle.buffer_ptrs])
        self._sigs = (C.c_void_p * self.world)(*[int(v) for v in self.handle.signal_pad_ptrs])
        if int(self._bases[self.rank]) != self.buffer.data_ptr():
            raise UsageError("symmetric memory: this rank's buffer pointer mismatch")
        n = int(_lib.lib().abcq_peer_state_bytes())
        self.state = torch.zeros(n // 4, dtype=torch.int32, device=dev)
        self.err = torch.zeros(1, dtype=torch.int32, device=dev)
        self._C, self._lib = C, _lib

    def plan(self, jobs) -> "PeerGemvPlan":
        return PeerGemvPlan(self, jobs)

    def wait(self, stream=None, timeout_s: float = 2.0) -> None:
        """Enqueue: publish this rank's latest launch, then block the stream
        until every rank's rows of its latest launch are in this rank's buffer
        (bounded: `err` = 1 + the late rank). Every rank calls it after the
        same launch."""
        from .device_model import _stream_handle
        self._lib.check(self._lib.lib().abcq_peer_wait(self._bases, self._sigs, self.world, self.rank,
                                                       self.state.data_ptr(), self.err.data_ptr(),
                                                       int(timeout_s * 1e9), _stream_handle(stream)),
                        "abcq_peer_wait")


class PeerGemvPlan:
    """A GemvBatchPlan whose launch also stores every output row into all
    ranks' PeerGather buffers (one launch: GEMV + all-gather)."""

    def __init__(self, gather: PeerGather, jobs):
        from .device_model import GemvBatchPlan
        lo = gather.local.data_ptr()
        hi = lo + gather.local.numel() * gather.local.element_size()
        for _, _, _, out in jobs:
            if not lo <= out.data_ptr() < hi:
                raise UsageError("PeerGemvPlan: every output must be a view of the gather's `local` rows")
        self.gather = gather
        self.base = GemvBatchPlan(jobs)

    def launch(self, stream=None):
        from .device_model import _stream_handle
        b, g = self.base, self.gather
        for dm, p, _, _ in b.jobs:
            if dm._level_ready:
                dm._order_after_upload(p, stream)
        sh = _stream_handle(stream)
        ws = b._ws.get(sh)
        if ws is None:
            from .device_model import stream_workspace
            ws = b._ws[sh] = stream_workspace(b.device, sh, b.need)
        nbytes = g.buffer.numel() * g.buffer.element_size()
        g._lib.check(b._L.abcq_gemv_batch_peer(b.arr, b.n, g.buffer.data_ptr(), nbytes, g._bases, g._sigs, g.world,
                                               g.rank, g.state.data_ptr(), ws.data_ptr(), ws.numel(), sh),
                     "abcq_gemv_batch_peer")
        return [j[3] for j in b.jobs]
