"""ABCQ model container: reader/writer compatible with the reference
(/root/reference/pkg/src/anybcq/model_format.py:1-154) and a GPU-resident
progressive loader.

Container layout (little-endian, model_format.py:1-15):

    b"ABCQ", u32 version (1), u32 header_len, header JSON (sorted keys,
    compact separators: rows, cols, group_size, mode, cycles, p_lo, p_hi,
    scale_width, creator), the p_hi planes ascending (each rows x ceil(cols/32)
    u32, row-major), the scale sets ascending precision (set p: p x rows x G in
    f32 or f16 per scale_width), the offsets ascending precision when
    asymmetric (rows x G each), u32 CRC32 of every preceding byte.

`serialize` writes byte-identical files to the reference's writer (checked
against files it wrote: tests/golden/container_*.abcq); `deserialize`
validates in the reference's order and raises its error classes (BadMagic,
BadVersion, FileFormat for header problems / trailing bytes, Truncated,
Checksum).

`ProgressiveLoader` is the serving loader: because planes
and scale sets are stored ascending, precision p_lo needs only planes
1..p_lo and set p_lo. The loader uploads level by level on a side stream --
level p_lo first, then each higher precision adds one plane and its set --
records a CUDA event per level and marks the DeviceModel, so a GEMV at p
waits device-side for exactly its own bytes and can run while higher planes
are still landing. With scale_width=2 the device keeps f16 scales, so the
scales the kernels read are bit-identical to the file's.
"""

from __future__ import annotations

import json
import mmap
import struct
import zlib
from dataclasses import dataclass

import numpy as np

from .errors import BadMagicError, BadVersionError, ChecksumError, FileFormatError, TruncatedError, UsageError
from .model import BitPlaneSet, MultiPrecisionModel, QuantConfig, ScaleTensor, group_count, words_per_row

ABCQ_MAGIC = b"ABCQ"
ABCQ_VERSION = 1
_PREFIX = struct.Struct("<4sII")
_CREATOR = "anybcq-0.1"  # the reference's creator tag: identical models -> identical bytes
_SCALE_DTYPES = {2: "<f2", 4: "<f4"}


@dataclass(frozen=True)
class ContainerLayout:
    """Header fields and the byte offset of every section of one container."""

    rows: int
    cols: int
    group_size: int
    mode: str
    cycles: int
    p_lo: int
    p_hi: int
    scale_width: int
    header_end: int

    @property
    def asymmetric(self) -> bool:
        return self.mode == "asymmetric"

    @property
    def groups(self) -> int:
        return group_count(self.cols, self.group_size)

    @property
    def plane_bytes(self) -> int:
        return self.rows * words_per_row(self.cols) * 4

    def plane_offset(self, i: int) -> int:
        return self.header_end + i * self.plane_bytes

    def set_offset(self, p: int) -> int:
        """Byte offset of scale set p (sets p_lo..p-1 precede it)."""
        before = sum(q for q in range(self.p_lo, p)) * self.rows * self.groups * self.scale_width
        return self.header_end + self.p_hi * self.plane_bytes + before

    def offsets_offset(self, p: int) -> int:
        sets = sum(range(self.p_lo, self.p_hi + 1)) * self.rows * self.groups * self.scale_width
        return (self.header_end + self.p_hi * self.plane_bytes + sets
                + (p - self.p_lo) * self.rows * self.groups * self.scale_width)

    @property
    def total_bytes(self) -> int:
        n_off = (self.p_hi - self.p_lo + 1) if self.asymmetric else 0
        return self.offsets_offset(self.p_lo + n_off) + 4


def serialize(model, path, scale_width: int = 4) -> None:
    """Write `model` as a container (model_format.py:46-79). scale_width=4
    round-trips f32 scales bit-exactly; 2 stores f16 (the deployment width)."""
    if scale_width not in _SCALE_DTYPES:
        raise UsageError(f"scale_width must be one of {sorted(_SCALE_DTYPES)}")
    dt = _SCALE_DTYPES[scale_width]
    header = {"rows": model.shape[0], "cols": model.shape[1], "group_size": model.config.group_size,
              "mode": model.config.mode, "cycles": model.config.cycles, "p_lo": model.p_lo,
              "p_hi": model.p_hi, "scale_width": scale_width, "creator": _CREATOR}
    head = json.dumps(header, sort_keys=True, separators=(",", ":")).encode()
    body = bytearray(_PREFIX.pack(ABCQ_MAGIC, ABCQ_VERSION, len(head)))
    body += head
    body += np.ascontiguousarray(model.bitplanes.words, dtype="<u4").tobytes()
    for p in model.precisions:
        body += np.asarray(model.scale_sets[p].alpha).astype(dt).tobytes()
    if model.config.asymmetric:
        for p in model.precisions:
            body += np.asarray(model.scale_sets[p].offset).astype(dt).tobytes()
    body += struct.pack("<I", zlib.crc32(bytes(body)))
    with open(path, "wb") as fh:
        fh.write(bytes(body))


def read_layout(raw, path="<buffer>") -> ContainerLayout:
    """Parse and validate the prefix + header (model_format.py:82-96,99-121)."""
    if len(raw) < _PREFIX.size:
        raise TruncatedError(f"{path}: shorter than the fixed prefix")
    magic, version, hlen = _PREFIX.unpack_from(raw)
    if magic != ABCQ_MAGIC:
        raise BadMagicError(f"{path}: bad magic {bytes(magic)!r}")
    if version != ABCQ_VERSION:
        raise BadVersionError(f"{path}: unsupported version {version}")
    if len(raw) < _PREFIX.size + hlen:
        raise TruncatedError(f"{path}: header extends past end of file")
    try:
        h = json.loads(bytes(raw[_PREFIX.size:_PREFIX.size + hlen]))
    except ValueError as exc:
        raise FileFormatError(f"{path}: unreadable header ({exc})") from exc
    try:
        lay = ContainerLayout(int(h["rows"]), int(h["cols"]), int(h["group_size"]), str(h["mode"]),
                              int(h.get("cycles", 0)), int(h["p_lo"]), int(h["p_hi"]),
                              int(h["scale_width"]), _PREFIX.size + hlen)
    except (KeyError, TypeError, ValueError) as exc:
        raise FileFormatError(f"{path}: header missing fields ({exc})") from exc
    if lay.scale_width not in _SCALE_DTYPES:
        raise FileFormatError(f"{path}: unsupported scale width {lay.scale_width}")
    if lay.rows < 1 or lay.cols < 1 or lay.group_size < 1 or not 1 <= lay.p_lo <= lay.p_hi:
        raise FileFormatError(f"{path}: invalid geometry in header")
    expected = lay.total_bytes
    if len(raw) < expected:
        raise TruncatedError(f"{path}: {len(raw)} bytes, layout requires {expected}")
    if len(raw) > expected:
        raise FileFormatError(f"{path}: {len(raw) - expected} trailing bytes")
    return lay


def _verify_crc(raw, lay: ContainerLayout, path) -> None:
    end = lay.total_bytes - 4
    stored = struct.unpack_from("<I", raw, end)[0]
    if zlib.crc32(memoryview(raw)[:end]) != stored:
        raise ChecksumError(f"{path}: checksum mismatch")


def _planes(raw, lay: ContainerLayout, first: int, count: int) -> np.ndarray:
    wpr = words_per_row(lay.cols)
    return np.frombuffer(raw, dtype="<u4", count=count * lay.rows * wpr,
                         offset=lay.plane_offset(first)).reshape(count, lay.rows, wpr)


def _scale_set(raw, lay: ContainerLayout, p: int):
    dt = _SCALE_DTYPES[lay.scale_width]
    a = np.frombuffer(raw, dtype=dt, count=p * lay.rows * lay.groups, offset=lay.set_offset(p))
    a = a.astype(np.float32).reshape(p, lay.rows, lay.groups)
    z = None
    if lay.asymmetric:
        z = np.frombuffer(raw, dtype=dt, count=lay.rows * lay.groups, offset=lay.offsets_offset(p))
        z = z.astype(np.float32).reshape(lay.rows, lay.groups)
    return a, z


def deserialize(path) -> MultiPrecisionModel:
    """Read a container into host types (model_format.py:99-154)."""
    with open(path, "rb") as fh:
        raw = fh.read()
    lay = read_layout(raw, path)
    _verify_crc(raw, lay, path)
    words = _planes(raw, lay, 0, lay.p_hi).copy()
    sets = {p: ScaleTensor(*_scale_set(raw, lay, p), lay.group_size) for p in range(lay.p_lo, lay.p_hi + 1)}
    cfg = QuantConfig(group_size=lay.group_size, mode=lay.mode, cycles=lay.cycles)
    return MultiPrecisionModel(BitPlaneSet(lay.p_hi, lay.rows, lay.cols, words), sets, lay.p_lo, lay.p_hi, cfg)


class ProgressiveLoader:
    """Upload a container to the GPU precision level by level.

        loader = ProgressiveLoader("m.abcq")        # header + CRC checked, nothing uploaded
        loader.load_level()                         # planes 1..p_lo + set p_lo (async)
        y = loader.model.gemv(loader.model.p_lo, x) # may run before higher planes land
        loader.load_all()                           # remaining planes + sets

    Uploads run on `stream` (default: a new side stream); each level records an
    event that launches reading that precision wait on device-side
    (DeviceModel.mark_level_ready). scale_dtype defaults to the file's width
    ("f16" for scale_width=2: bit-exact), "f32" otherwise.
    """

    def __init__(self, path, device=None, scale_dtype=None, stream=None, verify_crc: bool = True):
        import torch

        from .device_model import DeviceModel

        self.path = path
        with open(path, "rb") as fh:
            self._mm = mmap.mmap(fh.fileno(), 0, access=mmap.ACCESS_READ)
        self.layout = read_layout(self._mm, path)
        if verify_crc:
            _verify_crc(self._mm, self.layout, path)
        lay = self.layout
        if scale_dtype is None:
            scale_dtype = "f16" if lay.scale_width == 2 else "f32"
        self.model = DeviceModel(lay.rows, lay.cols, lay.group_size, lay.p_lo, lay.p_hi, lay.asymmetric,
                                 scale_dtype=scale_dtype, device=device)
        self.stream = stream if stream is not None else torch.cuda.Stream(device=self.model.device)
        # the model's buffers were allocated (zero-filled) on the current stream
        self.stream.wait_stream(torch.cuda.current_stream(self.model.device))
        self.loaded = 0  # highest servable precision uploaded (0: none)

    @property
    def config(self) -> QuantConfig:
        return QuantConfig(self.layout.group_size, self.layout.mode, self.layout.cycles)

    def load_level(self) -> int:
        """Upload the next precision level; returns it (0 when complete)."""
        import torch

        lay, dm = self.layout, self.model
        p = lay.p_lo if self.loaded == 0 else self.loaded + 1
        if p > lay.p_hi:
            return 0
        first = 0 if self.loaded == 0 else p - 1
        with torch.cuda.device(dm.device), torch.cuda.stream(self.stream):
            words = torch.from_numpy(_planes(self._mm, lay, first, p - first).view(np.int32).copy())
            dm.load_planes(words.pin_memory().to(dm.device, non_blocking=True), first=first)
            a, z = _scale_set(self._mm, lay, p)
            dm.load_scale_set(p, a, z)
            ev = torch.cuda.Event()
            ev.record(self.stream)
        dm.mark_level_ready(p, ev)
        self.loaded = p
        return p

    def load_all(self):
        while self.load_level():
            pass
        return self.model

    def close(self) -> None:
        self._mm.close()


def load_device_model(path, device=None, scale_dtype=None):
    """Whole container -> DeviceModel (all levels queued; serving order kept)."""
    return ProgressiveLoader(path, device=device, scale_dtype=scale_dtype).load_all()
