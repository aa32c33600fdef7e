"""Host-side model types -- the data formats either side of the GEMV path.

Mirrors the reference's public types so a reference user can hand over the
same objects (the engine also accepts the reference's own instances, duck
typed on the attributes below):

  * QuantConfig          bcq.py:31-47
  * BitPlaneSet          packing.py:40-93 (normative packing packing.py:1-37)
  * ScaleTensor          bcq.py:50-96
  * MultiPrecisionModel  progressive.py:32-79, precision_view :82-86

These are plain numpy containers (no compute); all arithmetic on them runs
in the CUDA library (DeviceModel / GemvEngine). Fitting (greedy/LS/BS,
progressive expansion) is an offline producer and out of scope.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import NonFiniteError, UsageError

MAX_PLANES = 16  # bcq.py:22


def words_per_row(cols: int) -> int:
    """ceil(cols/32) (packing.py:18-19)."""
    return (cols + 31) // 32


def group_count(cols: int, group_size: int) -> int:
    """bcq.py:124-125."""
    return (cols + group_size - 1) // group_size


def group_bounds(cols: int, group_size: int) -> list[tuple[int, int]]:
    """Column range of each group, last one possibly ragged (bcq.py:128-130)."""
    return [(lo, min(lo + group_size, cols)) for lo in range(0, cols, group_size)]


def pack_signs(codes: np.ndarray) -> np.ndarray:
    """(..., cols) {-1,+1} -> (..., ceil(cols/32)) LE u32; bit j of word w is
    column 32w+j, stored 1 means +1, padding bits zero (packing.py:22-30)."""
    codes = np.asarray(codes)
    cols = codes.shape[-1]
    wpr = words_per_row(cols)
    bits = np.zeros(codes.shape[:-1] + (wpr * 32,), dtype=np.uint8)
    bits[..., :cols] = codes > 0
    packed = np.packbits(bits, axis=-1, bitorder="little")
    return np.ascontiguousarray(packed).view("<u4").reshape(codes.shape[:-1] + (wpr,))


def unpack_signs(words: np.ndarray, cols: int) -> np.ndarray:
    """Inverse of pack_signs -> int8 codes (packing.py:33-37)."""
    by = np.ascontiguousarray(words, dtype="<u4").view(np.uint8)
    bits = np.unpackbits(by, axis=-1, bitorder="little", count=cols)
    return (bits.astype(np.int8) << 1) - 1


@dataclass(frozen=True)
class QuantConfig:
    group_size: int = 128
    mode: str = "symmetric"
    cycles: int = 20

    def __post_init__(self):
        if self.group_size < 1:
            raise UsageError(f"group_size must be >= 1, got {self.group_size}")
        if self.mode not in ("symmetric", "asymmetric"):
            raise UsageError(f"mode must be symmetric or asymmetric, got {self.mode!r}")
        if self.cycles < 0:
            raise UsageError(f"cycles must be >= 0, got {self.cycles}")

    @property
    def asymmetric(self) -> bool:
        return self.mode == "asymmetric"


@dataclass(frozen=True, eq=False)
class BitPlaneSet:
    """`planes` packed planes over (rows, cols); words (planes, rows, wpr) u32."""

    planes: int
    rows: int
    cols: int
    words: np.ndarray

    def __post_init__(self):
        if self.planes < 1:
            raise UsageError("plane count must be >= 1")
        expect = (self.planes, self.rows, words_per_row(self.cols))
        if tuple(self.words.shape) != expect:
            raise UsageError(f"packed words shape {self.words.shape} != {expect}")

    @classmethod
    def from_codes(cls, codes: np.ndarray) -> "BitPlaneSet":
        codes = np.asarray(codes)
        if codes.ndim != 3:
            raise UsageError(f"codes must be 3-D, got shape {codes.shape}")
        q, rows, k = codes.shape
        return cls(q, rows, k, pack_signs(codes))

    def codes(self, plane: int | None = None) -> np.ndarray:
        if plane is None:
            return unpack_signs(self.words, self.cols)
        return unpack_signs(self.words[plane], self.cols)

    def prefix(self, p: int) -> "BitPlaneSet":
        """Zero-copy view over the first p planes (packing.py:74-78)."""
        if not 1 <= p <= self.planes:
            raise UsageError(f"prefix {p} out of range [1, {self.planes}]")
        return BitPlaneSet(p, self.rows, self.cols, self.words[:p])

    def plane_bytes(self) -> int:
        return self.rows * words_per_row(self.cols) * 4

    def tobytes(self) -> bytes:
        return np.ascontiguousarray(self.words, dtype="<u4").tobytes()

    def __eq__(self, other) -> bool:
        # duck-typed: equal to the reference's BitPlaneSet with the same words too
        if not all(hasattr(other, a) for a in ("planes", "rows", "cols", "words")):
            return NotImplemented
        return ((self.planes, self.rows, self.cols) == (other.planes, other.rows, other.cols)
                and np.array_equal(self.words, other.words))


@dataclass(frozen=True, eq=False)
class ScaleTensor:
    """alpha (planes, rows, groups) f32; offset (rows, groups) f32 or None."""

    alpha: np.ndarray
    offset: np.ndarray | None
    group_size: int

    def __post_init__(self):
        if self.alpha.ndim != 3:
            raise UsageError(f"alpha must be 3-D, got shape {self.alpha.shape}")
        if not np.isfinite(self.alpha).all():
            raise NonFiniteError("scales contain NaN or Inf")
        if self.offset is not None:
            if self.offset.shape != self.alpha.shape[1:]:
                raise UsageError(f"offset shape {self.offset.shape} != {self.alpha.shape[1:]}")
            if not np.isfinite(self.offset).all():
                raise NonFiniteError("offsets contain NaN or Inf")

    @property
    def planes(self) -> int:
        return self.alpha.shape[0]

    @property
    def rows(self) -> int:
        return self.alpha.shape[1]

    @property
    def groups(self) -> int:
        return self.alpha.shape[2]

    def __eq__(self, other) -> bool:
        # bcq.py:87-96, duck-typed (a reference ScaleTensor with equal arrays is equal)
        if not all(hasattr(other, a) for a in ("alpha", "offset", "group_size")):
            return NotImplemented
        if self.group_size != other.group_size or not np.array_equal(self.alpha, other.alpha):
            return False
        if (self.offset is None) != (other.offset is None):
            return False
        return self.offset is None or np.array_equal(self.offset, other.offset)


@dataclass(frozen=True, eq=False)
class MultiPrecisionModel:
    """Shared planes plus one independent scale set per p in [p_lo, p_hi]."""

    bitplanes: BitPlaneSet
    scale_sets: dict
    p_lo: int
    p_hi: int
    config: QuantConfig

    def __post_init__(self):
        if not 1 <= self.p_lo <= self.p_hi <= MAX_PLANES:
            raise UsageError(f"invalid precision range [{self.p_lo}, {self.p_hi}]")
        if self.bitplanes.planes != self.p_hi:
            raise UsageError(f"{self.bitplanes.planes} planes stored but p_hi={self.p_hi}")
        expected = set(range(self.p_lo, self.p_hi + 1))
        if set(self.scale_sets) != expected:
            raise UsageError(f"scale sets {sorted(self.scale_sets)} != {sorted(expected)}")
        for p, st in self.scale_sets.items():
            if st.planes != p:
                raise UsageError(f"scale set {p} holds {st.planes} plane scales")
            if st.rows != self.bitplanes.rows:
                raise UsageError(f"scale set {p} row count mismatch")
            if st.groups != group_count(self.bitplanes.cols, self.config.group_size):
                raise UsageError(f"scale set {p} group count mismatch")
            if (st.offset is not None) != self.config.asymmetric:
                raise UsageError(f"scale set {p} offset does not match mode")

    @property
    def shape(self) -> tuple[int, int]:
        return self.bitplanes.rows, self.bitplanes.cols

    @property
    def precisions(self) -> range:
        return range(self.p_lo, self.p_hi + 1)


def precision_view(model, p: int):
    """(planes 0..p-1, scale set p) of a model (progressive.py:82-86)."""
    if p not in model.precisions:
        raise UsageError(f"precision {p} outside [{model.p_lo}, {model.p_hi}]")
    return model.bitplanes.prefix(p), model.scale_sets[p]
