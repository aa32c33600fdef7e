"""CPU oracle for the AnyBCQ bit-plane GEMV hot path -- TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference package's algorithm
for the path named by BASELINE.json's north_star (`anybcq.GemvEngine.lut`
and friends). It exists to CHECK the CUDA product path:

  * only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline /
    `--impl reference` leg may import it;
  * nothing under `paper_2510_10467_b200/` imports, links or executes it.

Parity pinning: every function below is checked against the reference's own
golden vectors (restated in tests/test_oracle.py) AND against outputs of the
real reference package (`/root/reference/pkg`, imported in the build
container by tests/golden/make_golden.py; vectors committed under
tests/golden/). See DESIGN.md §Oracle.

Each function cites the reference file:line it restates; paths are relative
to /root/reference/pkg/src/anybcq/.
"""

from __future__ import annotations

import numpy as np

# ---------------------------------------------------------------------------
# portable PRNG -- tensor_io.py:91-128
# ---------------------------------------------------------------------------

GOLDEN = 0x9E3779B97F4A7C15
MIX1 = 0xBF58476D1CE4E5B9
MIX2 = 0x94D049BB133111EB
_U64 = np.uint64


def splitmix64(state: np.ndarray) -> np.ndarray:
    """splitmix64 finalizer on a uint64 array (tensor_io.py:98-102)."""
    z = np.asarray(state, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> _U64(30))) * _U64(MIX1)
        z = (z ^ (z >> _U64(27))) * _U64(MIX2)
    return z ^ (z >> _U64(31))


def random_gaussian(rows: int, cols: int, seed: int) -> np.ndarray:
    """Seeded N(0,1) f32 matrix: counter i -> splitmix64(seed + (i+1)*GOLDEN),
    top 53 bits, Box-Muller (radius from even, angle from odd positions;
    cos then sin). Restates tensor_io.py:105-128."""
    if rows < 1 or cols < 1:
        raise ValueError(f"dimensions must be >= 1, got {rows}x{cols}")
    total = rows * cols
    pairs = (total + 1) // 2
    ctr = np.arange(1, 2 * pairs + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = splitmix64(_U64(seed & 0xFFFFFFFFFFFFFFFF) + ctr * _U64(GOLDEN))
    top = (z >> _U64(11)).astype(np.float64)
    u1 = (top[0::2] + 1.0) * (2.0 ** -53)
    u2 = top[1::2] * (2.0 ** -53)
    rad = np.sqrt(-2.0 * np.log(u1))
    ang = 2.0 * np.pi * u2
    out = np.empty(2 * pairs, dtype=np.float64)
    out[0::2] = rad * np.cos(ang)
    out[1::2] = rad * np.sin(ang)
    return out[:total].astype(np.float32).reshape(rows, cols)


def random_words(planes: int, rows: int, cols: int, seed: int) -> np.ndarray:
    """Synthetic packed planes for throughput shapes: one
    splitmix64 draw per 32-bit word (low half), padding bits past `cols`
    zeroed as packing.py:1-7 requires."""
    wpr = words_per_row(cols)
    n = planes * rows * wpr
    ctr = np.arange(1, n + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = splitmix64(_U64(seed & 0xFFFFFFFFFFFFFFFF) + ctr * _U64(GOLDEN))
    words = (z & _U64(0xFFFFFFFF)).astype(np.uint32).reshape(planes, rows, wpr)
    tail = cols - 32 * (wpr - 1)
    if tail < 32:
        words[:, :, -1] &= np.uint32((1 << tail) - 1)
    return words


# ---------------------------------------------------------------------------
# packing -- packing.py:18-37
# ---------------------------------------------------------------------------

def words_per_row(cols: int) -> int:
    """ceil(cols/32) little-endian u32 words per row (packing.py:18-19)."""
    return (cols + 31) // 32


def pack_signs(codes: np.ndarray) -> np.ndarray:
    """(..., cols) {-1,+1} -> (..., ceil(cols/32)) u32; bit j of word w is
    column 32w+j, 1 <-> +1, padding zero (packing.py:22-30)."""
    codes = np.asarray(codes)
    cols = codes.shape[-1]
    wpr = words_per_row(cols)
    bits = np.zeros(codes.shape[:-1] + (wpr * 32,), dtype=np.uint8)
    bits[..., :cols] = codes > 0
    by = np.packbits(bits, axis=-1, bitorder="little")
    return np.ascontiguousarray(by).view("<u4").reshape(codes.shape[:-1] + (wpr,))


def unpack_signs(words: np.ndarray, cols: int) -> np.ndarray:
    """Inverse of pack_signs -> int8 {-1,+1} (packing.py:33-37)."""
    by = np.ascontiguousarray(words, dtype="<u4").view(np.uint8)
    bits = np.unpackbits(by, axis=-1, bitorder="little", count=cols)
    return (bits.astype(np.int8) << 1) - 1


# ---------------------------------------------------------------------------
# groups -- bcq.py:124-130
# ---------------------------------------------------------------------------

def group_count(cols: int, group_size: int) -> int:
    return (cols + group_size - 1) // group_size


def group_bounds(cols: int, group_size: int) -> list[tuple[int, int]]:
    """Column ranges of each group, final group possibly ragged (bcq.py:128-130)."""
    return [(lo, min(lo + group_size, cols)) for lo in range(0, cols, group_size)]


# ---------------------------------------------------------------------------
# lookup table -- gemv.py:55-81
# ---------------------------------------------------------------------------

def lut_build(x: np.ndarray, chunk_width: int) -> np.ndarray:
    """T[c, t] = sum_j (bit j of t ? +x : -x)[c*mu + j] in f32, built by
    doubling in ascending j with the tail zero-padded (gemv.py:67-81).
    The f32 rounding sequence equals ((((0 -/+ x0) -/+ x1) ...) -/+ x_{mu-1})."""
    if not 1 <= chunk_width <= 8:
        raise ValueError(f"chunk width must be in [1, 8], got {chunk_width}")
    x = np.asarray(x, dtype=np.float32).ravel()
    chunks = (len(x) + chunk_width - 1) // chunk_width
    padded = np.zeros(chunks * chunk_width, dtype=np.float32)
    padded[: len(x)] = x
    padded = padded.reshape(chunks, chunk_width)
    t = np.zeros((chunks, 1), dtype=np.float32)
    for j in range(chunk_width):
        xj = padded[:, j: j + 1]
        t = np.concatenate([t - xj, t + xj], axis=1)
    return np.ascontiguousarray(t)


def chunk_indices(words: np.ndarray, cols: int, chunk_width: int) -> np.ndarray:
    """(planes, rows, chunks) u8 table indices: plane bytes for mu=8,
    nibbles (low first) for mu=4 (gemv.py:130-146)."""
    planes, rows, _ = words.shape
    by = np.ascontiguousarray(words, dtype="<u4").view(np.uint8).reshape(planes, rows, -1)
    nb = (cols + 7) // 8
    by = by[:, :, :nb]
    if chunk_width == 8:
        return np.ascontiguousarray(by)
    chunks = (cols + chunk_width - 1) // chunk_width
    idx = np.empty((planes, rows, 2 * nb), dtype=np.uint8)
    idx[:, :, 0::2] = by & 0x0F
    idx[:, :, 1::2] = by >> 4
    return np.ascontiguousarray(idx[:, :, :chunks])


# ---------------------------------------------------------------------------
# GEMV paths -- gemv.py:170-250
# ---------------------------------------------------------------------------

def _group_sums_f64(x64: np.ndarray, cols: int, group_size: int) -> np.ndarray:
    return np.array([x64[lo:hi].sum() for lo, hi in group_bounds(cols, group_size)])


def gemv_lut(words, cols, group_size, alpha, offset, p, x, chunk_width=8):
    """LUT path (gemv.py:188-250): f32 table; per (plane, row, group) an f32
    sum of table entries over the group's chunks; f64 accumulation of
    alpha*s; asymmetric term offset(f64) @ gx(f64). Groups whose edges are
    not chunk aligned take the naive per-column route on the ragged columns
    (gemv.py:224-250). Returns y f64 (rows,)."""
    x64 = np.asarray(x, dtype=np.float64).ravel()
    planes, rows, _ = words.shape
    mu = chunk_width
    table = lut_build(x64, mu)
    flat = table.ravel()
    chunks = table.shape[0]
    idx = chunk_indices(words, cols, mu)
    a64 = np.asarray(alpha, dtype=np.float32).astype(np.float64)
    y = np.zeros(rows, dtype=np.float64)
    groups = group_bounds(cols, group_size)
    aligned = group_size % mu == 0 or len(groups) == 1
    for gi, (lo, hi) in enumerate(groups):
        if aligned:
            per = group_size // mu if len(groups) > 1 else chunks
            c0 = gi * per
            c1 = min((gi + 1) * per, chunks) if gi < len(groups) - 1 else chunks
            ragged = []
        else:
            c0 = (lo + mu - 1) // mu
            c1 = chunks if hi == cols else hi // mu
            if c1 > c0:
                ragged = [(lo, c0 * mu), (c1 * mu if hi < cols else hi, hi)]
            else:
                c0 = c1 = 0
                ragged = [(lo, hi)]
        for i in range(p):
            part = np.zeros(rows, dtype=np.float64)
            if c1 > c0:
                gidx = idx[i, :, c0:c1].astype(np.intp) + (np.arange(c0, c1, dtype=np.intp) << mu)
                vals = flat[gidx]
                if aligned:
                    # numba kernel (gemv.py:86-95): sequential f32 group sum s;
                    # alpha(f32)*s(f32) is an f32 product added into the f64 acc
                    s = np.zeros(rows, dtype=np.float32)
                    for c in range(vals.shape[1]):
                        s += vals[:, c]
                    y += (np.asarray(alpha, dtype=np.float32)[i, :, gi] * s).astype(np.float64)
                    continue
                else:
                    # numpy route sums the gathered entries in f64 (gemv.py:244)
                    part += vals.sum(axis=1, dtype=np.float64)
            for clo, chi in ragged:
                if chi > clo:
                    codes = unpack_signs(words[i], cols)[:, clo:chi]
                    part += (codes * x64[clo:chi]).sum(axis=1)
            y += a64[i, :, gi] * part
    if offset is not None:
        y = y + np.asarray(offset, dtype=np.float32).astype(np.float64) @ _group_sums_f64(
            x64, cols, group_size)
    return y


def gemv_naive(words, cols, group_size, alpha, offset, p, x):
    """Naive path (gemv.py:170-186): unpack plane i, per-group f64 dot,
    y += alpha * partial; offset term as in the LUT path."""
    x64 = np.asarray(x, dtype=np.float64).ravel()
    rows = words.shape[1]
    a64 = np.asarray(alpha, dtype=np.float32).astype(np.float64)
    y = np.zeros(rows, dtype=np.float64)
    bounds = group_bounds(cols, group_size)
    for i in range(p):
        codes = unpack_signs(words[i], cols)
        for gi, (lo, hi) in enumerate(bounds):
            y += a64[i, :, gi] * (codes[:, lo:hi] * x64[lo:hi]).sum(axis=1)
    if offset is not None:
        y += np.asarray(offset, dtype=np.float32).astype(np.float64) @ _group_sums_f64(
            x64, cols, group_size)
    return y


def dequantize(words, cols, group_size, alpha, offset, p) -> np.ndarray:
    """Dense f32 reconstruction from planes 0..p-1 and scale set p:
    f64 einsum per group plus offset, cast to f32 (bcq.py:137-152,372-378)."""
    codes = unpack_signs(words[:p], cols).astype(np.float64)
    a64 = np.asarray(alpha, dtype=np.float32).astype(np.float64)
    rows = words.shape[1]
    recon = np.zeros((rows, cols), dtype=np.float64)
    for gi, (lo, hi) in enumerate(group_bounds(cols, group_size)):
        block = np.einsum("ink,in->nk", codes[:, :, lo:hi], a64[:p, :, gi])
        if offset is not None:
            block += np.asarray(offset, dtype=np.float32).astype(np.float64)[:, gi][:, None]
        recon[:, lo:hi] = block
    return recon.astype(np.float32)


def dequant_oracle(words, cols, group_size, alpha, offset, p, x) -> np.ndarray:
    """Dense-reconstruction product, f64 matvec (gemv.py:272-277)."""
    dense = dequantize(words, cols, group_size, alpha, offset, p).astype(np.float64)
    return dense @ np.asarray(x, dtype=np.float64).ravel()


def gemv_stats(p, rows, cols, group_size, asymmetric, lut_builds=1):
    """Exact traffic counters (gemv.py:158-168): plane bytes p*N*ceil(K/32)*4,
    scale bytes p*N*G*4 (+N*G*4 asymmetric)."""
    groups = group_count(cols, group_size)
    scale = p * rows * groups * 4 + (rows * groups * 4 if asymmetric else 0)
    return {
        "plane_bytes_fetched": p * rows * words_per_row(cols) * 4,
        "scale_bytes_fetched": scale,
        "lut_build_count": lut_builds,
    }


def rel_dev(a, b) -> float:
    """max|a-b| / max(max|b|, 1e-12) -- the reference's tolerance metric
    (tests/test_gemv.py:20-22)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    scale = max(float(np.max(np.abs(b))) if b.size else 0.0, 1e-12)
    return float(np.max(np.abs(a - b)) / scale) if a.size else 0.0


# ---------------------------------------------------------------------------
# thread policy -- parallel.py:14-30
# ---------------------------------------------------------------------------

def row_chunks(n_rows: int, workers: int) -> list[tuple[int, int]]:
    workers = max(1, min(workers, n_rows))
    step = (n_rows + workers - 1) // workers
    return [(lo, min(lo + step, n_rows)) for lo in range(0, n_rows, step)]
