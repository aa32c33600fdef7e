"""numpy statement of the B200 tiled plane/scale layout --
test infrastructure: the GPU packer must reproduce it bit for bit."""

import numpy as np


def tiled_planes(words: np.ndarray, rows: int, cols: int) -> np.ndarray:
    """(planes, rows, wpr) u32 -> (planes, NS, NRT, 32 lanes, 16 bytes) u8."""
    planes = words.shape[0]
    nrt, ns = -(-rows // 16), -(-cols // 256)
    wpr = words.shape[2]
    pad = np.zeros((planes, nrt * 16, ns * 8), dtype=np.uint32)
    pad[:, :rows, :wpr] = words
    by = pad.view(np.uint8).reshape(planes, nrt, 16, ns, 2, 16)     # i, rt, r, s, half, byte
    out = np.empty_like(by)
    for r in range(16):
        out[:, :, r] = np.roll(by[:, :, r], -r, axis=-1)              # stored j = ref (j + r) & 15
    return np.ascontiguousarray(out.transpose(0, 3, 1, 4, 2, 5)).reshape(planes, ns, nrt, 32, 16)


def tiled_scales(alpha: np.ndarray, rows: int, cols: int) -> np.ndarray:
    """alpha (p, rows, G) -> (p, NS, NRT, 32 lanes) with lane = half*16 + r."""
    p, _, G = alpha.shape
    nrt, ns = -(-rows // 16), -(-cols // 256)
    pad = np.zeros((p, nrt * 16, ns * 2), dtype=alpha.dtype)
    pad[:, :rows, :G] = alpha
    t = pad.reshape(p, nrt, 16, ns, 2)                                 # i, rt, r, s, half
    return np.ascontiguousarray(t.transpose(0, 3, 1, 4, 2)).reshape(p, ns, nrt, 32)


def tiled_offsets(offset: np.ndarray, rows: int, cols: int) -> np.ndarray:
    return tiled_scales(offset[None], rows, cols)[0]
