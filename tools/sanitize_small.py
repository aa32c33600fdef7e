"""Small launches of the round-2 kernels (a quick crash / hang check; compute-sanitizer is closed on this pool):
cluster GEMV (every geometry on a ragged asymmetric shape), the fused-norm
GEMV, the quantizer, argmax.
    python tools/sanitize_small.py
"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2510_10467_b200 as P  # noqa: E402
from paper_2510_10467_b200 import _lib  # noqa: E402
from paper_2510_10467_b200.decode import _Argmax  # noqa: E402

torch.cuda.set_device(0)
L = _lib.lib()
g = torch.Generator(device="cuda").manual_seed(0)
for rows, cols, asym in ((300, 1000, True), (64, 4096, False), (1000, 2048, False)):
    dm = P.DeviceModel(rows, cols, 128, 1, 4, asym, scale_dtype="f16")
    wpr = (cols + 31) // 32
    w = torch.randint(-2**31, 2**31 - 1, (4, rows, wpr), dtype=torch.int32, device="cuda", generator=g)
    if cols % 32:
        w[..., -1] &= (1 << (cols % 32)) - 1
    dm.load_planes(w)
    G = (cols + 127) // 128
    for p in range(1, 5):
        dm.load_scale_set(p, torch.rand((p, rows, G), device="cuda", generator=g) * 0.1,
                          torch.randn((rows, G), device="cuda", generator=g) * 0.1 if asym else None)
    x = torch.randn(cols, device="cuda", generator=g).half()
    L.abcq_debug_set_mode(27)
    for force in (5000, 5112, 5122, 5162, 5262, 5221):
        L.abcq_debug_set_mode(force)
        for p in (1, 3, 4):
            dm.gemv(p, x)
    L.abcq_debug_set_mode(5000)
    L.abcq_debug_set_mode(0)
    if cols <= 8192 and not asym:
        y = torch.empty(rows, device="cuda", dtype=torch.float16)
        xo = torch.empty_like(x)
        dm.gemv_add_rmsnorm(2, x, x.clone(), torch.ones_like(x), 1e-5, out=y, x_out=xo)
wq = np.random.default_rng(0).standard_normal((40, 200)).astype(np.float32)
P.build_multiprecision(wq, 1, 3, P.QuantConfig(group_size=40, mode="asymmetric", cycles=2))
P.bs_recalibrate_codes(wq, P.ScaleTensor(np.abs(np.random.default_rng(1).standard_normal((13, 40, 5))).astype(np.float32),
                                          None, 40))
am = _Argmax(torch.device("cuda"))
out = torch.empty((), device="cuda", dtype=torch.int64)
am(torch.randn(50000, device="cuda").half(), out)
torch.cuda.synchronize()
print("ok")
