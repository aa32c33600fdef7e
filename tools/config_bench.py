"""BASELINE.json configs 1, 3 and 5 on one B200 (config 2 = bench.py, config 4 =
tools/decode_bench.py), one JSON object on stdout:

  1. single BCQ linear 4096x4096, g=128, batch 1, p in {2,3,4}: device us per
     call (CUDA graph of back-to-back calls over weight copies > L2), GB/s of
     algorithmic bytes, fraction of the measured HBM peak, the cuBLAS fp16 GEMV
     of the same shape, and the C port of the reference on the host cores.
  3. small-batch GEMM B=1..16, mixed per-request p, Llama-3-8B MLP block
     (gate, up 14336x4096; down 4096x14336): tensor-core GEMM vs the batched
     LUT GEMV (B jobs in one launch); us per block and request-blocks/s.
  5. Llama-3-70B-shaped layers (gate/up 28672x8192, down 8192x28672) at p=2 and
     p=4 on ONE GPU (this pool has one GPU per call; the row-sharded 2/4/8-GPU
     path is bench.py --gpus N under torchrun).

    python tools/config_bench.py > profiles/r1_configs.json
"""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2510_10467_b200 as P  # noqa: E402
from paper_2510_10467_b200.device_model import gemv_batch  # noqa: E402

torch.cuda.set_device(0)
dev = torch.device("cuda", 0)
st = torch.cuda.Stream()
gen = torch.Generator(device="cuda").manual_seed(0)


def peak_gbs():
    try:
        d = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
        for k in ("hbm_gbs", "hbm_copy_gbs", "copy_gbs"):
            if k in d:
                return float(d[k])
    except Exception:
        pass
    return 6537.3


PEAK = peak_gbs()


def model(rows, cols, p_lo=2, p_hi=4):
    dm = P.DeviceModel(rows, cols, 128, p_lo, p_hi, False, scale_dtype="f16")
    dm.load_planes(torch.randint(-2**31, 2**31 - 1, (p_hi, rows, cols // 32), dtype=torch.int32, device=dev,
                                 generator=gen))
    for p in range(p_lo, p_hi + 1):
        dm.load_scale_set(p, 0.01 + 0.1 * torch.randn(p, rows, cols // 128, device=dev, generator=gen).abs())
    return dm


def algo_bytes(rows, cols, p):
    return p * rows * cols // 8 + p * rows * (cols // 128) * 2 + cols * 2 + rows * 2


def graph_us(fn, calls, reps=5):
    with torch.cuda.stream(st):
        fn(0)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for i in range(calls):
            fn(i)
    with torch.cuda.stream(st):
        g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(reps):
            g.replay()
        b.record(st)
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / (reps * calls)


out = {"device": torch.cuda.get_device_name(0), "hbm_peak_gbs": PEAK, "timing":
       "CUDA graph of back-to-back calls, CUDA events; weight copies rotate so the working set exceeds L2"}

# ---- config 1 ----------------------------------------------------------------
rows = cols = 4096
copies = [model(rows, cols) for _ in range(16)]  # 16 x 9.4 MB (p_hi=4 planes + scales) > 126 MB L2
x = torch.randn(cols, device=dev).half()
ys = [torch.empty(rows, device=dev, dtype=torch.float16) for _ in copies]
c1 = {"shape": [rows, cols], "g": 128, "batch": 1}
for p in (2, 3, 4):
    us = graph_us(lambda i: copies[i % len(copies)].gemv(p, x, out=ys[i % len(copies)], stream=st), 32)
    gbs = algo_bytes(rows, cols, p) / (us * 1e-6) / 1e9
    c1[f"p{p}"] = {"us": round(us, 3), "GBps": round(gbs, 1), "roofline_frac": round(gbs / PEAK, 4)}
dense = [torch.randn(rows, cols, device=dev, dtype=torch.float16, generator=gen) for _ in range(4)]
yd = torch.empty(rows, device=dev, dtype=torch.float16)
with torch.cuda.stream(st):
    torch.mv(dense[0], x, out=yd)
us = graph_us(lambda i: torch.mv(dense[i % 4], x, out=yd), 16)
c1["fp16_cublas"] = {"us": round(us, 3), "GBps": round((rows * cols * 2 + cols * 2 + rows * 2) / (us * 1e-6) / 1e9, 1)}
c1["speedup_vs_fp16"] = {f"p{p}": round(us / c1[f"p{p}"]["us"], 2) for p in (2, 3, 4)}
del dense
try:  # the reference algorithm on the host cores (C port, all threads)
    from oracle import c_oracle  # noqa: E402  (cpu baseline only)
    from oracle import anybcq_oracle as O  # noqa: E402
    words = O.random_words(4, rows, cols, seed=1)
    xs = np.random.default_rng(1).standard_normal(cols)
    thr = c_oracle.cpu_threads()
    c1["cpu_reference_port"] = {"threads": thr}
    for p in (2, 3, 4):
        al = np.full((p, rows, cols // 128), 0.05, np.float32)
        c_oracle.lut_gemv(words, cols, 128, al, None, p, xs, thr)
        t0 = time.perf_counter()
        for _ in range(5):
            c_oracle.lut_gemv(words, cols, 128, al, None, p, xs, thr)
        c1["cpu_reference_port"][f"p{p}_us"] = round((time.perf_counter() - t0) / 5 * 1e6, 1)
except Exception as e:  # noqa: BLE001
    c1["cpu_reference_port"] = {"unavailable": str(e)[:120]}
out["config1_single_linear_4096"] = c1
del copies

# ---- config 3 ----------------------------------------------------------------
mlp = {n: model(r, c) for n, r, c in (("gate", 14336, 4096), ("up", 14336, 4096), ("down", 4096, 14336))}
pat = [2, 3, 4]
c3 = {"block": "Llama-3-8B MLP (gate, up 14336x4096; down 4096x14336)", "p_pattern": pat}
for B in (1, 2, 4, 8, 16):
    ps = [pat[b % 3] for b in range(B)]
    X = {c: torch.randn(B, c, device=dev).half() for c in (4096, 14336)}
    outs = {n: torch.empty(B, m.rows, device=dev, dtype=torch.float32) for n, m in mlp.items()}

    def gemm(i):
        for n, m in mlp.items():
            m.gemm_mixedp(ps, X[m.cols], stream=st)

    def luts(i):
        for n, m in mlp.items():
            gemv_batch([(m, ps[b], X[m.cols][b], outs[n][b]) for b in range(B)], st)
    ug, ul = graph_us(gemm, 4), graph_us(luts, 4)
    c3[f"B{B}"] = {"tensor_core_gemm_us": round(ug, 2), "lut_gemv_batch_us": round(ul, 2),
                   "best": "gemm" if ug < ul else "lut_batch",
                   "request_blocks_per_s": round(B / (min(ug, ul) * 1e-6), 0)}
out["config3_small_batch_gemm"] = c3
del mlp

# ---- config 5 (single GPU) ---------------------------------------------------
c5 = {"note": "one GPU; row-sharded N-GPU runs: bench.py --gpus N under torchrun"}
for n, r, c in (("gate_up_70b", 28672, 8192), ("down_70b", 8192, 28672)):
    ms = [model(r, c, 2, 4) for _ in range(2)]
    xx = torch.randn(c, device=dev).half()
    yy = torch.empty(r, device=dev, dtype=torch.float16)
    for p in (2, 4):
        us = graph_us(lambda i: ms[i % 2].gemv(p, xx, out=yy, stream=st), 8)
        gbs = algo_bytes(r, c, p) / (us * 1e-6) / 1e9
        c5[f"{n}_p{p}"] = {"us": round(us, 2), "GBps": round(gbs, 1), "roofline_frac": round(gbs / PEAK, 4)}
    del ms
out["config5_70b_layers_1gpu"] = c5
print(json.dumps(out, indent=1))
