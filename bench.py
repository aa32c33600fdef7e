#!/usr/bin/env python
"""Benchmark: AnyBCQ bit-plane GEMV on B200 (BASELINE.json configs[1]).

One *step* = the Llama-3-8B layer-shape sweep (q, k, v, o, gate, up, down)
GEMV at batch 1 for every precision p in {2, 3, 4} (21 GEMVs), on synthetic
packed planes (splitmix64 words) and fp16 scales, x in fp16, y in fp16.

  value  = algorithmic bytes of the step / device time  [GB/s]
           (bytes = p-plane bytes + scale-set-p bytes + x + y)
  e2e    = the same through the public API with pinned HOST x/y
           (H2D of x + D2H of y per GEMV inside the timed region)
  roofline: the LUT kernel is the only kernel in the step; achieved =
           algorithmic bytes / kernel time, peak = MEASURED_PEAKS.json hbm_gbs
  cpu_baseline: the reference's LUT algorithm restated in C (oracle/),
           all host threads, on a bounded sample of the same workload

L2: three copies of the layer set (one per precision) so that every plane
byte is re-read only after a full step (>= 245 MB > 126 MB L2).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
For N > 1 (torchrun): each rank holds a 1/N row shard of layers N x taller
(per-rank work = the 1-GPU step, weak scaling) and every GEMV output is
all-gathered over NCCL.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

LAYERS = [("q", 4096, 4096), ("k", 1024, 4096), ("v", 1024, 4096), ("o", 4096, 4096),
          ("gate", 14336, 4096), ("up", 14336, 4096), ("down", 4096, 14336)]
# The timed step runs the 21 independent GEMVs of the sweep (7 layers x
# p=2,3,4 -- per-request precision, the AnyBCQ serving case) as ONE persistent
# mixed-precision batched launch (abcq_gemv_batch). Also reported: the same
# step as one launch per precision, grouped as a decoder issues it
# ([q,k,v] [o] [gate,up] [down] per p), and as 21 single-GEMV launches.
STEP_GROUPS = [tuple(range(7))]
DECODER_GROUPS = [(0, 1, 2), (3,), (4, 5), (6,)]
PRECISIONS = (2, 3, 4)
P_LO, P_HI = 2, 4
SCALE_BYTES = 2   # fp16 scales
XY_BYTES = 2      # fp16 x and y
METRIC = "bit-plane GEMV HBM GB/s (Llama-3-8B layer sweep, p=2/3/4, batch 1)"
WORKLOAD = ("Llama-3-8B layer sweep q/k/v/o/gate/up/down GEMV, batch 1, p=2,3,4 per step, g=128, fp16 "
            "scales/x/y; the 21 independent GEMVs (per-request precision) run as one persistent "
            "mixed-precision batched launch + one split-K reduce launch")


def algo_bytes(rows: int, cols: int, p: int) -> int:
    """p*N*K/8 + p*N*(K/128)*s_w + K*2 + N*2 (symmetric)."""
    G = -(-cols // 128)
    return p * rows * cols // 8 + p * rows * G * SCALE_BYTES + cols * XY_BYTES + rows * XY_BYTES


def step_bytes() -> int:
    return sum(algo_bytes(r, c, p) for p in PRECISIONS for _, r, c in LAYERS)


# ---------------------------------------------------------------------------
def read_peaks():
    try:
        d = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region: an NVML
    polling thread (nvidia_ml_py) while the timed steps run on the device;
    falls back to `nvidia-smi -lms 100` when NVML is unavailable."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4}

    def __init__(self, gpu_index: int):
        self.idx, self.rows, self.stop = gpu_index, [], threading.Event()
        self.nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(gpu_index)
            self.max_sm = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
        except Exception:
            self.nvml = None

    def _poll(self):
        p = self.nvml
        while not self.stop.is_set():
            try:
                ts = time.perf_counter()
                sm = float(p.nvmlDeviceGetClockInfo(self.h, p.NVML_CLOCK_SM))
                try:
                    rs = int(p.nvmlDeviceGetCurrentClocksEventReasons(self.h))
                except Exception:
                    rs = int(p.nvmlDeviceGetCurrentClocksThrottleReasons(self.h))
                self.rows.append((sm, rs, ts, time.perf_counter()))  # (query interval [ts, te])
            except Exception:
                return
            time.sleep(0)  # (yield the GIL; the timed region can be only a few ms long)

    def __enter__(self):
        if self.nvml is not None:
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        if self.nvml is not None:
            self.t.join(timeout=2)

    def mark(self, begin: bool):
        """host time at the start / end of the timed region"""
        if begin:
            self.t0 = time.perf_counter()
        else:
            self.t1 = time.perf_counter()

    def summary(self):
        t0, t1 = getattr(self, "t0", 0.0), getattr(self, "t1", float("inf"))
        # a query counts when its interval overlaps the region (an NVML query can
        # outlast a few-ms region, so 'completed inside' alone can find none)
        rows = [r for r in self.rows if r[2] <= t1 and r[3] >= t0]
        if not rows:
            return self._smi_once()
        sm = [r[0] for r in rows]
        reasons = sorted({n for _, rs, _, _ in rows for n, bit in self.REASONS.items() if rs & bit})
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": self.max_sm, "reasons": reasons,
                "samples": len(rows), "source": "nvml during the timed region"}

    def _smi_once(self):
        try:
            out = subprocess.run(["nvidia-smi", "-i", str(self.idx), "--query-gpu=clocks.sm,clocks.max.sm",
                                  "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                 timeout=10).stdout.strip().split(",")
            return {"sm_mhz": float(out[0]), "sm_max_mhz": float(out[1]), "reasons": ["unsampled-during-run"],
                    "source": "nvidia-smi after the run"}
        except Exception:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}


# ---------------------------------------------------------------------------
def make_layer_models(P, row_scale: int, copies: int, seed0: int = 0, p_lo: int = P_LO, p_hi: int = P_HI):
    """copies x 7 DeviceModels (p p_lo:p_hi, fp16 scales), synthetic planes/scales
    generated on the host from splitmix64."""
    from paper_2510_10467_b200.tensor_io import random_words  # (the GPU leg never imports oracle/)

    models = []
    for c in range(copies):
        row = []
        for li, (name, r, k) in enumerate(LAYERS):
            rows = r * row_scale
            seed = seed0 + 1000 * c + li
            dm = P.DeviceModel(rows, k, 128, p_lo, p_hi, False, scale_dtype="f16")
            dm.load_planes(random_words(p_hi, rows, k, seed=seed))
            rng = np.random.default_rng(seed)
            for p in range(p_lo, p_hi + 1):
                a = (0.01 + 0.1 * np.abs(rng.standard_normal((p, rows, k // 128)))).astype(np.float32)
                dm.load_scale_set(p, a)
            row.append(dm)
        models.append(row)
    return models


def run_gpu(args):
    import torch
    import torch.distributed as dist

    import paper_2510_10467_b200 as P

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    copies = len(PRECISIONS)
    models = make_layer_models(P, 1, copies, seed0=17 * rank)
    xs = {k: (torch.randn(k, device=dev) * 1.0).half() for k in {c for _, _, c in LAYERS}}
    ys = [[torch.empty(m.rows, dtype=torch.float16, device=dev) for m in row] for row in models]
    # multi-GPU step: the 21 row-sharded outputs of a step live in ONE flat
    # buffer, all-gathered by ONE NCCL call that overlaps the next step's
    # GEMV launch (two buffer sets; a step waits only for the gather that last
    # read its buffer)
    mp = world > 1 or os.environ.get("ABCQ_BENCH_FORCE_MP") == "1"
    if mp and not dist.is_initialized():
        dist.init_process_group("nccl", device_id=dev)

    stream = torch.cuda.Stream(device=dev)

    from paper_2510_10467_b200.device_model import gemv_batch

    def grouped_launches(groups):  # (rank 0 only: local launches, no collectives)
        for pi, p in enumerate(PRECISIONS):
            for grp in groups:
                gemv_batch([(models[pi][li], p, xs[models[pi][li].cols], ys[pi][li]) for li in grp], stream)

    all_jobs = [(pi, p, li) for pi, p in enumerate(PRECISIONS) for li in range(len(LAYERS))]

    def step_launches():  # single GPU (multi-GPU: step_mp)
        gemv_batch([(models[pi][li], p, xs[models[pi][li].cols], ys[pi][li]) for pi, p, li in all_jobs], stream)

    mp_rows = sum(models[pi][li].rows for pi, p, li in all_jobs)
    mp_y = [torch.empty(mp_rows, dtype=torch.float16, device=dev) for _ in range(2)] if mp else None
    mp_g = [torch.empty(mp_rows * world, dtype=torch.float16, device=dev) for _ in range(2)] if mp else None
    mp_views = []
    if mp:
        for b in range(2):
            off, v = 0, []
            for pi, p, li in all_jobs:
                v.append(mp_y[b][off:off + models[pi][li].rows])
                off += models[pi][li].rows
            mp_views.append(v)
    mp_work = [None, None]
    mp_plan = [P.GemvBatchPlan([(models[pi][li], p, xs[models[pi][li].cols], mp_views[b][n])
                                for n, (pi, p, li) in enumerate(all_jobs)]) for b in range(2)] if mp else None

    def step_mp(i):
        b = i & 1
        if mp_work[b] is not None:
            mp_work[b].wait()  # (stream waits for the gather that last read mp_y[b])
        mp_plan[b].launch(stream)
        mp_work[b] = dist.all_gather_into_tensor(mp_g[b], mp_y[b], async_op=True)

    def mp_drain():
        for b in range(2):
            if mp_work[b] is not None:
                mp_work[b].wait()
                mp_work[b] = None

    def single_launches():
        for pi, p in enumerate(PRECISIONS):
            for li, m in enumerate(models[pi]):
                m.gemv(p, xs[m.cols], out=ys[pi][li], stream=stream)

    def time_graph(fn, reps=10):
        with torch.cuda.stream(stream):
            fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            fn()
        with torch.cuda.stream(stream):
            g.replay()
            torch.cuda.synchronize()
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            for _ in range(reps):
                g.replay()
            a1.record(stream)
        torch.cuda.synchronize()
        return a0.elapsed_time(a1) / reps

    # warm up (allocates per-stream workspaces), then capture the K timed steps
    # as CUDA graphs of up to 50 consecutive steps each (a graph per step would
    # leave a replay gap between steps)
    with torch.cuda.stream(stream):
        for i in range(max(args.warmup, 3)):
            step_mp(i) if mp else step_launches()
        if mp:
            mp_drain()
    torch.cuda.synchronize()
    use_graph = not mp
    plan = []  # (graph, steps in it), replayed in order: exactly K steps
    if use_graph:
        per = min(args.steps, 50)
        sizes = [per] * (args.steps // per) + ([args.steps % per] if args.steps % per else [])
        built = {}
        for n in sizes:
            if n not in built:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=stream):
                    for _ in range(n):
                        step_launches()
                built[n] = g
            plan.append((built[n], n))
        with torch.cuda.stream(stream):
            for g in built.values():  # (untimed: first replays)
                g.replay()
            for _ in range(args.warmup):
                step_launches()
        torch.cuda.synchronize()

    # ---- timed region: K steps, events on the launching stream ------------
    if mp:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        time.sleep(0.02)  # poller running before the region starts
        clk.mark(True)
        with torch.cuda.stream(stream):
            ev0.record(stream)
            if use_graph:
                for g, _ in plan:
                    g.replay()
            else:
                for i in range(args.steps):
                    step_mp(i)
                mp_drain()  # the last steps' gathers complete inside the timed region
            ev1.record(stream)
        torch.cuda.synchronize()
        clk.mark(False)
    ms = ev0.elapsed_time(ev1)
    if mp:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    ms_step = ms / args.steps
    total_bytes = step_bytes() * world
    value = total_bytes / (ms_step * 1e-3) / 1e9

    # ---- the same step issued as a decoder would, and as 21 single launches --
    variants = {}
    if rank == 0:
        for name, fn in (("one_launch_per_precision", lambda: grouped_launches(STEP_GROUPS)),
                         ("decoder_grouped", lambda: grouped_launches(DECODER_GROUPS)),
                         ("single_launch_per_gemv", single_launches)):
            vms = time_graph(fn)
            variants[name] = {"ms_per_step": round(vms, 4), "GBps": round(step_bytes() / (vms * 1e-3) / 1e9, 1)}

    # ---- per-shape breakdown (device time, back-to-back launches) ----------
    per_shape = {}
    if rank == 0:
        reps = 20
        for li, (name, r, k) in enumerate(LAYERS):
            for pi, p in enumerate(PRECISIONS):
                g2 = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g2, stream=stream):
                    for j in range(reps):
                        models[j % copies][li].gemv(p, xs[k], out=ys[j % copies][li], stream=stream)
                with torch.cuda.stream(stream):   # replay() launches on the current stream
                    g2.replay()
                    torch.cuda.synchronize()
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record(stream)
                    for _ in range(5):
                        g2.replay()
                    b.record(stream)
                torch.cuda.synchronize()
                us = a.elapsed_time(b) * 1e3 / (5 * reps)
                per_shape[f"{name}_{r}x{k}_p{p}"] = {
                    "us": round(us, 3), "GBps": round(algo_bytes(r, k, p) / (us * 1e-6) / 1e9, 1)}

        # ---- p=2 sweep vs the cuBLAS fp16 GEMV sweep, every variant rotating
        # over weight copies whose total exceeds 2x L2 (5 p=2-only layer sets,
        # 272 MB; 2 dense fp16 sets, 235 MB), graphs of back-to-back sweeps
        pool = make_layer_models(P, 1, 5, seed0=500, p_lo=2, p_hi=2)
        ys2 = [[torch.empty(m.rows, dtype=torch.float16, device=dev) for m in row] for row in pool]
        dense = [[torch.randn(r, k, device=dev, dtype=torch.float16) * 0.01 for _, r, k in LAYERS] for _ in range(2)]
        yd = [torch.empty(r, device=dev, dtype=torch.float16) for _, r, _ in LAYERS]
        fused_w = [{g: torch.cat([d[i] for i in g]) for g in DECODER_GROUPS} for d in dense]
        fused_y = {g: torch.empty(fused_w[0][g].shape[0], device=dev, dtype=torch.float16) for g in DECODER_GROUPS}

        def per_sweep(fn, n):  # us per sweep: graph of sweeps over copies 0..n-1
            return 1e3 * time_graph(lambda: [fn(c) for c in range(n)], reps=10) / n

        with torch.cuda.stream(stream):  # cuBLAS handle/workspace before capture
            torch.mv(dense[0][0], xs[LAYERS[0][2]], out=yd[0])
        torch.cuda.synchronize()
        fp16_us = per_sweep(lambda c: [torch.mv(dense[c][li], xs[k], out=yd[li])
                                       for li, (_, r, k) in enumerate(LAYERS)], 2)
        fp16g_us = per_sweep(lambda c: [torch.mv(fused_w[c][g], xs[LAYERS[g[0]][2]], out=fused_y[g])
                                        for g in DECODER_GROUPS], 2)
        p2_us = per_sweep(lambda c: [m.gemv(2, xs[m.cols], out=ys2[c][li], stream=stream)
                                     for li, m in enumerate(pool[c])], 5)
        p2b_us = per_sweep(lambda c: gemv_batch([(m, 2, xs[m.cols], ys2[c][li]) for li, m in enumerate(pool[c])],
                                                stream), 5)
        p2g_us = per_sweep(lambda c: [gemv_batch([(pool[c][li], 2, xs[pool[c][li].cols], ys2[c][li]) for li in g],
                                                 stream) for g in DECODER_GROUPS], 5)
        # decoder-grouped with q/k/v and gate/up as row-stacked AnyBCQ models (one
        # GEMV per group, as the decode harness runs them; cuBLAS likewise on
        # the concatenated fp16 weights) -- BCQ is per row and group: exact
        from paper_2510_10467_b200.tensor_io import random_words
        stacked = []
        for c in range(5):
            row = []
            for gi, g in enumerate(DECODER_GROUPS):
                r, k = sum(LAYERS[i][1] for i in g), LAYERS[g[0]][2]
                dm = P.DeviceModel(r, k, 128, 2, 2, False, scale_dtype="f16")
                dm.load_planes(random_words(2, r, k, seed=900 + 10 * c + gi))
                dm.load_scale_set(2, (0.01 + 0.1 * np.abs(np.random.default_rng(c).standard_normal(
                    (2, r, k // 128)))).astype(np.float32))
                row.append(dm)
            stacked.append(row)
        ys_st = [torch.empty(m.rows, dtype=torch.float16, device=dev) for m in stacked[0]]
        p2s_us = per_sweep(lambda c: [m.gemv(2, xs[m.cols], out=ys_st[gi], stream=stream)
                                      for gi, m in enumerate(stacked[c])], 5)
        del stacked
        fp16_bytes = sum(r * k * 2 + k * 2 + r * 2 for _, r, k in LAYERS)
        fp16 = {"us_per_sweep": round(fp16_us, 2), "GBps": round(fp16_bytes / (fp16_us * 1e-6) / 1e9, 1),
                "abcq_p2_us_per_sweep": round(p2_us, 2), "speedup_p2": round(fp16_us / p2_us, 2),
                "abcq_p2_batched_us_per_sweep": round(p2b_us, 2), "speedup_p2_batched": round(fp16_us / p2b_us, 2),
                "decoder_grouped": {"cublas_fp16_us": round(fp16g_us, 2), "abcq_p2_us": round(p2g_us, 2),
                                    "speedup_p2": round(fp16g_us / p2g_us, 2),
                                    "abcq_p2_stacked_us": round(p2s_us, 2),
                                    "speedup_p2_stacked": round(fp16g_us / p2s_us, 2),
                                    "stacked": "q/k/v and gate/up as one row-stacked AnyBCQ model each "
                                               "(4 single GEMVs per sweep, as tools/decode_bench.py runs them)",
                                    "launches": "4 per sweep each: [q,k,v] [o] [gate,up] [down] (cuBLAS on "
                                                "concatenated fp16 weights)"},
                "note": "7 layers at p=2 vs fp16: cuBLAS 7 torch.mv; abcq 7 single launches / 1 gemv_batch / "
                        "4 decoder-grouped gemv_batch; weights rotate over copies > 2x L2"}
        del pool, fused_w
        del dense

    # ---- per shape, launch latency amortised: one gemv_batch of 8 independent
    # same-shape GEMVs (8 distinct weight sets, e.g. 8 adapters / requests on
    # different models), back to back over 2 such groups (> 2x L2 for the big
    # shapes; the small ones are partly L2-resident -- reported as measured)
    per_shape_b8 = {}
    if rank == 0 and not args.no_cpu:
        peak8, _ = read_peaks()
        for li, (name, r, k) in enumerate(LAYERS):
            if name in ("k", "v", "o", "up"):  # same shapes as q / gate
                continue
            pool8 = []
            for c in range(16):
                dm = P.DeviceModel(r, k, 128, P_LO, P_HI, False, scale_dtype="f16")
                dm.load_planes(torch.randint(-2**31, 2**31 - 1, (P_HI, r, k // 32), dtype=torch.int32, device=dev))
                for pp in PRECISIONS:
                    dm.load_scale_set(pp, 0.01 + 0.1 * torch.rand(pp, r, k // 128, device=dev))
                pool8.append(dm)
            yb = [torch.empty(r, dtype=torch.float16, device=dev) for _ in range(16)]
            for pp in PRECISIONS:
                us = 1e3 * time_graph(lambda: [gemv_batch([(pool8[8 * h + j], pp, xs[k], yb[8 * h + j]) for j in range(8)],
                                                          stream) for h in range(2)], reps=10) / 2
                gbps = 8 * algo_bytes(r, k, pp) / (us * 1e-6) / 1e9
                per_shape_b8[f"{name}_{r}x{k}_p{pp}"] = {"us_per_launch": round(us, 2), "GBps": round(gbps, 1),
                                                         "roofline_frac": round(gbps / peak8, 4)}
            del pool8, yb

    # ---- e2e: public API with pinned host buffers, copies in the timed region
    e2e = None
    if rank == 0:
        # one pinned staging buffer each way per step: x of both input widths
        # in, the 21 outputs out (views of one device buffer) -- one copy per
        # direction and step. Serving-style pipeline: two buffer sets, the H2D
        # of step i+1 and the D2H of step i on their own streams overlap the
        # GEMV launch of step i (event-ordered; every step still moves its
        # own bytes both ways inside the timed region)
        kx = sorted(xs)
        hx = torch.cat([xs[k].cpu() for k in kx]).pin_memory()
        n_out = sum(models[pi][li].rows for pi, p, li in all_jobs)
        sets = []
        for _ in range(2):
            dxa = torch.empty_like(hx, device=dev)
            dx, off = {}, 0
            for k in kx:
                dx[k] = dxa[off:off + k]
                off += k
            dya = torch.empty(n_out, dtype=torch.float16, device=dev)
            dys, off = [], 0
            for pi, p, li in all_jobs:
                dys.append(dya[off:off + models[pi][li].rows])
                off += models[pi][li].rows
            sets.append({"dxa": dxa, "dx": dx, "dya": dya, "dys": dys,
                         "hy": torch.empty(n_out, dtype=torch.float16).pin_memory(),
                         "in": torch.cuda.Event(), "comp": torch.cuda.Event(), "out": torch.cuda.Event()})
        for S in sets:  # the public API's repeated-launch form (validated and marshalled once)
            S["plan"] = P.GemvBatchPlan([(models[pi][li], p, S["dx"][models[pi][li].cols], S["dys"][n])
                                         for n, (pi, p, li) in enumerate(all_jobs)])
        s_in, s_out = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
        h2d = d2h = 0

        def e2e_step(i):
            nonlocal h2d, d2h
            S = sets[i & 1]
            with torch.cuda.stream(s_in):
                s_in.wait_event(S["comp"])  # the GEMV that last read this x buffer is done
                S["dxa"].copy_(hx, non_blocking=True)
                S["in"].record(s_in)
            h2d += hx.numel() * 2
            stream.wait_event(S["in"])
            stream.wait_event(S["out"])  # the D2H that last read this y buffer is done
            S["plan"].launch(stream)
            S["comp"].record(stream)
            with torch.cuda.stream(s_out):
                s_out.wait_event(S["comp"])
                S["hy"].copy_(S["dya"], non_blocking=True)
                S["out"].record(s_out)
            d2h += S["dya"].numel() * 2

        with torch.cuda.stream(stream):
            for S in sets:
                for e in ("in", "comp", "out"):
                    S[e].record(stream)
            for i in range(4):
                e2e_step(i)
            torch.cuda.synchronize()
            h2d = d2h = 0
            n_e2e = max(4, min(args.steps, 50))
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            s_in.wait_stream(stream)
            s_out.wait_stream(stream)
            for i in range(n_e2e):
                e2e_step(i)
            stream.wait_stream(s_out)
            b.record(stream)
            torch.cuda.synchronize()
        e2e_ms = a.elapsed_time(b) / n_e2e
        e2e = {"value": round(step_bytes() / (e2e_ms * 1e-3) / 1e9, 1), "unit": "GB/s",
               "ms_per_step": round(e2e_ms, 4), "h2d_bytes_per_step": h2d // n_e2e,
               "d2h_bytes_per_step": d2h // n_e2e,
               "api": "GemvBatchPlan.launch of the 21 GEMVs (one C-ABI abcq_gemv_batch call per step), eager; "
                      "pinned host x in and y out, one copy each way per step, copies of neighbouring steps "
                      "overlapped on two side streams"}

    if rank == 0:
        peak, peak_kind = read_peaks()
        kernel_bytes = step_bytes()
        achieved = kernel_bytes / (ms_step * 1e-3) / 1e9
        traffic = None
        tf = ROOT / "profiles" / "ncu_traffic.json"
        if tf.exists():  # ncu dram__bytes_read+write per launch of the batched kernel (profiles/)
            try:
                traffic = int(json.loads(tf.read_text())["traffic_bytes_per_launch"])
            except Exception:
                traffic = None
        cpu = cpu_baseline() if world == 1 and not args.no_cpu else None
        line = {
            "metric": METRIC, "value": round(value, 1), "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 5),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic (splitmix64 planes, |N(0,1)| fp16 scales, N(0,1) fp16 x)",
            "config": {"workload": WORKLOAD,
                       "layers": {n: [r, k] for n, r, k in LAYERS}, "precisions": list(PRECISIONS),
                       "bytes_per_step": kernel_bytes,
                       "l2": "inputs larger than L2: 3 plane-set copies, reuse distance = 1 step "
                             f"({kernel_bytes / 1e6:.0f} MB) > 126 MB",
                       "timing": ("the K steps captured as CUDA graphs of <= 50 steps, CUDA events on the launch stream"
                                  if not mp else "eager steps, one NCCL all-gather of the step's 21 outputs per "
                                  "step overlapping the next step (double-buffered), CUDA events, max over ranks"),
                       "parallelism": f"row-shard x{world}" if world > 1 else "single GPU"},
            # per step: the persistent batched GEMV kernel + the split-K reduce kernel
            "gpu_launches": args.steps * 2,  # (+ one NCCL all-gather per step when multi-GPU)
            "step_variants": variants,
            "e2e": e2e,
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "peak_kind": peak_kind,
                         "kernel": "abcq::gemv_batch_kernel (+ batch_reduce_kernel)", "traffic": traffic,
                         "algorithmic_bytes_per_step": kernel_bytes},
            "cpu_baseline": cpu,
            "clocks": clk.summary(),
            "per_shape": per_shape,
            "per_shape_batched8": per_shape_b8,
            "per_shape_batched8_note": "one gemv_batch of 8 independent same-shape GEMVs (distinct weights) per "
                                       "launch, back to back: the per-shape kernel rate with the launch latency "
                                       "amortised",
            "per_shape_note": "single launches, graph of 20 back-to-back launches rotating 3 weight copies "
                              "(the smaller layers can be partly L2-resident)",
            "fp16_cublas": fp16,
        }
        print(json.dumps(line))
    if mp:
        dist.destroy_process_group()


# ---------------------------------------------------------------------------
def _cpu_sample_models():
    from oracle import anybcq_oracle as O
    out = []
    for li, (name, r, k) in enumerate(LAYERS):
        words = O.random_words(P_HI, r, k, seed=li)
        rng = np.random.default_rng(li)
        alphas = {p: (0.01 + 0.1 * np.abs(rng.standard_normal((p, r, k // 128)))).astype(np.float16)
                  .astype(np.float32) for p in PRECISIONS}
        out.append((name, r, k, words, alphas))
    return out


def cpu_baseline(repeats: int = 2):
    """The reference LUT algorithm (C port of gemv.py:67-95,188-222) on all host
    cores, over the full layer sweep (the GPU step's workload), `repeats` times."""
    from oracle import c_oracle

    threads = c_oracle.cpu_threads()
    models = _cpu_sample_models()
    x = {k: np.random.default_rng(k).standard_normal(k).astype(np.float16).astype(np.float64)
         for k in {c for _, _, c in LAYERS}}
    for name, r, k, words, alphas in models[:1]:
        c_oracle.lut_gemv(words, k, 128, alphas[2], None, 2, x[k], threads)  # warm
    t0 = time.perf_counter()
    for _ in range(repeats):
        for p in PRECISIONS:
            for name, r, k, words, alphas in models:
                c_oracle.lut_gemv(words, k, 128, alphas[p], None, p, x[k], threads)
    dt = (time.perf_counter() - t0) / repeats
    return {"value": round(step_bytes() / dt / 1e9, 3), "unit": "GB/s", "cores": threads, "kind": "port",
            "ms_per_step": round(dt * 1e3, 1),
            "sample": f"full layer sweep (21 GEMVs) x{repeats}, C restatement of GemvEngine.lut, "
                      f"{threads} pthreads"}


def run_reference(args):
    """--impl reference: the reference's CPU algorithm (C port) on this workload."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import c_oracle

    threads = c_oracle.cpu_threads()
    models = _cpu_sample_models()
    x = {k: np.random.default_rng(k).standard_normal(k).astype(np.float16).astype(np.float64)
         for k in {c for _, _, c in LAYERS}}

    def one_step():
        for p in PRECISIONS:
            for name, r, k, words, alphas in models:
                c_oracle.lut_gemv(words, k, 128, alphas[p], None, p, x[k], threads)

    for _ in range(args.warmup):
        one_step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        one_step()
    dt = (time.perf_counter() - t0) / args.steps
    value = round(step_bytes() / dt / 1e9, 3)
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s",
        "n_gpus": int(os.environ.get("WORLD_SIZE", "1")),
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt * 1e3, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic", "config": {"workload": WORKLOAD, "implementation": "reference CPU algorithm "
                                        "(C restatement of GemvEngine.lut, all host threads)"},
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": threads, "kind": "port",
                         "sample": "full layer sweep per step (C restatement of GemvEngine.lut; "
                                   "reference is Python+numba, no compiled sources to build)"},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
