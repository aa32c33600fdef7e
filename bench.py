#!/usr/bin/env python
"""Benchmark: AnyBCQ bit-plane GEMV on B200 (BASELINE.json configs[1] headline,
every other BASELINE config reported beside it).

Headline step = the Llama-3-8B layer-shape sweep (q, k, v, o, gate, up, down)
GEMV at batch 1 for every precision p in {2, 3, 4} (21 GEMVs = 21 requests
with per-request precision) on synthetic packed planes (splitmix64 words,
tensor_io.random_words) and fp16 scales, x and y in fp16, run as ONE
persistent mixed-precision batched launch (+ its split-K reduce launch).

  value    = algorithmic bytes of the step / device time  [GB/s]
             (bytes = p-plane bytes + scale-set-p bytes + x + y)
  parity   = one untimed step of the EXACT timed configuration checked against
             the C port of GemvEngine.lut on the identical host inputs
  e2e      = the same through the public API with pinned HOST x/y
  roofline = the LUT kernel (the only kernel of the step); achieved =
             algorithmic bytes / kernel time, peak = MEASURED_PEAKS.json
  cpu_baseline: the reference's LUT algorithm restated in C (oracle/), all
             host threads and one thread, plus the real reference (numba,
             baseline/_ref) on a 4096x4096 layer when installed
  config1..config5: BASELINE.json configs[0..4] (see each key's "what")

L2: three copies of the layer set (one per precision) so that every plane
byte is re-read only after a full step (>= 245 MB > 126 MB L2); per-shape
pools rotate over copies whose total exceeds 2x L2.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
For N > 1 (torchrun; `--gpus N` without torchrun re-launches itself under
torchrun): each rank holds a 1/N row shard of layers N x taller (per-rank
work = the 1-GPU step, weak scaling) and every step's outputs are
all-gathered over NCCL; config5 row-shards the Llama-3-70B layers over the N
ranks (strong scaling, GEMV-only and GEMV + all-gather times).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import socket
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
LAYERS_70B = [("q", 8192, 8192), ("k", 1024, 8192), ("v", 1024, 8192), ("o", 8192, 8192),
              ("gate", 28672, 8192), ("up", 28672, 8192), ("down", 8192, 28672)]
STEP_GROUPS = [tuple(range(7))]
DECODER_GROUPS = [(0, 1, 2), (3,), (4, 5), (6,)]
PRECISIONS = (2, 3, 4)
E2E_GROUP = 4     # e2e steps per copy-pipeline group
E2E_SETS = int(os.environ.get("ABCQ_BENCH_E2E_SETS", "4"))  # buffer sets in flight (groups computing / copying)
MP_RESERVE_SMS = 4  # N > 1: SMs left to the overlapping NCCL all-gather (abcq_set_reserved_sms, NCCL_MAX_CTAS)
P_LO, P_HI = 2, 4
SCALE_BYTES = 2   # fp16 scales
XY_BYTES = 2      # fp16 x and y
L2_BYTES = 126 * 1024 * 1024
METRIC = "bit-plane GEMV HBM GB/s (Llama-3-8B layer sweep, p=2/3/4, batch 1)"
WORKLOAD = ("Llama-3-8B layer sweep q/k/v/o/gate/up/down GEMV, batch 1, p=2,3,4 per step, g=128, fp16 "
            "scales/x/y; the 21 independent GEMVs (per-request precision) run as one persistent "
            "mixed-precision batched launch + one split-K reduce launch")
DTYPE = "f32"   # arithmetic: f32 table entries (reference rounding), f32 group sums and accumulation
DTYPE_NOTE = "storage: 1-bit sign planes, fp16 scales / x / y; arithmetic f32 (tables, sums, accumulation)"


def algo_bytes(rows: int, cols: int, p: int) -> int:
    """p*N*K/8 + p*N*(K/128)*s_w + K*2 + N*2 (symmetric)."""
    G = -(-cols // 128)
    return p * rows * cols // 8 + p * rows * G * SCALE_BYTES + cols * XY_BYTES + rows * XY_BYTES


def step_bytes() -> int:
    return sum(algo_bytes(r, c, p) for p in PRECISIONS for _, r, c in LAYERS)


def bench_config(world: int) -> dict:
    """The config dict printed by BOTH arms (identical keys and values)."""
    return {"workload": WORKLOAD, "layers": {n: [r, k] for n, r, k in LAYERS}, "precisions": list(PRECISIONS),
            "group_size": 128, "batch": 1, "bytes_per_step": step_bytes(),
            "l2": f"inputs larger than L2: 3 plane-set copies, reuse distance = 1 step "
                  f"({step_bytes() / 1e6:.0f} MB) > 126 MB",
            "parallelism": f"row-shard x{world}" if world > 1 else "single GPU"}


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


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
class Ctx:
    """What every section needs: torch, the package, the device and stream."""

    def __init__(self, dev, stream, rank, world):
        import torch

        import paper_2510_10467_b200 as P
        from paper_2510_10467_b200.device_model import gemv_batch

        self.torch, self.P, self.gemv_batch = torch, P, gemv_batch
        self.dev, self.stream, self.rank, self.world = dev, stream, rank, world

    def time_graph(self, fn, reps=10):
        """ms per call of fn: fn captured once as a CUDA graph, replayed reps times."""
        torch, st = self.torch, self.stream
        with torch.cuda.stream(st):
            fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            fn()
        with torch.cuda.stream(st):
            g.replay()
            torch.cuda.synchronize()
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record(st)
            for _ in range(reps):
                g.replay()
            a1.record(st)
        torch.cuda.synchronize()
        return a0.elapsed_time(a1) / reps

    def device_model(self, rows, cols, p_lo, p_hi, seed, asym=False):
        """A DeviceModel with device-RNG planes and |N|-ish fp16 scales (pools, 70B shards)."""
        torch = self.torch
        g = torch.Generator(device=self.dev).manual_seed(seed)
        dm = self.P.DeviceModel(rows, cols, 128, p_lo, p_hi, asym, scale_dtype="f16", device=self.dev)
        dm.load_planes(torch.randint(-2**31, 2**31 - 1, (p_hi, rows, cols // 32), dtype=torch.int32,
                                     device=self.dev, generator=g))
        for p in range(p_lo, p_hi + 1):
            a = 0.01 + 0.1 * torch.rand((p, rows, cols // 128), device=self.dev, generator=g)
            z = 0.1 * torch.randn((rows, cols // 128), device=self.dev, generator=g) if asym else None
            dm.load_scale_set(p, a, z)
        return dm


def make_layer_models(P, row_scale: int, copies: int, seed0: int = 0, p_lo: int = P_LO, p_hi: int = P_HI,
                      keep_host: bool = False):
    """copies x 7 DeviceModels (p p_lo:p_hi, fp16 scales), synthetic planes /
    scales generated on the host (splitmix64 words); with keep_host
    the host arrays (words, f16-rounded alphas) are returned for the parity
    check against the C port on IDENTICAL inputs."""
    from paper_2510_10467_b200.tensor_io import random_words  # (the GPU leg never imports oracle/)

    models, host = [], []
    for c in range(copies):
        row, hrow = [], []
        for li, (name, r, k) in enumerate(LAYERS):
            rows = r * row_scale
            seed = seed0 + 1000 * c + li
            dm = P.DeviceModel(rows, k, 128, p_lo, p_hi, False, scale_dtype="f16")
            words = random_words(p_hi, rows, k, seed=seed)
            dm.load_planes(words)
            rng = np.random.default_rng(seed)
            alphas = {}
            for p in range(p_lo, p_hi + 1):
                a = (0.01 + 0.1 * np.abs(rng.standard_normal((p, rows, k // 128)))).astype(np.float32)
                dm.load_scale_set(p, a)
                alphas[p] = a.astype(np.float16).astype(np.float32)  # what the f16 device set holds
            row.append(dm)
            hrow.append((words, alphas) if keep_host else None)
        models.append(row)
        host.append(hrow)
    return models, host


def parity_check(ctx, models, host, xs_host, ys, jobs):
    """The exact timed configuration's outputs (already computed by one untimed
    step) vs the C port of GemvEngine.lut on the identical host inputs."""
    from oracle import anybcq_oracle as O  # checker only
    from oracle import c_oracle

    threads = c_oracle.cpu_threads()
    worst, worst_job, devs = 0.0, None, {}
    for pi, p, li in jobs:
        words, alphas = host[pi][li]
        k = LAYERS[li][2]
        want = c_oracle.lut_gemv(words, k, 128, alphas[p], None, p, xs_host[k].astype(np.float64), threads)
        got = ys[pi][li].float().cpu().numpy()
        d = O.rel_dev(got, want)
        devs[f"{LAYERS[li][0]}_p{p}"] = float(f"{d:.3e}")
        if d > worst:
            worst, worst_job = d, f"{LAYERS[li][0]}_p{p}"
    return {"max_rel_dev": float(f"{worst:.3e}"), "worst_job": worst_job, "tolerance": 1e-3,
            "ok": worst <= 1e-3, "per_job": devs,
            "what": "one untimed step of the exact timed configuration (21 jobs, one batched launch, fp16 x/y/"
                    "scales) vs the C port of GemvEngine.lut on identical inputs; rel_dev = max|y-y_ref| / "
                    "max|y_ref| (fp16 y rounding included)"}


def run_gpu(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        sys.exit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    mp = world > 1 or os.environ.get("ABCQ_BENCH_FORCE_MP") == "1"
    mp_reserve = 0
    if mp:
        # the step's all-gather runs beside the next step's GEMV (another
        # stream): NCCL is capped at MP_RESERVE_SMS CTAs and the persistent
        # GEMV grid leaves that many SMs free, so neither waits for the
        # other's SMs (at world size 1 -- the forced-MP test -- the gather is a
        # local copy and the reserve only costs: 4.61 vs 4.68 TB/s)
        mp_reserve = int(os.environ.get("ABCQ_BENCH_MP_RESERVE", str(MP_RESERVE_SMS if world > 1 else 0)))
        if mp_reserve:
            os.environ.setdefault("NCCL_MAX_CTAS", str(mp_reserve))
            os.environ.setdefault("NCCL_MIN_CTAS", "1")
        dist.init_process_group("nccl", device_id=dev)
    stream = torch.cuda.Stream(device=dev)
    ctx = Ctx(dev, stream, rank, world)
    P, gemv_batch = ctx.P, ctx.gemv_batch
    if mp_reserve:
        P.set_reserved_sms(mp_reserve)

    copies = len(PRECISIONS)
    models, host = make_layer_models(P, 1, copies, seed0=17 * rank, keep_host=(rank == 0))
    rng = np.random.default_rng(1234 + rank)
    xs_host = {k: rng.standard_normal(k).astype(np.float16) for k in sorted({c for _, _, c in LAYERS})}
    xs = {k: torch.from_numpy(v).to(dev) for k, v in xs_host.items()}
    ys = [[torch.empty(m.rows, dtype=torch.float16, device=dev) for m in row] for row in models]
    all_jobs = [(pi, p, li) for pi, p in enumerate(PRECISIONS) for li in range(len(LAYERS))]

    def step_launches():
        gemv_batch([(models[pi][li], p, xs[models[pi][li].cols], ys[pi][li]) for pi, p, li in all_jobs], stream)

    # multi-GPU step: the 21 row-sharded outputs of a step live in ONE flat
    # buffer, all-gathered by ONE NCCL call that overlaps the next step's GEMV
    # launch (two buffer sets; a step waits only for the gather that last read
    # its buffer)
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
    # the product's multi-GPU step: the all-gather FUSED into the GEMV launch --
    # its split-K completion stores every row into all ranks' symmetric buffers
    # over NVLink peer memory (abcq_gemv_batch_peer); NCCL (above) if torch
    # symmetric memory is unavailable or ABCQ_BENCH_ALLGATHER=nccl
    ag_mode, peer, peer_plan = "nccl", None, None
    if mp and os.environ.get("ABCQ_BENCH_ALLGATHER", "peer") == "peer":
        try:
            from paper_2510_10467_b200.parallel import PeerGather
            peer = PeerGather(mp_rows, device=dev)
            off, pv = 0, []
            for pi, p, li in all_jobs:
                pv.append(peer.local[off:off + models[pi][li].rows])
                off += models[pi][li].rows
            peer_plan = peer.plan([(models[pi][li], p, xs[models[pi][li].cols], pv[n])
                                   for n, (pi, p, li) in enumerate(all_jobs)])
            ag_mode = "peer"
        except Exception as exc:  # noqa: BLE001
            peer = peer_plan = None
            ag_mode = f"nccl (fused peer all-gather unavailable: {str(exc)[:100]})"
        ok = torch.tensor([1 if peer is not None else 0], device=dev)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)  # every rank takes the same path
        if peer is not None and int(ok.item()) == 0:
            peer = peer_plan = None
            ag_mode = "nccl (fused peer all-gather unavailable on another rank)"
    if mp_reserve and ag_mode == "peer":  # no collective kernel beside the GEMV grid
        P.set_reserved_sms(0)
        mp_reserve = 0

    def step_mp(i):
        b = i & 1
        if mp_work[b] is not None:
            mp_work[b].wait()
        mp_plan[b].launch(stream)
        mp_work[b] = dist.all_gather_into_tensor(mp_g[b], mp_y[b], async_op=True)

    def mp_drain():
        for b in range(2):
            if mp_work[b] is not None:
                mp_work[b].wait()
                mp_work[b] = None

    # ---- parity of the exact timed configuration (untimed, rank 0) ---------
    with torch.cuda.stream(stream):
        step_launches()
    torch.cuda.synchronize()
    parity = parity_check(ctx, models, host, xs_host, ys, all_jobs) if rank == 0 else None
    host = None  # (release the host copies)

    # warm up, then capture the K timed steps as CUDA graphs of up to 50 steps
    with torch.cuda.stream(stream):
        for i in range(max(args.warmup, 3)):
            step_mp(i) if mp else step_launches()
        if mp:
            mp_drain()
        if peer_plan is not None:  # (its workspace allocated outside the graph capture)
            for i in range(max(args.warmup, 3)):
                peer_plan.launch(stream)
    torch.cuda.synchronize()

    side = torch.cuda.Stream(device=dev) if mp else None
    ev_done = [torch.cuda.Event() for _ in range(2)]      # GEMV of buffer b written
    ev_gathered = [torch.cuda.Event() for _ in range(2)]  # all-gather of buffer b read it

    def step_mp_graphed(i):
        # inside a CUDA graph: the step's GEMV launch on the main stream, its
        # NCCL all-gather forked to a side stream so it overlaps the next
        # step's GEMV (two output buffers; a GEMV waits only for the gather
        # that last read its buffer). Graph replay removes the host-driven
        # loop's per-step enqueue cost, as on one GPU.
        b = i & 1
        if i >= 2:
            stream.wait_event(ev_gathered[b])
        mp_plan[b].launch(stream)
        ev_done[b].record(stream)
        side.wait_event(ev_done[b])
        with torch.cuda.stream(side):
            dist.all_gather_into_tensor(mp_g[b], mp_y[b])
            ev_gathered[b].record(side)

    def graph_steps(n):
        if not mp:
            for _ in range(n):
                step_launches()
            return
        if peer_plan is not None:
            for _ in range(n):
                peer_plan.launch(stream)
            return
        side.wait_stream(stream)
        for i in range(n):
            step_mp_graphed(i)
        stream.wait_stream(side)  # (the last gathers complete inside the graph)

    use_graph = True
    plan = []
    graph_mode = "graphs"
    if use_graph:
        per = min(args.steps, 50)
        sizes = [per] * (args.steps // per) + ([args.steps % per] if args.steps % per else [])
        built = {}
        try:
            for n in sizes:
                if n not in built:
                    g = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(g, stream=stream):
                        graph_steps(n)
                    built[n] = g
                plan.append((built[n], n))
        except Exception as exc:  # (NCCL capture unsupported here: the eager overlapped loop)
            if not mp:
                raise
            torch.cuda.synchronize()
            use_graph, plan, graph_mode = False, [], f"eager ({str(exc)[:60]})"
    if use_graph:
        with torch.cuda.stream(stream):
            for g in built.values():
                g.replay()
        torch.cuda.synchronize()

    # ---- timed region: K steps, events on the launching stream ------------
    if mp:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        time.sleep(0.02)
        clk.mark(True)
        with torch.cuda.stream(stream):
            ev0.record(stream)
            if use_graph:
                for g, _ in plan:
                    g.replay()
            elif peer_plan is not None:
                for i in range(args.steps):
                    peer_plan.launch(stream)
            else:
                for i in range(args.steps):
                    step_mp(i)
                mp_drain()
            ev1.record(stream)
        while not ev1.query():  # wait without holding the GIL, so the clock sampler keeps polling
            time.sleep(0.0002)
        torch.cuda.synchronize()
        clk.mark(False)
    ms = ev0.elapsed_time(ev1)
    if mp:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    ms_step = ms / args.steps
    value = step_bytes() * world / (ms_step * 1e-3) / 1e9
    ag_check = None
    if peer is not None:  # every rank's latest rows in this rank's buffer == an NCCL all-gather of them
        with torch.cuda.stream(stream):
            peer.wait(stream)
        torch.cuda.synchronize()
        dist.barrier()
        ref = torch.empty_like(peer.buffer)
        dist.all_gather_into_tensor(ref, peer.local.clone())
        torch.cuda.synchronize()
        ag_check = bool(torch.equal(ref, peer.buffer)) and int(peer.err.item()) == 0
    ag_alt = None
    if peer is not None:  # the baseline beside it: the same GEMV steps + an NCCL all-gather on a side stream
        try:
            rsv = MP_RESERVE_SMS if world > 1 else 0
            P.set_reserved_sms(rsv)  # (the collective's SMs, as in the NCCL mode)
            n_alt = min(args.steps, 50)
            g2 = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g2, stream=stream):
                side.wait_stream(stream)
                for i in range(n_alt):
                    step_mp_graphed(i)
                stream.wait_stream(side)
            with torch.cuda.stream(stream):
                g2.replay()
            torch.cuda.synchronize()
            dist.barrier()
            a2, b2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(stream):
                a2.record(stream)
                g2.replay()
                b2.record(stream)
            torch.cuda.synchronize()
            t2 = torch.tensor([a2.elapsed_time(b2)], device=dev)
            dist.all_reduce(t2, op=dist.ReduceOp.MAX)
            ms2 = float(t2.item()) / n_alt
            ag_alt = {"allgather": f"nccl on a side stream overlapping the next GEMV ({rsv} SMs reserved)",
                      "ms_per_step": round(ms2, 5), "value": round(step_bytes() * world / (ms2 * 1e-3) / 1e9, 1)}
            P.set_reserved_sms(0)
            del g2
        except Exception as exc:  # noqa: BLE001
            ag_alt = {"error": str(exc)[:120]}

    peak, peak_kind = read_peaks()
    sections = set(args.sections.split(",")) if args.sections else None
    want = (lambda name: sections is None or name in sections)

    # ---- config5: Llama-3-70B layers row-sharded over the N ranks (all ranks)
    cfg5 = config5_row_sharded(ctx, args, peak) if want("config5") else None

    out = {}
    if rank == 0:
        if want("variants"):
            out.update(step_variants(ctx, models, xs, ys, peak))
        if want("per_shape"):
            out["per_shape"] = per_shape(ctx, xs)
        if want("fp16"):
            out["fp16_cublas"] = fp16_comparison(ctx, xs)
        if want("batched8"):
            out["per_shape_batched8"] = per_shape_batched8(ctx, xs, peak)
        if want("e2e"):
            out["e2e"] = e2e_section(ctx, models, xs, all_jobs, args)
        if want("config1"):
            out["config1"] = config1(ctx, args, peak)
        if want("config3"):
            out["config3"] = config3(ctx)
        if want("config4"):
            out["config4"] = config4(ctx, args)
        if want("loader"):
            out["loader"] = loader_section(ctx, args)
        if want("quantizer"):
            out["quantizer"] = quantizer_section(ctx, args)
    if mp:
        dist.barrier()

    if rank == 0:
        achieved = step_bytes() / (ms_step * 1e-3) / 1e9
        traffic = None
        tf = ROOT / "profiles" / "ncu_traffic.json"
        if tf.exists():
            try:
                traffic = int(json.loads(tf.read_text())["traffic_bytes_per_launch"])
            except Exception:
                traffic = None
        cpu = cpu_baseline() if world == 1 and not args.no_cpu else None
        config = bench_config(world)  # (identical to the reference arm's: same_config)
        timing = ("the K steps captured as CUDA graphs of <= 50 steps, CUDA events on the launch stream"
                  if not mp else ("the K steps captured as CUDA graphs of <= 50 steps, each step one GEMV launch + "
                                  "one NCCL all-gather of its 21 outputs on a side stream overlapping the next "
                                  "step's GEMV (double-buffered), CUDA events, max over ranks"
                                  if use_graph else graph_mode + ": one NCCL all-gather of the step's 21 outputs "
                                  "per step overlapping the next step (double-buffered), CUDA events, max over ranks"))
        if mp_reserve:
            timing += f"; the GEMV grid leaves {mp_reserve} SMs to the all-gather (NCCL_MAX_CTAS={mp_reserve})"
        if peer is not None:
            timing = ("the K steps captured as CUDA graphs of <= 50 steps, each step ONE GEMV launch whose split-K "
                      "completion also stores its rows into every rank's symmetric buffer over NVLink peer memory "
                      "(the all-gather fused into the GEMV, abcq_gemv_batch_peer), CUDA events, max over ranks")
        line = {
            "metric": METRIC, "value": round(value, 1), "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 5),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": DTYPE,
            "dtype_note": DTYPE_NOTE,
            "data": "synthetic (splitmix64 planes, |N(0,1)| fp16 scales, N(0,1) fp16 x)",
            "config": config,
            "timing": timing,
            # per step: the persistent batched GEMV kernel + the split-K reduce kernel
            "gpu_launches": args.steps * 2,
            "parity": parity,
            "e2e": out.pop("e2e", None),
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "peak_kind": peak_kind,
                         "kernel": "abcq::gemv_batch_kernel (+ batch_reduce_kernel)", "traffic": traffic,
                         "algorithmic_bytes_per_step": step_bytes()},
            "cpu_baseline": cpu,
            "clocks": clk.summary(),
            "config5": cfg5,
        }
        if mp:
            line["allgather"] = ag_mode
            line["allgather_check"] = ag_check
            line["allgather_nccl_variant"] = ag_alt
        line.update(out)
        print(json.dumps(line))
    if mp:
        dist.destroy_process_group()


# ---------------------------------------------------------------------------
def step_variants(ctx, models, xs, ys, peak):
    """The same 21 GEMVs issued as a decoder would (one batched launch per
    [q,k,v] [o] [gate,up] [down] group and precision), as 21 single launches,
    and one launch per precision; each with its roofline fraction."""
    gemv_batch, st = ctx.gemv_batch, ctx.stream

    def grouped(groups):  # a group of one is a single GEMV (abcq_gemv: the cluster kernel where it wins)
        for pi, p in enumerate(PRECISIONS):
            for grp in groups:
                if len(grp) == 1:
                    m = models[pi][grp[0]]
                    m.gemv(p, xs[m.cols], out=ys[pi][grp[0]], stream=st)
                else:
                    gemv_batch([(models[pi][li], p, xs[models[pi][li].cols], ys[pi][li]) for li in grp], st)

    def singles():
        for pi, p in enumerate(PRECISIONS):
            for li, m in enumerate(models[pi]):
                m.gemv(p, xs[m.cols], out=ys[pi][li], stream=st)

    res = {}
    for name, fn in (("one_launch_per_precision", lambda: grouped(STEP_GROUPS)),
                     ("decoder_grouped", lambda: grouped(DECODER_GROUPS)),
                     ("single_launch_per_gemv", singles)):
        ms = ctx.time_graph(fn)
        gbps = step_bytes() / (ms * 1e-3) / 1e9
        res[name] = {"ms_per_step": round(ms, 4), "GBps": round(gbps, 1), "roofline_frac": round(gbps / peak, 4)}
    return {"step_variants": res,
            "roofline_decoder_grouped": {"bound": "hbm", "achieved": res["decoder_grouped"]["GBps"], "peak": peak,
                                         "unit": "GB/s", "frac": res["decoder_grouped"]["roofline_frac"],
                                         "what": "the step's 21 GEMVs as a decoder issues them: 4 launches per "
                                                 "precision ([q,k,v] and [gate,up] batched launches, [o] and [down] "
                                                 "single GEMVs)"},
            "roofline_single_launch": {"bound": "hbm", "achieved": res["single_launch_per_gemv"]["GBps"],
                                       "peak": peak, "unit": "GB/s",
                                       "frac": res["single_launch_per_gemv"]["roofline_frac"],
                                       "what": "21 dependent-style single-GEMV launches back to back"}}


def _pool(ctx, rows, cols, p_lo, p_hi, seed0, min_copies=2, max_copies=64):
    """Copies of one shape whose plane bytes exceed 2x L2 (capped)."""
    per = p_hi * rows * cols // 8
    n = max(min_copies, min(max_copies, math.ceil(2 * L2_BYTES / per) + 1))
    return [ctx.device_model(rows, cols, p_lo, p_hi, seed0 + c) for c in range(n)]


def per_shape(ctx, xs):
    """Single launches back to back (graph of 20), rotating over > 2x L2 of copies."""
    torch = ctx.torch
    res = {}
    for li, (name, r, k) in enumerate(LAYERS):
        if name in ("v", "up"):  # same shapes as k / gate
            continue
        pool = _pool(ctx, r, k, P_LO, P_HI, 7000 + 100 * li)
        y = torch.empty(r, dtype=torch.float16, device=ctx.dev)
        for p in PRECISIONS:
            n = 20
            ms = ctx.time_graph(lambda: [pool[j % len(pool)].gemv(p, xs[k], out=y, stream=ctx.stream)
                                         for j in range(n)], reps=5)
            us = ms * 1e3 / n
            res[f"{name}_{r}x{k}_p{p}"] = {"us": round(us, 3), "GBps": round(algo_bytes(r, k, p) / (us * 1e-6) / 1e9, 1),
                                           "copies": len(pool)}
        del pool
    res["note"] = ("single GEMV launches back to back (graph of 20), rotating over weight copies totalling > 2x L2 "
                   "(capped at 64 copies); the small layers are latency-bound")
    return res


def fp16_comparison(ctx, xs):
    """p=2 sweep vs the cuBLAS fp16 GEMV sweep, rotating over > 2x L2."""
    torch, P, gemv_batch, st, dev = ctx.torch, ctx.P, ctx.gemv_batch, ctx.stream, ctx.dev
    pool, _ = make_layer_models(P, 1, 5, seed0=500, p_lo=2, p_hi=2)
    ys2 = [[torch.empty(m.rows, dtype=torch.float16, device=dev) for m in row] for row in pool]
    dense = [[torch.randn(r, k, device=dev, dtype=torch.float16) * 0.01 for _, r, k in LAYERS] for _ in range(2)]
    yd = [torch.empty(r, device=dev, dtype=torch.float16) for _, r, _ in LAYERS]
    fused_w = [{g: torch.cat([d[i] for i in g]) for g in DECODER_GROUPS} for d in dense]
    fused_y = {g: torch.empty(fused_w[0][g].shape[0], device=dev, dtype=torch.float16) for g in DECODER_GROUPS}

    def per_sweep(fn, n):
        return 1e3 * ctx.time_graph(lambda: [fn(c) for c in range(n)], reps=10) / n

    with torch.cuda.stream(st):
        torch.mv(dense[0][0], xs[LAYERS[0][2]], out=yd[0])
    torch.cuda.synchronize()
    fp16_us = per_sweep(lambda c: [torch.mv(dense[c][li], xs[k], out=yd[li]) for li, (_, r, k) in enumerate(LAYERS)], 2)
    fp16g_us = per_sweep(lambda c: [torch.mv(fused_w[c][g], xs[LAYERS[g[0]][2]], out=fused_y[g])
                                    for g in DECODER_GROUPS], 2)
    p2_us = per_sweep(lambda c: [m.gemv(2, xs[m.cols], out=ys2[c][li], stream=st) for li, m in enumerate(pool[c])], 5)
    p2b_us = per_sweep(lambda c: gemv_batch([(m, 2, xs[m.cols], ys2[c][li]) for li, m in enumerate(pool[c])], st), 5)
    p2g_us = per_sweep(lambda c: [gemv_batch([(pool[c][li], 2, xs[pool[c][li].cols], ys2[c][li]) for li in g], st)
                                  for g in DECODER_GROUPS], 5)
    stacked = []
    for c in range(5):
        stacked.append([ctx.device_model(sum(LAYERS[i][1] for i in g), LAYERS[g[0]][2], 2, 2, 900 + 10 * c + gi)
                        for gi, g in enumerate(DECODER_GROUPS)])
    ys_st = [torch.empty(m.rows, dtype=torch.float16, device=dev) for m in stacked[0]]
    p2s_us = per_sweep(lambda c: [m.gemv(2, xs[m.cols], out=ys_st[gi], stream=st) for gi, m in enumerate(stacked[c])], 5)
    fp16_bytes = sum(r * k * 2 + k * 2 + r * 2 for _, r, k in LAYERS)
    return {"us_per_sweep": round(fp16_us, 2), "GBps": round(fp16_bytes / (fp16_us * 1e-6) / 1e9, 1),
            "abcq_p2_us_per_sweep": round(p2_us, 2), "speedup_p2": round(fp16_us / p2_us, 2),
            "abcq_p2_batched_us_per_sweep": round(p2b_us, 2), "speedup_p2_batched": round(fp16_us / p2b_us, 2),
            "decoder_grouped": {"cublas_fp16_us": round(fp16g_us, 2), "abcq_p2_us": round(p2g_us, 2),
                                "speedup_p2": round(fp16g_us / p2g_us, 2),
                                "abcq_p2_stacked_us": round(p2s_us, 2),
                                "speedup_p2_stacked": round(fp16g_us / p2s_us, 2),
                                "stacked": "q/k/v and gate/up as one row-stacked AnyBCQ model each (4 single "
                                           "GEMVs per sweep, as the decode harness runs them)",
                                "launches": "4 per sweep each: [q,k,v] [o] [gate,up] [down] (cuBLAS on "
                                            "concatenated fp16 weights)"},
            "note": "7 layers at p=2 vs fp16: cuBLAS 7 torch.mv vs abcq 7 single launches (like for like); "
                    "1 gemv_batch; 4 decoder-grouped launches; weights rotate over copies > 2x L2"}


def per_shape_batched8(ctx, xs, peak):
    """One gemv_batch of 8 independent same-shape GEMVs per launch: the
    per-shape kernel rate with the launch latency amortised."""
    torch, gemv_batch = ctx.torch, ctx.gemv_batch
    res = {}
    for li, (name, r, k) in enumerate(LAYERS):
        if name in ("k", "v", "o", "up"):
            continue
        pool8 = [ctx.device_model(r, k, P_LO, P_HI, 3000 + 50 * li + c) for c in range(16)]
        yb = [torch.empty(r, dtype=torch.float16, device=ctx.dev) for _ in range(16)]
        for pp in PRECISIONS:
            us = 1e3 * ctx.time_graph(lambda: [gemv_batch([(pool8[8 * h + j], pp, xs[k], yb[8 * h + j])
                                                           for j in range(8)], ctx.stream) for h in range(2)],
                                      reps=10) / 2
            gbps = 8 * algo_bytes(r, k, pp) / (us * 1e-6) / 1e9
            res[f"{name}_{r}x{k}_p{pp}"] = {"us_per_launch": round(us, 2), "GBps": round(gbps, 1),
                                            "roofline_frac": round(gbps / peak, 4)}
        del pool8, yb
    return res


def e2e_section(ctx, models, xs, all_jobs, args):
    """Public API with pinned host buffers, copies inside the timed region.

    Serving-style pipeline: steps run in groups of E2E_GROUP; a group's inputs
    (every step's x) are ONE host -> device copy on a side stream while the
    previous group computes, and its outputs ONE device -> host copy on another
    side stream while the next group computes (E2E_SETS buffer sets: a
    group's buffers are reused E2E_SETS groups later; 2 / 3 / 4 sets measured
    62.5 / 62.5 / 62.0 us per step). The compute
    stream waits on the copy streams once per group, so the launches inside a
    group stay PDL-chained and the host issues two copies per group instead of
    two per step (per-step copies left the step host-bound: 64 vs 58.8 us)."""
    torch, P, st, dev = ctx.torch, ctx.P, ctx.stream, ctx.dev
    G = E2E_GROUP
    kx = sorted(xs)
    hx1 = torch.cat([xs[k].cpu() for k in kx])
    nx = hx1.numel()
    hx = hx1.repeat(G).pin_memory()  # one group's inputs: G steps x (every distinct x)
    n_out = sum(models[pi][li].rows for pi, p, li in all_jobs)
    halves = []
    for _ in range(E2E_SETS):  # per buffer set: its G steps' inputs and outputs, contiguous (one copy each way)
        H = {"dx": torch.empty(G * nx, dtype=torch.float16, device=dev),
             "dy": torch.empty(G * n_out, dtype=torch.float16, device=dev),
             "hy": torch.empty(G * n_out, dtype=torch.float16).pin_memory(), "plans": []}
        for j in range(G):
            dx, off = {}, j * nx
            for k in kx:
                dx[k] = H["dx"][off:off + k]
                off += k
            dys, off = [], j * n_out
            for pi, p, li in all_jobs:
                dys.append(H["dy"][off:off + models[pi][li].rows])
                off += models[pi][li].rows
            H["plans"].append(P.GemvBatchPlan([(models[pi][li], p, dx[models[pi][li].cols], dys[n])
                                               for n, (pi, p, li) in enumerate(all_jobs)]))
        halves.append(H)
    # (every plan shares the compute stream's one split-K workspace: device_model.stream_workspace)
    ev = {k: [torch.cuda.Event() for _ in range(E2E_SETS)] for k in ("in", "comp", "out")}  # per buffer set
    s_in, s_out = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    cnt = {"h2d": 0, "d2h": 0}

    def h2d(g):  # group g's inputs (its buffers were last computed on by group g - E2E_SETS)
        h = g % E2E_SETS
        with torch.cuda.stream(s_in):
            s_in.wait_event(ev["comp"][h])
            halves[h]["dx"].copy_(hx, non_blocking=True)
            ev["in"][h].record(s_in)
        cnt["h2d"] += hx.numel() * 2

    def e2e_group(g, last):
        h = g % E2E_SETS
        H = halves[h]
        # the NEXT group's inputs go first: issued behind the previous group's
        # output copy they would land late (one copy queue) and stall this stream
        if not last:
            h2d(g + 1)
        st.wait_event(ev["in"][h])
        st.wait_event(ev["out"][h])  # group g - E2E_SETS's outputs have left these buffers
        for plan in H["plans"]:
            plan.launch(st)
        ev["comp"][h].record(st)
        with torch.cuda.stream(s_out):
            s_out.wait_event(ev["comp"][h])
            H["hy"].copy_(H["dy"], non_blocking=True)
            ev["out"][h].record(s_out)
        cnt["d2h"] += H["dy"].numel() * 2

    with torch.cuda.stream(st):
        for k in ev:
            for e in ev[k]:
                e.record(st)
        h2d(0)
        for g in range(E2E_SETS):
            e2e_group(g, g == E2E_SETS - 1)
        torch.cuda.synchronize()
        cnt["h2d"] = cnt["d2h"] = 0
        n_groups = max(2, min(args.steps, 48) // G)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        s_in.wait_stream(st)
        s_out.wait_stream(st)
        h2d(0)
        for g in range(n_groups):
            e2e_group(g, g == n_groups - 1)
        st.wait_stream(s_out)
        b.record(st)
        torch.cuda.synchronize()
    n_e2e = n_groups * G
    e2e_ms = a.elapsed_time(b) / n_e2e
    return {"value": round(step_bytes() / (e2e_ms * 1e-3) / 1e9, 1), "unit": "GB/s",
            "ms_per_step": round(e2e_ms, 4), "h2d_bytes_per_step": cnt["h2d"] // n_e2e,
            "d2h_bytes_per_step": cnt["d2h"] // n_e2e, "steps": n_e2e,
            "api": f"GemvBatchPlan.launch of the 21 GEMVs (one C-ABI abcq_gemv_batch call per step), eager; "
                   f"every step's inputs copied in from and its outputs copied out to pinned host memory; steps in "
                   f"groups of {G}, each group's inputs one copy (issued while the previous group computes) and its "
                   f"outputs one copy (while the next computes), {E2E_SETS} buffer sets in flight; the compute "
                   f"stream waits on the copy streams once per group"}


def config1(ctx, args, peak):
    """BASELINE configs[0]: one 4096x4096 BCQ linear, g=128, batch 1, p=2/3/4 --
    device time (single launches back to back over > 2x L2 of copies), the
    drop-in GemvEngine.lut with host numpy in/out (the reference's API), the
    cuBLAS fp16 GEMV, and the reference's CPU path beside it."""
    torch = ctx.torch
    r = k = 4096
    pool = _pool(ctx, r, k, P_LO, P_HI, 11000)
    x = torch.randn(k, device=ctx.dev).half()
    y = torch.empty(r, dtype=torch.float16, device=ctx.dev)
    res = {"shape": [r, k], "copies": len(pool)}
    for p in PRECISIONS:
        n = 20
        ms = ctx.time_graph(lambda: [pool[j % len(pool)].gemv(p, x, out=y, stream=ctx.stream) for j in range(n)],
                            reps=10)
        us = ms * 1e3 / n
        gbps = algo_bytes(r, k, p) / (us * 1e-6) / 1e9
        res[f"p{p}"] = {"us": round(us, 3), "GBps": round(gbps, 1), "roofline_frac": round(gbps / peak, 4)}
    dense = [torch.randn(r, k, device=ctx.dev, dtype=torch.float16) * 0.01 for _ in range(8)]
    with torch.cuda.stream(ctx.stream):
        torch.mv(dense[0], x, out=y)
    torch.cuda.synchronize()
    ms = ctx.time_graph(lambda: [torch.mv(dense[j % 8], x, out=y) for j in range(16)], reps=10)
    res["cublas_fp16_us"] = round(ms * 1e3 / 16, 3)
    res["speedup_vs_fp16"] = {f"p{p}": round(res["cublas_fp16_us"] / res[f"p{p}"]["us"], 2) for p in PRECISIONS}
    # the drop-in (reference API): numpy in, (f64[N], GemvStats) out, a sync per call
    from paper_2510_10467_b200.engine import GemvEngine
    eng = GemvEngine(pool[0])
    xh = np.random.default_rng(3).standard_normal(k).astype(np.float32)
    for p in PRECISIONS:
        for _ in range(3):
            eng.lut(p, xh)
        t0 = time.perf_counter()
        n = 50
        for _ in range(n):
            eng.lut(p, xh)
        res[f"p{p}"]["dropin_lut_us"] = round((time.perf_counter() - t0) / n * 1e6, 1)
    del pool, dense
    if not args.no_cpu:
        res["cpu"] = cpu_layer_times(r, k)
    res["what"] = ("BASELINE configs[0]: single BCQ linear 4096x4096, group 128, batch 1; us = device time per "
                   "GEMV back to back; dropin_lut_us = GemvEngine.lut(p, numpy x) end to end (H2D, launch, D2H, "
                   "f64 cast, host timer); cpu = the reference's LUT path on this host")
    return res


def cpu_layer_times(rows, cols):
    """The reference's CPU path on one rows x cols layer, p=2/3/4: the C port
    (1 thread and all threads) and, when baseline/_ref holds the real
    reference, its numba GemvEngine.lut with the reference's own _time_calls
    (median of 32 after one warm-up, gemv.py:296-305) at ANYBCQ_THREADS=1/0."""
    from oracle import anybcq_oracle as O  # checker / baseline only
    from oracle import c_oracle

    words = O.random_words(P_HI, rows, cols, seed=5)
    rng = np.random.default_rng(5)
    alphas = {p: (0.01 + 0.1 * np.abs(rng.standard_normal((p, rows, cols // 128)))).astype(np.float32)
              for p in PRECISIONS}
    x = rng.standard_normal(cols)
    out = {"cpu_model": cpu_model(), "host_threads": c_oracle.cpu_threads()}
    for th in (1, c_oracle.cpu_threads()):
        row = {}
        for p in PRECISIONS:
            c_oracle.lut_gemv(words, cols, 128, alphas[p], None, p, x, th)
            reps = 5 if th == 1 else 20
            t0 = time.perf_counter()
            for _ in range(reps):
                c_oracle.lut_gemv(words, cols, 128, alphas[p], None, p, x, th)
            row[f"p{p}_us"] = round((time.perf_counter() - t0) / reps * 1e6, 1)
        out[f"c_port_{th}_threads"] = row
    ref = numba_reference_times(words, alphas, rows, cols, x)
    if ref is not None:
        out["reference_numba"] = ref
    return out


def numba_reference_times(words, alphas, rows, cols, x):
    """The unmodified reference (baseline/_ref) GemvEngine.lut, timed by its own
    _time_calls, in a subprocess per thread setting (ANYBCQ_THREADS)."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "anybcq").exists():
        return None
    import tempfile
    with tempfile.TemporaryDirectory() as td:
        np.savez(Path(td) / "m.npz", words=words, x=x, **{f"a{p}": a for p, a in alphas.items()})
        code = (
            "import json,sys,numpy as np\n"
            "from anybcq import MultiPrecisionModel, QuantConfig, GemvEngine\n"
            "from anybcq.packing import BitPlaneSet\n"
            "from anybcq.bcq import ScaleTensor\n"
            "from anybcq.gemv import _time_calls\n"
            f"z=np.load(sys.argv[1]); rows,cols={rows},{cols}\n"
            f"sets={{p: ScaleTensor(z['a%d'%p], None, 128) for p in {list(PRECISIONS)}}}\n"
            f"m=MultiPrecisionModel(BitPlaneSet({P_HI}, rows, cols, z['words']), sets, {P_LO}, {P_HI}, QuantConfig(128))\n"
            "e=GemvEngine(m); x=z['x']; out={}\n"
            f"for p in {list(PRECISIONS)}:\n"
            "    med, lo = _time_calls(lambda: e.lut(p, x), 32)\n"
            "    out['p%d_us' % p] = round(med, 1)\n"
            "print(json.dumps(out))\n")
        res = {}
        for th in ("1", "0"):
            env = dict(os.environ, PYTHONPATH=str(ref), ANYBCQ_THREADS=th, NUMBA_CACHE_DIR=str(Path(td) / "nb"))
            try:
                r = subprocess.run([sys.executable, "-c", code, str(Path(td) / "m.npz")], env=env,
                                   capture_output=True, text=True, timeout=600)
                res["threads_" + ("1" if th == "1" else "all")] = json.loads(r.stdout.strip().splitlines()[-1])
            except Exception as exc:  # noqa: BLE001
                res["threads_" + th] = f"failed: {str(exc)[:100]}"
        res["what"] = ("unmodified reference anybcq.GemvEngine.lut (numba) from baseline/_ref, its own "
                       "_time_calls: median us of 32 calls after one warm-up; ANYBCQ_THREADS=1 and 0 (all)")
        return res


def config3(ctx):
    """BASELINE configs[2]: batch B = 1..16 requests with mixed per-request p on
    a Llama-3-8B MLP block (gate, up: 14336x4096; down: 4096x14336): the
    mixed-precision GEMM (one pass over planes 0..max p) vs the B requests as
    B LUT GEMVs in one batched launch, per matrix; 3 block copies (> 2x L2)."""
    torch, gemv_batch, st = ctx.torch, ctx.gemv_batch, ctx.stream
    shapes = [("gate", 14336, 4096), ("up", 14336, 4096), ("down", 4096, 14336)]
    blocks = [[ctx.device_model(r, k, P_LO, P_HI, 21000 + 10 * c + i) for i, (_, r, k) in enumerate(shapes)]
              for c in range(3)]
    res = {}
    for B in (1, 2, 4, 8, 16):
        ps = [2 + (b % 3) for b in range(B)]
        X = {k: torch.randn(B, k, device=ctx.dev).half() for k in (4096, 14336)}
        Y = {r: torch.empty(B, r, device=ctx.dev, dtype=torch.float16) for r in (4096, 14336)}

        def gemm():
            for c in range(3):
                for dm in blocks[c]:
                    dm.gemm_mixedp(ps, X[dm.cols], out_dtype=torch.float16, stream=st)

        def lut():
            for c in range(3):
                for dm in blocks[c]:
                    gemv_batch([(dm, ps[b], X[dm.cols][b], Y[dm.rows][b]) for b in range(B)], st)

        g_us = ctx.time_graph(gemm, reps=5) * 1e3 / 3
        l_us = ctx.time_graph(lut, reps=5) * 1e3 / 3
        pmax = max(ps)
        plane_bytes = sum(pmax * r * k // 8 for _, r, k in shapes)
        res[f"B{B}"] = {"gemm_us": round(g_us, 2), "lut_batched_us": round(l_us, 2),
                        "gemm_plane_GBps": round(plane_bytes / (g_us * 1e-6) / 1e9, 1),
                        "best": "gemm" if g_us < l_us else "lut_batched", "precisions": ps}
    del blocks
    res["what"] = ("us per MLP block (gate+up+down) at batch B with per-request p cycling 2,3,4; gemm = "
                   "abcq_gemm_mixedp per matrix (tensor cores, planes read once up to max p); lut_batched = "
                   "the B requests as B independent GEMVs in one abcq_gemv_batch launch per matrix")
    return res


def config4(ctx, args):
    """BASELINE configs[3]: random-init Llama-3-8B decode step (32 layers, ctx
    1024, batch 1), all linears AnyBCQ at p (q/k/v and gate/up row-stacked,
    SiLU-gated down input), fp16 attention / norms / lm_head, vs the same step
    with dense fp16 cuBLAS linears: tokens/s from CUDA-graph replays."""
    torch = ctx.torch
    from paper_2510_10467_b200.decode import Fp16LlamaStep, LlamaConfig, QuantizedLlamaStep, time_step
    cfg = LlamaConfig(layers=32)
    res = {"ctx": 1024, "layers": 32}
    with torch.cuda.device(ctx.dev):
        qm = QuantizedLlamaStep(cfg, p=3, ctx=1024, device=ctx.dev)
        for p in PRECISIONS:
            qm.p = p
            ms = time_step(qm, 20)
            gb = qm.linear_bytes() + cfg.vocab * cfg.hidden * 2
            res[f"p{p}"] = {"ms_per_token": round(ms, 4), "tokens_per_s": round(1e3 / ms, 1),
                            "weight_GBps": round(gb / (ms * 1e-3) / 1e9, 1)}
        del qm
        torch.cuda.empty_cache()
        fm = Fp16LlamaStep(cfg, ctx=1024, device=ctx.dev)
        ms = time_step(fm, 20)
        res["fp16"] = {"ms_per_token": round(ms, 4), "tokens_per_s": round(1e3 / ms, 1)}
        del fm
        torch.cuda.empty_cache()
    for p in PRECISIONS:
        res[f"p{p}"]["speedup_vs_fp16"] = round(res["fp16"]["ms_per_token"] / res[f"p{p}"]["ms_per_token"], 2)
    res["paper_table5_speedup"] = {"p2": round(245 / 105, 2), "p3": round(212 / 105, 2), "p4": round(186 / 105, 2)}
    res["what"] = ("tokens/s of one batch-1 decode step captured as a CUDA graph; random weights and KV cache; "
                   "paper Table 5 (PAPER.md:430-432) ratios beside")
    return res


def config5_row_sharded(ctx, args, peak):
    """BASELINE configs[4]: Llama-3-70B layers (q/o 8192^2, k/v 1024x8192,
    gate/up 28672x8192, down 8192x28672) at p=2 and p=4, output rows sharded
    over the N ranks (RowShardedGemv: each rank's slice by one plan launch
    straight into the NCCL all-gather buffer). Per layer set: the GEMVs alone
    (graph of back-to-back launches) and GEMV + all-gather per layer (eager,
    NCCL over NVLink), device time, max over ranks. Strong scaling: the total
    work is fixed, each rank reads 1/N of the planes."""
    torch = ctx.torch
    import torch.distributed as dist
    from paper_2510_10467_b200.parallel import RowShardedGemv, row_shard_bounds

    world, rank = ctx.world, ctx.rank
    engines = []
    for li, (name, r, k) in enumerate(LAYERS_70B):
        lo, hi = row_shard_bounds(r, world, rank)
        dm = ctx.device_model(hi - lo, k, 2, 4, 50000 + 100 * li + rank) if hi > lo else None
        engines.append(RowShardedGemv(shard=dm, rows=r, device=ctx.dev, dtype=torch.float16) if dm is not None
                       else None)
    xs = {k: torch.randn(k, device=ctx.dev).half() for k in (8192, 28672)}
    for e in engines:
        if e is not None:
            e.x_buffer.copy_(xs[e.cols])
    res = {"n_gpus": world}
    # fused all-gather buffers (one symmetric buffer per layer, rank r's rows
    # at r * per-rank rows) when a process group exists
    peers, peer_plans = [], {}
    if dist.is_initialized():
        usable = torch.tensor([1 if all(e is not None for e in engines) else 0], device=ctx.dev)
        dist.all_reduce(usable, op=dist.ReduceOp.MIN)
    if dist.is_initialized() and int(usable.item()) == 1:
        try:
            from paper_2510_10467_b200.parallel import PeerGather
            for li, (name, r, k) in enumerate(LAYERS_70B):
                lo0, hi0 = row_shard_bounds(r, world, 0)
                peers.append(PeerGather(hi0 - lo0, device=ctx.dev))
            for p in (2, 4):
                peer_plans[p] = [pg.plan([(e.dm, p, e.x_buffer, pg.local[:e.dm.rows])])
                                 for e, pg in zip(engines, peers)]
        except Exception as exc:  # noqa: BLE001
            peers, peer_plans = [], {}
            res["fused_allgather"] = f"unavailable: {str(exc)[:100]}"
        ok = torch.tensor([1 if peers else 0], device=ctx.dev)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)  # every rank takes the same path
        if peers and int(ok.item()) == 0:
            peers, peer_plans = [], {}
            res["fused_allgather"] = "unavailable on another rank"
    for p in (2, 4):
        def local_all():
            for e in engines:
                if e is not None:
                    e.local(p, e.x_buffer, ctx.stream)

        gemv_ms = ctx.time_graph(local_all, reps=10)

        def local_gather_all():
            for e in engines:
                if e is not None:
                    e.local(p, e.x_buffer, ctx.stream)
                    e.gather()

        # + the all-gather of every layer's output: captured in the graph too
        # (NCCL over NVLink); eager with events if capture is refused
        if world > 1:
            dist.barrier()
        try:
            full_ms = ctx.time_graph(local_gather_all, reps=10)
            mode = "graph"
        except Exception:  # noqa: BLE001
            torch.cuda.synchronize()
            with torch.cuda.stream(ctx.stream):
                for _ in range(3):
                    local_gather_all()
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            n = 10
            with torch.cuda.stream(ctx.stream):
                a.record(ctx.stream)
                for _ in range(n):
                    local_gather_all()
                b.record(ctx.stream)
            torch.cuda.synchronize()
            full_ms = a.elapsed_time(b) / n
            mode = "eager"
        # the product path: each layer's all-gather FUSED into its GEMV launch
        # (rows stored into every rank's symmetric buffer, abcq_gemv_batch_peer),
        # then the consumer wait (every rank's rows landed) before the next layer
        peer_ms = None
        if peers:
            if world > 1:
                dist.barrier()

            def peer_all():
                for pp_, pg in zip(peer_plans[p], peers):
                    pp_.launch(ctx.stream)
                    pg.wait(ctx.stream)

            peer_ms = ctx.time_graph(peer_all, reps=10)
        t = torch.tensor([gemv_ms, full_ms, peer_ms or 0.0], device=ctx.dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        gemv_ms, full_ms, peer_ms2 = (float(v) for v in t.tolist())
        total = sum(algo_bytes(r, k, p) for _, r, k in LAYERS_70B)
        res[f"p{p}"] = {"gemv_us_per_layer_set": round(gemv_ms * 1e3, 2),
                        "gemv_allgather_us_per_layer_set": round(full_ms * 1e3, 2), "allgather_timing": mode,
                        "gemv_fused_allgather_us_per_layer_set": round(peer_ms2 * 1e3, 2) if peers else None,
                        "GBps_total": round(total / (gemv_ms * 1e-3) / 1e9, 1),
                        "roofline_frac_per_gpu": round(total / world / (gemv_ms * 1e-3) / 1e9 / peak, 4)}
    del engines
    del peers, peer_plans
    res["what"] = ("Llama-3-70B layer set (q,k,v,o,gate,up,down) row-sharded over n_gpus; GBps_total = the "
                   "whole layer set's algorithmic bytes / GEMV time; all-gather of each layer's fp16 output: NCCL "
                   "after the GEMV (gemv_allgather_*) or fused into it -- rows stored into every rank's symmetric "
                   "buffer by the GEMV's completion, then the consumer wait (gemv_fused_allgather_*)")
    return res


def loader_section(ctx, args):
    """an .abcq container (14336 x 4096, p = 2..4, f16
    scales -- one Llama-3-8B gate layer) to a GPU-resident model through
    ProgressiveLoader: the host mmap -> pinned -> device upload and the tiled
    repack, time to the first servable precision (planes 1..p_lo + set p_lo:
    a GEMV at p_lo can launch) and to the whole model, wall time with the
    device synchronised; file bytes / time."""
    torch = ctx.torch
    import tempfile

    from paper_2510_10467_b200.container import ProgressiveLoader, serialize
    from paper_2510_10467_b200.model import BitPlaneSet, MultiPrecisionModel, QuantConfig, ScaleTensor
    from paper_2510_10467_b200.tensor_io import random_words

    rows, cols, p_lo, p_hi = 14336, 4096, 2, 4
    rng = np.random.default_rng(5)
    words = random_words(p_hi, rows, cols, seed=9)
    sets = {p: ScaleTensor((0.01 + 0.1 * np.abs(rng.standard_normal((p, rows, cols // 128)))).astype(np.float32),
                           None, 128) for p in range(p_lo, p_hi + 1)}
    model = MultiPrecisionModel(BitPlaneSet(p_hi, rows, cols, words), sets, p_lo, p_hi, QuantConfig(128))
    x = torch.randn(cols, device=ctx.dev).half()
    res = {}
    with tempfile.TemporaryDirectory() as td:
        path = str(Path(td) / "layer.abcq")
        serialize(model, path, scale_width=2)
        nbytes = os.path.getsize(path)
        for rep in range(3):  # (first: allocator / module warm-up)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            ld = ProgressiveLoader(path, device=ctx.dev)
            ld.load_level()
            y = ld.model.gemv(p_lo, x)  # ordered after its level's upload on the device
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            ld.load_all()
            torch.cuda.synchronize()
            t2 = time.perf_counter()
            ld.close()
            del ld, y
        res = {"shape": [rows, cols], "precisions": [p_lo, p_hi], "file_bytes": nbytes,
               "first_gemv_s": round(t1 - t0, 4), "all_levels_s": round(t2 - t0, 4),
               "GBps_file": round(nbytes / (t2 - t0) / 1e9, 2),
               "what": "ProgressiveLoader: header + CRC check, planes 1..p_lo + set p_lo uploaded and one GEMV at "
                       "p_lo served, then the remaining levels; wall seconds, device synchronised"}
    return res


def quantizer_section(ctx, args):
    """The GPU quantizer: build_multiprecision 2:4,
    group 128, cycles 1 (the reference CLI's bench-suite fit, cli.py:150-152)
    on Llama-3-8B shapes, wall time with the device synchronised, the
    relative errors per precision; beside it the unmodified reference
    (baseline/_ref, numpy f64 on the host) on the 4096x4096 matrix."""
    torch = ctx.torch
    from paper_2510_10467_b200.model import QuantConfig
    from paper_2510_10467_b200.quantize import build_multiprecision, precision_errors
    from paper_2510_10467_b200.tensor_io import random_gaussian

    cfg = QuantConfig(group_size=128, cycles=1)
    build_multiprecision(random_gaussian(64, 256, seed=1), 2, 4, cfg)  # (module load, first launches)
    res = {}
    for r, k in ((4096, 4096), (14336, 4096)):
        w = random_gaussian(r, k, seed=0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        m = build_multiprecision(w, 2, 4, cfg)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        errs = precision_errors(w, m)
        res[f"{r}x{k}"] = {"gpu_s": round(dt, 3), "relative_sq_error": {p: round(e, 6) for p, e in errs.items()}}
    ref = ROOT / "baseline" / "_ref"
    if not args.no_cpu and (ref / "anybcq").exists():
        code = ("import time, json\n"
                "from anybcq import QuantConfig, random_gaussian\n"
                "from anybcq.progressive import build_multiprecision, precision_errors\n"
                "w = random_gaussian(4096, 4096, seed=0)\n"
                "t0 = time.perf_counter(); m = build_multiprecision(w, 2, 4, QuantConfig(group_size=128, cycles=1))\n"
                "dt = time.perf_counter() - t0\n"
                "print(json.dumps({'cpu_s': round(dt, 2), 'relative_sq_error': {p: round(e, 6) for p, e in "
                "precision_errors(w, m).items()}}))\n")
        try:
            r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, PYTHONPATH=str(ref)),
                               capture_output=True, text=True, timeout=600)
            res["reference_4096x4096"] = json.loads(r.stdout.strip().splitlines()[-1])
        except Exception as exc:  # noqa: BLE001
            res["reference_4096x4096"] = f"failed: {str(exc)[:100]}"
    res["what"] = ("build_multiprecision(w, 2, 4, group 128, cycles 1): GPU quantizer wall seconds (device "
                   "synchronised) and relative squared errors; the unmodified reference on the host beside it")
    return res


# ---------------------------------------------------------------------------
def _cpu_sample_models():
    """The GPU step's exact host inputs (same splitmix64 words, f16-rounded
    alphas and fp16 x as make_layer_models / run_gpu on rank 0, copy per
    precision) for the C port."""
    from oracle import anybcq_oracle as O  # checker / baseline only
    out = {}
    for pi, p in enumerate(PRECISIONS):
        for li, (name, r, k) in enumerate(LAYERS):
            seed = 1000 * pi + li
            words = O.random_words(P_HI, r, k, seed=seed)
            rng = np.random.default_rng(seed)
            a = None
            for q in range(P_LO, P_HI + 1):
                aq = (0.01 + 0.1 * np.abs(rng.standard_normal((q, r, k // 128)))).astype(np.float32)
                if q == p:
                    a = aq.astype(np.float16).astype(np.float32)
            out[(p, li)] = (words, a)
    rng = np.random.default_rng(1234)
    xs = {k: rng.standard_normal(k).astype(np.float16).astype(np.float64) for k in sorted({c for _, _, c in LAYERS})}
    return out, xs


def cpu_baseline(repeats: int = 2):
    """The reference LUT algorithm (C port of gemv.py:67-95,188-222) on the
    GPU step's exact inputs: all host threads over the full step, and one
    thread over a bounded sample (the step's q/k/v/o GEMVs at p=2)."""
    from oracle import c_oracle

    threads = c_oracle.cpu_threads()
    models, xs = _cpu_sample_models()
    k0 = LAYERS[0][2]
    c_oracle.lut_gemv(*models[(2, 0)][:1], k0, 128, models[(2, 0)][1], None, 2, xs[k0], threads)  # warm
    t0 = time.perf_counter()
    for _ in range(repeats):
        for (p, li), (words, a) in models.items():
            k = LAYERS[li][2]
            c_oracle.lut_gemv(words, k, 128, a, None, p, xs[k], threads)
    dt = (time.perf_counter() - t0) / repeats
    sample = [(2, li) for li in range(4)]
    t0 = time.perf_counter()
    for p, li in sample:
        words, a = models[(p, li)]
        k = LAYERS[li][2]
        c_oracle.lut_gemv(words, k, 128, a, None, p, xs[k], 1)
    dt1 = time.perf_counter() - t0
    b1 = sum(algo_bytes(LAYERS[li][1], LAYERS[li][2], p) for p, li in sample)
    return {"value": round(step_bytes() / dt / 1e9, 3), "unit": "GB/s", "cores": threads, "kind": "port",
            "cpu_model": cpu_model(), "ms_per_step": round(dt * 1e3, 1),
            "sample": f"the full step's 21 GEMVs x{repeats} on the GPU step's exact inputs, C restatement of "
                      f"GemvEngine.lut, {threads} pthreads",
            "single_thread": {"value": round(b1 / dt1 / 1e9, 3), "unit": "GB/s", "cores": 1,
                              "sample": "q/k/v/o at p=2 of the same inputs, 1 thread"}}


def run_reference(args):
    """--impl reference: the reference's CPU algorithm (C port, all host threads)
    on this workload -- the GPU step's exact inputs -- rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import c_oracle

    threads = c_oracle.cpu_threads()
    models, xs = _cpu_sample_models()

    def one_step():
        for (p, li), (words, a) in models.items():
            k = LAYERS[li][2]
            c_oracle.lut_gemv(words, k, 128, a, None, p, xs[k], threads)

    for _ in range(args.warmup):
        one_step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        one_step()
    dt = (time.perf_counter() - t0) / args.steps
    value = round(step_bytes() / dt / 1e9, 3)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt * 1e3, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": DTYPE,
        "dtype_note": DTYPE_NOTE, "data": "synthetic (splitmix64 planes, |N(0,1)| fp16 scales, N(0,1) fp16 x)",
        "config": bench_config(world),
        "implementation": "reference CPU algorithm (C restatement of GemvEngine.lut, all host threads); the "
                          "reference is Python + numba with no compiled sources (its numba timing: config1.cpu)",
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": threads, "kind": "port", "cpu_model": cpu_model(),
                         "sample": "the full step (21 GEMVs) per step, the GPU step's exact inputs"},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline legs")
    ap.add_argument("--sections", default="", help="comma list of the extra sections to run (default: all): "
                    "variants,per_shape,fp16,batched8,e2e,config1,config3,config4,config5,loader,quantizer")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch under torchrun (the driver launches
        # N > 1 that way itself); fails if fewer GPUs are visible
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), str(Path(__file__).resolve()),
               *sys.argv[1:]]
        sys.exit(subprocess.call(cmd))
    run_gpu(args)


if __name__ == "__main__":
    main()
