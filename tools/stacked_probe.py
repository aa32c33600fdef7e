"""Hypothesis check for multi-job rounds: the bench step's 21 GEMVs as issued
(q,k,v,o,gate,up,down x p=2,3,4: 21 jobs) vs the same bytes with the six
x-sharing layers of each precision row-stacked into one model (6 jobs):
same x, same planes per row -- only the (job, slice) piece count differs.
    python tools/stacked_probe.py"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2510_10467_b200 as P  # noqa: E402
from paper_2510_10467_b200.device_model import GemvBatchPlan  # noqa: E402

torch.cuda.set_device(0)
dev = torch.device("cuda", 0)
g = torch.Generator(device="cuda").manual_seed(0)


def model(rows, cols):
    dm = P.DeviceModel(rows, cols, 128, 2, 4, False, scale_dtype="f16", device=dev)
    dm.load_planes(torch.randint(-2**31, 2**31 - 1, (4, rows, cols // 32), dtype=torch.int32, device="cuda", generator=g))
    for p in (2, 3, 4):
        dm.load_scale_set(p, 0.01 + 0.01 * torch.rand((p, rows, cols // 128), device="cuda", generator=g))
    return dm


x = {k: torch.randn(k, device="cuda").half() for k in (4096, 14336)}
sets = []
for copy in range(3):  # > L2 rotation as in the bench
    sep = [[model(r, c) for _, r, c in bench.LAYERS] for _ in bench.PRECISIONS]
    stk = [[model(4096 + 1024 + 1024 + 4096 + 14336 + 14336, 4096), model(4096, 14336)] for _ in bench.PRECISIONS]
    sets.append((sep, stk))


def plans(kind):
    out = []
    for sep, stk in sets:
        jobs = []
        for pi, p in enumerate(bench.PRECISIONS):
            ms = sep[pi] if kind == "separate" else stk[pi]
            for m in ms:
                jobs.append((m, p, x[m.cols], torch.empty(m.rows, device="cuda", dtype=torch.float16)))
        out.append(GemvBatchPlan(jobs))
    return out


st = torch.cuda.Stream()
for kind in ("separate", "stacked", "separate", "stacked"):
    pl = plans(kind)
    with torch.cuda.stream(st):
        for q in pl:
            q.launch(st)
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=st):
            for i in range(30):
                pl[i % 3].launch(st)
        gr.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        gr.replay()
        b.record(st)
    torch.cuda.synchronize()
    us = a.elapsed_time(b) * 1e3 / 30
    print(f"{kind}: {len(pl[0].jobs)} jobs, {us:.2f} us/step, {bench.step_bytes() / us / 1e3:.0f} GB/s", flush=True)
