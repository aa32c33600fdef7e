"""Host and device cost of GemvBatchPlan.launch when a loop rotates over
several plans (different x / y buffers, same models) -- the e2e pipeline's
pattern -- against one plan launched repeatedly.
    python tools/plan_rotation_probe.py"""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2510_10467_b200 as P  # noqa: E402

torch.cuda.set_device(0)
models, _ = bench.make_layer_models(P, 1, len(bench.PRECISIONS))
st = torch.cuda.Stream()


def make_plan():
    xs = {k: torch.randn(k, device="cuda").half() for k in {c for _, _, c in bench.LAYERS}}
    return P.GemvBatchPlan([(models[pi][li], p, xs[models[pi][li].cols],
                             torch.empty(models[pi][li].rows, dtype=torch.float16, device="cuda"))
                            for pi, p in enumerate(bench.PRECISIONS) for li in range(len(bench.LAYERS))])


plans = [make_plan() for _ in range(8)]
for nplans in (1, 2, 8):
    with torch.cuda.stream(st):
        for k in range(16):
            plans[k % nplans].launch(st)
        torch.cuda.synchronize()
        for n in (40, 200):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            t0 = time.perf_counter()
            for k in range(n):
                plans[k % nplans].launch(st)
            t1 = time.perf_counter()
            b.record(st)
            torch.cuda.synchronize()
            print(f"{nplans} plan(s), n={n}: host {1e6 * (t1 - t0) / n:.1f} us/launch, "
                  f"device {1e3 * a.elapsed_time(b) / n:.1f} us/step")
