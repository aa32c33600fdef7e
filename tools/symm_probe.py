import os, socket, sys, torch
sys.path.insert(0, "/root/repo")
import torch.distributed as dist
import bench
import paper_2510_10467_b200 as P
from paper_2510_10467_b200.parallel import PeerGather
s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
models, _ = bench.make_layer_models(P, 1, 3)
xs = {k: torch.randn(k, device="cuda").half() for k in {c for _, _, c in bench.LAYERS}}
all_jobs = [(pi, p, li) for pi, p in enumerate(bench.PRECISIONS) for li in range(len(bench.LAYERS))]
R = sum(models[pi][li].rows for pi, p, li in all_jobs)
g = PeerGather(R)
reg = torch.empty(R, dtype=torch.float16, device="cuda")
def views(buf):
    off, v = 0, []
    for pi, p, li in all_jobs:
        v.append(buf[off:off + models[pi][li].rows]); off += models[pi][li].rows
    return v
jobs_reg = [(models[pi][li], p, xs[models[pi][li].cols], v) for (pi, p, li), v in zip(all_jobs, views(reg))]
jobs_sym = [(models[pi][li], p, xs[models[pi][li].cols], v) for (pi, p, li), v in zip(all_jobs, views(g.local))]
plan_reg = P.GemvBatchPlan(jobs_reg)
plan_sym = P.GemvBatchPlan(jobs_sym)
plan_peer = g.plan(jobs_sym)
st = torch.cuda.Stream()
def t(fn, n=100):
    with torch.cuda.stream(st):
        for _ in range(5): fn()
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=st):
            for _ in range(n): fn()
        gr.replay(); torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st); gr.replay(); b.record(st)
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / n
from paper_2510_10467_b200 import _lib
for _ in range(2):
    print("regular buffer, plain launch %.2f us" % t(lambda: plan_reg.launch(st)))
    print("symm buffer, plain launch    %.2f us" % t(lambda: plan_sym.launch(st)))
    print("symm buffer, peer launch     %.2f us" % t(lambda: plan_peer.launch(st)))
    for m in (37, 38):
        _lib.lib().abcq_debug_set_mode(m)
        print("symm buffer, peer launch, mode %d %.2f us" % (m, t(lambda: plan_peer.launch(st))))
        _lib.lib().abcq_debug_set_mode(0)
dist.destroy_process_group()
