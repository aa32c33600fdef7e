import sys, time, torch
sys.path.insert(0, "/root/repo")
import bench
import paper_2510_10467_b200 as P
torch.cuda.set_device(0)
models, _ = bench.make_layer_models(P, 1, 3)
xs = {k: torch.randn(k, device="cuda").half() for k in {c for _, _, c in bench.LAYERS}}
jobs = []
ys = []
for pi, p in enumerate(bench.PRECISIONS):
    for li in range(len(bench.LAYERS)):
        m = models[pi][li]
        y = torch.empty(m.rows, dtype=torch.float16, device="cuda"); ys.append(y)
        jobs.append((m, p, xs[m.cols], y))
plan = P.GemvBatchPlan(jobs)
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    for _ in range(20): plan.launch(st)
torch.cuda.synchronize()
for n in (50, 200):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        a.record(st)
        t0 = time.perf_counter()
        for _ in range(n): plan.launch(st)
        t1 = time.perf_counter()
        b.record(st)
    torch.cuda.synchronize()
    print(f"n={n}: host {1e6*(t1-t0)/n:.1f} us/launch, device {1e3*a.elapsed_time(b)/n:.1f} us/step")

# e2e-style groups: which part costs? (G launches per group, waits / copies toggled)
G = 4
hx = torch.randn(G * 9216, dtype=torch.float16).pin_memory()
dx = torch.empty_like(hx, device="cuda")
n_out = sum(j[0].rows for j in jobs)
dy = torch.empty(G * n_out, dtype=torch.float16, device="cuda")
hy = torch.empty(G * n_out, dtype=torch.float16).pin_memory()
s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
e_in, e_comp, e_out = torch.cuda.Event(), torch.cuda.Event(), torch.cuda.Event()


def run(variant, groups=12):
    with torch.cuda.stream(st):
        for e in (e_in, e_comp, e_out):
            e.record(st)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        s_in.wait_stream(st)
        s_out.wait_stream(st)
        for g in range(groups):
            if "h2d" in variant:
                with torch.cuda.stream(s_in):
                    dx.copy_(hx, non_blocking=True)
                    e_in.record(s_in)
            if "wait" in variant:
                st.wait_event(e_in)
                st.wait_event(e_out)
            if "inwait" in variant:
                st.wait_event(e_in)
            for _ in range(G):
                plan.launch(st)
            e_comp.record(st)
            if "d2h" in variant:
                with torch.cuda.stream(s_out):
                    s_out.wait_event(e_comp)
                    if "small" in variant:
                        hy[:n_out].copy_(dy[:n_out], non_blocking=True)
                    else:
                        hy.copy_(dy, non_blocking=True)
                    e_out.record(s_out)
        st.wait_stream(s_out)
        b.record(st)
    torch.cuda.synchronize()
    return 1e3 * a.elapsed_time(b) / (groups * G)


for v in ("", "d2h", "d2h+small", "d2h+wait", "d2h+small+wait", "h2d+d2h+inwait", ""):
    run(v)
    print(f"variant [{v}]: {run(v):.1f} us/step")

# the output copy's own duration: alone, and under the GEMV stream
def d2h_time(under_compute):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if under_compute:
        with torch.cuda.stream(st):
            for _ in range(30):
                plan.launch(st)
    with torch.cuda.stream(s_out):
        a.record(s_out)
        hy.copy_(dy, non_blocking=True)
        b.record(s_out)
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3


for uc in (False, True, False, True):
    t = d2h_time(uc)
    print(f"D2H of {hy.numel() * 2 / 1e6:.2f} MB {'under the GEMV' if uc else 'alone'}: {t:.1f} us = {hy.numel() * 2 / t / 1e3:.1f} GB/s")
