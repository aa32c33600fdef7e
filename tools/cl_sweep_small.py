import sys, json, math
sys.path.insert(0, "/root/repo/tools"); sys.argv = ["x", "--shapes", "4096x4096"]
exec(open("/root/repo/tools/cl_probe.py").read().split("out = {\"shapes\": {}}")[0])
res = {}
for (rows, cols) in [(4096, 4096), (1024, 4096), (6144, 4096)]:
    per_copy = 4 * rows * cols // 8
    ncopy = max(3, min(48, math.ceil(300e6 / per_copy)))
    models = [make(rows, cols, 100 + c) for c in range(ncopy)]
    x = torch.randn(cols, device="cuda").half(); y = torch.empty(rows, device="cuda", dtype=torch.float16)
    for p in (2, 3, 4):
        row = {}
        for name, modes in [("auto", (5000, 6000)), ("s1w16", (5162, 6016)), ("s1w8", (5162, 6008)), ("s2w8", (5262, 6008))]:
            L.abcq_debug_set_mode(27)
            for m in modes: L.abcq_debug_set_mode(m)
            try:
                row[name] = round(min(time_graph(models, p, x, y, 20) for _ in range(3)), 3)
            except Exception as e:
                row[name] = str(e)[:40]
        L.abcq_debug_set_mode(5000); L.abcq_debug_set_mode(6000); L.abcq_debug_set_mode(0)
        res[f"{rows}x{cols}_p{p}"] = row
        print(rows, cols, p, row, flush=True)
