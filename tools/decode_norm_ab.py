import json, statistics, sys
sys.path.insert(0, "/root/repo")
import torch
import paper_2510_10467_b200.decode as D
torch.cuda.set_device(0)
qm = D.QuantizedLlamaStep(D.LlamaConfig(), p=3, ctx=1024)
res = {}
for r in range(3):
    for name, fn, fo in (("separate", False, False), ("fuse_norm", True, False), ("fuse_norm_out", False, True)):
        qm.fuse_norm, qm.fuse_norm_out = fn, fo
        for p in (2, 3, 4):
            qm.p = p
            res.setdefault(name, {}).setdefault(p, []).append(D.time_step(qm, 30))
print(json.dumps({k: {f"p{p}": round(statistics.median(v), 4) for p, v in d.items()} for k, d in res.items()}))
