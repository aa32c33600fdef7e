import sys, time, cProfile, pstats, io
sys.path.insert(0, "/root/repo")
import torch
from paper_2510_10467_b200.model import QuantConfig
from paper_2510_10467_b200.quantize import build_multiprecision
from paper_2510_10467_b200.tensor_io import random_gaussian
cfg = QuantConfig(group_size=128, cycles=1)
build_multiprecision(random_gaussian(64, 256, seed=1), 2, 4, cfg)
for r, k in ((4096, 4096), (14336, 4096), (4096, 4096)):
    w = random_gaussian(r, k, seed=0)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    m = build_multiprecision(w, 2, 4, cfg)
    torch.cuda.synchronize(); print(r, k, round(time.perf_counter() - t0, 3))
w = random_gaussian(4096, 4096, seed=0)
pr = cProfile.Profile(); pr.enable()
m = build_multiprecision(w, 2, 4, cfg); torch.cuda.synchronize()
pr.disable()
s = io.StringIO(); pstats.Stats(pr, stream=s).sort_stats("cumulative").print_stats(25); print(s.getvalue()[:6000])
