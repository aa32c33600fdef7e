"""One Llama-3-8B decode step (eager, 4 layers) for an ncu launch list:
    ncu --metrics gpu__time_duration.sum --csv --log-file l.csv python tools/decode_launches.py
"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2510_10467_b200.decode import LlamaConfig, QuantizedLlamaStep  # noqa: E402

torch.cuda.set_device(0)
m = QuantizedLlamaStep(LlamaConfig(layers=4), p=3, ctx=1024)
for _ in range(3):
    m.step()
torch.cuda.synchronize()
