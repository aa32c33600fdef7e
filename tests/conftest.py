import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def load_case(name):
    """Golden case written by tests/golden/make_golden.py from the real reference."""
    with np.load(GOLDEN / f"{name}.npz") as z:
        return {k: z[k] for k in z.files}


GOLDEN_CASES = [
    "g32_32x128", "asym_g40_16x80", "g128_64x256", "single_col_1x4",
    "asym_g25_16x100", "g128_ragged_37x200", "asym_g128_128x1024", "g128_512x4096",
]


@pytest.fixture(scope="session")
def cuda_available():
    import torch
    return torch.cuda.is_available()
