"""Host-side logic on CPU: model types mirror the reference's, validation
comes first, and the product fails loudly without a GPU (no CPU fallback)."""

import numpy as np
import pytest
import torch

import paper_2510_10467_b200 as P
from conftest import load_case


def test_pack_signs_matches_reference_golden():
    with np.load("tests/golden/packing.npz") as z:
        assert np.array_equal(P.pack_signs(z["codes"]), z["words"])
        assert np.array_equal(P.unpack_signs(z["words"], 100), z["codes"])


def test_bitplaneset_prefix_is_view():
    rng = np.random.default_rng(9)
    codes = np.where(rng.random((4, 5, 45)) < 0.5, -1, 1).astype(np.int8)
    bp = P.BitPlaneSet.from_codes(codes)
    two = bp.prefix(2)
    assert two.words.base is not None and np.array_equal(two.codes(), codes[:2])
    with pytest.raises(P.UsageError):
        bp.prefix(5)


def test_model_validation_mirrors_reference():
    c = load_case("g32_32x128")
    bp = P.BitPlaneSet(4, 32, 128, c["words"])
    sets = {p: P.ScaleTensor(c[f"alpha_{p}"], None, 32) for p in (2, 3, 4)}
    m = P.MultiPrecisionModel(bp, sets, 2, 4, P.QuantConfig(32))
    assert list(m.precisions) == [2, 3, 4] and m.shape == (32, 128)
    with pytest.raises(P.UsageError):
        P.MultiPrecisionModel(bp, {2: sets[2]}, 2, 4, P.QuantConfig(32))
    with pytest.raises(P.NonFiniteError):
        P.ScaleTensor(np.full((1, 1, 1), np.nan, np.float32), None, 8)
    with pytest.raises(P.UsageError):
        P.precision_view(m, 1)


@pytest.mark.skipif(torch.cuda.is_available(), reason="CPU-only behaviour")
def test_engine_fails_loudly_without_gpu():
    c = load_case("g32_32x128")
    bp = P.BitPlaneSet(4, 32, 128, c["words"])
    m = P.MultiPrecisionModel(bp, {p: P.ScaleTensor(c[f"alpha_{p}"], None, 32) for p in (2, 3, 4)},
                              2, 4, P.QuantConfig(32))
    with pytest.raises(P.UsageError):
        P.GemvEngine(m, chunk_width=5)          # argument checks first (gemv.py:107-108)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        P.GemvEngine(m)


def test_product_package_never_imports_oracle():
    import pathlib
    pkg = pathlib.Path(P.__file__).parent
    for f in pkg.rglob("*.py"):
        text = f.read_text()
        assert "import oracle" not in text and "from oracle" not in text, f


# --- torch.ops.anybcq_b200 (SURVEY §8b device operator) -------------------------

class _Shape:  # stands in for a DeviceModel: the fake kernels read only rows/cols
    rows, cols = 48, 256


def test_torch_ops_registered_and_trace_shapes():
    from torch._subclasses.fake_tensor import FakeTensorMode
    from paper_2510_10467_b200 import ops
    for name in ("gemv", "gemm_mixedp", "dequantize"):
        assert hasattr(torch.ops.anybcq_b200, name)
    h = ops.register(_Shape())
    try:
        with FakeTensorMode():
            x = torch.empty(256, dtype=torch.float16)
            assert torch.ops.anybcq_b200.gemv(h, x, 3).shape == (48,)
            assert torch.ops.anybcq_b200.gemv(h, x, 3).dtype == torch.float16
            X = torch.empty(3, 256)
            Y = torch.ops.anybcq_b200.gemm_mixedp(h, X, [2, 4, 3])
            assert Y.shape == (3, 48) and Y.dtype == torch.float32
            assert torch.ops.anybcq_b200.dequantize(h, 2, X).shape == (48, 256)
            with pytest.raises(P.UsageError):
                torch.ops.anybcq_b200.gemv(h, torch.empty(255), 3)
            with pytest.raises(P.UsageError):
                torch.ops.anybcq_b200.gemm_mixedp(h, X, [2, 4])
    finally:
        ops.unregister(h)
    with pytest.raises(P.UsageError):
        ops.model(h)
    with pytest.raises(P.UsageError):
        ops.register(object())


def test_synthetic_words_match_the_oracle_generator():
    from oracle import anybcq_oracle as O
    from paper_2510_10467_b200.tensor_io import random_words
    for planes, rows, cols, seed in ((4, 16, 4096, 3), (2, 5, 100, 7), (1, 3, 31, 0)):
        assert np.array_equal(random_words(planes, rows, cols, seed), O.random_words(planes, rows, cols, seed))
