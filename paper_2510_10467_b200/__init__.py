"""anybcq-b200: B200-native (sm_100a) AnyBCQ bit-plane matmul.

Drop-in for the reference package's GEMV path (`anybcq.gemv`): the same
entry points backed by hand-written CUDA in libanybcq_b200.so (C ABI:
include/anybcq_b200.h). See DESIGN.md.
"""

from .errors import (AnyBcqError, BadMagicError, BadVersionError, ChecksumError, FileFormatError,
                     NonFiniteError, TruncatedError, UnsupportedDtypeError, UsageError)
from .model import (BitPlaneSet, MultiPrecisionModel, QuantConfig, ScaleTensor, group_bounds,
                    group_count, pack_signs, precision_view, unpack_signs, words_per_row)

__version__ = "0.1.0"


def __getattr__(name):
    # torch-dependent modules load lazily so the host types import without CUDA
    if name in ("GemvEngine", "GemvStats", "LookupTable", "BenchRow", "bench", "gemv_lut",
                "gemv_naive", "dequant_oracle", "dense_gemv_reference", "render_bench_text",
                "render_bench_csv"):
        from . import engine
        return getattr(engine, name)
    if name in ("DeviceModel", "GemvBatchPlan", "gemv_batch", "set_reserved_sms"):
        from . import device_model
        return getattr(device_model, name)
    if name in ("QuantizedMatrix", "greedy_init", "ls_update_scales", "bs_recalibrate_codes", "alternate_fit",
                "expand_step", "build_multiprecision", "precision_errors", "relative_reconstruction_error"):
        from . import quantize
        return getattr(quantize, name)
    raise AttributeError(name)
