"""pytest plugin: route the reference package's GEMV engine to this repo's
drop-in before the reference's own test modules import it.

Loaded with `-p ref_dropin_plugin` by tests/test_reference_suite_gpu.py, which
runs the reference's unchanged test files (installed under baseline/_ref by
tools/install_reference.sh) on the B200 engine. This is the reference-side
binding a maintainer would add: the engine class, bench() and the fitting API
(the GPU quantizer) are swapped, and the drop-in's
argument errors surface as the reference's own anybcq.UsageError (the
reference's CLI exit codes and HTTP 400 mapping catch that class,
cli.py:247-266, service/server.py:107-109).
"""

import functools

import anybcq
import anybcq.cli
import anybcq.errors
import anybcq.gemv
import anybcq.bcq
import anybcq.progressive
import anybcq.service.server

import paper_2510_10467_b200.engine as b200
import paper_2510_10467_b200.quantize as b200q
from paper_2510_10467_b200.errors import NonFiniteError as B200NonFiniteError
from paper_2510_10467_b200.errors import UsageError as B200UsageError


def _ref_errors(fn):
    @functools.wraps(fn)
    def wrapped(*a, **k):
        try:
            return fn(*a, **k)
        except B200UsageError as exc:
            raise anybcq.errors.UsageError(str(exc)) from exc
        except B200NonFiniteError as exc:
            raise anybcq.errors.NonFiniteError(str(exc)) from exc
    return wrapped


class GemvEngine(b200.GemvEngine):
    __init__ = _ref_errors(b200.GemvEngine.__init__)
    lut = _ref_errors(b200.GemvEngine.lut)
    naive = _ref_errors(b200.GemvEngine.naive)


def gemv_lut(model, p, x, chunk_width=8):
    return GemvEngine(model, chunk_width).lut(p, x)


def gemv_naive(model, p, x):
    return GemvEngine(model).naive(p, x)


bench = _ref_errors(b200.bench)   # device-timed (CUDA events), same rows and counters

for _mod in (anybcq, anybcq.gemv, anybcq.cli, anybcq.service.server):
    _mod.GemvEngine = GemvEngine
    _mod.bench = bench
for _mod in (anybcq, anybcq.gemv):
    _mod.gemv_lut = gemv_lut
    _mod.gemv_naive = gemv_naive

# the GPU quantizer (quantize.py) behind the reference's fitting API
for _name in ("greedy_init", "ls_update_scales", "bs_recalibrate_codes", "alternate_fit", "dequantize",
              "expand_step", "build_multiprecision", "precision_errors"):
    _fn = _ref_errors(getattr(b200q, _name))
    for _mod in (anybcq, anybcq.bcq, anybcq.progressive, anybcq.cli):
        if hasattr(_mod, _name):
            setattr(_mod, _name, _fn)
