"""Command-line surface of the drop-in engine: `quantize`, `gemv` and `bench`,
with the reference CLI's flags, outputs and exit codes (/root/reference/pkg/
src/anybcq/cli.py:75-158,184-247): 0 success, 2 bad flags or validation
(UsageError), 3 file / I-O problems (FileFormatError, OSError), 4 numeric
failure (NonFiniteError). Errors go to stderr only.

    python -m paper_2510_10467_b200.cli quantize --random 4096x4096 --bits 2:4 --out m.abcq
    python -m paper_2510_10467_b200.cli gemv --model m.abcq --bits 3 --x x.fmat --out y.fmat
    python -m paper_2510_10467_b200.cli bench --model m.abcq --bits all --repeats 32 --format csv
    python -m paper_2510_10467_b200.cli bench --shapes 4096x14336 --format csv

The model is loaded with the progressive GPU loader (container.py). `gemv`
runs every row of x at precision --bits through ONE batched launch per 32
rows (abcq_gemv_batch; bitwise equal to per-row calls) and prints the CRC32
of the f32 outputs plus the reference's traffic counters. `--path naive`
uses the f64 per-column kernel (GemvEngine.naive). `quantize` and `bench
--shapes` fit on the GPU (quantize.py: the reference's greedy / least-squares
/ recalibration / progressive expansion as CUDA kernels). The reference's
refine / inspect commands (calibration, footprint accounting) are not part
of this path.
"""

from __future__ import annotations

import argparse
import sys
import zlib

import numpy as np

from . import __version__
from .errors import AnyBcqError, FileFormatError, NonFiniteError, UsageError


def _cmd_gemv(args) -> int:
    import torch

    from . import _lib
    from .container import ProgressiveLoader
    from .device_model import gemv_batch
    from .engine import GemvEngine
    from .tensor_io import load_matrix, save_matrix

    x = load_matrix(args.x)
    loader = ProgressiveLoader(args.model)
    dm = loader.model
    if x.shape[1] != dm.cols:
        raise UsageError(f"input cols {x.shape[1]} != model cols {dm.cols}")
    if args.bits not in dm.precisions:
        raise UsageError(f"precision {args.bits} outside [{dm.p_lo}, {dm.p_hi}]")
    loader.load_all()
    st = GemvEngine(dm)._stats(args.bits, 1 if args.path == "lut" else 0, 0.0)
    xd = torch.from_numpy(np.array(x)).to(dm.device)
    if args.path == "lut" and dm.layout == _lib.LAYOUT_TILED:
        ys = torch.empty(x.shape[0], dm.rows, dtype=torch.float32, device=dm.device)
        gemv_batch([(dm, args.bits, xd[s], ys[s]) for s in range(x.shape[0])])
    else:
        run = dm.gemv if args.path == "lut" else dm.gemv_naive
        ys = torch.stack([run(args.bits, xd[s]) for s in range(x.shape[0])])
    y = ys.cpu().numpy().astype(np.float32)
    save_matrix(y, args.out)
    print(f"checksum=0x{zlib.crc32(y.astype('<f4').tobytes()):08x}")
    print(f"plane_bytes={st.plane_bytes_fetched * x.shape[0]} scale_bytes={st.scale_bytes_fetched * x.shape[0]} "
          f"path={args.path}")
    return 0


BENCH_SUITE = ((4096, 14336), (5120, 17920), (8192, 28672))  # cli.py:33-34
_MODES = {"sym": "symmetric", "asym": "asymmetric", "symmetric": "symmetric", "asymmetric": "asymmetric"}


def _parse_bits(spec: str) -> tuple[int, int]:
    """P or L:H (cli.py:40-51)."""
    try:
        if ":" in spec:
            lo_s, hi_s = spec.split(":", 1)
            lo, hi = int(lo_s), int(hi_s)
        else:
            lo = hi = int(spec)
    except ValueError as exc:
        raise UsageError(f"--bits expects P or L:H, got {spec!r}") from exc
    if not 1 <= lo <= hi:
        raise UsageError(f"--bits range must satisfy 1 <= L <= H, got {spec!r}")
    return lo, hi


def _parse_shape(spec: str) -> tuple[int, int]:
    """RxC (cli.py:54-62)."""
    try:
        rows_s, cols_s = spec.lower().split("x", 1)
        rows, cols = int(rows_s), int(cols_s)
    except ValueError as exc:
        raise UsageError(f"expected RxC, got {spec!r}") from exc
    if rows < 1 or cols < 1:
        raise UsageError(f"shape dims must be >= 1, got {spec!r}")
    return rows, cols


def _cmd_quantize(args) -> int:
    """Fit a multi-precision model on the GPU (quantize.build_multiprecision)
    and write an ABCQ container (cli.py:75-93: same flags, output lines)."""
    from .container import serialize
    from .model import QuantConfig
    from .quantize import build_multiprecision, precision_errors
    from .tensor_io import load_matrix, random_gaussian

    if args.input is None and args.random is None:
        raise UsageError("one of --input or --random is required")
    if args.input is not None and args.random is not None:
        raise UsageError("--input and --random are mutually exclusive")
    w = load_matrix(args.input) if args.input is not None else random_gaussian(*_parse_shape(args.random), args.seed)
    p_lo, p_hi = _parse_bits(args.bits)
    cfg = QuantConfig(group_size=args.group, mode=_MODES[args.mode], cycles=args.cycles)
    model = build_multiprecision(w, p_lo, p_hi, cfg)
    serialize(model, args.out, scale_width=args.scale_width)
    errs = precision_errors(w, model)
    if args.format == "csv":
        print("p,relative_sq_error")
        for p in model.precisions:
            print(f"{p},{errs[p]:.8f}")
    else:
        print(f"{'p':>3}  relative_sq_error")
        for p in model.precisions:
            print(f"{p:>3}  {errs[p]:.8f}")
        print(f"wrote {args.out}")
    return 0


def _cmd_bench(args) -> int:
    """--model: a container; --shapes: the reference's synthetic suite
    (cli.py:135-158), each shape fitted on the GPU (build_multiprecision
    2:4, cycles 1) and benched with its dense weights as the dense row."""
    from .container import deserialize
    from .engine import bench, render_bench_csv, render_bench_text
    from .model import QuantConfig
    from .tensor_io import random_gaussian

    if (args.model is None) == (args.shapes is None):
        raise UsageError("exactly one of --model or --shapes is required")
    if args.repeats < 1:
        raise UsageError("--repeats must be >= 1")

    def bits(default):
        if args.bits == "all":
            return default
        try:
            return [int(b) for b in args.bits.split(",")]
        except ValueError as exc:
            raise UsageError(f"--bits expects 'all' or a comma list, got {args.bits!r}") from exc

    rows = []
    if args.model is not None:
        model = deserialize(args.model)
        x = random_gaussian(1, model.shape[1], args.seed).ravel()
        rows += bench(model, bits(list(model.precisions)), x, repeats=args.repeats, include_dense=args.dense)
    else:
        from .quantize import build_multiprecision
        for spec in args.shapes.split(","):
            shape = _parse_shape(spec)
            w = random_gaussian(*shape, seed=args.seed)
            model = build_multiprecision(w, 2, 4, QuantConfig(group_size=args.group, cycles=1))
            x = random_gaussian(1, shape[1], args.seed + 1).ravel()
            rows += bench(model, bits([2, 3, 4]), x, repeats=args.repeats, include_dense=args.dense,
                          dense_weights=w)
    print(render_bench_csv(rows) if args.format == "csv" else render_bench_text(rows))
    return 0


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="anybcq-b200", description="AnyBCQ bit-plane GEMV on B200 (sm_100a)")
    ap.add_argument("--version", action="version", version=f"anybcq-b200 {__version__}")
    sub = ap.add_subparsers(dest="command", required=True)
    q = sub.add_parser("quantize", help="fit a multi-precision model (on the GPU)")
    q.add_argument("--input", help="FMAT weight matrix")
    q.add_argument("--random", metavar="NxK", help="generate a seeded Gaussian matrix")
    q.add_argument("--seed", type=int, default=0)
    q.add_argument("--bits", required=True, help="P for fixed precision or L:H for progressive")
    q.add_argument("--group", type=int, default=128)
    q.add_argument("--cycles", type=int, default=20)
    q.add_argument("--mode", choices=sorted(_MODES), default="asym")
    q.add_argument("--scale-width", type=int, choices=(2, 4), default=4)
    q.add_argument("--out", required=True)
    q.add_argument("--format", choices=("text", "csv"), default="text")
    q.set_defaults(func=_cmd_quantize)
    g = sub.add_parser("gemv", help="run the engine at a chosen precision")
    g.add_argument("--model", required=True)
    g.add_argument("--bits", type=int, required=True)
    g.add_argument("--x", required=True, help="FMAT input (one vector per row)")
    g.add_argument("--out", required=True)
    g.add_argument("--path", choices=("lut", "naive"), default="lut")
    g.set_defaults(func=_cmd_gemv)
    b = sub.add_parser("bench", help="time the engine paths")
    b.add_argument("--model")
    b.add_argument("--shapes", help="synthetic suite, e.g. " + ",".join(f"{r}x{c}" for r, c in BENCH_SUITE))
    b.add_argument("--bits", default="all")
    b.add_argument("--group", type=int, default=128)
    b.add_argument("--repeats", type=int, default=32)
    b.add_argument("--seed", type=int, default=0)
    b.add_argument("--dense", action="store_true", help="add the dense f32 GEMV row (reference contract)")
    b.add_argument("--format", choices=("text", "csv"), default="text")
    b.set_defaults(func=_cmd_bench)
    return ap


def main(argv=None) -> int:
    parser = build_parser()
    try:
        args = parser.parse_args(argv)
    except SystemExit as exc:  # argparse: 2 on bad flags, 0 on --help / --version
        return int(exc.code or 0)
    try:
        return args.func(args)
    except UsageError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2
    except (FileFormatError, OSError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 3
    except NonFiniteError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 4
    except AnyBcqError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
