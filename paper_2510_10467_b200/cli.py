"""Command-line surface of the drop-in engine: `gemv` and `bench`, with the
reference CLI's flags, outputs and exit codes (/root/reference/pkg/src/
anybcq/cli.py:113-158,184-247): 0 success, 2 bad flags or validation
(UsageError), 3 file / I-O problems (FileFormatError, OSError), 4 numeric
failure (NonFiniteError). Errors go to stderr only.

    python -m paper_2510_10467_b200.cli gemv --model m.abcq --bits 3 --x x.fmat --out y.fmat
    python -m paper_2510_10467_b200.cli bench --model m.abcq --bits all --repeats 32 --format csv

The model is loaded with the progressive GPU loader (container.py). `gemv`
runs every row of x at precision --bits through ONE batched launch per 32
rows (abcq_gemv_batch; bitwise equal to per-row calls) and prints the CRC32
of the f32 outputs plus the reference's traffic counters. `--path naive`
uses the f64 per-column kernel (GemvEngine.naive). `bench --shapes` (the
reference's quantize-then-bench suite) is not offered: quantization is out
of scope; bench a container instead.
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


def _cmd_bench(args) -> int:
    from .container import deserialize
    from .engine import bench, render_bench_csv, render_bench_text
    from .tensor_io import random_gaussian

    if args.model is None:
        raise UsageError("--model is required (quantizing a synthetic --shapes suite is out of scope)")
    if args.repeats < 1:
        raise UsageError("--repeats must be >= 1")
    model = deserialize(args.model)
    if args.bits == "all":
        precisions = list(model.precisions)
    else:
        try:
            precisions = [int(b) for b in args.bits.split(",")]
        except ValueError as exc:
            raise UsageError(f"--bits expects 'all' or a comma list, got {args.bits!r}") from exc
    x = random_gaussian(1, model.shape[1], args.seed).ravel()
    rows = bench(model, precisions, x, repeats=args.repeats, include_dense=args.dense)
    print(render_bench_csv(rows) if args.format == "csv" else render_bench_text(rows))
    return 0


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="anybcq-b200", description="AnyBCQ bit-plane GEMV on B200 (sm_100a)")
    ap.add_argument("--version", action="version", version=f"anybcq-b200 {__version__}")
    sub = ap.add_subparsers(dest="command", required=True)
    g = sub.add_parser("gemv", help="run the engine at a chosen precision")
    g.add_argument("--model", required=True)
    g.add_argument("--bits", type=int, required=True)
    g.add_argument("--x", required=True, help="FMAT input (one vector per row)")
    g.add_argument("--out", required=True)
    g.add_argument("--path", choices=("lut", "naive"), default="lut")
    g.set_defaults(func=_cmd_gemv)
    b = sub.add_parser("bench", help="time the engine paths")
    b.add_argument("--model")
    b.add_argument("--bits", default="all")
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
