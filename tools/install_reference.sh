#!/usr/bin/env bash
# Install the UNMODIFIED reference package (anybcq) into baseline/_ref -- the
# reference arm of bench.py and the drop-in test of the reference's own test
# files (tests/test_reference_suite_gpu.py). Run in the build container, where
# /root/reference exists; baseline/_ref is git-ignored but travels to the GPU
# box with gpurun. The install needs no network: numpy / numba / fastapi /
# pydantic are already in the image, so dependency resolution is skipped
# (--no-deps); the build runs from a copy because /root/reference is read-only.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC=/root/reference/pkg
[ -d "$SRC" ] || { echo "no $SRC here (GPU box?): keep the prebuilt baseline/_ref" >&2; exit 0; }
TMP="$(mktemp -d)"
cp -r "$SRC" "$TMP/pkg"
rm -rf "$ROOT/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$ROOT/baseline/_ref" "$TMP/pkg"
# the reference's own test files, run unchanged against the drop-in
cp -r "$SRC/tests" "$ROOT/baseline/_ref/anybcq_tests"
rm -rf "$TMP"
echo "installed: $ROOT/baseline/_ref"
