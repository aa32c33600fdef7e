"""Compile the C oracle (oracle/c/abcq_oracle.c) -> oracle/build/libabcq_oracle.so.

Test / baseline infrastructure only. The reference itself is Python + numba
(no C/C++ sources), so there is no `oracle/_ref` build: the reference arm
runs this restatement ("port"), see DESIGN.md §Oracle.
"""

from __future__ import annotations

import subprocess
from pathlib import Path

HERE = Path(__file__).resolve().parent
SRC = HERE / "c" / "abcq_oracle.c"
OUT = HERE / "build" / "libabcq_oracle.so"


def build(force: bool = False) -> Path:
    if not force and OUT.exists() and OUT.stat().st_mtime >= SRC.stat().st_mtime:
        return OUT
    OUT.parent.mkdir(exist_ok=True)
    cmd = ["gcc", "-O3", "-std=c11", "-fPIC", "-shared", "-pthread", str(SRC), "-o", str(OUT)]
    subprocess.run(cmd, check=True)
    return OUT


if __name__ == "__main__":
    print(build(force=True))
