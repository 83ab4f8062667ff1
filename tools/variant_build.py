#!/usr/bin/env python3
"""Build a variant of the product library from a patched copy of one source file, into
paper_2411_12788_b200/lib_<name>/ (for A/B timing with SPLAT_B200_LIB; not used by the product).

    python tools/variant_build.py <name> <source.cu> <sed-expression | file:<path>>
"""
import shutil
import subprocess
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2411_12788_b200 import build as b  # noqa: E402

name, src, expr = sys.argv[1:4]
work = Path("/tmp") / f"variant_{name}"
if work.exists():
    shutil.rmtree(work)
shutil.copytree(b.CSRC, work)
if expr.startswith("file:"):  # replace the source by another file (e.g. a copy from git history)
    shutil.copy(expr[5:], work / src)
else:
    subprocess.run(["sed", "-i", expr, str(work / src)], check=True)
b.CSRC = work
b.HEADERS = [work / "common.cuh", work / "internal.h"] + b.HEADERS[2:]
b.OBJ = b.PKG / f"build_{name}"
b.LIB = b.PKG / f"lib_{name}" / "libsplat_b200.so"
b.COMMON = [a.replace(str(b.PKG / "csrc"), str(work)) for a in b.COMMON]
print(b.build(verbose=False))
