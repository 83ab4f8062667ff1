#!/usr/bin/env python3
"""Instrumented build of the product library (-DSPLAT_STATS) into paper_2411_12788_b200/lib_stats/,
for traversal-statistics experiments (tools/traversal_stats.py). Not used by the product."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2411_12788_b200 import build as b  # noqa: E402

b.OBJ = b.PKG / "build_stats"
b.LIB = b.PKG / "lib_stats" / "libsplat_b200.so"
print(b.build(verbose=False, extra_flags=("-DSPLAT_STATS",)))
