#!/usr/bin/env python3
"""Instrumented build of the product library (-DSPLAT_STATS) into paper_2411_12788_b200/lib_stats/,
for traversal-statistics experiments (tools/traversal_stats.py). Not used by the product.

    python tools/stats_build.py [bwd]   # bwd: instrument the backward only (the forward's counters
                                        # fault at 1 M Gaussians, see tools/traversal_stats.py)"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2411_12788_b200 import build as b  # noqa: E402

b.OBJ = b.PKG / "build_stats"
b.LIB = b.PKG / "lib_stats" / "libsplat_b200.so"
if "bwd" in sys.argv[1:]:
    b.SOURCES = dict(b.SOURCES)
    b.SOURCES["backward.cu"] = b.SOURCES["backward.cu"] + ["-DSPLAT_STATS"]
    print(b.build(verbose=False, force=True))
else:
    print(b.build(verbose=False, extra_flags=("-DSPLAT_STATS",)))
