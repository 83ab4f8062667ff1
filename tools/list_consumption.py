#!/usr/bin/env python3
"""How much of the per-tile lists the blend forward reads (it stops a block at saturation), for
one config-1 view: entries offered to staging / tile-list entries, over all 8 x 8 blocks (each
block walks its tile's list).  Needs the instrumented variant built from a forward with the
g_consumed counters (level-2 bypass estimate)."""
import ctypes as C
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2411_12788_b200 import scenes  # noqa: E402
from paper_2411_12788_b200.rasterizer import Context, DeviceGaussians, render  # noqa: E402

ctx = Context.default(0)
s = scenes.make_gaussians(1_000_000, seed=0)
ds = DeviceGaussians.from_host(s, 0)
buf = (C.c_ulonglong * 4)()
ctx.lib.splat_debug_consumed.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
for k in range(4):
    cam = scenes.ring_camera(k * 16, 64)
    ctx.lib.splat_debug_consumed(buf, 1)
    render(ds, cam, want_depth=False, ctx=ctx)
    torch.cuda.synchronize()
    ctx.lib.splat_debug_consumed(buf, 1)
    print(f"view {k * 16}: offered {buf[0]:,} of {buf[1]:,} list entries walked by the blocks "
          f"({100 * buf[0] / max(buf[1], 1):.1f} %), staged {buf[2]:,}")
