#!/usr/bin/env python3
"""How deep the blend forward walks each tile list (config 1): per tile, the deepest list position
any of its 8x8 blocks staged before saturating, against the list length.  Needs the instrumented
variant: python tools/variant_build.py walk forward.cu file:<forward.cu with g_walk + splat_debug_walk>
and SPLAT_B200_LIB=paper_2411_12788_b200/lib_walk/libsplat_b200.so."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2411_12788_b200 import scenes  # noqa: E402
from paper_2411_12788_b200.rasterizer import Context, DeviceGaussians, render  # noqa: E402

ctx = Context.default(0)
s = scenes.make_gaussians(1_000_000, seed=0)
ds = DeviceGaussians.from_host(s, 0)
buf = np.zeros(2 * 65536, np.uint32)
ctx.lib.splat_debug_walk.argtypes = [C.c_void_p, C.c_int]
ctx.lib.splat_debug_walk(buf.ctypes.data, 0)
for k in ([int(a) for a in sys.argv[1:]] or (0, 16, 32, 48)):
    cam = scenes.ring_camera(k, 64)
    render(ds, cam, want_depth=False, ctx=ctx)
    torch.cuda.synchronize()
    ctx.lib.splat_debug_walk(buf.ctypes.data, 0)
    tiles = ((cam.width + 15) // 16) * ((cam.height + 15) // 16)
    walked = buf[:65536][: 4 * tiles].reshape(tiles, 4).max(1).astype(np.int64)
    length = buf[65536:][: 4 * tiles].reshape(tiles, 4).max(1).astype(np.int64)
    if len(sys.argv) > 5:
        print(f"view {k}: walked max {walked.max()}, list max {length.max()}")
        continue
    print(f"view {k}: tiles {tiles}, list entries {length.sum():,}, walked (deepest block per tile) {walked.sum():,} "
          f"({100 * walked.sum() / length.sum():.1f} %); list length p50/p90/max {np.percentile(length, 50):.0f}/"
          f"{np.percentile(length, 90):.0f}/{length.max()}, walked p50/p90/p99/max {np.percentile(walked, 50):.0f}/"
          f"{np.percentile(walked, 90):.0f}/{np.percentile(walked, 99):.0f}/{walked.max()}")
    for K in (128, 256, 512, 1024, 2048):
        over = (walked > K - 64) & (length > K)  # may need entries past a K-entry prefix
        print(f"   prefix {K:5d}: entries built {np.minimum(length, K).sum():,} "
              f"({100 * np.minimum(length, K).sum() / length.sum():.1f} %), tiles that may run past it "
              f"{over.sum()} ({100 * over.mean():.2f} %), their entries {length[over].sum():,}")
