#!/usr/bin/env python3
"""Forward / backward traversal statistics of one config-1 view (instrumented build, SPLAT_B200_LIB).

Known issue: with the forward counters compiled in (-DSPLAT_STATS in forward.cu) the instrumented
forward faults at 1 M Gaussians (fine at 20 K); build with the forward counters renamed out
(SPLAT_STATS_FWD) to read the backward counters at full size.

    python tools/stats_build.py   # here
    SPLAT_B200_LIB=paper_2411_12788_b200/lib_stats/libsplat_b200.so python tools/traversal_stats.py
"""
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
cam = scenes.ring_camera(0, 64)
render(ds, cam, want_depth=False, ctx=ctx)
buf = (C.c_ulonglong * 12)()
lib = ctx.lib
lib.splat_debug_stats.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
rc0 = lib.splat_debug_stats(buf, 1)
print("forward stats:", "on" if rc0 == 0 else f"off (rc {rc0})")
from paper_2411_12788_b200 import capi  # noqa: E402
from paper_2411_12788_b200.rasterizer import render_backward  # noqa: E402
lib.splat_debug_bstats.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
bbuf = (C.c_ulonglong * 12)()
render(ds, cam, want_depth=False, ctx=ctx)
torch.cuda.synchronize()
lib.splat_debug_stats(buf, 1)
lib.splat_debug_bstats(bbuf, 1)
d_color = torch.full((cam.height, cam.width, 3), 1e-6, device="cuda:0")
render_backward(ds, cam, capi.RasterConfig(), d_color, ctx=ctx)
torch.cuda.synchronize()
lib.splat_debug_bstats(bbuf, 1)
bv = list(bbuf)
bnames = ["bwd half-entries evaluated", "  with >=1 commit", "  eligible lanes (idx <= last)",
          "  committing lanes", "  pair iterations (past the skip test)", "  entries reduced",
          "  reductions with one entry committing", "  half evaluations with one eligible entry"]
for n, x in zip(bnames, bv):
    print(f"{n:45s} {x:,}")
print(f"bwd eligible lanes per evaluation {bv[2] / max(bv[0], 1):.1f}, committing {bv[3] / max(bv[1], 1):.1f} per reduction")
v = list(buf)
names = ["warp-entries evaluated", "  of which exact 8x4 patch test fails", "  of which >=1 lane gate passes",
         "  exact patch passes but no lane passes", "entries staged (block cull kept)", "lanes active at eval (sum)",
         "entries offered to staging", "warp-batches with active lanes", "warp-batches needed (packed)",
         "active pixel-batches", "CTA batches"]
for n, x in zip(names, v):
    print(f"{n:45s} {x:,}")
print(f"mean active lanes per evaluation {v[5] / max(v[0], 1):.1f}")
