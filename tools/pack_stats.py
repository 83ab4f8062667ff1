"""Forward warp-packing potential (variant build lib_pack): pair iterations per batch and warp,
and the share spent in batches that start with <= 32 active pixels (one warp could hold them)."""
import ctypes as C
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2411_12788_b200 import scenes  # noqa: E402
from paper_2411_12788_b200.rasterizer import Context, DeviceGaussians, render  # noqa: E402

ctx = Context.default(0)
s = scenes.make_gaussians(1_000_000, seed=0)
ds = DeviceGaussians.from_host(s, 0)
buf = (C.c_ulonglong * 8)()
ctx.lib.splat_debug_pack.argtypes = [C.POINTER(C.c_ulonglong)]
for k in range(3):
    render(ds, scenes.ring_camera(k, 64), want_depth=False, ctx=ctx)
    torch.cuda.synchronize()
    ctx.lib.splat_debug_pack(buf)
    v = list(buf)
    print(f"view {k}: pair iterations (both warps) {v[0]:,}; in batches with <= 32 active pixels {v[2]:,} "
          f"({v[2] / max(v[0], 1):.1%}); saved by packing there (>= min of the warps) {v[1]:,} ({v[1] / max(v[0], 1):.1%}); "
          f"batches {v[3]:,}, packable {v[4]:,}")
