import sys, torch
sys.path.insert(0, "/root/repo")
from paper_2411_12788_b200 import scenes, capi
from paper_2411_12788_b200.rasterizer import Context, DeviceGaussians, render, render_backward
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
ctx = Context.default(0)
s = scenes.make_gaussians(n, seed=0)
ds = DeviceGaussians.from_host(s, 0)
cam = scenes.ring_camera(0, 64)
render(ds, cam, want_depth=False, ctx=ctx); torch.cuda.synchronize(); print("render ok")
d_color = torch.full((cam.height, cam.width, 3), 1e-6, device="cuda:0")
render_backward(ds, cam, capi.RasterConfig(), d_color, ctx=ctx); torch.cuda.synchronize(); print("backward ok")
