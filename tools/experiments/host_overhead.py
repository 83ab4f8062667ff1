"""Host-side cost of one ViewTrainer.step_host call on the B200 box: the end-to-end step time and
the Python wrapper alone (the C-ABI call stubbed), config 1."""
import time, sys
sys.path.insert(0, '.')
import torch, numpy as np
from paper_2411_12788_b200 import capi, scenes
from paper_2411_12788_b200.rasterizer import Context, DeviceGaussians, render
from paper_2411_12788_b200.trainer import ViewTrainer
torch.cuda.set_device(0)
ctx = Context.default(0)
s = scenes.make_gaussians(1_000_000, seed=0)
ds = DeviceGaussians.from_host(s, 0)
dt = DeviceGaussians.from_host(scenes.perturbed(s), 0)
cams = [scenes.ring_camera(k, 64) for k in range(64)]
targets = [render(dt, c, want_depth=False, ctx=ctx).color.clone() for c in cams]
host_t = [t.cpu().pin_memory() for t in targets]
tr = ViewTrainer(ds, capi.AdamConfig(), group_mask=capi.GROUP_CENTERS, ctx=ctx)
for k in range(10): tr.step_host([cams[k]], [host_t[k]])
torch.cuda.synchronize()
# host-only overhead of the Python wrapper: time _native's prologue by monkeypatching the lib call
N=200
t0=time.perf_counter()
for k in range(N): tr.step_host([cams[k % 64]], [host_t[k % 64]])
t1=time.perf_counter()
print("e2e per step us", (t1-t0)/N*1e6)
lib = ctx.lib
real = lib.splat_train_step
class Fake:
    def __call__(self, *a): return 0
lib.splat_train_step = Fake()
t0=time.perf_counter()
for k in range(N): tr.step_host([cams[k % 64]], [host_t[k % 64]])
t1=time.perf_counter()
print("python wrapper only per step us", (t1-t0)/N*1e6)
lib.splat_train_step = real
