#!/usr/bin/env python3
"""GPU timeline of one config-4 step (3 M Gaussians, 8 views, Adam on every group; CUPTI kernel
records through torch.profiler): per stream, busy time and the idle gaps, to see how the twin
context overlaps one view's front end with the other view's blend kernels."""
import json
import sys
import tempfile
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2411_12788_b200 import capi, scenes  # noqa: E402
from paper_2411_12788_b200.rasterizer import Context, DeviceGaussians, render  # noqa: E402
from paper_2411_12788_b200.trainer import ViewTrainer  # noqa: E402

torch.cuda.set_device(0)
ctx = Context.default(0)
s = scenes.make_gaussians(3_000_000, seed=0)
ds = DeviceGaussians.from_host(s, 0)
dt = DeviceGaussians.from_host(scenes.perturbed(s), 0)
cams = [scenes.ring_camera(k, 256) for k in range(256)]
targets = [render(dt, c, want_depth=False, ctx=ctx).color.clone() for c in cams[:32]]
del dt
tr = ViewTrainer(ds, capi.AdamConfig(scene_extent=3.3), group_mask=capi.GROUP_ALL, ctx=ctx, max_views=8)
for k in range(2):
    tr.step(cams[8 * k:8 * k + 8], targets[8 * k:8 * k + 8])
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    tr.step(cams[16:24], targets[16:24])
    torch.cuda.synchronize()
path = Path(tempfile.mkdtemp()) / "trace.json"
prof.export_chrome_trace(str(path))
ev = json.load(open(path))["traceEvents"]
ks = sorted([e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")], key=lambda e: e["ts"])
t0 = ks[0]["ts"]
end = max(e["ts"] + e["dur"] for e in ks)
print(f"step span {end - t0:.0f} us")
# union of busy intervals over all streams, and per kernel family time
iv = sorted((e["ts"], e["ts"] + e["dur"]) for e in ks)
busy, cur_s, cur_e = 0.0, None, None
for a, b in iv:
    if cur_e is None or a > cur_e:
        if cur_e is not None:
            busy += cur_e - cur_s
        cur_s, cur_e = a, b
    else:
        cur_e = max(cur_e, b)
busy += cur_e - cur_s
print(f"GPU busy (any stream) {busy:.0f} us, idle {end - t0 - busy:.0f} us")
fam = {}
for e in ks:
    nm = e["name"].replace("void ", "").replace("splat_b200::", "").replace("(anonymous namespace)::", "").split("(")[0].split("<")[0]
    fam[nm] = fam.get(nm, 0.0) + e["dur"]
for k, v in sorted(fam.items(), key=lambda x: -x[1])[:16]:
    print(f"  {k:40s} {v:8.0f} us")
for e in ks:
    nm = e["name"].replace("void ", "").replace("splat_b200::", "").replace("(anonymous namespace)::", "").split("(")[0][:34]
    print(f"{e['ts'] - t0:9.1f} {e['dur']:8.1f} s{e.get('args', {}).get('stream', '?')} {nm}")
