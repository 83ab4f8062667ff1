#!/usr/bin/env python3
"""One config-1 training view bracketed by cudaProfilerStart/Stop, for ncu captures.

    ncu --set full --import-source on --clock-control none --profile-from-start off \
        -o gpurun_out/step python profiles/capture_step.py
    ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
        python profiles/capture_step.py

Same workload as bench.py (1M Gaussians, seed 0, 1237x822 ring views, L1 vs perturbed targets,
all 59 gradients, Adam on means); three unprofiled warm-up views first.
"""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2411_12788_b200 import capi, scenes  # noqa: E402
from paper_2411_12788_b200.rasterizer import Context, DeviceGaussians, render  # noqa: E402
from paper_2411_12788_b200.trainer import ViewTrainer  # noqa: E402


def main(views: int = 1, warmup: int = 3):
    torch.cuda.set_device(0)
    ctx = Context.default(0)
    s = scenes.make_gaussians(1_000_000, seed=0)
    ds = DeviceGaussians.from_host(s, 0)
    dt = DeviceGaussians.from_host(scenes.perturbed(s), 0)
    cams = [scenes.ring_camera(k, 64) for k in range(warmup + views)]
    targets = [render(dt, c, want_depth=False, ctx=ctx).color.clone() for c in cams]
    del dt
    tr = ViewTrainer(ds, capi.AdamConfig(), group_mask=capi.GROUP_CENTERS, ctx=ctx)
    for k in range(warmup):
        tr.step([cams[k]], [targets[k]])
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    for k in range(warmup, warmup + views):
        tr.step([cams[k]], [targets[k]])
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print("captured", views, "view(s);", tr.pairs_last_step[-1], "pairs")


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 1)
