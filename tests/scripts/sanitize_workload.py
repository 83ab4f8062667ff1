"""A config-0-sized pass over every kernel family, for compute-sanitizer (tests/test_gpu_sanitizer.py):
render with all outputs + importance, the fused L1 backward, Adam, a 2-view training step with host
targets (twin context, copy stream), the depth sort at a size that takes the cooperative path,
depth unprojection, visibility pass, densify / simplify kernels and SSIM."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path[:0] = [str(ROOT)]
from paper_2411_12788_b200 import capi, densify as D, scenes  # noqa: E402
from paper_2411_12788_b200 import rasterizer as R  # noqa: E402
from paper_2411_12788_b200.trainer import ViewTrainer  # noqa: E402

s = scenes.make_gaussians(20_000, seed=0)
cams = [scenes.ring_camera(k, 4, width=256, height=192) for k in range(4)]
ds = R.DeviceGaussians.from_host(s)
out, rep = R.render(ds, cams[0], report=True)
tgt = [R.render(R.DeviceGaussians.from_host(scenes.perturbed(s)), c, want_depth=False).color.clone() for c in cams]
tr = ViewTrainer(ds, capi.AdamConfig(), group_mask=capi.GROUP_ALL, max_views=2)
tr.step(cams[:2], tgt[:2])
tr.step_host(cams[2:], [t.cpu().pin_memory() for t in tgt[2:]])
R.depth_points(ds, cams[:2], stride=4)
R.visibility_pass(ds, cams[:2])
crit, _ = D.identify_critical(ds, cams[:2], "max-weight", 0.5)
grown, ms = D.aggressive_clone(ds, crit)
D.importance_sample(ds, torch.rand(s.n, dtype=torch.float64, device="cuda"), 5000, 3)
R.ssim(tgt[0], tgt[1])
torch.cuda.synchronize()
print("sanitize workload ok")
