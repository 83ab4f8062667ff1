"""Tile lists materialised only up to a prefix (binning.cu bin_emit, StagePipe tails): with the
prefix cut to 64 / 256 entries every block walks into the supertile-list tails, in the forward
(training and importance), in the backward's re-culling paths (the one-pixel-per-thread backward
re-culls every tile list) and after the bit-exact getter completed the lists; results must be the
oracle's as with complete lists.  Separate processes: the prefix is fixed at context creation."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.timeout(600)
@pytest.mark.parametrize("env", [{"SPLAT_LIST_PREFIX": "64"}, {"SPLAT_LIST_PREFIX": "256", "SPLAT_BWD_PX2": "0"},
                                 {"SPLAT_LIST_PREFIX": "100", "SPLAT_BLEND_PERSISTENT": "0"}])
def test_parity_with_list_tails(env):
    r = subprocess.run([sys.executable, str(ROOT / "tests" / "scripts" / "tails_check.py")], capture_output=True,
                       text=True, timeout=550, env=dict(os.environ, **env), cwd=str(ROOT))
    assert r.returncode == 0 and "tails check ok" in r.stdout, (r.stdout + r.stderr)[-4000:]


def test_default_prefix_on_deep_walks(oracle):
    """Default (adaptive) prefix on a scene whose pixels never saturate: 12 K faint Gaussians all
    over a 64 x 64 image give every tile a ~12 K-entry list that the blend walks to its end, past
    the 4096-entry prefix (the first view reads the tails, later views a doubled prefix); images
    and gradients stay the oracle's."""
    import numpy as np
    from helpers import assert_bitwise, assert_grads_close
    from paper_2411_12788_b200 import rasterizer as R
    from paper_2411_12788_b200 import scenes
    from paper_2411_12788_b200.capi import RasterConfig
    s = scenes.make_gaussians(12_000, seed=7, radius=0.6, log_scale_mean=np.log(0.3))
    s.opacity_logits[:] = np.float32(-4.0)  # alpha ~ 0.018: transmittance stays above the floor
    cam = scenes.front_camera(64, 64)
    want = oracle.render(s, cam, report=False)
    for view in range(3):
        out = R.render(s, cam)
        for key in ("color", "alpha", "transmittance", "max_contributor"):
            assert_bitwise(getattr(out, key), want[key], f"view {view} {key}")
    target = oracle.render(scenes.perturbed(s), cam, report=False)["color"]
    _, d_color = oracle.l1_loss(want["color"], target)
    assert_grads_close(R.render_backward(s, cam, RasterConfig(), d_color), oracle.render_backward(s, cam, d_color),
                       what="deep walks")
    fw = R.forward_debug()
    lens = fw["ranges"][:, 1] - fw["ranges"][:, 0]
    assert lens.max() > 4096, lens.max()
