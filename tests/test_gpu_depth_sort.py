"""The forward's depth sort on skewed depth distributions, CUDA path vs the oracle's
std::sort by (depth, index) (rasterizer.cpp:85-88): the survivor order bit-exact.

With the front camera (depth = z + 4 exactly) the scenes put thousands of Gaussians on one
plane of identical depth (ties: the stable LSD sort must keep them in index order) or on a slab of
distinct depths a few ulps apart (long runs of keys that differ only in the low digits), mixed
with the uniform ball, back to back on one context with changing Gaussian counts (the sort's
zero-at-rest histogram and its trivial-pass skipping must re-arm between views).
"""
import numpy as np
import pytest

from helpers import assert_bitwise
from paper_2411_12788_b200 import rasterizer as R
from paper_2411_12788_b200 import scenes

pytestmark = pytest.mark.gpu


def _scene(n, seed, kind):
    s = scenes.make_gaussians(n, seed=seed)
    rng = np.random.default_rng(seed)
    c = s.centers.copy()
    if kind == "plane":  # 5000 Gaussians at one depth
        c[:5000, 2] = np.float32(-0.3)
    elif kind == "slab":  # 6000 distinct depths 16 ulps apart
        d = (np.float32(3.7).view(np.uint32) + 16 * np.arange(6000, dtype=np.uint32)).view(np.float32)
        c[:6000, 2] = (d.astype(np.float64) - 4.0).astype(np.float32)
    elif kind == "all_plane":  # every Gaussian at one depth: one key for the whole sort
        c[:, 2] = np.float32(0.25)
    perm = rng.permutation(n)
    return scenes.GaussianSet(c[perm], s.log_scales[perm], s.rotations[perm], s.opacity_logits[perm], s.sh[perm],
                              s.active_sh_degree)


def test_depth_order_on_skewed_scenes(oracle):
    cam = scenes.front_camera(640, 480)
    for step, (kind, n) in enumerate([("uniform", 150_000), ("plane", 120_000), ("uniform", 120_000),
                                      ("slab", 160_000), ("all_plane", 60_000), ("plane", 90_000),
                                      ("slab", 90_000), ("uniform", 200_000)]):
        s = _scene(n, step, kind)
        R.render(s, cam)
        fw = R.forward_debug()
        po = oracle.project(s, cam)
        assert fw["n_survivors"] == po["n_survivors"], kind
        assert_bitwise(fw["order"], po["order"], f"{kind} (view {step}) depth order")
