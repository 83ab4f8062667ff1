"""Depth re-initialisation tail on device (csrc/spatial.cu, densify.depth_reinitialize) vs the
reference build: third-nearest-neighbour distances bit-exact (grid k-NN on device vs the
reference's grid index), and the fresh set bit-exact given the reference's own sample draw."""
import numpy as np
import pytest
import torch

from helpers import assert_bitwise
from paper_2411_12788_b200 import densify as D
from paper_2411_12788_b200 import scenes

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("m", [0, 1, 2, 3, 200, 256, 257, 5000, 300_000])
def test_third_neighbor_distances(ref, m):
    rng = np.random.default_rng(m)
    p = rng.random((m, 3)).astype(np.float32)
    if m > 10:
        p[5] = p[4]
    got = D.third_neighbor_distances(torch.from_numpy(p).cuda()).cpu().numpy()
    assert_bitwise(got, ref.third_neighbor_distances(p), f"nn3 m={m}")


def test_third_neighbor_distances_surface(ref):
    rng = np.random.default_rng(2)
    v = rng.normal(size=(400_000, 3))
    p = (v / np.linalg.norm(v, axis=1, keepdims=True)).astype(np.float32)
    p[:1000, 2] = 0.0  # a flat patch too
    got = D.third_neighbor_distances(torch.from_numpy(p).cuda()).cpu().numpy()
    assert_bitwise(got, ref.third_neighbor_distances(p), "nn3 sphere shell")


def test_depth_reinitialize_matches_reference(oracle, ref):
    s = scenes.make_gaussians(3000, seed=8, log_scale_mean=np.log(0.03))
    cams = [scenes.ring_camera(k, 3, width=48, height=40) for k in range(3)]
    rng = np.random.default_rng(1)
    images = np.stack([rng.random((40, 48, 3)).astype(np.float32) for _ in cams])
    want = ref.depth_reinitialize_views(s, cams, list(images), sample_count=900, seed=5)
    pool = sum(int((oracle.render(s, c)["max_contributor"] >= 0).sum()) for c in cams)
    idx = ref.fisher_yates(5, pool, min(900, pool))
    fed = D.depth_reinitialize(s, cams, torch.from_numpy(images).cuda(), 900,
                               sample=torch.from_numpy(idx).cuda()).to_host()
    # default draw: the library's own std::mt19937 partial Fisher-Yates (splat_pool_sample)
    drawn = D.depth_reinitialize(s, cams, torch.from_numpy(images).cuda(), 900, rng=D.Rng(5)).to_host()
    for fresh, how in ((fed, "fed the reference's draw"), (drawn, "library draw")):
        for a, b, name in zip((fresh.centers, fresh.log_scales, fresh.rotations, fresh.opacity_logits, fresh.sh),
                              want, ("centers", "log_scales", "rotations", "opacity_logits", "sh")):
            assert_bitwise(a, b, f"fresh {name} ({how})")
    # a set that renders nothing: std::runtime_error in the reference (densify.cpp:223-225)
    empty = s.select(np.zeros(0, np.int64))
    with pytest.raises(RuntimeError):
        D.depth_reinitialize(empty, cams[:1], torch.from_numpy(images[:1]).cuda(), 10)
