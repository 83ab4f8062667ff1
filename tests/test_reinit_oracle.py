"""Depth re-initialisation tail on CPU: the C restatement of
third_neighbor_distances (brute force) and of depth_reinitialize's fresh set, pinned bitwise to
the reference's own spatial.cpp (grid index for n > 256) and depth_reinitialize."""
import numpy as np

from paper_2411_12788_b200 import scenes


def test_third_neighbor_distances_pinned(oracle, ref):
    rng = np.random.default_rng(0)
    for m in (0, 1, 2, 3, 4, 100, 256, 257, 3000):
        p = rng.random((m, 3)).astype(np.float32)
        if m > 10:
            p[5] = p[4]  # a duplicate: distance 0 floored at min_dist
        got = oracle.third_neighbor_distances(p)
        want = ref.third_neighbor_distances(p)
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), m
    # surface-like cloud (a sphere shell), as depth points are
    v = rng.normal(size=(4000, 3))
    p = (v / np.linalg.norm(v, axis=1, keepdims=True)).astype(np.float32)
    assert np.array_equal(oracle.third_neighbor_distances(p).view(np.uint32),
                          ref.third_neighbor_distances(p).view(np.uint32))


def test_depth_reinitialize_pinned(oracle, ref):
    s = scenes.make_gaussians(3000, seed=8, log_scale_mean=np.log(0.03))
    cams = [scenes.ring_camera(k, 3, width=48, height=40) for k in range(3)]
    rng = np.random.default_rng(1)
    images = [rng.random((40, 48, 3)).astype(np.float32) for _ in cams]
    want = ref.depth_reinitialize_views(s, cams, images, sample_count=900, seed=5)
    # the pool in the reference's order: per view, raster order, pixels with a max contributor
    pts, cols = [], []
    for k, cam in enumerate(cams):
        r = oracle.render(s, cam)
        p, x = oracle.unproject(cam, r["max_contributor"], r["alpha"], r["depth"], rule=0, alpha_threshold=0.5,
                                view_index=k, stride=1, seed=0)
        pts.append(p)
        cols.append(images[k].reshape(-1, 3)[x])
    pts, cols = np.concatenate(pts), np.concatenate(cols)
    idx = ref.fisher_yates(5, pts.shape[0], min(900, pts.shape[0]))
    got = oracle.reinit_gaussians(pts[idx], cols[idx])
    for a, b, name in zip(got, want, ("centers", "log_scales", "rotations", "opacity_logits", "sh")):
        assert a.shape == b.shape and np.array_equal(a.view(np.uint32), b.view(np.uint32)), name
