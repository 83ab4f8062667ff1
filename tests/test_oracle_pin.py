"""Pins the C restatement (oracle/splat_oracle.c) to the reference's own sources compiled in place
(oracle/_ref): bit-identical on every output, on scenes beyond the committed fixtures."""
import numpy as np
import pytest

from helpers import assert_bitwise, exact_cfg, small_scene
from paper_2411_12788_b200 import scenes
from paper_2411_12788_b200.capi import AdamConfig, RasterConfig

GRADS = ("d_centers", "d_log_scales", "d_rotations", "d_opacity_logits", "d_sh", "grad2d_accum", "grad2d_count")


def _pin_all(oracle, ref, s, cam, cfg, mask=None, bg=(0.0, 0.0, 0.0), seed=0):
    a = oracle.render(s, cam, cfg, mask=mask, bg=bg)
    b = ref.render(s, cam, cfg, mask=mask, bg=bg)
    for k in ("color", "alpha", "depth", "transmittance", "max_contributor", "importance", "max_weight",
              "max_pixel_count"):
        assert_bitwise(a[k], b[k], k)
    ta, tb = oracle.tiles(s, cam, cfg, mask=mask), ref.tiles(s, cam, cfg, mask=mask)
    assert_bitwise(ta["ranges"], tb["ranges"], "ranges")
    assert_bitwise(ta["gaussian"], tb["gaussian"], "lists")
    pa, pb = oracle.project(s, cam, cfg, mask=mask), ref.project(s, cam, cfg, mask=mask)
    for k in ("order", "rect", "depth", "mean2d", "conic", "color", "opacity"):
        assert_bitwise(pa[k], pb[k], k)
    d_color = np.random.default_rng(seed).uniform(-1, 1, size=(cam.height, cam.width, 3)).astype(np.float32)
    ga = oracle.render_backward(s, cam, d_color, cfg, mask=mask, bg=bg)
    gb = ref.render_backward(s, cam, d_color, cfg, mask=mask, bg=bg)
    for k in GRADS:
        assert_bitwise(ga[k], gb[k], k)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_pin_random_scenes(oracle, ref, seed):
    s, cam = small_scene(n=700, seed=40 + seed, w=80, h=60)
    _pin_all(oracle, ref, s, cam, RasterConfig(), seed=seed)


def test_pin_config0(oracle, ref):
    s = scenes.make_gaussians(20_000, seed=0)
    cam = scenes.config0_camera()
    _pin_all(oracle, ref, s, cam, RasterConfig())


@pytest.mark.parametrize("tile", [8, 16, 32, 64])
def test_pin_tile_sizes(oracle, ref, tile):
    s, cam = small_scene(n=300, seed=50, w=50, h=38)
    _pin_all(oracle, ref, s, cam, RasterConfig(tile_size=tile), bg=(0.1, 0.2, 0.3))


def test_pin_exact_mode_mask_degrees(oracle, ref):
    s, cam = small_scene(n=50, seed=51, w=32, h=32, sh_degree=1)
    _pin_all(oracle, ref, s, cam, exact_cfg())
    s, cam = small_scene(n=400, seed=52, sh_degree=2)
    mask = (np.random.default_rng(9).uniform(size=s.n) < 0.5).astype(np.uint8)
    _pin_all(oracle, ref, s, cam, RasterConfig(), mask=mask)


def test_pin_mode_a(ref):
    """The two exp modes of the C restatement and of the reference agree pairwise."""
    from oracle_lib import OracleLib
    oa = OracleLib("oracle", "A")
    ra = OracleLib("ref", "A")
    s, cam = small_scene(n=500, seed=53)
    a, b = oa.render(s, cam), ra.render(s, cam)
    for k in ("color", "alpha", "max_contributor"):
        assert_bitwise(a[k], b[k], k)


def test_pin_adam(oracle, ref):
    rng = np.random.default_rng(3)
    s = scenes.make_gaussians(300, seed=3)
    grads = dict(d_centers=rng.normal(size=(300, 3)).astype(np.float32),
                 d_log_scales=rng.normal(size=(300, 3)).astype(np.float32),
                 d_rotations=rng.normal(size=(300, 4)).astype(np.float32),
                 d_opacity_logits=rng.normal(size=300).astype(np.float32),
                 d_sh=rng.normal(size=(300, 48)).astype(np.float32))
    cfg = AdamConfig(scene_extent=3.3)
    hs, m, v, t = s, np.zeros(59 * 300, np.float32), np.zeros(59 * 300, np.float32), 0
    for _ in range(4):
        hs, m, v, t = oracle.adam_step(hs, grads, m, v, cfg, t)
    want = ref.adam_steps(s, grads, cfg, 4)
    for k in ("centers", "log_scales", "rotations", "opacity_logits", "sh"):
        assert_bitwise(getattr(hs, k), getattr(want, k), k)
    for step in (0, 1, 9000, 18000, 50000):
        assert oracle.lr_at(cfg, step) == ref.lr_at(cfg, step)


def test_pin_l1(oracle, ref):
    rng = np.random.default_rng(4)
    a = rng.uniform(size=3000).astype(np.float32)
    b = rng.uniform(size=3000).astype(np.float32)
    b[::7] = a[::7]  # exact ties give a zero gradient
    la, ga = oracle.l1_loss(a, b)
    lb, gb = ref.l1_loss(a, b)
    assert la == lb
    assert_bitwise(ga, gb, "l1 grad")
    assert np.all(ga[::7] == 0)


def test_pin_unprojection_against_depth_reinitialize(oracle, ref):
    """densify.cpp:207-222: with sample_count >= pool, depth_reinitialize's fresh centres are a
    permutation of every unprojected argmax pixel."""
    s, cam = small_scene(n=600, seed=54, w=48, h=40)
    r = oracle.render(s, cam)
    pts, pix = oracle.unproject(cam, r["max_contributor"], r["alpha"], r["depth"], rule=0, stride=1)
    img = np.random.default_rng(0).uniform(size=(cam.height, cam.width, 3)).astype(np.float32)
    fresh = ref.depth_reinitialize(s, cam, img, sample_count=cam.width * cam.height, seed=1)
    assert fresh.shape == pts.shape
    key = lambda a: a[np.lexsort(a.T[::-1])]  # noqa: E731
    assert_bitwise(key(fresh), key(pts), "unprojected points")


def test_pin_global_importance(oracle, ref):
    """simplify.cpp:13-34: fp64 sum over views of importance and of argmax counts."""
    s = scenes.make_gaussians(3000, seed=55)
    cams = [scenes.ring_camera(k, 4, width=96, height=64) for k in range(4)]
    acc, cnt = ref.global_importance(s, cams)
    want_acc = np.zeros(s.n)
    want_cnt = np.zeros(s.n, np.int64)
    for c in cams:
        r = oracle.render(s, c)
        want_acc += r["importance"].astype(np.float64)
        want_cnt += r["max_pixel_count"]
    assert_bitwise(acc, want_acc, "accum_weight")
    assert np.array_equal(cnt, want_cnt)
