"""Known-answer tests of the reference's own suite (test_rasterizer.cpp, test_gradients.cpp,
test_optimizer.cpp) restated on the CPU oracle, in both exp modes."""
import numpy as np
import pytest

from helpers import exact_cfg
from paper_2411_12788_b200 import scenes
from paper_2411_12788_b200.capi import AdamConfig, RasterConfig

MODES = ["B", "A"]


@pytest.fixture(params=MODES)
def lib(request):
    from oracle_lib import OracleLib
    return OracleLib("oracle", request.param)


def test_empty_set_renders_background(lib):  # test_rasterizer.cpp:148-163
    cam = scenes.front_camera(16, 16)
    r = lib.render(scenes.GaussianSet.empty(0), cam, bg=(0.25, 0.5, 0.75))
    assert np.all(r["color"][..., 0] == 0.25) and np.all(r["color"][..., 1] == 0.5)
    assert np.all(r["alpha"] == 0) and np.all(r["depth"] == 0) and np.all(r["max_contributor"] == -1)


def test_single_gaussian_alpha_and_cap(lib):  # test_rasterizer.cpp:165-203
    cam = scenes.front_camera(64, 64, 4.0)
    s = scenes.GaussianSet.empty(1)
    off = 4.0 * (31.5 - cam.cx) / cam.fx
    s.centers[0] = (-off, -off, 0.0)
    s.log_scales[0] = np.log(0.2)
    s.opacity_logits[0] = np.log(4.0)
    s.sh[0, :3] = (np.array([0.9, 0.1, 0.1]) - 0.5) / 0.28209479177387814
    s.active_sh_degree = 0
    r = lib.render(s, cam, bg=(0.0, 0.0, 1.0))
    assert abs(r["alpha"][31, 31] - 0.8) < 1e-6
    assert abs(r["color"][31, 31, 0] - 0.72) < 1e-6 and abs(r["color"][31, 31, 2] - 0.28) < 1e-6
    assert r["max_contributor"][31, 31] == 0
    s.opacity_logits[0] = 12.0
    assert abs(lib.render(s, cam, bg=(0, 0, 1))["alpha"][31, 31] - 0.99) < 1e-6
    assert lib.render(s, cam, exact_cfg())["alpha"][31, 31] > 0.9999


def test_occlusion_pair_importance(lib):  # test_rasterizer.cpp:335-358
    cam = scenes.front_camera(33, 33, 4.0)
    s = scenes.GaussianSet.empty(2)
    s.centers[0], s.centers[1] = (0, 0, 1), (0, 0, -1)
    s.log_scales[:] = np.log(0.25)
    s.opacity_logits[:] = np.log(1.5)
    s.sh[:, 0] = 0.3
    r = lib.render(s, cam, exact_cfg())
    assert abs(r["max_weight"][1] - 0.6) < 1e-6 and abs(r["max_weight"][0] - 0.24) < 1e-6
    assert r["importance"][1] > r["importance"][0]
    assert r["max_pixel_count"][1] > 0 and r["max_pixel_count"][0] == 0


def test_weights_plus_transmittance_is_one(lib):  # test_rasterizer.cpp:123-146
    s = scenes.make_gaussians(8, seed=22, log_scale_mean=np.log(0.2))
    cam = scenes.fov_camera(24, 24, 60.0, (0.0, 0.0, -3.0))
    r = lib.render(s, cam, exact_cfg())
    assert np.allclose(r["alpha"] + r["transmittance"], 1.0, atol=1e-6)
    assert abs(r["importance"].sum(dtype=np.float64) - r["alpha"].sum(dtype=np.float64)) < 1e-3


def test_depth_image_and_near_plane(lib):  # test_rasterizer.cpp:244-261, 306-315
    cam = scenes.front_camera(32, 32, 4.0)
    s = scenes.GaussianSet.empty(2)
    s.log_scales[0] = np.log(0.3)
    s.opacity_logits[0] = 2.0
    s.sh[0, :3] = 0.5
    s.centers[1] = (0, 0, -5)  # behind the camera
    r = lib.render(s, cam)
    assert r["max_contributor"][15, 15] == 0 and abs(r["depth"][15, 15] - 4.0) < 4e-2
    p = lib.project(s, cam)
    assert p["n_survivors"] == 1 and p["order"][0] == 0


def test_zero_gradient_cases(lib):  # test_gradients.cpp:125-146
    cam = scenes.front_camera(16, 16, 4.0)
    s = scenes.GaussianSet.empty(1)
    s.centers[0] = (0, 0, -50)
    g = lib.render_backward(s, cam, np.ones((16, 16, 3), np.float32))
    assert np.all(g["d_centers"] == 0) and g["grad2d_count"][0] == 0
    s.centers[0] = (0, 0, 0)
    s.opacity_logits[0] = 1.0
    g = lib.render_backward(s, cam, np.zeros((16, 16, 3), np.float32))
    assert np.all(g["d_centers"] == 0) and g["d_sh"][0, 0] == 0


def test_backward_linear_in_upstream(lib):  # test_gradients.cpp:148-171
    s = scenes.make_gaussians(4, seed=33, log_scale_mean=np.log(0.2), sh_degree=2)
    cam = scenes.fov_camera(24, 24, 60.0, (0.0, 0.0, -3.0))
    rng = np.random.default_rng(0)
    d1 = rng.uniform(-1, 1, (24, 24, 3)).astype(np.float32)
    d2 = rng.uniform(-1, 1, (24, 24, 3)).astype(np.float32)
    g1, g2 = lib.render_backward(s, cam, d1), lib.render_backward(s, cam, d2)
    gm = lib.render_backward(s, cam, (2 * d1 - 0.5 * d2).astype(np.float32))
    for k in ("d_centers", "d_opacity_logits"):
        want = 2 * g1[k].astype(np.float64) - 0.5 * g2[k]
        assert np.allclose(gm[k], want, rtol=1e-4, atol=1e-6 * np.abs(want).max())


def test_adam_first_step_and_noop(lib):  # test_optimizer.cpp:107-159
    cfg = AdamConfig(scene_extent=2.0)
    s = scenes.GaussianSet.empty(1)
    z = lambda *sh: np.zeros(sh, np.float32)  # noqa: E731
    g = dict(d_centers=np.array([[1, -1, 0.5]], np.float32), d_log_scales=np.array([[-2, 0, 0]], np.float32),
             d_rotations=z(1, 4), d_opacity_logits=np.array([3.0], np.float32), d_sh=z(1, 48))
    g["d_sh"][0, 0], g["d_sh"][0, 5] = 1.0, -1.0
    out, _, _, t = lib.adam_step(s, g, z(59), z(59), cfg, 0)
    lr_pos = 1.6e-4 * 2.0
    assert np.allclose(out.centers[0], [-lr_pos, lr_pos, -lr_pos], rtol=1e-5)
    assert abs(out.log_scales[0, 0] - cfg.lr_scale) < 1e-8 and out.log_scales[0, 1] == 0
    assert abs(out.opacity_logits[0] + cfg.lr_opacity) < 1e-7
    assert abs(out.sh[0, 0] + cfg.lr_sh_dc) < 1e-8 and abs(out.sh[0, 5] - cfg.lr_sh_rest) < 1e-9 and t == 1
    s2 = scenes.make_gaussians(3, seed=50)
    zero = {k: np.zeros_like(v) for k, v in g.items()}
    zero = dict(d_centers=z(3, 3), d_log_scales=z(3, 3), d_rotations=z(3, 4), d_opacity_logits=z(3), d_sh=z(3, 48))
    o2, _, _, _ = lib.adam_step(s2, zero, z(177), z(177), AdamConfig(), 0, group_mask=1 | 2 | 8 | 16)
    for k in ("centers", "log_scales", "opacity_logits", "sh"):
        assert np.array_equal(getattr(o2, k), getattr(s2, k))
