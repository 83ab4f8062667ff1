"""CUDA path vs the CPU oracle (mode B: shared splat_expf), through the C-ABI.

Bit-exact: survivor set, per-Gaussian rects / depth / 2D params / colour, per-tile lists and
ranges, forward images (colour, alpha, depth, transmittance), argmax, max_weight, argmax counts,
Adam, unprojected points and pixel indices.  Tolerance: importance sums and gradients (1e-4 rel).
"""
import numpy as np
import pytest

from helpers import assert_bitwise, assert_grads_close, cfg0_scene, exact_cfg, rel_err, small_scene
from paper_2411_12788_b200 import rasterizer as R
from paper_2411_12788_b200 import scenes
from paper_2411_12788_b200.capi import AdamConfig, RasterConfig

pytestmark = pytest.mark.gpu


def _render_both(oracle, s, cam, cfg=None, mask=None, bg=(0.0, 0.0, 0.0)):
    cfg = cfg or RasterConfig()
    out, rep = R.render(s, cam, cfg, mask=mask, background=bg, report=True)
    want = oracle.render(s, cam, cfg, mask=mask, bg=bg)
    return out, rep, want


def _check_render(out, rep, want, what):
    for k in ("color", "alpha", "depth", "transmittance", "max_contributor"):
        assert_bitwise(getattr(out, k), want[k], f"{what} {k}")
    assert_bitwise(rep.max_weight, want["max_weight"], f"{what} max_weight")
    assert_bitwise(rep.max_pixel_count, want["max_pixel_count"], f"{what} max_pixel_count")
    e = rel_err(rep.importance, want["importance"], floor_frac=1e-6)
    assert e <= 1e-4, f"{what} importance rel err {e:.3e}"


def test_config0_projection_and_tiles_bit_exact(oracle):
    s, cam = cfg0_scene()
    R.render(s, cam)
    dbg = R.project_debug(s.n)
    fw = R.forward_debug()
    po = oracle.project(s, cam)
    surv = np.zeros(s.n, bool)
    surv[po["order"]] = True
    assert_bitwise(dbg["survivor"], surv, "survivor set")
    assert fw["n_survivors"] == po["n_survivors"]
    assert_bitwise(fw["order"], po["order"], "depth order")
    for k in ("rect", "depth", "mean2d", "conic", "color", "opacity"):
        assert_bitwise(dbg[k][surv], po[k][surv], k)
    to = oracle.tiles(s, cam)
    assert fw["n_pairs"] == to["n_pairs"]
    assert_bitwise(fw["ranges"], to["ranges"], "tile ranges")
    assert_bitwise(fw["gaussian"], to["gaussian"], "per-tile lists")
    # sort keys (tile << 32 | float bits of depth) are then identical by construction; check order
    depth_bits = dbg["depth"].view(np.uint32).astype(np.uint64)
    keys = (fw["key_tile"].astype(np.uint64) << np.uint64(32)) | depth_bits[fw["gaussian"]]
    assert np.all(np.diff(keys.astype(np.int64)) >= 0), "sorted keys not monotone"


def test_config0_render_bit_exact(oracle):
    s, cam = cfg0_scene()
    out, rep, want = _render_both(oracle, s, cam)
    _check_render(out, rep, want, "cfg0")


def test_config0_backward_within_tolerance(oracle):
    s, cam = cfg0_scene()
    target = oracle.render(scenes.perturbed(s), cam)["color"]
    fwd = oracle.render(s, cam)
    _, d_color = oracle.l1_loss(fwd["color"], target)
    got = R.render_backward(s, cam, RasterConfig(), d_color)
    want = oracle.render_backward(s, cam, d_color)
    assert_grads_close(got, want, what="cfg0")
    e = rel_err(got["grad2d_accum"], want["grad2d_accum"])
    assert e <= 1e-4, f"grad2d_accum {e:.3e}"


def test_gradient_accuracy_vs_fp64(oracle, ref):
    """The GPU gradients are as close to the reference's fp64 instantiation (render_backward<double>)
    as the reference's own float path is: ||gpu - ref64|| <= 1.05 ||ref32 - ref64|| + 1e-6 ||ref64||."""
    s, cam = cfg0_scene()
    target = oracle.render(scenes.perturbed(s), cam)["color"]
    _, d_color = oracle.l1_loss(oracle.render(s, cam)["color"], target)
    g32 = oracle.render_backward(s, cam, d_color)
    g64 = ref.render_backward_f64(s, cam, d_color)
    gg = R.render_backward(s, cam, RasterConfig(), d_color)
    for k in g64:
        truth = np.asarray(g64[k], np.float64)
        e_gpu = np.linalg.norm(gg[k] - truth)
        e_ref = np.linalg.norm(g32[k] - truth)
        assert e_gpu <= 1.05 * e_ref + 1e-6 * np.linalg.norm(truth), f"{k}: gpu {e_gpu:.3e} vs ref32 {e_ref:.3e}"


def test_fused_l1_backward_matches_split(oracle):
    s, cam = cfg0_scene(n=5000, seed=3)
    target = oracle.render(scenes.perturbed(s), cam)["color"]
    want_loss, d_color = oracle.l1_loss(oracle.render(s, cam)["color"], target)
    want = oracle.render_backward(s, cam, d_color)
    import torch
    ctx = R.Context.default()
    ds = R.DeviceGaussians.from_host(s)
    cfg = RasterConfig()
    R.render(ds, cam, cfg, ctx=ctx, want_depth=False)
    grads = R.DeviceGrads(s.n)
    tgt = torch.from_numpy(target).cuda()
    loss = torch.zeros(1, device="cuda")
    import ctypes as C
    from paper_2411_12788_b200.capi import as_fp
    ctx.bind_stream()
    ctx.check(ctx.lib.splat_render_backward_l1(ctx.h, C.byref(ds.struct()), C.byref(cam), C.byref(cfg),
                                               as_fp(tgt.data_ptr()), None, (C.c_float * 3)(0, 0, 0),
                                               C.byref(grads.struct()), 0, as_fp(loss.data_ptr())))
    got = grads.to_host()
    assert_grads_close(got, want, what="fused")
    assert abs(loss.item() - want_loss) <= 1e-5 * abs(want_loss)


@pytest.mark.parametrize("tile", [8, 16, 32, 48, 64])  # 48: non-power-of-two tile division path
def test_tile_sizes(oracle, tile):
    s, cam = small_scene(n=400, w=50, h=38)  # not tile-aligned
    cfg = RasterConfig(tile_size=tile)
    out, rep, want = _render_both(oracle, s, cam, cfg)
    _check_render(out, rep, want, f"tile{tile}")
    fw = R.forward_debug()
    to = oracle.tiles(s, cam, cfg)
    assert_bitwise(fw["ranges"], to["ranges"], "ranges")
    assert_bitwise(fw["gaussian"], to["gaussian"], "lists")
    # tile size does not change the image (test_rasterizer.cpp:105-121)
    base = R.render(s, cam, RasterConfig())
    assert_bitwise(out.color, base.color, "tile invariance")


@pytest.mark.parametrize("deg", [0, 1, 2, 3])
def test_sh_degrees_and_background(oracle, deg):
    s, cam = small_scene(n=500, sh_degree=deg, seed=11 + deg)
    out, rep, want = _render_both(oracle, s, cam, bg=(0.25, 0.5, 0.75))
    _check_render(out, rep, want, f"deg{deg}")
    d_color = np.random.default_rng(deg).uniform(-1, 1, size=(cam.height, cam.width, 3)).astype(np.float32)
    got = R.render_backward(s, cam, RasterConfig(), d_color, background=(0.25, 0.5, 0.75))
    want_g = oracle.render_backward(s, cam, d_color, bg=(0.25, 0.5, 0.75))
    assert_grads_close(got, want_g, what=f"deg{deg}")


def test_exact_mode(oracle):
    s, cam = small_scene(n=60, w=32, h=32, seed=21)
    out, rep, want = _render_both(oracle, s, cam, exact_cfg())
    _check_render(out, rep, want, "exact")
    d_color = np.random.default_rng(1).uniform(-1, 1, size=(32, 32, 3)).astype(np.float32)
    got = R.render_backward(s, cam, exact_cfg(), d_color)
    want_g = oracle.render_backward(s, cam, d_color, cfg=exact_cfg())
    assert_grads_close(got, want_g, what="exact")


def test_mask_equals_subset(oracle):
    s, cam = small_scene(n=800, seed=31)
    mask = (np.random.default_rng(7).uniform(size=s.n) < 0.6).astype(np.uint8)
    out, rep, want = _render_both(oracle, s, cam, mask=mask)
    _check_render(out, rep, want, "masked")
    sub = R.render(s.select(np.flatnonzero(mask)), cam)
    assert_bitwise(out.color, sub.color, "mask == subset")
    d_color = np.random.default_rng(2).uniform(-1, 1, size=(cam.height, cam.width, 3)).astype(np.float32)
    got = R.render_backward(s, cam, RasterConfig(), d_color, mask=mask)
    want_g = oracle.render_backward(s, cam, d_color, mask=mask)
    assert_grads_close(got, want_g, what="masked")
    assert np.all(got["d_centers"][mask == 0] == 0)
    with pytest.raises(ValueError):
        R.render(s, cam, mask=mask[:10])


def test_empty_and_all_culled(oracle):
    cam = scenes.front_camera(16, 16)
    out = R.render(scenes.GaussianSet.empty(0), cam, background=(0.25, 0.5, 0.75))
    assert np.all(out.color[..., 0] == 0.25) and np.all(out.color[..., 2] == 0.75)
    assert np.all(out.alpha == 0) and np.all(out.depth == 0) and np.all(out.max_contributor == -1)
    s = scenes.GaussianSet.empty(3)
    s.centers[:] = (0.0, 0.0, -50.0)  # behind the camera
    out, rep, want = _render_both(oracle, s, cam)
    _check_render(out, rep, want, "culled")
    d = np.ones((16, 16, 3), np.float32)
    g = R.render_backward(s, cam, RasterConfig(), d)
    assert np.all(g["d_centers"] == 0) and np.all(g["grad2d_count"] == 0)


def test_adam_bit_exact(oracle):
    rng = np.random.default_rng(4)
    s = scenes.make_gaussians(1000, seed=4)
    grads = dict(d_centers=rng.normal(size=(1000, 3)).astype(np.float32),
                 d_log_scales=rng.normal(size=(1000, 3)).astype(np.float32),
                 d_rotations=rng.normal(size=(1000, 4)).astype(np.float32),
                 d_opacity_logits=rng.normal(size=1000).astype(np.float32),
                 d_sh=rng.normal(size=(1000, 48)).astype(np.float32))
    cfg = AdamConfig(scene_extent=3.3)
    ds = R.DeviceGaussians.from_host(s)
    dg = R.DeviceGrads(1000)
    import torch
    for k, v in grads.items():
        getattr(dg, k).copy_(torch.from_numpy(v))
    opt = R.OptimState(cfg, 1000)
    hs, m, v, t = s, np.zeros(59 * 1000, np.float32), np.zeros(59 * 1000, np.float32), 0
    for _ in range(3):
        opt.step(ds, dg)
        hs, m, v, t = oracle.adam_step(hs, grads, m, v, cfg, t)
    got = ds.to_host()
    for k in ("centers", "log_scales", "rotations", "opacity_logits", "sh"):
        assert_bitwise(getattr(got, k), getattr(hs, k), f"adam {k}")
    assert_bitwise(opt.m.cpu().numpy(), m, "adam m")
    assert_bitwise(opt.v.cpu().numpy(), v, "adam v")
    assert opt.step_count() == t == 3


def test_adam_zero_gradients_and_tail(oracle):
    """Zero / negative-zero gradients (the mf == 0 shortcut) and a count that is not a multiple of
    4 (the scalar tail of the 4-wide kernel), over steps with and without gradients."""
    n = 1003
    rng = np.random.default_rng(6)
    s = scenes.make_gaussians(n, seed=6)
    shapes = dict(d_centers=(n, 3), d_log_scales=(n, 3), d_rotations=(n, 4), d_opacity_logits=(n,), d_sh=(n, 48))
    import torch
    ds = R.DeviceGaussians.from_host(s)
    dg = R.DeviceGrads(n)
    opt = R.OptimState(AdamConfig(scene_extent=2.0), n)
    hs, m, v, t = s, np.zeros(59 * n, np.float32), np.zeros(59 * n, np.float32), 0
    for step in range(4):
        grads = {}
        for k, shp in shapes.items():
            g = rng.normal(size=shp).astype(np.float32)
            g[rng.random(shp) < 0.5] = 0.0
            g[rng.random(shp) < 0.1] = -0.0
            if step == 2:
                g[:] = 0.0
            grads[k] = g
            getattr(dg, k).copy_(torch.from_numpy(g))
        opt.step(ds, dg)
        hs, m, v, t = oracle.adam_step(hs, grads, m, v, AdamConfig(scene_extent=2.0), t)
    got = ds.to_host()
    for k in ("centers", "log_scales", "rotations", "opacity_logits", "sh"):
        assert_bitwise(getattr(got, k), getattr(hs, k), f"adam {k}")
    assert_bitwise(opt.m.cpu().numpy(), m, "adam m")
    assert_bitwise(opt.v.cpu().numpy(), v, "adam v")


def test_adam_means_only(oracle):
    rng = np.random.default_rng(5)
    s = scenes.make_gaussians(200, seed=5)
    grads = dict(d_centers=rng.normal(size=(200, 3)).astype(np.float32),
                 d_log_scales=np.zeros((200, 3), np.float32), d_rotations=np.zeros((200, 4), np.float32),
                 d_opacity_logits=np.zeros(200, np.float32), d_sh=np.zeros((200, 48), np.float32))
    ds = R.DeviceGaussians.from_host(s)
    dg = R.DeviceGrads(200)
    import torch
    dg.d_centers.copy_(torch.from_numpy(grads["d_centers"]))
    opt = R.OptimState(AdamConfig(), 200)
    opt.step(ds, dg, group_mask=1)
    hs, _, _, _ = oracle.adam_step(s, grads, np.zeros(59 * 200, np.float32), np.zeros(59 * 200, np.float32),
                                   AdamConfig(), 0, group_mask=1)
    got = ds.to_host()
    assert_bitwise(got.centers, hs.centers, "means")
    assert_bitwise(got.rotations, s.rotations, "rotations untouched")


@pytest.mark.parametrize("rule,stride", [(0, 1), (1, 4)])
def test_unproject(oracle, rule, stride):
    s, cam = cfg0_scene(n=8000, seed=9)
    out = R.render(s, cam)
    want = oracle.render(s, cam)
    pts, pix, k = R.unproject_depth(cam, rule=rule, alpha_threshold=0.5, view_index=3, stride=stride, seed=1)
    wp, wx = oracle.unproject(cam, want["max_contributor"], want["alpha"], want["depth"], rule=rule,
                              alpha_threshold=0.5, view_index=3, stride=stride, seed=1)
    assert k == wx.size
    assert_bitwise(pix.cpu().numpy(), wx, "pixel indices")
    assert_bitwise(pts.cpu().numpy(), wp, "points")


def test_kat_single_gaussian_alpha(oracle):
    """test_rasterizer.cpp:165-203: alpha = 0.8 at the pixel centre; 0.99 cap."""
    cam = scenes.front_camera(64, 64, 4.0)
    s = scenes.GaussianSet.empty(1)
    off = 4.0 * (31.5 - cam.cx) / cam.fx
    s.centers[0] = (-off, -off, 0.0)
    s.log_scales[0] = np.log(0.2)
    s.opacity_logits[0] = np.log(4.0)
    red = np.array([0.9, 0.1, 0.1])
    s.sh[0, :3] = (red - 0.5) / 0.28209479177387814
    s.active_sh_degree = 0
    out = R.render(s, cam, background=(0.0, 0.0, 1.0))
    assert abs(out.alpha[31, 31] - 0.8) < 1e-6
    assert abs(out.color[31, 31, 0] - 0.72) < 1e-6 and abs(out.color[31, 31, 2] - 0.28) < 1e-6
    assert out.max_contributor[31, 31] == 0
    s.opacity_logits[0] = 12.0
    capped = R.render(s, cam, background=(0.0, 0.0, 1.0))
    assert abs(capped.alpha[31, 31] - 0.99) < 1e-6
    assert R.render(s, cam, exact_cfg()).alpha[31, 31] > 0.9999


def test_kat_occlusion_pair():
    """test_rasterizer.cpp:335-358: max_weight = {0.24, 0.6}; only the front one is argmax."""
    cam = scenes.front_camera(33, 33, 4.0)
    s = scenes.GaussianSet.empty(2)
    s.centers[0] = (0, 0, 1)
    s.centers[1] = (0, 0, -1)
    s.log_scales[:] = np.log(0.25)
    s.opacity_logits[:] = np.log(1.5)
    s.sh[:, 0] = 0.3
    rep = R.accumulate_importance(s, cam, exact_cfg())
    assert abs(rep.max_weight[1] - 0.6) < 1e-6 and abs(rep.max_weight[0] - 0.24) < 1e-6
    assert rep.importance[1] > rep.importance[0]
    assert rep.is_max_contributor(1) and not rep.is_max_contributor(0)


def test_depth_kat():
    """test_rasterizer.cpp:244-261: central pixel depth ~ camera distance."""
    cam = scenes.front_camera(32, 32, 4.0)
    s = scenes.GaussianSet.empty(1)
    s.log_scales[0] = np.log(0.3)
    s.opacity_logits[0] = 2.0
    s.sh[0, :3] = 0.5
    out = R.render(s, cam)
    assert out.max_contributor[15, 15] == 0
    assert abs(out.depth[15, 15] - 4.0) < 4e-2


def test_invalid_arguments():
    s, cam = small_scene(n=10)
    bad = scenes.fov_camera(16, 16, 60.0, (0, 0, -3))
    bad.rotation[0] = 2.0
    with pytest.raises(ValueError):
        R.render(s, bad)
    with pytest.raises(ValueError):
        R.render_backward(s, cam, RasterConfig(), np.zeros((3, 3, 3), np.float32))
    with pytest.raises(ValueError):
        R.render(s, cam, RasterConfig(tile_size=12))


@pytest.mark.parametrize("tile", [16, 32])
def test_traversal_counts_equal_oracle(oracle, tile):
    """V (list visits) and C (commits) of traverse_pixel, counted on the GPU over the forward's
    lists, equal the oracle's counts exactly (SURVEY.md §8d workload symbols)."""
    s, cam = cfg0_scene()
    cfg = RasterConfig()
    cfg.tile_size = tile
    R.render(s, cam, cfg)
    v, c = R.traversal_counts()
    want = oracle.render(s, cam, cfg, report=False)
    assert (v, c) == (want["visits"], want["commits"])
    assert 0 < c < v


@pytest.mark.parametrize("exact", [False, True])
def test_project_records_equal_oracle(oracle, exact):
    """splat_project (project<float>): survivors in (depth, index) order with their rects, radii,
    depths, 2D means, conics, colours and opacities bit-exact; cov2d is the matrix the conic was
    inverted from (the reference's inv_det multiply reproduces the conic bit for bit)."""
    s, cam = cfg0_scene()
    cfg = exact_cfg() if exact else RasterConfig()
    got = R.project(s, cam, cfg)
    want = oracle.project(s, cam, cfg)
    order = want["order"][: want["n_survivors"]]
    assert_bitwise(got["index"], order, "survivor order")
    rect = np.stack([got["x0"], got["x1"], got["y0"], got["y1"]], 1)
    assert_bitwise(rect, want["rect"][order], "rects")
    assert_bitwise(got["radius"], want["radius"][order], "radius")
    assert_bitwise(got["depth_mean"], want["depth"][order], "depth")
    assert_bitwise(got["mean2d"], want["mean2d"][order], "mean2d")
    assert_bitwise(got["conic"], want["conic"][order], "conic")
    assert_bitwise(got["color"], want["color"][order], "colour")
    assert_bitwise(got["opacity"], want["opacity"][order], "opacity")
    c = got["cov2d"].astype(np.float32)
    det = c[:, 0] * c[:, 2] - c[:, 1] * c[:, 1]
    inv = np.float32(1.0) / det
    assert_bitwise(np.stack([c[:, 2] * inv, -c[:, 1] * inv, c[:, 0] * inv], 1), got["conic"], "conic from cov2d")
    assert_bitwise(got["center_world"], s.centers[order], "centre")
