"""BASELINE configs 2, 3 and 4 at reduced scale, CUDA path vs the CPU oracle.

cfg 2: depth rendering + unprojection over ring views, alpha > 0.5, seeded stride-4 selection:
       point indices bit-exact, positions bit-exact (tolerance 1e-5 in the spec).
cfg 3: per-view visibility bitmasks (max blend weight > 1e-3) bit-exact, global importance (fp64
       sum over views) within 1e-4, argmax counts exact; culled fwd/bwd vs oracle, and culled vs
       unculled fidelity (MAE < 1/255, test_simplify_visibility.cpp:198-219).
cfg 4: view-parallel training step (batch of views, gradients summed = ParamGrads::add, Adam on
       all parameters) vs the oracle's step.
"""
import numpy as np
import pytest

from helpers import assert_bitwise, assert_grads_close
from paper_2411_12788_b200 import capi, scenes
from paper_2411_12788_b200 import rasterizer as R
from paper_2411_12788_b200.capi import AdamConfig, RasterConfig

pytestmark = pytest.mark.gpu


def _ring(k, count, w=320, h=214):
    return scenes.ring_camera(k, count, width=w, height=h)


def test_config2_depth_unprojection_multi_view(oracle):
    s = scenes.make_gaussians(30_000, seed=2, log_scale_mean=np.log(0.01))
    cams = [_ring(k, 6) for k in range(6)]
    pts, views, pix = R.depth_points(s, cams, rule=capi.DEPTH_RULE_ALPHA, alpha_threshold=0.5, stride=4, seed=7)
    pts, views, pix = pts.cpu().numpy(), views.cpu().numpy(), pix.cpu().numpy()
    want_p, want_v, want_x = [], [], []
    for k, cam in enumerate(cams):
        r = oracle.render(s, cam)
        p, x = oracle.unproject(cam, r["max_contributor"], r["alpha"], r["depth"], rule=1, alpha_threshold=0.5,
                                view_index=k, stride=4, seed=7)
        want_p.append(p)
        want_x.append(x)
        want_v.append(np.full(x.size, k, np.int32))
    assert_bitwise(views, np.concatenate(want_v), "view of each point")
    assert_bitwise(pix, np.concatenate(want_x), "pixel of each point")
    assert_bitwise(pts, np.concatenate(want_p), "points")
    assert pts.shape[0] > 1000


def test_config3_visibility_and_global_importance(oracle):
    s = scenes.make_gaussians(20_000, seed=3)
    cams = [_ring(k, 8) for k in range(8)]
    masks, accum, counts = R.visibility_pass(s, cams, threshold=1e-3)
    masks = masks.cpu().numpy()
    want_acc = np.zeros(s.n)
    want_cnt = np.zeros(s.n, np.int64)
    for k, cam in enumerate(cams):
        r = oracle.render(s, cam)
        assert_bitwise(R.unpack_mask(masks[k], s.n), r["max_weight"] > 1e-3, f"view {k} mask")
        want_acc += r["importance"].astype(np.float64)
        want_cnt += r["max_pixel_count"]
    acc = accum.cpu().numpy()
    assert np.abs(acc - want_acc).max() <= 1e-4 * np.abs(want_acc).max()
    assert np.array_equal(counts.cpu().numpy(), want_cnt)


def test_config3_culled_forward_backward(oracle):
    s = scenes.make_gaussians(20_000, seed=4)
    cam = _ring(0, 8)
    masks, _, _ = R.visibility_pass(s, [cam], threshold=1e-3)
    mask = R.unpack_mask(masks[0].cpu().numpy(), s.n).astype(np.uint8)
    assert 0 < mask.sum() < s.n
    out, rep = R.render(s, cam, mask=mask, report=True)
    want = oracle.render(s, cam, mask=mask)
    for k in ("color", "alpha", "depth", "max_contributor"):
        assert_bitwise(getattr(out, k), want[k], k)
    full = R.render(s, cam)
    assert np.abs(out.color.astype(np.float64) - full.color).mean() < 1.0 / 255
    target = oracle.render(scenes.perturbed(s), cam)["color"]
    _, d_color = oracle.l1_loss(want["color"], target)
    got = R.render_backward(s, cam, RasterConfig(), d_color, mask=mask)
    want_g = oracle.render_backward(s, cam, d_color, mask=mask)
    assert_grads_close(got, want_g, what="culled")


def test_config4_batched_step_all_parameters(oracle):
    import torch
    from paper_2411_12788_b200.trainer import ViewTrainer, pack_grads, unpack_grads
    s = scenes.make_gaussians(20_000, seed=5)
    t_set = scenes.perturbed(s)
    cams = [_ring(k, 16) for k in range(16)]
    targets = [oracle.render(t_set, c)["color"] for c in cams]
    adam = AdamConfig(scene_extent=3.3)
    ds = R.DeviceGaussians.from_host(s)
    tr = ViewTrainer(ds, adam, group_mask=capi.GROUP_ALL)
    hs, m, v, t = s, np.zeros(59 * s.n, np.float32), np.zeros(59 * s.n, np.float32), 0
    for step in range(2):
        idx = [4 * step + j for j in range(4)]
        loss = tr.step([cams[i] for i in idx], [torch.from_numpy(targets[i]).cuda() for i in idx]).cpu().numpy()
        flat = np.zeros(59 * s.n, np.float32)
        want_loss = []
        for i in idx:
            r = oracle.render(hs, cams[i])
            lo, dc = oracle.l1_loss(r["color"], targets[i])
            want_loss.append(lo)
            flat += pack_grads(oracle.render_backward(hs, cams[i], dc))
        assert np.allclose(loss, want_loss, rtol=1e-5)
        g_host = tr.grads.to_host()
        assert_grads_close(g_host, unpack_grads(flat, s.n), what=f"step {step} summed grads")
        hs, m, v, t = oracle.adam_step(hs, unpack_grads(flat, s.n), m, v, adam, t)
    got = ds.to_host()
    for k in ("centers", "log_scales", "rotations", "opacity_logits", "sh"):
        a, b = getattr(got, k).astype(np.float64), getattr(hs, k)
        # Adam normalises each update by sqrt(v) (first steps ~ lr * sign(g)): elements whose
        # gradient is pure cancellation noise can differ by up to 2 lr per step; everything else
        # must agree to 1e-3 lr.  Bound both.
        lr = {"centers": 1.6e-4 * 3.3, "log_scales": 5e-3, "rotations": 1e-3, "opacity_logits": 5e-2, "sh": 2.5e-3}[k]
        d = np.abs(a - b)
        assert d.max() <= 4 * lr + 1e-6, k
        assert (d > 1e-3 * lr).mean() < 1e-3, f"{k}: {(d > 1e-3 * lr).mean():.2e} of elements off"


def test_view_parallel_passes_single_rank_match(oracle):
    """multiview.visibility_pass_views / depth_points_views (the NCCL view-parallel passes) on one
    rank equal the plain passes; the max blend weight over views equals the oracle's."""
    from paper_2411_12788_b200 import multiview as MV
    s = scenes.make_gaussians(20_000, seed=4)
    cams = [_ring(k, 4) for k in range(4)]
    masks, accum, counts, mx = MV.visibility_pass_views(s, cams)
    m0, a0, c0 = R.visibility_pass(s, cams)
    assert_bitwise(masks.cpu().numpy(), m0.cpu().numpy(), "view-parallel masks")
    # per-view importance is an atomic float sum (order varies run to run): tolerance, not bits
    assert np.allclose(accum.cpu().numpy(), a0.cpu().numpy(), rtol=1e-5, atol=1e-9), "view-parallel accum"
    assert_bitwise(counts.cpu().numpy(), c0.cpu().numpy(), "view-parallel counts")
    want = np.max(np.stack([oracle.render(s, c)["max_weight"] for c in cams]), 0)
    assert_bitwise(mx.cpu().numpy(), want, "max blend weight over views")
    p, v, x = MV.depth_points_views(s, cams, stride=3, seed=1)
    p0, v0, x0 = R.depth_points(s, cams, stride=3, seed=1)
    for a, b, what in ((p, p0, "points"), (v, v0, "views"), (x, x0, "pixels")):
        assert_bitwise(a.cpu().numpy(), b.cpu().numpy(), f"view-parallel {what}")


def test_native_passes_reject_a_bad_view_and_recover(oracle):
    """A camera the validation rejects in the middle of a multi-view call: the call raises with the
    reference's exception type, the helper contexts' queued work is joined, and the next call on
    the same context returns the per-view loop's results."""
    from paper_2411_12788_b200 import multiview as MV
    s = scenes.make_gaussians(20_000, seed=9)
    cams = [_ring(k, 4) for k in range(4)]
    bad = list(cams)
    bad[2] = scenes.fov_camera(0, 16, 60.0, (0.0, 0.0, -3.0))  # zero width
    with pytest.raises(ValueError):  # std::invalid_argument
        MV.depth_points_views(s, bad, stride=3, seed=1)
    with pytest.raises(ValueError):
        MV.visibility_pass_views(s, bad)
    p, v, x = MV.depth_points_views(s, cams, stride=3, seed=1)
    p0, v0, x0 = R.depth_points(s, cams, stride=3, seed=1)
    for a, b, what in ((p, p0, "points"), (v, v0, "views"), (x, x0, "pixels")):
        assert_bitwise(a.cpu().numpy(), b.cpu().numpy(), f"after an error: {what}")
    masks, _, counts, _ = MV.visibility_pass_views(s, cams)
    m0, _, c0 = R.visibility_pass(s, cams)
    assert_bitwise(masks.cpu().numpy(), m0.cpu().numpy(), "after an error: masks")
    assert_bitwise(counts.cpu().numpy(), c0.cpu().numpy(), "after an error: counts")
