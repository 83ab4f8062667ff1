"""Device state that persists between calls (SURVEY.md §8b boundary, capi.cu): the survivor /
pair counters, the persistent kernels' work queues, the depth sort's histogram, the binning scan's
look-back words and the alternating touched-list counters are all re-zeroed by the kernels that
consume them instead of by memsets.  Interleave every entry point over changing set sizes, image
shapes and tile sizes (buffers regrow, the sort changes tiles per CTA) and check each result
against the oracle, so a counter left dirty by one call shows up in the next."""
import numpy as np
import pytest

from helpers import assert_bitwise, assert_grads_close
from paper_2411_12788_b200 import capi, scenes
from paper_2411_12788_b200 import rasterizer as R
from paper_2411_12788_b200.capi import AdamConfig, RasterConfig
from paper_2411_12788_b200.trainer import ViewTrainer

pytestmark = pytest.mark.gpu


def _forward_matches(oracle, s, cam, cfg, what):
    out = R.render(s, cam, cfg)
    want = oracle.render(s, cam, cfg)
    for k in ("color", "alpha", "transmittance", "max_contributor"):
        assert_bitwise(getattr(out, k), want[k], f"{what} {k}")
    return want


@pytest.mark.parametrize("seed", [0, 1])
def test_interleaved_calls_over_changing_sizes(oracle, seed):
    rng = np.random.default_rng(seed)
    plan = [(12_000, 160, 120, 16), (40_000, 256, 192, 16), (3_000, 96, 64, 8), (25_000, 200, 150, 32),
            (0, 64, 64, 16), (30_000, 256, 256, 16)]
    for i, (n, w, h, ts) in enumerate(plan):
        cfg = RasterConfig(tile_size=ts)
        cam = scenes.fov_camera(w, h, 60.0, (0.3 * float(rng.normal()), 0.2, -3.0))
        if n == 0:  # an empty set between populated ones
            out = R.render(scenes.GaussianSet.empty(0), cam, cfg)
            assert np.all(out.alpha == 0)
            continue
        s = scenes.make_gaussians(n, seed=seed * 10 + i)
        want = _forward_matches(oracle, s, cam, cfg, f"step {i} render")
        target = oracle.render(scenes.perturbed(s), cam, cfg)["color"]
        _, d_color = oracle.l1_loss(want["color"], target)
        got = R.render_backward(s, cam, cfg, d_color)
        ref = oracle.render_backward(s, cam, d_color, cfg)
        assert_grads_close(got, ref, what=f"step {i} backward")
        # the same forward again right after a backward: queues and counters are back at zero
        _forward_matches(oracle, s, cam, cfg, f"step {i} render again")


def test_training_steps_then_render(oracle):
    """Native training steps (host and device targets), then a plain render of the updated set:
    equal to the oracle's render of the same parameters."""
    import torch
    s = scenes.make_gaussians(15_000, seed=3)
    cams = [scenes.fov_camera(192, 128, 60.0, (0.2 * k, 0.1, -3.0)) for k in range(3)]
    targets = [oracle.render(scenes.perturbed(s), c)["color"] for c in cams]
    ds = R.DeviceGaussians.from_host(s)
    tr = ViewTrainer(ds, AdamConfig(), group_mask=capi.GROUP_ALL)
    for k in range(3):
        tr.step_host([cams[k]], [np.ascontiguousarray(targets[k])])
        tr.step([cams[(k + 1) % 3]], [torch.from_numpy(targets[(k + 1) % 3]).cuda()])
    torch.cuda.synchronize()
    updated = ds.to_host()
    _forward_matches(oracle, updated, cams[0], RasterConfig(), "after training")


@pytest.mark.parametrize("lam", [0.0, 0.2])
def test_overlapped_multi_view_step_host_targets(oracle, lam):
    """A 10-view step with host targets: views alternate between the context and its twin (own
    stream, chains ordered by events) and the 8 target staging slots are refilled once a view's
    backward ran.  The per-view losses and the summed gradients equal the oracle's."""
    from paper_2411_12788_b200.trainer import ViewTrainer, pack_grads, unpack_grads
    s = scenes.make_gaussians(8_000, seed=11)
    cams = [scenes.ring_camera(k, 10, width=96, height=72) for k in range(10)]
    targets = [np.ascontiguousarray(oracle.render(scenes.perturbed(s), c)["color"]) for c in cams]
    ds = R.DeviceGaussians.from_host(s)
    tr = ViewTrainer(ds, AdamConfig(), group_mask=0, lambda_dssim=lam)  # no optimiser step
    loss = tr.step_host(cams, targets)
    flat = np.zeros(59 * s.n, np.float32)
    want = []
    for cam, tgt in zip(cams, targets):
        r = oracle.render(s, cam)
        if lam > 0:
            lo, dc = oracle.photometric_loss(r["color"], tgt, lam)
        else:
            lo, dc = oracle.l1_loss(r["color"], tgt)
        want.append(lo)
        flat += pack_grads(oracle.render_backward(s, cam, dc))
    # the device's SSIM means are fp64 sums, the oracle's float sums (test_gpu_ssim.py): the loss
    # values agree to the oracle's own summation error, the gradients are the strict check
    assert np.allclose(loss, want, rtol=1e-4 if lam == 0 else 1e-3, atol=1e-7)
    assert_grads_close(tr.grads.to_host(), unpack_grads(flat, s.n), what=f"10-view summed grads (lambda {lam})")


def test_reuse_forward_requires_identical_inputs(oracle):
    """render_backward(reuse_forward = 1) / the fused L1 backward reuse the preceding forward only
    when every input matches: the full camera, the raster config, every parameter pointer and the
    SH degree.  Otherwise the fused call reports SPLAT_ERR_NO_FORWARD_STATE and the
    reuse call re-renders (its gradients equal a fresh backward)."""
    import ctypes as C
    import torch
    s = scenes.make_gaussians(3000, seed=4)
    cam = scenes.fov_camera(96, 80, 60.0, (0.0, 0.0, -3.0))
    ctx = R.Context.default()
    ds = R.DeviceGaussians.from_host(s)
    tgt = torch.zeros(cam.height, cam.width, 3, device="cuda")
    g = R.DeviceGrads(s.n)
    loss = torch.zeros(1, device="cuda")

    def fused(cam_, cfg_, ds_):
        ctx.bind_stream()
        return ctx.lib.splat_render_backward_l1(ctx.h, C.byref(ds_.struct()), C.byref(cam_), C.byref(cfg_),
                                                capi.as_fp(tgt.data_ptr()), None, R._bg((0, 0, 0)),
                                                C.byref(g.struct()), 0, capi.as_fp(loss.data_ptr()))

    base = RasterConfig()
    R.render(ds, cam, base)
    assert fused(cam, base, ds) == 0
    variants = []
    c2 = scenes.fov_camera(96, 80, 60.0, (0.0, 0.0, -3.0))
    c2.fx *= 1.01
    variants.append((c2, base, ds))
    c3 = scenes.fov_camera(96, 80, 60.0, (0.0, 0.0, -3.0))
    c3.cx += 0.5
    variants.append((c3, base, ds))
    cfg2 = RasterConfig()
    cfg2.contribution_min = 2.0 / 255.0
    variants.append((cam, cfg2, ds))
    cfg3 = RasterConfig()
    cfg3.tile_size = 32
    variants.append((cam, cfg3, ds))
    ds2 = R.DeviceGaussians.from_host(s)
    ds2.active_sh_degree = 1
    variants.append((cam, base, ds2))
    for k, (c_, f_, d_) in enumerate(variants):
        R.render(ds, cam, base)
        assert fused(c_, f_, d_) == capi.SPLAT_ERR_NO_FORWARD_STATE, k
    # reuse_forward with a changed camera re-renders: equal to a fresh backward on that camera
    want = oracle.render_backward(s, c2, np.ones((80, 96, 3), np.float32), base)
    R.render(ds, cam, base)
    got = R.render_backward(ds, c2, base, torch.ones(80, 96, 3, device="cuda"), reuse_forward=True).to_host()
    assert_grads_close(got, want, what="reuse after a camera change")
