"""Out-of-bounds writes, checked without compute-sanitizer (disabled on this GPU pool): every output
buffer the C-ABI writes is a view into a larger allocation whose head and tail guard zones hold a
sentinel bit pattern, and the zones must be intact after the call.  Image sizes that are not
multiples of the 8 x 8 blocks or the tiles, tile sizes 8 / 16 / 32, masks, the fused L1 backward,
unprojection with an exact-size output and a two-view training step with host targets."""
import ctypes as C

import numpy as np
import pytest
import torch

from paper_2411_12788_b200 import capi, scenes
from paper_2411_12788_b200 import rasterizer as R
from paper_2411_12788_b200.capi import ImportanceOutputs, ParamGrads, RasterConfig, RenderOutputs, as_fp, as_ip

pytestmark = pytest.mark.gpu
GUARD = 4096  # elements on each side
SENT_F = np.uint32(0x7FC0DEAD)  # a NaN payload no kernel writes
SENT_I = np.uint32(0x5A5A5A5A)


class Guarded:
    def __init__(self, numel, dtype=torch.float32):
        self.numel = int(numel)
        want = SENT_F if dtype == torch.float32 else SENT_I
        raw = np.full(self.numel + 2 * GUARD, want, np.uint32).view(np.int32)
        self.buf = torch.from_numpy(raw).cuda().view(dtype)
        self.t = self.buf[GUARD:GUARD + self.numel]

    def ptr(self):
        return self.t.data_ptr()

    def check(self, what):
        raw = self.buf.view(torch.int32).cpu().numpy().view(np.uint32)
        want = SENT_F if self.buf.dtype == torch.float32 else SENT_I
        head, tail = raw[:GUARD], raw[GUARD + self.numel:]
        assert (head == want).all(), f"{what}: write before the buffer"
        assert (tail == want).all(), f"{what}: write past the buffer (first at +{np.argmax(tail != want)})"


def _ctx():
    ctx = R.Context.default()
    ctx.bind_stream()
    return ctx


@pytest.mark.parametrize("w,h,tile", [(203, 117, 16), (256, 192, 32), (97, 61, 8), (1237, 822, 16)])
def test_forward_and_backward_write_inside_their_buffers(w, h, tile):
    ctx = _ctx()
    n = 20_000 if w < 1000 else 200_000
    s = scenes.make_gaussians(n, seed=w)
    ds = R.DeviceGaussians.from_host(s)
    cam = scenes.fov_camera(w, h, 60.0, (0.0, 0.5, -3.0))
    cfg = RasterConfig()
    cfg.tile_size = tile
    hw = w * h
    col, alp, dep, tr = Guarded(3 * hw), Guarded(hw), Guarded(hw), Guarded(hw)
    mc = Guarded(hw, torch.int32)
    imp, mw, mpc = Guarded(n), Guarded(n), Guarded(n, torch.int32)
    mask = torch.from_numpy((np.arange(n) % 5 != 0).astype(np.uint8)).cuda()
    outs = RenderOutputs(as_fp(col.ptr()), as_fp(alp.ptr()), as_fp(dep.ptr()), as_fp(tr.ptr()), as_ip(mc.ptr()))
    rep = ImportanceOutputs(as_fp(imp.ptr()), as_fp(mw.ptr()), as_ip(mpc.ptr()))
    ctx.check(ctx.lib.splat_render(ctx.h, C.byref(ds.struct()), C.byref(cam), C.byref(cfg),
                                   capi.as_u8p(mask.data_ptr()), R._bg((0.1, 0.2, 0.3)), C.byref(outs), C.byref(rep)))
    torch.cuda.synchronize()
    for g, what in ((col, "colour"), (alp, "alpha"), (dep, "depth"), (tr, "transmittance"), (mc, "argmax"),
                    (imp, "importance"), (mw, "max weight"), (mpc, "argmax counts")):
        g.check(what)
    # training forward (no report) then the fused L1 backward into guarded gradient blocks
    ctx.check(ctx.lib.splat_render(ctx.h, C.byref(ds.struct()), C.byref(cam), C.byref(cfg), None,
                                   R._bg((0, 0, 0)), C.byref(outs), None))
    grads = [Guarded(k * n) for k in (3, 3, 4, 1, 48)] + [Guarded(n), Guarded(n, torch.int32)]
    pg = ParamGrads(*[as_fp(g.ptr()) for g in grads[:6]], as_ip(grads[6].ptr()))
    target = torch.rand(h, w, 3, device="cuda")
    loss = Guarded(1)
    ctx.check(ctx.lib.splat_render_backward_l1(ctx.h, C.byref(ds.struct()), C.byref(cam), C.byref(cfg),
                                               as_fp(target.data_ptr()), None, R._bg((0, 0, 0)), C.byref(pg), 0,
                                               as_fp(loss.ptr())))
    # unprojection into an output of exactly the point count
    cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
    probe_p, probe_x = torch.empty(3 * hw, device="cuda"), torch.empty(hw, dtype=torch.int32, device="cuda")
    R.render(ds, cam, cfg)
    ctx.check(ctx.lib.splat_depth_unproject(ctx.h, C.byref(cam), capi.DEPTH_RULE_ARGMAX, 0.5, 0, 1, 0,
                                            as_fp(probe_p.data_ptr()), as_ip(probe_x.data_ptr()), hw,
                                            as_ip(cnt.data_ptr())))
    torch.cuda.synchronize()
    m = int(cnt.item())
    pts, pix = Guarded(3 * m), Guarded(m, torch.int32)
    ctx.check(ctx.lib.splat_depth_unproject(ctx.h, C.byref(cam), capi.DEPTH_RULE_ARGMAX, 0.5, 0, 1, 0,
                                            as_fp(pts.ptr()), as_ip(pix.ptr()), m, as_ip(cnt.data_ptr())))
    torch.cuda.synchronize()
    for g, what in zip(grads, ("d_centers", "d_log_scales", "d_rotations", "d_opacity", "d_sh", "grad2d_accum",
                               "grad2d_count")):
        g.check(what)
    loss.check("loss")
    pts.check("points")
    pix.check("pixels")
    assert m > 0


def test_training_step_writes_inside_its_buffers():
    from paper_2411_12788_b200.trainer import ViewTrainer
    ctx = _ctx()
    n = 30_000
    s = scenes.make_gaussians(n, seed=1)
    cams = [scenes.ring_camera(k, 4, width=333, height=211) for k in range(4)]
    tgts = [torch.rand(c.height, c.width, 3) .pin_memory() for c in cams]
    ds = R.DeviceGaussians.from_host(s)
    tr = ViewTrainer(ds, capi.AdamConfig(), group_mask=capi.GROUP_ALL, ctx=ctx, max_views=4)
    # guard the packed parameter / gradient / moment buffers: replace them by guarded views
    for obj, name in ((tr.params, "flat"), (tr.grads, "flat"), (tr.opt, "m"), (tr.opt, "v")):
        g = Guarded(getattr(obj, name).numel())
        g.t.copy_(getattr(obj, name))
        setattr(obj, name + "_guard", g)
        setattr(obj, name, g.t)
    tr.params._views()
    tr.grads = R.DeviceGrads(n)
    gg = Guarded(tr.grads.flat.numel())
    tr.grads.flat = gg.t
    o = 0
    for nm, k in (("d_centers", 3), ("d_log_scales", 3), ("d_rotations", 4), ("d_opacity_logits", 1), ("d_sh", 48)):
        setattr(tr.grads, nm, gg.t[o:o + k * n].view(n, k) if k > 1 else gg.t[o:o + n])
        o += k * n
    tr._gr = tr.grads.struct()
    tr.step_host(cams[:2], tgts[:2])
    tr.step_host(cams[2:], tgts[2:])
    torch.cuda.synchronize()
    tr.params.flat_guard.check("parameters")
    tr.opt.m_guard.check("Adam m")
    tr.opt.v_guard.check("Adam v")
    gg.check("gradients")
