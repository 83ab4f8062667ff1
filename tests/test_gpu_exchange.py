"""splat_adam_step_range (the sharded optimiser step of the view-parallel exchange) against the
full splat_adam_step: shards cut anywhere in the packed layout (mid-row in SH, across group
boundaries, odd n) give bit-identical parameters and moments once the rotations are renormalised,
and padding elements are never touched."""
import ctypes as C

import numpy as np
import pytest
import torch

from paper_2411_12788_b200 import capi
from paper_2411_12788_b200.exchange import padded_len
from paper_2411_12788_b200.rasterizer import Context, DeviceGaussians, DeviceGrads, OptimState

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,world,buckets,mask", [(1001, 2, 3, capi.GROUP_ALL), (4097, 8, 4, capi.GROUP_ALL),
                                                  (777, 3, 1, capi.GROUP_CENTERS | capi.GROUP_SH),
                                                  (50_000, 8, 4, capi.GROUP_ALL)])
def test_sharded_adam_equals_full_step(n, world, buckets, mask):
    from paper_2411_12788_b200 import scenes
    ctx = Context.default()
    ctx.bind_stream()
    rng = np.random.default_rng(n)
    s = scenes.make_gaussians(n, seed=n % 97)
    L = padded_len(n, world, buckets)
    full = DeviceGaussians.from_host(s)
    shard = DeviceGaussians.from_host(s)
    shard.ensure_flat_len(L)
    grads = DeviceGrads(n, flat_len=L)
    g = torch.from_numpy(rng.normal(0, 1e-3, 59 * n).astype(np.float32)).cuda()
    g[rng.random(59 * n) < 0.2] = 0.0
    grads.flat[: 59 * n] = g
    opt_full = OptimState(capi.AdamConfig(), n)
    m = torch.zeros(L, device="cuda")
    v = torch.zeros(L, device="cuda")
    cfg = capi.AdamConfig()
    bucket = L // buckets
    sl = bucket // world
    for step in range(3):
        opt_full.step(full, grads, mask, ctx)
        for b in range(buckets):
            for r in range(world):
                b0 = b * bucket + r * sl
                ctx.check(ctx.lib.splat_adam_step_range(ctx.h, shard.flat.data_ptr(), grads.flat[b0:].data_ptr(),
                                                        m.data_ptr(), v.data_ptr(), n, b0, sl, C.byref(cfg), step,
                                                        mask))
        if mask & capi.GROUP_ROTATIONS:
            ctx.check(ctx.lib.splat_quat_normalize(ctx.h, shard.rotations.data_ptr(), n))
    torch.cuda.synchronize()
    assert torch.equal(shard.flat[: 59 * n], full.flat[: 59 * n])
    assert torch.equal(m[: 59 * n], opt_full.m[: 59 * n]) and torch.equal(v[: 59 * n], opt_full.v[: 59 * n])
    assert not shard.flat[59 * n:].any() and not m[59 * n:].any()


@pytest.mark.parametrize("mask", [capi.GROUP_ALL, capi.GROUP_CENTERS])
def test_native_nccl_exchange_single_rank_equals_plain_step(mask):
    """splat_train_step with the library's own NCCL communicator (one rank here: reduce-scatter and
    all-gather over a 1-rank communicator, sharded Adam over its one shard per bucket) equals the
    plain step bit for bit — this runs the C-ABI's NCCL exchange path end to end."""
    from paper_2411_12788_b200 import scenes
    from paper_2411_12788_b200.rasterizer import render
    from paper_2411_12788_b200.trainer import ViewTrainer
    s = scenes.make_gaussians(30_001, seed=4)
    cams = [scenes.ring_camera(k, 6, width=320, height=214) for k in range(6)]
    ctx_plain, ctx_comm = Context(0), Context(0)
    pert = DeviceGaussians.from_host(scenes.perturbed(s))
    targets = [render(pert, c, want_depth=False, ctx=ctx_plain).color.clone() for c in cams]
    out = []
    for ctx, native in ((ctx_plain, False), (ctx_comm, True)):
        tr = ViewTrainer(DeviceGaussians.from_host(s), capi.AdamConfig(), group_mask=mask, ctx=ctx, max_views=3,
                         buckets=3, native_comm=native)
        tr.step(cams[:3], targets[:3])
        tr.step_host(cams[3:], [t.cpu().pin_memory() for t in targets[3:]])
        torch.cuda.synchronize()
        out.append((tr.params.flat[: 59 * s.n].clone(), tr.opt.t))
    assert out[0][1] == out[1][1] == 2
    # the blend backward's float atomics make the summed gradients run-to-run different in the last
    # bits, so the two trainers agree to rounding (the exchange itself is checked bitwise below)
    d = (out[0][0] - out[1][0]).abs()
    assert float((d > 1e-6).float().mean()) <= 1e-4 and float(d.max()) <= 0.2
    ctx_comm.check(ctx_comm.lib.splat_comm_destroy(ctx_comm.h))


def test_native_nccl_exchange_step_bitwise():
    """splat_exchange_step over a 1-rank NCCL communicator == splat_adam_step, bit for bit."""
    from paper_2411_12788_b200 import scenes
    n, buckets = 40_003, 5
    ctx_plain, ctx_comm = Context(0), Context(0)
    uid = (C.c_char * 128)()
    ctx_comm.check(ctx_comm.lib.splat_comm_unique_id(uid))
    ctx_comm.check(ctx_comm.lib.splat_comm_init(ctx_comm.h, 1, 0, uid, buckets))
    L = int(ctx_comm.lib.splat_exchange_len(n, 1, buckets))
    assert L == padded_len(n, 1, buckets)
    s = scenes.make_gaussians(n, seed=9)
    rng = np.random.default_rng(1)
    a = DeviceGaussians.from_host(s)
    b = DeviceGaussians.from_host(s)
    b.ensure_flat_len(L)
    grads = DeviceGrads(n, flat_len=L)
    grads.flat[: 59 * n] = torch.from_numpy(rng.normal(0, 1e-3, 59 * n).astype(np.float32)).cuda()
    opt = OptimState(capi.AdamConfig(), n)
    m, v = torch.zeros(L, device="cuda"), torch.zeros(L, device="cuda")
    cfg = capi.AdamConfig()
    t = C.c_int32(0)
    for _ in range(3):
        ctx_plain.bind_stream()
        opt.step(a, grads, capi.GROUP_ALL, ctx_plain)
        ctx_comm.bind_stream()
        ctx_comm.check(ctx_comm.lib.splat_exchange_step(ctx_comm.h, b.flat.data_ptr(), grads.flat.data_ptr(),
                                                        m.data_ptr(), v.data_ptr(), n, L, C.byref(cfg), C.byref(t),
                                                        capi.GROUP_ALL))
    torch.cuda.synchronize()
    assert t.value == 3
    assert torch.equal(a.flat[: 59 * n], b.flat[: 59 * n])
    assert torch.equal(opt.m[: 59 * n], m[: 59 * n]) and torch.equal(opt.v[: 59 * n], v[: 59 * n])
    ctx_comm.check(ctx_comm.lib.splat_comm_destroy(ctx_comm.h))
