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
