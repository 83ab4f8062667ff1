"""The hand-written sm_100a primitives behind the tile lists: stable radix sort and the single-pass
scan, against numpy (stable argsort / cumsum), including sizes that take the reduce-then-scan
radix path and key ranges with constant digits (trivial passes)."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _sort(keys, vals, begin, end):
    import torch
    from paper_2411_12788_b200.rasterizer import Context
    ctx = Context.default()
    k = torch.from_numpy(keys.view(np.int32)).cuda()
    v = torch.from_numpy(vals.view(np.int32)).cuda()
    ka, va = torch.empty_like(k), torch.empty_like(v)
    alt = C.c_int()
    ctx.bind_stream()
    ctx.check(ctx.lib.splat_sort_pairs(ctx.h, k.data_ptr(), v.data_ptr(), ka.data_ptr(), va.data_ptr(), keys.size,
                                       begin, end, C.byref(alt)))
    if alt.value:
        k, v = ka, va
    return k.cpu().numpy().view(np.uint32), v.cpu().numpy().view(np.uint32)


@pytest.mark.parametrize("n,bits,spread", [(1000, 32, 1), (1_000_000, 32, 1), (1_000_000, 32, 0),
                                          (3_500_000, 9, 1), (5000, 9, 1), (777_777, 13, 1),
                                          # 32-bit sorts run as one cooperative kernel while the
                                          # 4096-key tiles fit one wave at <= 6 tiles per CTA
                                          # (multi-tile CTAs from ~1.2 M keys); 4 M keys fall back
                                          (1, 32, 1), (2048, 32, 1), (2049, 32, 0), (3_000_000, 32, 1),
                                          (100_000, 32, 2), (2_000_003, 32, 0), (2_500_000, 32, 2),
                                          (4_000_000, 32, 1)])
def test_radix_sort_is_stable(n, bits, spread):
    rng = np.random.default_rng(n + bits)
    if spread == 2:  # all keys equal: every pass trivial
        keys = np.full(n, 0x40123456, np.uint32)
    elif spread:
        keys = rng.integers(0, 1 << bits, size=n, dtype=np.uint64).astype(np.uint32)
    else:  # depth-like keys: float bits of values in one binade (top byte constant) with ties
        keys = np.round(rng.uniform(2.1, 3.9, size=n), 3).astype(np.float32).view(np.uint32)
    vals = np.arange(n, dtype=np.uint32)
    k, v = _sort(keys, vals, 0, bits)
    order = np.argsort(keys, kind="stable")
    assert np.array_equal(v, order)
    assert np.array_equal(k, keys[order])


@pytest.mark.parametrize("n", [1, 4095, 4096, 4097, 1_000_003])
def test_exclusive_scan(n):
    import torch
    from paper_2411_12788_b200.rasterizer import Context
    ctx = Context.default()
    x = np.random.default_rng(n).integers(0, 50, size=n).astype(np.uint32)
    t = torch.from_numpy(x.view(np.int32)).cuda()
    out = torch.empty_like(t)
    tot = torch.zeros(1, dtype=torch.int32, device="cuda")
    ctx.bind_stream()
    ctx.check(ctx.lib.splat_exclusive_scan(ctx.h, t.data_ptr(), out.data_ptr(), n, tot.data_ptr()))
    want = np.concatenate([[0], np.cumsum(x, dtype=np.uint64)[:-1]]).astype(np.uint32)
    assert np.array_equal(out.cpu().numpy().view(np.uint32), want)
    assert int(tot.item()) == int(x.sum())
