"""View-parallel passes over many views (BASELINE configs 2 and 3; config 4's training step is
trainer.ViewTrainer).  SURVEY.md §8e: one process per GPU, every rank holds a replica of the
Gaussians, views are partitioned in contiguous blocks (rank r: views [r V / W, (r+1) V / W)), the
per-view work is local, and the only exchanges are:

  config 3 (importance / visibility, accumulate_importance rasterizer.cpp:184-193 +
  global_importance simplify.cpp:13-34):
      accum_weight  fp64 all-reduce SUM   (each rank sums its views in order, then ranks are summed)
      intersections int64 all-reduce SUM  (argmax counts: exact)
      max_weight    fp32 all-reduce MAX   (per-Gaussian maximum blend weight over all views: exact)
      per-view visibility bitmasks: all-gather, reassembled in view order (exact)
  config 2 (depth rendering + unprojection, densify.cpp:207-222):
      per-rank point counts all-gathered, points gathered in view order; a point is identified by
      (view, pixel), so indices are bit-exact independent of the number of ranks.

The collective logic takes the per-view work as a callable, so the same code runs the CUDA path
over NCCL and, in tests/test_multiview.py, an oracle stand-in over gloo on CPU.  Only the fp64
importance sum depends on the partition (rounding of the rank partial sums); everything else is
identical to the single-process result.
"""
from __future__ import annotations

import ctypes as C
from typing import Callable, Optional, Sequence

from . import capi
from .capi import ImportanceOutputs, RasterConfig, as_fp, as_ip
from .rasterizer import Context, _device_set, _torch, render, unproject_depth


def _torch_any():
    """torch for the collective plumbing (also on CPU tensors for the gloo tests); the per-view
    CUDA work below goes through rasterizer._torch, which refuses to run without a GPU."""
    import torch
    return torch


def _dist():
    import torch.distributed as dist
    return dist if dist.is_available() and dist.is_initialized() else None


def rank_world(pg=None) -> tuple[int, int]:
    d = _dist()
    if d is None:
        return 0, 1
    return d.get_rank(pg), d.get_world_size(pg)


def view_block(n_views: int, rank: int, world: int) -> range:
    """Contiguous block of views of `rank` (sizes differ by at most one)."""
    return range(rank * n_views // world, (rank + 1) * n_views // world)


def _gather_rows(local, n_views: int, world: int, pg=None):
    """All-gather per-view rows (local: [len(block), ...]) into [n_views, ...] in view order."""
    torch = _torch_any()
    d = _dist()
    if d is None or world == 1:
        return local
    per = (n_views + world - 1) // world
    pad = torch.zeros((per, *local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    parts = [torch.empty_like(pad) for _ in range(world)]
    d.all_gather(parts, pad, group=pg)
    rows = [parts[r][: len(view_block(n_views, r, world))] for r in range(world)]
    return torch.cat(rows, 0)


def importance_views(view_fn: Callable, n_views: int, n: int, device, pg=None, block_fn: Optional[Callable] = None):
    """Config-3 pass.  view_fn(k, mask_row, accum, counts, max_all) adds view k's importance into
    the running fp64 accum / int64 counts / fp32 max_all (in place) and writes its bitmask words
    into mask_row; or block_fn(block, masks, accum, counts, max_all) does the rank's whole block of
    views at once (the native pass).  Returns (masks [n_views, ceil(n/32)] int32, accum f64 [n],
    counts i64 [n], max_all f32 [n]) on every rank."""
    torch = _torch_any()
    rank, world = rank_world(pg)
    block = view_block(n_views, rank, world)
    words = max((n + 31) // 32, 1)
    masks = torch.zeros((len(block), words), dtype=torch.int32, device=device)
    accum = torch.zeros(max(n, 1), dtype=torch.float64, device=device)
    counts = torch.zeros(max(n, 1), dtype=torch.int64, device=device)
    max_all = torch.zeros(max(n, 1), dtype=torch.float32, device=device)
    if block_fn is not None:
        block_fn(block, masks, accum, counts, max_all)
    else:
        for j, k in enumerate(block):
            view_fn(k, masks[j], accum, counts, max_all)
    d = _dist()
    if d is not None and world > 1:
        d.all_reduce(accum, op=d.ReduceOp.SUM, group=pg)
        d.all_reduce(counts, op=d.ReduceOp.SUM, group=pg)
        d.all_reduce(max_all, op=d.ReduceOp.MAX, group=pg)
    masks = _gather_rows(masks, n_views, world, pg)
    return masks, accum[:n], counts[:n], max_all[:n]


def points_views(view_fn: Callable, n_views: int, device, pg=None, block_fn: Optional[Callable] = None):
    """Config-2 pass.  view_fn(k) returns (points [m, 3] f32, pixels [m] i32) of view k; or
    block_fn(block) returns (points, views, pixels) of the rank's whole block of views in view order
    (the native pass).  Returns (points [M, 3], views [M] i32, pixels [M] i32) in view order on every
    rank."""
    torch = _torch_any()
    rank, world = rank_world(pg)
    if block_fn is not None:
        pts, vws, pix = block_fn(view_block(n_views, rank, world))
    else:
        pts, pix, vws = [], [], []
        for k in view_block(n_views, rank, world):
            p, x = view_fn(k)
            pts.append(p)
            pix.append(x)
            vws.append(torch.full((x.shape[0],), k, dtype=torch.int32, device=device))
        cat = lambda xs, shape, dt: torch.cat(xs) if xs else torch.zeros(shape, dtype=dt, device=device)  # noqa: E731
        pts = cat(pts, (0, 3), torch.float32)
        pix = cat(pix, (0,), torch.int32)
        vws = cat(vws, (0,), torch.int32)
    d = _dist()
    if d is None or world == 1:
        return pts, vws, pix
    cnt = torch.tensor([pix.shape[0]], dtype=torch.int64, device=device)
    cnts = [torch.empty_like(cnt) for _ in range(world)]
    d.all_gather(cnts, cnt, group=pg)
    cnts = [int(c.item()) for c in cnts]
    m = max(cnts)
    packed = torch.zeros((m, 5), dtype=torch.float32, device=device)  # x, y, z, view, pixel (as bits)
    packed[: pts.shape[0], :3] = pts
    packed[: pts.shape[0], 3] = vws.view(torch.float32)
    packed[: pts.shape[0], 4] = pix.view(torch.float32)
    parts = [torch.empty_like(packed) for _ in range(world)]
    d.all_gather(parts, packed, group=pg)
    allp = torch.cat([parts[r][: cnts[r]] for r in range(world)], 0)
    return (allp[:, :3].contiguous(), allp[:, 3].contiguous().view(torch.int32),
            allp[:, 4].contiguous().view(torch.int32))


# ---- the CUDA per-view work ------------------------------------------------------------------
def visibility_pass_views(set_, cams: Sequence[capi.Camera], cfg: Optional[RasterConfig] = None,
                          threshold: float = 1e-3, ctx: Optional[Context] = None, pg=None, per_view: bool = False):
    """Config 3 over `cams`, view-parallel across the ranks of `pg` (single process without one):
    the rank's views through splat_visibility_pass (accumulate_importance + visibility_update_max
    per view, consecutive views overlapped on a twin context; per_view: one C-ABI call per view),
    then the reductions above."""
    torch = _torch()
    ctx = ctx or Context.default()
    cfg = cfg or RasterConfig()
    ds, _ = _device_set(set_, ctx.device)
    n = ds.n
    dev = f"cuda:{ctx.device}"
    rep = dict(importance=torch.zeros(max(n, 1), dtype=torch.float32, device=dev),
               max_weight=torch.zeros(max(n, 1), dtype=torch.float32, device=dev),
               max_pixel_count=torch.zeros(max(n, 1), dtype=torch.int32, device=dev))
    out = ImportanceOutputs(as_fp(rep["importance"].data_ptr()), as_fp(rep["max_weight"].data_ptr()),
                            as_ip(rep["max_pixel_count"].data_ptr()))
    g = ds.struct()
    ctx.bind_stream()

    def view_fn(k, mask_row, accum, counts, max_all):
        ctx.check(ctx.lib.splat_accumulate_importance(ctx.h, C.byref(g), C.byref(cams[k]), C.byref(cfg), None,
                                                      C.byref(out)))
        ctx.check(ctx.lib.splat_visibility_update_max(ctx.h, C.byref(out), n, threshold, mask_row.data_ptr(),
                                                      accum.data_ptr(), counts.data_ptr(), max_all.data_ptr()))

    def block_fn(block, masks, accum, counts, max_all):  # the native pass over the block (twin overlap)
        if len(block) == 0:
            return
        cam_arr = (capi.Camera * len(block))(*[cams[k] for k in block])
        ctx.check(ctx.lib.splat_visibility_pass(ctx.h, C.byref(g), cam_arr, len(block), C.byref(cfg), threshold,
                                                masks.data_ptr(), masks.shape[1], accum.data_ptr(), counts.data_ptr(),
                                                max_all.data_ptr()))

    return importance_views(view_fn, len(cams), n, dev, pg, block_fn=None if per_view else block_fn)


def depth_points_views(set_, cams: Sequence[capi.Camera], cfg: Optional[RasterConfig] = None,
                       rule: int = capi.DEPTH_RULE_ALPHA, alpha_threshold: float = 0.5, stride: int = 4,
                       seed: int = 0, ctx: Optional[Context] = None, pg=None, per_view: bool = False):
    """Config 2 over `cams`, view-parallel across the ranks of `pg`: the rank's views through
    splat_depth_points (depth render + unprojection per view, points appended in view order,
    consecutive views overlapped on a twin context; per_view: render + rasterizer.unproject_depth per
    view), gathered in view order."""
    ctx = ctx or Context.default()
    cfg = cfg or RasterConfig()
    ds, _ = _device_set(set_, ctx.device)

    def view_fn(k):
        render(ds, cams[k], cfg, ctx=ctx, want_depth=True)
        p, px, _ = unproject_depth(cams[k], rule=rule, alpha_threshold=alpha_threshold, view_index=k,
                                   stride=stride, seed=seed, ctx=ctx)
        return p.clone(), px.clone()

    def block_fn(block):  # the native pass over the block (twin overlap, points appended in view order)
        torch = _torch()
        dev = f"cuda:{ctx.device}"
        if len(block) == 0:
            return (torch.zeros((0, 3), dtype=torch.float32, device=dev),
                    torch.zeros(0, dtype=torch.int32, device=dev), torch.zeros(0, dtype=torch.int32, device=dev))
        cam_arr = (capi.Camera * len(block))(*[cams[k] for k in block])
        cap = max(sum(cams[k].width * cams[k].height for k in block) // stride + len(block), 1)
        pts = torch.empty((cap, 3), dtype=torch.float32, device=dev)
        vws = torch.empty(cap, dtype=torch.int32, device=dev)
        pix = torch.empty(cap, dtype=torch.int32, device=dev)
        cnt = torch.zeros(1, dtype=torch.int32, device=dev)
        ctx.bind_stream()
        ctx.check(ctx.lib.splat_depth_points(ctx.h, C.byref(ds.struct()), cam_arr, len(block), C.byref(cfg), rule,
                                             alpha_threshold, block[0], stride, seed, pts.data_ptr(), vws.data_ptr(),
                                             pix.data_ptr(), cap, cnt.data_ptr()))
        m = int(cnt.item())
        if m > cap:  # (cannot happen: at most one pixel in `stride` per view is selected)
            raise RuntimeError(f"depth_points: {m} points exceed the capacity {cap}")
        return pts[:m], vws[:m], pix[:m]

    return points_views(view_fn, len(cams), f"cuda:{ctx.device}", pg, block_fn=None if per_view else block_fn)
