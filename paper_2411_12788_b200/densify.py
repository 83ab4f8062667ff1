"""On-device densification and simplification, mirroring the
reference's API over the C-ABI (include/splat_b200.h):

  build_masks          visibility.cpp:9-37       per-view quantile masks (VisibilityTable)
  view_statistics      densify.cpp:41-53         max blend weight / ever-max / summed importance
  identify_critical    densify.cpp:32-103        MaxWeight, Opacity, AccumWeight, Random criteria
  aggressive_clone     densify.cpp:105-130 + apply_densify_plan densify.cpp:159-195
  importance_prune     simplify.cpp:94-107       select_above_quantile on global importance
  select / remap       gaussian_set.hpp:96-110, OptimState::remap optimizer.cpp:73-108
  quantile_threshold   quantile.hpp:16-28
  third_neighbor_distances / depth_reinitialize   spatial.cpp:101-121, densify.cpp:198-252

Everything per Gaussian runs in CUDA (csrc/densify.cu + the radix sort); the host reads back
only the scalars the reference's control flow branches on.  No CPU fallback.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Sequence

from . import capi
from .capi import ImportanceOutputs, RasterConfig, as_fp, as_ip
from .rasterizer import Context, DeviceGaussians, OptimState, _device_set, _torch

CRITERIA = {"random": capi.CRITERION_RANDOM, "opacity": capi.CRITERION_OPACITY,
            "accum-weight": capi.CRITERION_ACCUM_WEIGHT, "max-weight": capi.CRITERION_MAX_WEIGHT}


def _crit(criterion) -> int:
    """ident_criterion_from_string (densify.cpp:14-20) or an int."""
    if isinstance(criterion, str):
        if criterion not in CRITERIA:
            raise ValueError(f"unknown identification criterion: {criterion}")
        return CRITERIA[criterion]
    return int(criterion)


def quantile_threshold(values, keep_q: float, sel=None, ctx: Optional[Context] = None):
    """quantile_threshold over a CUDA float32 / float64 tensor (entries with sel != 0). Returns
    (tau, selected count)."""
    torch = _torch()
    ctx = ctx or Context.default()
    ctx.bind_stream()
    cnt = C.c_int32()
    sp = sel.data_ptr() if sel is not None else None
    if values.dtype == torch.float64:
        tau = C.c_double()
        ctx.check(ctx.lib.splat_quantile_threshold_f64(ctx.h, values.data_ptr(), sp, values.numel(), keep_q,
                                                       C.byref(tau), C.byref(cnt)))
    else:
        tau = C.c_float()
        ctx.check(ctx.lib.splat_quantile_threshold(ctx.h, values.data_ptr(), sp, values.numel(), keep_q,
                                                   C.byref(tau), C.byref(cnt)))
    return tau.value, cnt.value


class _Report:
    def __init__(self, n, dev):
        torch = _torch()
        self.importance = torch.zeros(max(n, 1), dtype=torch.float32, device=dev)
        self.max_weight = torch.zeros(max(n, 1), dtype=torch.float32, device=dev)
        self.max_pixel_count = torch.zeros(max(n, 1), dtype=torch.int32, device=dev)
        self.struct = ImportanceOutputs(as_fp(self.importance.data_ptr()), as_fp(self.max_weight.data_ptr()),
                                        as_ip(self.max_pixel_count.data_ptr()))


def build_masks(set_, cams: Sequence[capi.Camera], keep_q: float, cfg: Optional[RasterConfig] = None,
                ctx: Optional[Context] = None):
    """build_masks: [views, n] uint8 CUDA tensor, row k = VisibilityTable::mask_for(k)."""
    torch = _torch()
    ctx = ctx or Context.default()
    cfg = cfg or RasterConfig()
    ds, _ = _device_set(set_, ctx.device)
    n, dev = ds.n, f"cuda:{ctx.device}"
    masks = torch.zeros((len(cams), max(n, 1)), dtype=torch.uint8, device=dev)
    rep = _Report(n, dev)
    g = ds.struct()
    ctx.bind_stream()
    for k, cam in enumerate(cams):
        ctx.check(ctx.lib.splat_accumulate_importance(ctx.h, C.byref(g), C.byref(cam), C.byref(cfg), None,
                                                      C.byref(rep.struct)))
        ctx.check(ctx.lib.splat_visibility_mask(ctx.h, rep.importance.data_ptr(), n, keep_q, masks[k].data_ptr()))
    return masks[:, :n]


def view_statistics(set_, cams: Sequence[capi.Camera], cfg: Optional[RasterConfig] = None, masks=None,
                    ctx: Optional[Context] = None):
    """The per-view folds identify_critical makes (densify.cpp:41-53): (best_weight f32 = max over
    views of max_weight, max_count_sum i64 (> 0 iff ever the max contributor), summed importance
    f64), with optional per-view masks ([views, n] uint8 CUDA, as VisibilityTable)."""
    torch = _torch()
    ctx = ctx or Context.default()
    cfg = cfg or RasterConfig()
    ds, _ = _device_set(set_, ctx.device)
    n, dev = ds.n, f"cuda:{ctx.device}"
    best = torch.zeros(max(n, 1), dtype=torch.float32, device=dev)
    cnt = torch.zeros(max(n, 1), dtype=torch.int64, device=dev)
    summed = torch.zeros(max(n, 1), dtype=torch.float64, device=dev)
    rep = _Report(n, dev)
    g = ds.struct()
    ctx.bind_stream()
    for k, cam in enumerate(cams):
        mp = capi.as_u8p(masks[k].data_ptr()) if masks is not None else None
        ctx.check(ctx.lib.splat_accumulate_importance(ctx.h, C.byref(g), C.byref(cam), C.byref(cfg), mp,
                                                      C.byref(rep.struct)))
        ctx.check(ctx.lib.splat_visibility_update_max(ctx.h, C.byref(rep.struct), n, 0.0, None, summed.data_ptr(),
                                                      cnt.data_ptr(), best.data_ptr()))
    return best[:n], cnt[:n], summed[:n]


def identify_critical(set_, cams: Sequence[capi.Camera], criterion="max-weight", keep_q: float = 0.5,
                      cfg: Optional[RasterConfig] = None, random_scores=None, masks=None, stats=None,
                      ctx: Optional[Context] = None):
    """identify_critical.  Returns (critical uint8 CUDA tensor [n], CriticalSelection::count).
    random_scores: float64 CUDA tensor [n] for the Random criterion (the reference draws them from
    its std::mt19937).  stats: precomputed view_statistics (e.g. gathered across ranks by
    multiview.importance_views)."""
    torch = _torch()
    ctx = ctx or Context.default()
    ds, _ = _device_set(set_, ctx.device)
    c = _crit(criterion)
    best, cnt, summed = stats if stats is not None else view_statistics(ds, cams, cfg, masks, ctx)
    crit = torch.zeros(max(ds.n, 1), dtype=torch.uint8, device=f"cuda:{ctx.device}")
    count = C.c_int32()
    ctx.bind_stream()
    ctx.check(ctx.lib.splat_identify_critical(ctx.h, C.byref(ds.struct()), best.data_ptr(), cnt.data_ptr(),
                                              summed.data_ptr(), c, keep_q,
                                              random_scores.data_ptr() if random_scores is not None else None,
                                              crit.data_ptr(), C.byref(count)))
    return crit[:ds.n], count.value


class Rng:
    """The reference trainer's std::mt19937 (passed by reference to identify_critical,
    vanilla_clone_split and depth_reinitialize), held by the library as a splat_rng: the draws
    are the reference's own sequences (include/splat_rng.h)."""

    def __init__(self, seed: int = 5489, ctx: Optional[Context] = None):
        self.lib = (ctx or Context.default()).lib
        h = C.c_void_p()
        rc = self.lib.splat_rng_create(seed & 0xFFFFFFFF, C.byref(h))
        if rc:
            raise RuntimeError(f"splat_rng_create: status {rc}")
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.splat_rng_destroy(self.h)
            self.h = None

    def state(self):
        w = (C.c_uint32 * 625)()
        self.lib.splat_rng_get_state(self.h, w)
        return list(w)

    def set_state(self, words) -> None:
        w = (C.c_uint32 * 625)(*words)
        if self.lib.splat_rng_set_state(self.h, w):
            raise ValueError("splat_rng_set_state: bad state")


def random_scores(rng: Rng, n: int, ctx: Optional[Context] = None):
    """identify_critical's Random-criterion draws (densify.cpp:78-80) as a float64 CUDA tensor."""
    torch = _torch()
    ctx = ctx or Context.default()
    out = torch.empty(max(n, 1), dtype=torch.float64, device=f"cuda:{ctx.device}")
    ctx.bind_stream()
    ctx.check(ctx.lib.splat_random_scores(ctx.h, rng.h, n, out.data_ptr(), 1))
    return out[:n]


def importance_sample(params: DeviceGaussians, importance, target_count: int, seed: int,
                      ctx: Optional[Context] = None):
    """importance_sample (simplify.cpp:36-92) on a float64 CUDA importance tensor.  Returns
    (kept DeviceGaussians, kept indices int32 CUDA tensor, ascending)."""
    torch = _torch()
    ctx = ctx or Context.default()
    n = params.n
    kept = torch.empty(max(n, 1), dtype=torch.int32, device=params.flat.device)
    nk = C.c_int32()
    ctx.bind_stream()
    ctx.check(ctx.lib.splat_importance_sample(ctx.h, importance.data_ptr(), n, int(target_count),
                                              int(seed) & 0xFFFFFFFFFFFFFFFF, kept.data_ptr(), C.byref(nk)))
    kept = kept[: nk.value]
    return select(params, kept, ctx=ctx), kept


def vanilla_clone_split(params: DeviceGaussians, grad2d_accum, grad2d_count, grad_threshold: float,
                        scale_threshold: float, scene_extent: float, rng: Rng, ctx: Optional[Context] = None):
    """vanilla_clone_split + apply_densify_plan (Progressive mode, densify.cpp:132-163, 182-191).
    grad2d_accum / grad2d_count: the ParamGrads statistics (CUDA float32 / int32 [n]).  Returns
    (new DeviceGaussians, moment_source int32 CUDA tensor, clones, splits); rng advances exactly
    as the reference's std::mt19937 would."""
    torch = _torch()
    ctx = ctx or Context.default()
    ctx.bind_stream()
    ds, _ = _device_set(params, ctx.device)
    g = ds.struct()
    n_out, nc, ns = C.c_int32(), C.c_int32(), C.c_int32()
    dev = f"cuda:{ctx.device}"
    # sizing call: capacity 0 returns the row count without drawing or writing anything
    probe = DeviceGaussians(0, ds.active_sh_degree, ctx.device)
    rc = ctx.lib.splat_vanilla_clone_split(ctx.h, C.byref(g), grad2d_accum.data_ptr(), grad2d_count.data_ptr(),
                                           grad_threshold, scale_threshold, scene_extent, rng.h, C.byref(probe.mut()),
                                           0, None, C.byref(n_out), C.byref(nc), C.byref(ns))
    if rc not in (0, capi.SPLAT_ERR_INVALID_ARGUMENT) or (rc and "capacity" not in
                                                            (ctx.lib.splat_last_error(ctx.h) or b"").decode()):
        ctx.check(rc)
    need = n_out.value
    out = DeviceGaussians(need, ds.active_sh_degree, ctx.device)
    ms = torch.empty(max(need, 1), dtype=torch.int32, device=dev)
    ctx.check(ctx.lib.splat_vanilla_clone_split(ctx.h, C.byref(g), grad2d_accum.data_ptr(), grad2d_count.data_ptr(),
                                                grad_threshold, scale_threshold, scene_extent, rng.h,
                                                C.byref(out.mut()), need, ms.data_ptr(), C.byref(n_out),
                                                C.byref(nc), C.byref(ns)))
    return out, ms[:need], nc.value, ns.value


def _grow(params: DeviceGaussians, capacity: int) -> DeviceGaussians:
    """Copy of params in a layout with room for `capacity` rows (first params.n rows filled)."""
    out = DeviceGaussians(capacity, params.active_sh_degree, params.flat.device.index or 0)
    n = params.n
    out.centers[:n].copy_(params.centers)
    out.log_scales[:n].copy_(params.log_scales)
    out.rotations[:n].copy_(params.rotations)
    out.opacity_logits[:n].copy_(params.opacity_logits)
    out.sh[:n].copy_(params.sh)
    return out


def aggressive_clone(params: DeviceGaussians, critical, ctx: Optional[Context] = None):
    """aggressive_clone + apply_densify_plan.  Returns (new DeviceGaussians, moment_source int32
    CUDA tensor) — feed moment_source to OptimState.remap."""
    torch = _torch()
    ctx = ctx or Context.default()
    ctx.bind_stream()
    n = params.n
    n_out = C.c_int32()
    dev = f"cuda:{ctx.device}"
    # the row count the plan needs (the call returns it without modifying anything when short)
    rc = ctx.lib.splat_aggressive_clone(ctx.h, C.byref(params.mut()), n, critical.data_ptr(), None, C.byref(n_out))
    if rc not in (0, 1):
        ctx.check(rc)
    need = n_out.value
    grown = _grow(params, need) if need > n else params
    p = grown.mut()
    p.n = n
    ms = torch.empty(max(need, 1), dtype=torch.int32, device=dev)
    ctx.check(ctx.lib.splat_aggressive_clone(ctx.h, C.byref(p), need, critical.data_ptr(), ms.data_ptr(),
                                             C.byref(n_out)))
    return grown, ms[:need]


def select(params: DeviceGaussians, keep, n_rows: Optional[int] = None, ctx: Optional[Context] = None):
    """GaussianSetT::select with a CUDA int32 index tensor (or the first n_rows when keep is None)."""
    torch = _torch()
    ctx = ctx or Context.default()
    if keep is None:
        keep = torch.arange(n_rows, dtype=torch.int32, device=params.flat.device)
    m = int(keep.numel())
    out = DeviceGaussians(m, params.active_sh_degree, params.flat.device.index or 0)
    ctx.bind_stream()
    for src, dst, w in ((params.centers, out.centers, 3), (params.log_scales, out.log_scales, 3),
                        (params.rotations, out.rotations, 4), (params.opacity_logits, out.opacity_logits, 1),
                        (params.sh, out.sh, 48)):
        ctx.check(ctx.lib.splat_gather_rows(ctx.h, src.data_ptr(), w, keep.data_ptr(), m, dst.data_ptr()))
    return out


def remap(opt: OptimState, source, ctx: Optional[Context] = None) -> None:
    """OptimState::remap (optimizer.cpp:73-108): row r of every moment array takes old row
    source[r]; source[r] < 0 gives zero moments.  OptimState::keep is remap with kept indices."""
    torch = _torch()
    ctx = ctx or Context.default()
    n_old, n_new = opt.n, int(source.numel())
    dev = opt.m.device
    m = torch.zeros(max(59 * n_new, 1), dtype=torch.float32, device=dev)
    v = torch.zeros(max(59 * n_new, 1), dtype=torch.float32, device=dev)
    ctx.bind_stream()
    o_old = o_new = 0
    for w in (3, 3, 4, 1, 48):
        for src, dst in ((opt.m, m), (opt.v, v)):
            ctx.check(ctx.lib.splat_gather_rows(ctx.h, src.data_ptr() + 4 * o_old, w, source.data_ptr(), n_new,
                                                dst.data_ptr() + 4 * o_new))
        o_old += w * n_old
        o_new += w * n_new
    opt.m, opt.v, opt.n = m, v, n_new


def importance_prune(params: DeviceGaussians, importance, keep_q: float, ctx: Optional[Context] = None):
    """importance_prune on a float64 CUDA importance tensor (e.g. global importance).  Returns
    (kept DeviceGaussians, kept indices int32 CUDA tensor)."""
    torch = _torch()
    ctx = ctx or Context.default()
    n = params.n
    kept = torch.empty(max(n, 1), dtype=torch.int32, device=params.flat.device)
    nk = C.c_int32()
    ctx.bind_stream()
    ctx.check(ctx.lib.splat_importance_prune(ctx.h, importance.data_ptr(), n, keep_q, kept.data_ptr(), C.byref(nk)))
    kept = kept[: nk.value]
    return select(params, kept, ctx=ctx), kept


def third_neighbor_distances(points, min_dist: float = 1e-7, ctx: Optional[Context] = None):
    """third_neighbor_distances over a CUDA float32 tensor [m, 3] (grid k-NN on device)."""
    torch = _torch()
    ctx = ctx or Context.default()
    m = int(points.shape[0])
    out = torch.empty(max(m, 1), dtype=torch.float32, device=points.device)
    ctx.bind_stream()
    ctx.check(ctx.lib.splat_third_neighbor_distances(ctx.h, points.contiguous().data_ptr(), m, min_dist,
                                                     out.data_ptr()))
    return out[:m]


def depth_reinitialize(set_, cams: Sequence[capi.Camera], images, sample_count: int, sample=None,
                       cfg: Optional[RasterConfig] = None, min_dist: float = 1e-7, ctx: Optional[Context] = None,
                       rng: Optional[Rng] = None) -> DeviceGaussians:
    """depth_reinitialize (densify.cpp:198-252) on device: render each view, unproject every pixel
    with a max contributor (view-major, raster order = the reference's pool order), draw
    min(sample_count, pool) of them, and build the fresh set (3rd-NN isotropic scales, identity
    rotation, opacity 0.1, SH DC from the image colour).

    images: CUDA float32 [views, H, W, 3].  sample: optional CUDA int32 pool indices in draw
    order; default: the reference's own draw, a partial Fisher-Yates with
    uniform_int_distribution<int> over `rng` (a std::mt19937, default seed 5489), drawn by the
    library (splat_pool_sample).  Raises RuntimeError when no pixel has a valid depth
    (densify.cpp:223-225)."""
    torch = _torch()
    from .rasterizer import depth_points
    ctx = ctx or Context.default()
    if len(cams) == 0:
        raise ValueError("depth_reinitialize: no cameras")
    if images.shape[0] != len(cams):
        raise ValueError("depth_reinitialize: camera/image count mismatch")
    if sample_count < 1:
        raise ValueError("depth_reinitialize: sample_count < 1")
    ds, _ = _device_set(set_, ctx.device)
    pts, views, pix = depth_points(ds, cams, cfg, rule=capi.DEPTH_RULE_ARGMAX, stride=1, seed=0, ctx=ctx)
    pool = int(pts.shape[0])
    if pool == 0:
        raise RuntimeError("depth_reinitialize: no valid depth pixels (model renders nothing)")
    take = min(sample_count, pool)
    if sample is None:
        sample = torch.empty(take, dtype=torch.int32, device=pts.device)
        ctx.bind_stream()
        rng = rng or Rng(ctx=ctx)  # keep the engine alive across the call
        ctx.check(ctx.lib.splat_pool_sample(ctx.h, rng.h, pool, take, sample.data_ptr()))
    sample = sample[:take].contiguous()
    hw = images.shape[1] * images.shape[2]
    # colour of each pooled point: row (view * HW + pixel) of the [views * HW, 3] image rows
    src = (views.to(torch.int64) * hw + pix.to(torch.int64)).to(torch.int32)[sample.to(torch.int64)].contiguous()
    sampled = torch.empty((take, 3), dtype=torch.float32, device=pts.device)
    colors = torch.empty((take, 3), dtype=torch.float32, device=pts.device)
    ctx.bind_stream()
    ctx.check(ctx.lib.splat_gather_rows(ctx.h, pts.contiguous().data_ptr(), 3, sample.data_ptr(), take,
                                        sampled.data_ptr()))
    ctx.check(ctx.lib.splat_gather_rows(ctx.h, images.contiguous().data_ptr(), 3, src.data_ptr(), take,
                                        colors.data_ptr()))
    fresh = DeviceGaussians(take, ds.active_sh_degree, ctx.device)
    ctx.check(ctx.lib.splat_reinit_gaussians(ctx.h, sampled.data_ptr(), colors.data_ptr(), take, min_dist,
                                             C.byref(fresh.mut())))
    return fresh

