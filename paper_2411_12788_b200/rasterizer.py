"""Host-side mirror of the reference's rasterizer / gradients / optimizer API over the C-ABI.

Names, argument meaning and error behaviour follow the reference (paths relative to
/root/reference/proj):

  render(set, cam, cfg, mask, background, report)   rasterizer.hpp:72-76
  accumulate_importance(set, cam, cfg, mask)        rasterizer.hpp:79-82
  render_backward(set, cam, cfg, d_color, mask, bg) gradients.hpp:52-56
  l1_loss(a, b, want_grad)                          loss.hpp:9-10
  OptimState(config, n).step(set, grads)            optimizer.hpp:37-76
  unproject_depth(out, cam, ...)                    densify.cpp:207-222

Exceptions: std::invalid_argument -> ValueError, std::logic_error -> LogicError,
std::runtime_error -> RuntimeError.  Host (numpy) inputs give host outputs, like the reference's
std::vector storage; ``DeviceGaussians`` inputs keep everything resident in HBM (torch tensors).
There is no CPU fallback: every call goes through libsplat_b200.so on a CUDA device.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import capi
from .capi import (AdamConfig, AdamMoments, Camera, Gaussians, ImportanceOutputs, ParamGrads, ParamsMut,
                   RasterConfig, RenderOutputs, as_fp, as_ip, as_u8p)
from .scenes import GaussianSet


class LogicError(RuntimeError):
    """std::logic_error of the reference (e.g. parallel arrays out of sync)."""


class SplatCudaError(RuntimeError):
    pass


def _torch():
    import torch  # device memory, streams and torch.distributed only: plumbing, not the product
    if not torch.cuda.is_available():
        raise SplatCudaError("libsplat_b200 needs a CUDA device (no CPU fallback)")
    return torch


class Context:
    """One splat_ctx per device, bound to torch's current CUDA stream at each call."""

    _default: dict = {}

    def __init__(self, device: int = 0):
        self.lib = capi.load_library()
        self.device = device
        h = C.c_void_p()
        rc = self.lib.splat_ctx_create(device, C.byref(h))
        if rc != 0:
            raise SplatCudaError(f"splat_ctx_create failed ({rc})")
        self.h = h

    @classmethod
    def default(cls, device: int = 0) -> "Context":
        if device not in cls._default:
            cls._default[device] = cls(device)
        return cls._default[device]

    def bind_stream(self):
        torch = _torch()
        s = torch.cuda.current_stream(self.device).cuda_stream
        if s != getattr(self, "_bound_stream", None):  # one C call per stream change, not per step
            self.lib.splat_ctx_set_stream(self.h, C.c_void_p(s))
            self._bound_stream = s

    def check(self, rc: int):
        if rc == 0:
            return
        msg = (self.lib.splat_last_error(self.h) or b"").decode()
        if rc == capi.SPLAT_ERR_INVALID_ARGUMENT:
            raise ValueError(msg)
        if rc == capi.SPLAT_ERR_LOGIC:
            raise LogicError(msg)
        if rc == capi.SPLAT_ERR_RUNTIME:
            raise RuntimeError(msg)
        if rc == capi.SPLAT_ERR_NO_FORWARD_STATE:
            raise RuntimeError(msg)
        raise SplatCudaError(f"status {rc}: {msg}")

    def launches(self) -> int:
        return int(self.lib.splat_kernel_launches(self.h))

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.lib.splat_ctx_destroy(self.h)
        except Exception:
            pass


class DeviceGaussians:
    """GaussianSetT<float> resident in HBM: one contiguous float32 buffer of 59 floats per
    Gaussian laid out [centers 3N | log_scales 3N | rotations 4N | opacity N | sh 48N], so the
    packed gradient / all-reduce buffer has the same layout."""

    def __init__(self, n: int, active_sh_degree: int = 3, device: int = 0, flat_len: int = 0):
        torch = _torch()
        self.n = int(n)
        self.active_sh_degree = int(active_sh_degree)
        # flat_len > 59 n: zero padding after the packed groups (the sharded exchange splits the
        # buffer into equal per-rank pieces)
        self.flat = torch.zeros(max(59 * self.n, flat_len, 1), dtype=torch.float32, device=f"cuda:{device}")
        self._views()

    def ensure_flat_len(self, flat_len: int) -> None:
        """Grow the padding after the packed groups to flat_len floats (re-points the views)."""
        if self.flat.numel() >= flat_len:
            return
        torch = _torch()
        f = torch.zeros(flat_len, dtype=torch.float32, device=self.flat.device)
        f[: 59 * self.n].copy_(self.flat[: 59 * self.n])
        self.flat = f
        self._views()

    def _views(self):
        n = self.n
        f = self.flat
        o = 0
        self.centers = f[o:o + 3 * n].view(n, 3); o += 3 * n
        self.log_scales = f[o:o + 3 * n].view(n, 3); o += 3 * n
        self.rotations = f[o:o + 4 * n].view(n, 4); o += 4 * n
        self.opacity_logits = f[o:o + n]; o += n
        self.sh = f[o:o + 48 * n].view(n, 48)

    @classmethod
    def from_host(cls, s: GaussianSet, device: int = 0) -> "DeviceGaussians":
        torch = _torch()
        s.check_consistent()
        d = cls(s.n, s.active_sh_degree, device)
        host = np.concatenate([s.centers.reshape(-1), s.log_scales.reshape(-1), s.rotations.reshape(-1),
                               s.opacity_logits.reshape(-1), s.sh.reshape(-1)]).astype(np.float32)
        if host.size:
            d.flat[: host.size].copy_(torch.from_numpy(host))
        return d

    def to_host(self) -> GaussianSet:
        h = self.flat.cpu().numpy()
        n = self.n
        o = np.cumsum([0, 3 * n, 3 * n, 4 * n, n, 48 * n])
        return GaussianSet(h[o[0]:o[1]].reshape(n, 3).copy(), h[o[1]:o[2]].reshape(n, 3).copy(),
                           h[o[2]:o[3]].reshape(n, 4).copy(), h[o[3]:o[4]].copy(), h[o[4]:o[5]].reshape(n, 48).copy(),
                           self.active_sh_degree)

    def struct(self) -> Gaussians:
        return Gaussians(as_fp(self.centers.data_ptr()), as_fp(self.log_scales.data_ptr()),
                         as_fp(self.rotations.data_ptr()), as_fp(self.opacity_logits.data_ptr()),
                         as_fp(self.sh.data_ptr()), self.n, self.active_sh_degree)

    def mut(self) -> ParamsMut:
        return ParamsMut(as_fp(self.centers.data_ptr()), as_fp(self.log_scales.data_ptr()),
                         as_fp(self.rotations.data_ptr()), as_fp(self.opacity_logits.data_ptr()),
                         as_fp(self.sh.data_ptr()), self.n, self.active_sh_degree)


class DeviceGrads:
    """ParamGrads<float> in HBM with the DeviceGaussians packed layout (+ grad2d stats)."""

    def __init__(self, n: int, device: int = 0, flat_len: int = 0):
        torch = _torch()
        self.n = n
        self.flat = torch.zeros(max(59 * n, flat_len, 1), dtype=torch.float32, device=f"cuda:{device}")
        self.grad2d_accum = torch.zeros(max(n, 1), dtype=torch.float32, device=f"cuda:{device}")
        self.grad2d_count = torch.zeros(max(n, 1), dtype=torch.int32, device=f"cuda:{device}")
        f = self.flat
        o = 0
        self.d_centers = f[o:o + 3 * n].view(n, 3); o += 3 * n
        self.d_log_scales = f[o:o + 3 * n].view(n, 3); o += 3 * n
        self.d_rotations = f[o:o + 4 * n].view(n, 4); o += 4 * n
        self.d_opacity_logits = f[o:o + n]; o += n
        self.d_sh = f[o:o + 48 * n].view(n, 48)

    def struct(self) -> ParamGrads:
        return ParamGrads(as_fp(self.d_centers.data_ptr()), as_fp(self.d_log_scales.data_ptr()),
                          as_fp(self.d_rotations.data_ptr()), as_fp(self.d_opacity_logits.data_ptr()),
                          as_fp(self.d_sh.data_ptr()), as_fp(self.grad2d_accum.data_ptr()),
                          as_ip(self.grad2d_count.data_ptr()))

    def to_host(self) -> dict:
        n = self.n
        return dict(d_centers=self.d_centers.cpu().numpy(), d_log_scales=self.d_log_scales.cpu().numpy(),
                    d_rotations=self.d_rotations.cpu().numpy(), d_opacity_logits=self.d_opacity_logits.cpu().numpy(),
                    d_sh=self.d_sh.cpu().numpy(), grad2d_accum=self.grad2d_accum[:n].cpu().numpy(),
                    grad2d_count=self.grad2d_count[:n].cpu().numpy())


@dataclass
class RenderOutput:
    """RenderOutput<float> (rasterizer.hpp:43-51)."""

    width: int
    height: int
    color: object
    alpha: object
    depth: object
    transmittance: object
    max_contributor: object


@dataclass
class ImportanceReport:
    """ImportanceReport<float> (rasterizer.hpp:54-61)."""

    importance: object
    max_weight: object
    max_pixel_count: object

    def is_max_contributor(self, i: int) -> bool:
        return bool(self.max_pixel_count[i] > 0)


def _bg(background) -> "C.Array":
    b = (C.c_float * 3)(*[float(x) for x in (background if background is not None else (0.0, 0.0, 0.0))])
    return b


def _device_set(set_, device):
    if isinstance(set_, DeviceGaussians):
        return set_, True
    if not isinstance(set_, GaussianSet):
        raise TypeError("expected GaussianSet or DeviceGaussians")
    set_.check_consistent() if set_.n else None
    return DeviceGaussians.from_host(set_, device), False


def _device_mask(mask, n, device):
    if mask is None:
        return None
    torch = _torch()
    if isinstance(mask, torch.Tensor):
        if mask.numel() != n:
            raise ValueError("visibility mask size does not match Gaussian count")
        return mask.to(device=f"cuda:{device}", dtype=torch.uint8).contiguous()
    m = np.asarray(mask)
    if m.size != n:
        raise ValueError("visibility mask size does not match Gaussian count")
    return torch.from_numpy((m != 0).astype(np.uint8)).to(f"cuda:{device}")


def _alloc_render(torch, h, w, device, want_depth=True):
    dev = f"cuda:{device}"
    return dict(color=torch.empty((h, w, 3), dtype=torch.float32, device=dev),
                alpha=torch.empty((h, w), dtype=torch.float32, device=dev),
                depth=torch.empty((h, w), dtype=torch.float32, device=dev) if want_depth else None,
                transmittance=torch.empty((h, w), dtype=torch.float32, device=dev),
                max_contributor=torch.empty((h, w), dtype=torch.int32, device=dev))


def render(set_, cam: Camera, cfg: Optional[RasterConfig] = None, mask=None, background=(0.0, 0.0, 0.0),
           report: bool = False, ctx: Optional[Context] = None, want_depth: bool = True):
    """render<float>; returns RenderOutput (and ImportanceReport when report=True)."""
    torch = _torch()
    ctx = ctx or Context.default()
    cfg = cfg or RasterConfig()
    ds, resident = _device_set(set_, ctx.device)
    m = _device_mask(mask, ds.n, ctx.device)
    o = _alloc_render(torch, cam.height, cam.width, ctx.device, want_depth)
    outs = RenderOutputs(as_fp(o["color"].data_ptr()), as_fp(o["alpha"].data_ptr()),
                         as_fp(o["depth"].data_ptr()) if o["depth"] is not None else capi.fp(),
                         as_fp(o["transmittance"].data_ptr()), as_ip(o["max_contributor"].data_ptr()))
    rep = None
    if report:
        dev = f"cuda:{ctx.device}"
        r = dict(importance=torch.zeros(max(ds.n, 1), dtype=torch.float32, device=dev),
                 max_weight=torch.zeros(max(ds.n, 1), dtype=torch.float32, device=dev),
                 max_pixel_count=torch.zeros(max(ds.n, 1), dtype=torch.int32, device=dev))
        rep = ImportanceOutputs(as_fp(r["importance"].data_ptr()), as_fp(r["max_weight"].data_ptr()),
                                as_ip(r["max_pixel_count"].data_ptr()))
    ctx.bind_stream()
    rc = ctx.lib.splat_render(ctx.h, C.byref(ds.struct()), C.byref(cam), C.byref(cfg),
                              as_u8p(m.data_ptr()) if m is not None else capi.u8p(), _bg(background),
                              C.byref(outs), C.byref(rep) if rep is not None else None)
    ctx.check(rc)
    ctx.keep = (o, ds, m)  # the forward state (colour, alpha, depth, argmax) must outlive this call
    conv = (lambda t: t) if resident else (lambda t: t.cpu().numpy() if t is not None else None)
    out = RenderOutput(cam.width, cam.height, conv(o["color"]), conv(o["alpha"]), conv(o["depth"]),
                       conv(o["transmittance"]), conv(o["max_contributor"]))
    if not report:
        return out
    n = ds.n
    return out, ImportanceReport(conv(r["importance"][:n]), conv(r["max_weight"][:n]), conv(r["max_pixel_count"][:n]))


def accumulate_importance(set_, cam: Camera, cfg: Optional[RasterConfig] = None, mask=None,
                          ctx: Optional[Context] = None) -> ImportanceReport:
    """accumulate_importance<float> (rasterizer.cpp:184-193)."""
    torch = _torch()
    ctx = ctx or Context.default()
    cfg = cfg or RasterConfig()
    ds, resident = _device_set(set_, ctx.device)
    m = _device_mask(mask, ds.n, ctx.device)
    dev = f"cuda:{ctx.device}"
    r = dict(importance=torch.zeros(max(ds.n, 1), dtype=torch.float32, device=dev),
             max_weight=torch.zeros(max(ds.n, 1), dtype=torch.float32, device=dev),
             max_pixel_count=torch.zeros(max(ds.n, 1), dtype=torch.int32, device=dev))
    rep = ImportanceOutputs(as_fp(r["importance"].data_ptr()), as_fp(r["max_weight"].data_ptr()),
                            as_ip(r["max_pixel_count"].data_ptr()))
    ctx.bind_stream()
    ctx.check(ctx.lib.splat_accumulate_importance(ctx.h, C.byref(ds.struct()), C.byref(cam), C.byref(cfg),
                                                  as_u8p(m.data_ptr()) if m is not None else capi.u8p(),
                                                  C.byref(rep)))
    n = ds.n
    conv = (lambda t: t) if resident else (lambda t: t.cpu().numpy())
    return ImportanceReport(conv(r["importance"][:n]), conv(r["max_weight"][:n]), conv(r["max_pixel_count"][:n]))


def render_backward(set_, cam: Camera, cfg: Optional[RasterConfig], d_color, mask=None,
                    background=(0.0, 0.0, 0.0), ctx: Optional[Context] = None, grads: Optional[DeviceGrads] = None,
                    accumulate: bool = False, reuse_forward: bool = False):
    """render_backward<float> (gradients.cpp:45-222). Returns a dict of host arrays for host inputs,
    or the DeviceGrads for device inputs."""
    torch = _torch()
    ctx = ctx or Context.default()
    cfg = cfg or RasterConfig()
    ds, resident = _device_set(set_, ctx.device)
    m = _device_mask(mask, ds.n, ctx.device)
    if isinstance(d_color, np.ndarray):
        if d_color.shape != (cam.height, cam.width, 3):
            raise ValueError("render_backward: dLoss/dColor shape mismatch")
        dc = torch.from_numpy(np.ascontiguousarray(d_color, np.float32)).to(f"cuda:{ctx.device}")
    else:
        if tuple(d_color.shape) != (cam.height, cam.width, 3):
            raise ValueError("render_backward: dLoss/dColor shape mismatch")
        dc = d_color.contiguous()
    g = grads or DeviceGrads(ds.n, ctx.device)
    ctx.bind_stream()
    ctx.check(ctx.lib.splat_render_backward(ctx.h, C.byref(ds.struct()), C.byref(cam), C.byref(cfg),
                                            as_fp(dc.data_ptr()), as_u8p(m.data_ptr()) if m is not None else capi.u8p(),
                                            _bg(background), C.byref(g.struct()), int(accumulate), int(reuse_forward)))
    return g if resident else g.to_host()


def l1_loss(a, b, want_grad: bool = True, ctx: Optional[Context] = None):
    """l1_loss<float> (loss.cpp:63-76): returns (loss, grad)."""
    torch = _torch()
    ctx = ctx or Context.default()
    host = isinstance(a, np.ndarray)
    dev = f"cuda:{ctx.device}"
    ta = torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(dev) if host else a.contiguous()
    tb = torch.from_numpy(np.ascontiguousarray(b, np.float32)).to(dev) if isinstance(b, np.ndarray) else b.contiguous()
    if tuple(ta.shape) != tuple(tb.shape):
        raise ValueError("l1_loss: shape mismatch")
    grad = torch.empty_like(ta) if want_grad else None
    loss = torch.zeros(1, dtype=torch.float32, device=dev)
    ctx.bind_stream()
    ctx.check(ctx.lib.splat_l1_loss(ctx.h, as_fp(ta.data_ptr()), as_fp(tb.data_ptr()), ta.numel(),
                                    as_fp(grad.data_ptr()) if grad is not None else capi.fp(), as_fp(loss.data_ptr())))
    if host:
        return float(loss.item()), (grad.cpu().numpy() if grad is not None else None)
    return loss, grad


def _img_pair(a, b, ctx, what):
    torch = _torch()
    dev = f"cuda:{ctx.device}"
    host = isinstance(a, np.ndarray)
    ta = torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(dev) if host else a.contiguous()
    tb = torch.from_numpy(np.ascontiguousarray(b, np.float32)).to(dev) if isinstance(b, np.ndarray) else b.contiguous()
    if tuple(ta.shape) != tuple(tb.shape) or ta.dim() != 3:
        raise ValueError(f"{what}: shape mismatch")
    return ta, tb, host


def ssim(a, b, want_grad: bool = True, ctx: Optional[Context] = None):
    """ssim<float> (loss.cpp:78-134) of H x W x C images: returns (mean SSIM, d/da)."""
    return photometric_loss(a, b, -1.0, want_grad, ctx, _what="ssim")


def photometric_loss(rendered, target, lam: float, want_grad: bool = True, ctx: Optional[Context] = None,
                     _what: str = "photometric_loss"):
    """photometric_loss<float> (loss.cpp:136-147): (1 - lam) L1 + lam (1 - SSIM), and its gradient.
    (lam < 0 gives plain SSIM: see ssim.)"""
    torch = _torch()
    ctx = ctx or Context.default()
    ta, tb, host = _img_pair(rendered, target, ctx, _what)
    h, w, ch = ta.shape
    grad = torch.empty_like(ta) if want_grad else None
    val = torch.zeros(1, dtype=torch.float32, device=ta.device)
    ctx.bind_stream()
    ctx.check(ctx.lib.splat_photometric_loss(ctx.h, ta.data_ptr(), tb.data_ptr(), w, h, ch, lam,
                                             grad.data_ptr() if grad is not None else None, val.data_ptr()))
    if host:
        return float(val.item()), (grad.cpu().numpy() if grad is not None else None)
    return val, grad


class OptimState:
    """OptimState (optimizer.hpp:37-76): Adam moments in HBM with the packed parameter layout."""

    def __init__(self, config: Optional[AdamConfig] = None, n: int = 0, device: int = 0, flat_len: int = 0):
        torch = _torch()
        self.config = config or AdamConfig()
        self.n = n
        self.t = 0
        self.m = torch.zeros(max(59 * n, flat_len, 1), dtype=torch.float32, device=f"cuda:{device}")
        self.v = torch.zeros(max(59 * n, flat_len, 1), dtype=torch.float32, device=f"cuda:{device}")

    def size(self) -> int:
        return self.n

    def step_count(self) -> int:
        return self.t

    def _moments(self) -> AdamMoments:
        n = self.n
        offs = [0, 3 * n, 6 * n, 10 * n, 11 * n]
        mp, vp = self.m.data_ptr(), self.v.data_ptr()
        ptrs = []
        for o in offs:
            ptrs += [as_fp(mp + 4 * o), as_fp(vp + 4 * o)]
        return AdamMoments(*ptrs)

    def step(self, set_: DeviceGaussians, grads: DeviceGrads, group_mask: int = capi.GROUP_ALL,
             ctx: Optional[Context] = None) -> None:
        """OptimState::step (optimizer.cpp:40-71); set_ is updated in place."""
        ctx = ctx or Context.default()
        if set_.n != self.n or grads.n != self.n:
            raise LogicError("OptimState::step: moment/gradient rows out of sync with set")
        t = C.c_int32(self.t)
        ctx.bind_stream()
        ctx.check(ctx.lib.splat_adam_step(ctx.h, C.byref(set_.mut()), C.byref(grads.struct()), C.byref(self._moments()),
                                          C.byref(self.config), C.byref(t), group_mask))
        self.t = t.value


def unproject_depth(cam: Camera, rule: int = capi.DEPTH_RULE_ARGMAX, alpha_threshold: float = 0.5,
                    view_index: int = 0, stride: int = 1, seed: int = 0, ctx: Optional[Context] = None,
                    capacity: Optional[int] = None):
    """Unproject the preceding render's depth (densify.cpp:213-220) with the stride rule of
    splat_depth_unproject.  Returns (points [k,3], pixel [k]) as torch tensors on the device."""
    torch = _torch()
    ctx = ctx or Context.default()
    dev = f"cuda:{ctx.device}"
    cap = capacity if capacity is not None else cam.width * cam.height
    pts = torch.empty((max(cap, 1), 3), dtype=torch.float32, device=dev)
    pix = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
    cnt = torch.zeros(1, dtype=torch.int32, device=dev)
    ctx.bind_stream()
    ctx.check(ctx.lib.splat_depth_unproject(ctx.h, C.byref(cam), rule, alpha_threshold, view_index, stride, seed,
                                            as_fp(pts.data_ptr()), as_ip(pix.data_ptr()), cap, as_ip(cnt.data_ptr())))
    k = int(cnt.item())
    return pts[: min(k, cap)], pix[: min(k, cap)], k


def forward_debug(ctx: Optional[Context] = None) -> dict:
    """Bit-exact views of the preceding forward: per-Gaussian rects, depth order, sorted pairs,
    tile ranges (host arrays)."""
    ctx = ctx or Context.default()
    ns, npairs = C.c_int64(), C.c_int64()
    tx, ty = C.c_int32(), C.c_int32()
    ctx.check(ctx.lib.splat_forward_counts(ctx.h, C.byref(ns), C.byref(npairs), C.byref(tx), C.byref(ty)))
    P = npairs.value
    tiles = np.zeros(max(P, 1), np.int32)
    gauss = np.zeros(max(P, 1), np.int32)
    ranges = np.zeros((tx.value * ty.value, 2), np.int32)
    order = np.zeros(max(ns.value, 1), np.int32)
    ctx.check(ctx.lib.splat_tiles_debug(ctx.h, tiles.ctypes.data_as(capi.ip), gauss.ctypes.data_as(capi.ip),
                                        ranges.ctypes.data_as(capi.ip), order.ctypes.data_as(capi.ip)))
    return dict(n_survivors=ns.value, n_pairs=P, tiles_x=tx.value, tiles_y=ty.value, key_tile=tiles[:P],
                gaussian=gauss[:P], ranges=ranges, order=order[: ns.value])


def project(set_, cam: Camera, cfg: Optional[RasterConfig] = None, mask=None, ctx: Optional[Context] = None):
    """project<float> (rasterizer.cpp:10-90): the survivors' ProjectedGaussian records sorted by
    (depth, index), as a numpy structured array with capi.Projected's fields."""
    ctx = ctx or Context.default()
    cfg = cfg or RasterConfig()
    ds, _ = _device_set(set_, ctx.device)
    m = _device_mask(mask, ds.n, ctx.device)
    out = (capi.Projected * max(ds.n, 1))()
    cnt = C.c_int32()
    ctx.bind_stream()
    ctx.check(ctx.lib.splat_project(ctx.h, C.byref(ds.struct()), C.byref(cam), C.byref(cfg),
                                    as_u8p(m.data_ptr()) if m is not None else capi.u8p(), C.cast(out, C.c_void_p),
                                    max(ds.n, 1), C.byref(cnt)))
    arr = np.ctypeslib.as_array(out)[: cnt.value].copy()
    return arr


def traversal_counts(ctx: Optional[Context] = None) -> tuple[int, int]:
    """(V, C) of the preceding forward: traverse_pixel list visits and committed samples summed over
    the pixels (a measurement pass, synchronous)."""
    ctx = ctx or Context.default()
    v, c = C.c_int64(), C.c_int64()
    ctx.bind_stream()
    ctx.check(ctx.lib.splat_traversal_counts(ctx.h, C.byref(v), C.byref(c)))
    return v.value, c.value


def project_debug(n: int, ctx: Optional[Context] = None) -> dict:
    ctx = ctx or Context.default()
    rect = np.zeros((max(n, 1), 4), np.int32)
    radius = np.zeros(max(n, 1), np.int32)
    depth = np.zeros(max(n, 1), np.float32)
    surv = np.zeros(max(n, 1), np.uint8)
    mean2d = np.zeros((max(n, 1), 2), np.float32)
    conic = np.zeros((max(n, 1), 3), np.float32)
    color = np.zeros((max(n, 1), 3), np.float32)
    opac = np.zeros(max(n, 1), np.float32)
    ctx.check(ctx.lib.splat_project_debug(ctx.h, rect.ctypes.data_as(capi.ip), radius.ctypes.data_as(capi.ip),
                                          depth.ctypes.data_as(capi.fp), surv.ctypes.data_as(capi.u8p),
                                          mean2d.ctypes.data_as(capi.fp), conic.ctypes.data_as(capi.fp),
                                          color.ctypes.data_as(capi.fp), opac.ctypes.data_as(capi.fp)))
    return dict(rect=rect[:n], depth=depth[:n], survivor=surv[:n].astype(bool), mean2d=mean2d[:n], conic=conic[:n],
                color=color[:n], opacity=opac[:n])


def visibility_pass(set_, cams, cfg: Optional[RasterConfig] = None, threshold: float = 1e-3,
                    ctx: Optional[Context] = None):
    """BASELINE config 3 over views: accumulate_importance per view (rasterizer.cpp:184-193), the
    per-view visibility bitmask (max blend weight > threshold) and global_importance
    (simplify.cpp:13-34: fp64 sum of importance, sum of argmax counts, views in order).
    Returns (masks [views, ceil(n/32)] uint32 words, accum_weight float64 [n], intersections int64 [n])
    as torch CUDA tensors."""
    torch = _torch()
    ctx = ctx or Context.default()
    cfg = cfg or RasterConfig()
    ds, _ = _device_set(set_, ctx.device)
    n = ds.n
    dev = f"cuda:{ctx.device}"
    words = (n + 31) // 32
    masks = torch.zeros((len(cams), max(words, 1)), dtype=torch.int32, device=dev)
    accum = torch.zeros(max(n, 1), dtype=torch.float64, device=dev)
    counts = torch.zeros(max(n, 1), dtype=torch.int64, device=dev)
    r = dict(importance=torch.zeros(max(n, 1), dtype=torch.float32, device=dev),
             max_weight=torch.zeros(max(n, 1), dtype=torch.float32, device=dev),
             max_pixel_count=torch.zeros(max(n, 1), dtype=torch.int32, device=dev))
    rep = ImportanceOutputs(as_fp(r["importance"].data_ptr()), as_fp(r["max_weight"].data_ptr()),
                            as_ip(r["max_pixel_count"].data_ptr()))
    ctx.bind_stream()
    g = ds.struct()
    for k, cam in enumerate(cams):
        ctx.check(ctx.lib.splat_accumulate_importance(ctx.h, C.byref(g), C.byref(cam), C.byref(cfg), None,
                                                      C.byref(rep)))
        ctx.check(ctx.lib.splat_visibility_update(ctx.h, C.byref(rep), n, threshold, masks[k].data_ptr(),
                                                  accum.data_ptr(), counts.data_ptr()))
    return masks, accum[:n], counts[:n]


def unpack_mask(words, n: int) -> np.ndarray:
    """uint32 bitmask words -> bool [n] (bit i of word i // 32)."""
    w = np.asarray(words).astype(np.uint32)
    bits = (w[:, None] >> np.arange(32, dtype=np.uint32)[None, :]) & 1
    return bits.reshape(-1)[:n].astype(bool)


def depth_points(set_, cams, cfg: Optional[RasterConfig] = None, rule: int = capi.DEPTH_RULE_ALPHA,
                 alpha_threshold: float = 0.5, stride: int = 4, seed: int = 0, ctx: Optional[Context] = None):
    """BASELINE config 2 (aggressive densification's depth pass, densify.cpp:207-222): per view,
    render depth + alpha, select pixels with alpha > alpha_threshold (or argmax >= 0) and
    (view * H * W + pixel + seed) % stride == 0, unproject them.  Returns (points [k, 3],
    view [k], pixel [k]) as torch CUDA tensors, views in order, pixels in raster order."""
    torch = _torch()
    ctx = ctx or Context.default()
    cfg = cfg or RasterConfig()
    ds, _ = _device_set(set_, ctx.device)
    pts, views, pixels = [], [], []
    for k, cam in enumerate(cams):
        render(ds, cam, cfg, ctx=ctx, want_depth=True)
        p, px, cnt = unproject_depth(cam, rule=rule, alpha_threshold=alpha_threshold, view_index=k, stride=stride,
                                     seed=seed, ctx=ctx)
        pts.append(p.clone())
        pixels.append(px.clone())
        views.append(torch.full((p.shape[0],), k, dtype=torch.int32, device=p.device))
    return torch.cat(pts), torch.cat(views), torch.cat(pixels)
