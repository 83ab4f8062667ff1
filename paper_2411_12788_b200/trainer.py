"""View-parallel training step over the C-ABI: the caller side of the hot path.

One step (trainer.cpp:226-240 with lambda_dssim = 0, batched as BASELINE config 4):
  for each view of this rank's batch:
      render<float>                                   (splat_render)
      l1_loss + render_backward<float>, grads summed  (splat_render_backward_l1, ParamGrads::add)
        or, with lambda_dssim > 0, photometric_loss   (splat_render_backward_photometric)
  all-reduce of the packed gradient (torch.distributed / NCCL), only when world_size > 1:
      the 3N mean gradients when only means are optimised (config 1), all 59N floats otherwise
  OptimState::step on the selected parameter groups (splat_adam_step)

Views shard across ranks with no data-path collective other than that gradient exchange.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Sequence

import numpy as np

from . import capi
from .capi import Camera, RasterConfig, RenderOutputs, as_fp
from .rasterizer import Context, DeviceGaussians, DeviceGrads, OptimState, _torch


def views_for(step: int, rank: int, world: int, views_per_rank: int, ring: int) -> list[int]:
    """Ring-view indices rank `rank` trains at `step`: consecutive blocks of `views_per_rank`,
    rank-major within the step, wrapping around the ring (SURVEY.md §8e partitioning)."""
    base = step * world * views_per_rank + rank * views_per_rank
    return [(base + j) % ring for j in range(views_per_rank)]


def pack_grads(g: dict) -> np.ndarray:
    """ParamGrads as the packed all-reduce buffer [centers 3N | scales 3N | rot 4N | opac N | sh 48N]."""
    return np.concatenate([np.asarray(g[k], np.float32).reshape(-1) for k in
                           ("d_centers", "d_log_scales", "d_rotations", "d_opacity_logits", "d_sh")])


def unpack_grads(flat: np.ndarray, n: int) -> dict:
    o = np.cumsum([0, 3 * n, 3 * n, 4 * n, n, 48 * n])
    return dict(d_centers=flat[o[0]:o[1]].reshape(n, 3), d_log_scales=flat[o[1]:o[2]].reshape(n, 3),
                d_rotations=flat[o[2]:o[3]].reshape(n, 4), d_opacity_logits=flat[o[3]:o[4]],
                d_sh=flat[o[4]:o[5]].reshape(n, 48))


class ViewTrainer:
    def __init__(self, params: DeviceGaussians, adam: Optional[capi.AdamConfig] = None,
                 group_mask: int = capi.GROUP_ALL, cfg: Optional[RasterConfig] = None,
                 background=(0.0, 0.0, 0.0), ctx: Optional[Context] = None, max_views: int = 64,
                 process_group=None, lambda_dssim: float = 0.0):
        torch = _torch()
        self.torch = torch
        self.ctx = ctx or Context.default()
        self.params = params
        self.cfg = cfg or RasterConfig()
        self.bg = (C.c_float * 3)(*background)
        self.group_mask = group_mask
        self.grads = DeviceGrads(params.n, self.ctx.device)
        self.opt = OptimState(adam or capi.AdamConfig(), params.n, self.ctx.device)
        self.loss = torch.zeros(max_views, dtype=torch.float32, device=f"cuda:{self.ctx.device}")
        self.pg = process_group
        # photometric loss weight (trainer.hpp:46; 0 = the L1-only BASELINE configs)
        self.lambda_dssim = float(lambda_dssim)
        self.pairs_last_step: list[int] = []
        self.survivors_last_step: list[int] = []
        self._empty_out = RenderOutputs()
        self._gs = params.struct()
        self._gr = self.grads.struct()
        self._staging = None

    @property
    def world_size(self) -> int:
        import torch.distributed as dist
        return dist.get_world_size(self.pg) if dist.is_available() and dist.is_initialized() else 1

    def reduce_slice(self):
        """The part of the packed gradient that the optimiser consumes (the exchanged bytes)."""
        n = self.params.n
        if self.group_mask == capi.GROUP_CENTERS:
            return self.grads.flat[: 3 * n]
        return self.grads.flat[: 59 * n]

    def _views(self, cams: Sequence[Camera], targets, ready=None) -> None:
        """`ready[j]` (optional): an event the backward of view j waits for (its target's H2D
        copy), so the copy overlaps that view's forward."""
        lib, h = self.ctx.lib, self.ctx.h
        self.pairs_last_step = []
        self.survivors_last_step = []
        for j, (cam, tgt) in enumerate(zip(cams, targets)):
            self.ctx.check(lib.splat_render(h, C.byref(self._gs), C.byref(cam), C.byref(self.cfg), None, self.bg,
                                            C.byref(self._empty_out), None))
            ns_, np_ = C.c_int64(), C.c_int64()
            lib.splat_forward_counts(h, C.byref(ns_), C.byref(np_), None, None)
            self.pairs_last_step.append(np_.value)
            self.survivors_last_step.append(ns_.value)
            if ready is not None:
                self.torch.cuda.current_stream().wait_event(ready[j])
            if self.lambda_dssim > 0.0:  # photometric_loss -> render_backward (trainer.cpp:226-239)
                self.ctx.check(lib.splat_render_backward_photometric(
                    h, C.byref(self._gs), C.byref(cam), C.byref(self.cfg), as_fp(tgt.data_ptr()), None, self.bg,
                    C.byref(self._gr), 1 if j > 0 else 0, self.lambda_dssim, as_fp(self.loss.data_ptr() + 4 * j)))
            else:
                self.ctx.check(lib.splat_render_backward_l1(h, C.byref(self._gs), C.byref(cam), C.byref(self.cfg),
                                                            as_fp(tgt.data_ptr()), None, self.bg, C.byref(self._gr),
                                                            1 if j > 0 else 0, as_fp(self.loss.data_ptr() + 4 * j)))

    def _finish(self) -> None:
        if self.world_size > 1:
            import torch.distributed as dist
            dist.all_reduce(self.reduce_slice(), op=dist.ReduceOp.SUM, group=self.pg)
        self.opt.step(self.params, self.grads, self.group_mask, self.ctx)

    def step(self, cams: Sequence[Camera], targets, ready=None) -> "object":
        """Device-resident step: targets are CUDA tensors [H, W, 3]. Returns the per-view loss
        tensor (device); nothing is synchronised."""
        self.ctx.bind_stream()
        self._views(cams, targets, ready)
        self._finish()
        return self.loss[: len(cams)]

    def step_host(self, cams: Sequence[Camera], targets_host) -> np.ndarray:
        """End-to-end step through the public API: each view's target is copied host->device
        (pinned, async) inside the step and the per-view losses are read back to the host.

        The copies run on a side stream and each view's backward waits only for its own target,
        so the H2D transfer overlaps that view's forward (preprocess, sort, binning, blend)."""
        torch = self.torch
        k = len(cams)
        shape = tuple(targets_host[0].shape)
        if self._staging is None or self._staging.shape[0] < k or tuple(self._staging.shape[1:]) != shape:
            self._staging = torch.empty((k, *shape), dtype=torch.float32, device=f"cuda:{self.ctx.device}")
            self._copy_stream = torch.cuda.Stream(device=self.ctx.device)
            self._copy_events = [torch.cuda.Event() for _ in range(k)]
        compute = torch.cuda.current_stream(self.ctx.device)
        cs = self._copy_stream
        cs.wait_stream(compute)  # the staging buffer is free once the previous step's backward ran
        with torch.cuda.stream(cs):
            for j in range(k):
                self._staging[j].copy_(targets_host[j], non_blocking=True)
                self._copy_events[j].record(cs)
        self.step(cams, [self._staging[j] for j in range(k)], ready=self._copy_events[:k])
        return self.loss[:k].cpu().numpy()
