"""View-parallel training step over the C-ABI: the caller side of the hot path.

One step (trainer.cpp:226-240 with lambda_dssim = 0, batched as BASELINE config 4):
  for each view of this rank's batch:
      render<float>                                   (splat_render)
      l1_loss + render_backward<float>, grads summed  (splat_render_backward_l1, ParamGrads::add)
        or, with lambda_dssim > 0, photometric_loss   (splat_render_backward_photometric)
  one process: OptimState::step on the selected parameter groups (splat_adam_step)
  world_size > 1: the sharded exchange of the full 59N-float packed gradient (exchange.py:
      bucketed reduce-scatter -> Adam on this rank's shards -> all-gather of the parameters)

Views shard across ranks with no data-path collective other than that gradient exchange.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Sequence

import numpy as np

from . import capi
from .capi import Camera, RasterConfig
from .exchange import ShardedExchange, padded_len
from .rasterizer import Context, DeviceGaussians, DeviceGrads, LogicError, OptimState, _torch


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
                 process_group=None, lambda_dssim: float = 0.0, buckets: int = 4, native_comm: bool = False):
        """native_comm: the exchange runs inside splat_train_step over the library's own NCCL
        communicator (splat_comm_init; its unique id is broadcast through torch.distributed when
        world_size > 1) instead of through torch.distributed collectives (exchange.py)."""
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
        self.exchange: Optional[ShardedExchange] = None
        self.buckets = buckets
        self.native_comm = bool(native_comm)
        if self.native_comm:
            self._setup_native_comm()
        elif self.world_size > 1:
            self._setup_exchange()
        self._gr = self.grads.struct()

    def _pad_buffers(self, L: int) -> None:
        n = self.params.n
        self.params.ensure_flat_len(L)
        if self.grads.flat.numel() < L:
            self.grads = DeviceGrads(n, self.ctx.device, flat_len=L)
        if self.opt.m.numel() < L:
            torch = self.torch
            for name in ("m", "v"):
                old = getattr(self.opt, name)
                new = torch.zeros(L, dtype=torch.float32, device=old.device)
                new[: 59 * n].copy_(old[: 59 * n])
                setattr(self.opt, name, new)

    def _setup_native_comm(self) -> None:
        """The library's NCCL communicator on this context (one rank per process and GPU)."""
        world = self.world_size
        rank = 0
        uid = (C.c_char * 128)()
        if world > 1:
            import torch.distributed as dist
            rank = dist.get_rank(self.pg)
            if rank == 0:
                self.ctx.check(self.ctx.lib.splat_comm_unique_id(uid))
            obj = [bytes(uid)]
            dist.broadcast_object_list(obj, src=0, group=self.pg)
            uid = (C.c_char * 128).from_buffer_copy(obj[0])
        else:
            self.ctx.check(self.ctx.lib.splat_comm_unique_id(uid))
        self.ctx.check(self.ctx.lib.splat_comm_init(self.ctx.h, world, rank, uid, self.buckets))
        self._pad_buffers(int(self.ctx.lib.splat_exchange_len(self.params.n, world, self.buckets)))

    def _setup_exchange(self) -> None:
        """Packed buffers padded for the sharded exchange (params are re-pointed in place)."""
        import torch.distributed as dist
        n = self.params.n
        self._pad_buffers(padded_len(n, self.world_size, self.buckets))
        self.exchange = ShardedExchange(n, self.world_size, dist.get_rank(self.pg), self.pg, self.buckets)

    @property
    def world_size(self) -> int:
        import torch.distributed as dist
        return dist.get_world_size(self.pg) if dist.is_available() and dist.is_initialized() else 1

    def _native(self, cams: Sequence[Camera], ptrs, on_host: bool, group_mask: int, loss_host=None) -> None:
        """splat_train_step: the whole per-step loop (render, loss, backward summed over views,
        Adam on group_mask; group_mask 0 = no optimiser step) in one native call."""
        lib, h = self.ctx.lib, self.ctx.h
        v = len(cams)
        if v > self.loss.numel():
            raise ValueError("more views than max_views")
        cam_arr = (Camera * v)(*cams)
        tp = (C.c_void_p * v)(*ptrs)
        t = C.c_int32(self.opt.t)
        n = self.params.n
        if self.opt.n != n:  # optimizer.cpp:42-43
            raise LogicError("ViewTrainer: optimizer rows out of sync with the parameter set (remap the moments)")
        if self.grads.n != n:  # the set was densified / pruned: the gradient buffer follows its size
            self.grads = DeviceGrads(n, self.ctx.device)
            if self.native_comm:
                self._pad_buffers(int(lib.splat_exchange_len(n, self.world_size, self.buckets)))
            elif self.world_size > 1:
                self._setup_exchange()
            self._gr = self.grads.struct()
        # ctypes views of the parameter / moment buffers, rebuilt only when a buffer is replaced
        key = (id(self.params.flat), n, self.params.active_sh_degree, id(self.opt.m), id(self.opt.v))
        if key != getattr(self, "_ckey", None):
            self._ckey, self._pm, self._mo = key, self.params.mut(), self.opt._moments()
            self._loss_ptr = self.loss.data_ptr()
        self.ctx.check(lib.splat_train_step(
            h, C.byref(self._pm), C.byref(self._gr), C.byref(self._mo), C.byref(self.opt.config),
            C.byref(t), group_mask, cam_arr, v, tp, 1 if on_host else 0, C.byref(self.cfg), self.bg,
            self.lambda_dssim, self._loss_ptr, loss_host))
        if group_mask:
            self.opt.t = t.value
        self._views_last_step = v

    def _last_counts(self):
        ns_, np_ = C.c_int64(), C.c_int64()
        self.ctx.lib.splat_forward_counts(self.ctx.h, C.byref(ns_), C.byref(np_), None, None)  # the last view's
        return ns_.value, np_.value

    @property
    def pairs_last_step(self) -> list[int]:
        """Tile-Gaussian pairs of the last step's views (the last view's count, per view)."""
        return [self._last_counts()[1]] * getattr(self, "_views_last_step", 0)

    @property
    def survivors_last_step(self) -> list[int]:
        return [self._last_counts()[0]] * getattr(self, "_views_last_step", 0)

    def _views(self, cams: Sequence[Camera], targets) -> None:
        """Render + loss + backward of the views (gradients summed), no optimiser step."""
        self._native(cams, [t.data_ptr() for t in targets], False, 0)

    def _finish_distributed(self) -> None:
        """Sharded exchange + optimiser step of this rank's summed gradients (exchange.py)."""
        if self.exchange is None or self.exchange.n != self.params.n:
            self._setup_exchange()
            self._gr = self.grads.struct()
        self.exchange.step(self.params.flat, self.grads.flat, self.opt.m, self.opt.v, self.opt.config, self.opt.t,
                           self.group_mask, self.ctx)
        self.opt.t += 1

    def step(self, cams: Sequence[Camera], targets) -> "object":
        """Device-resident step: targets are CUDA tensors [H, W, 3]. Returns the per-view loss
        tensor (device); nothing is synchronised.  One process: a single splat_train_step call;
        several ranks: views + backward natively, NCCL all-reduce, then Adam."""
        self.ctx.bind_stream()
        ptrs = [t.data_ptr() for t in targets]
        if self.world_size > 1 and not self.native_comm:
            self._native(cams, ptrs, False, 0)
            self._finish_distributed()
        else:
            self._native(cams, ptrs, False, self.group_mask)
        return self.loss[: len(cams)]

    def step_host(self, cams: Sequence[Camera], targets_host) -> np.ndarray:
        """End-to-end step through the public API: each view's target is copied host->device
        (pinned, async, on the library's copy stream, overlapping that view's forward) inside the
        step and the per-view losses are read back to the host (the call returns after the step)."""
        self.ctx.bind_stream()
        ptrs = [t.data_ptr() if hasattr(t, "data_ptr") else t.ctypes.data for t in targets_host]
        out = np.zeros(len(cams), np.float32)
        if self.world_size > 1 and not self.native_comm:
            self._native(cams, ptrs, True, 0)
            self._finish_distributed()
            return self.loss[: len(cams)].cpu().numpy()
        self._native(cams, ptrs, True, self.group_mask, out.ctypes.data)
        return out
