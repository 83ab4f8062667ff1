"""View-parallel gradient exchange: reduce-scatter -> sharded Adam -> all-gather.

The reference trains one view per iteration (trainer.cpp:208-240) and sums per-view gradients
with ParamGrads::add (gradients.hpp:35-45); BASELINE config 4 batches views across ranks, each
holding a replica of the Gaussians.  After every rank has summed its own views' gradients into
the packed buffer [centers 3N | log_scales 3N | rotations 4N | opacity N | sh 48N] (+ zero
padding to a multiple of `world * buckets * 4` floats):

  for each bucket b (issued back to back on the communicator):
      reduce-scatter(sum) of bucket b      -> this rank's shard of the summed gradient
  for each bucket b:
      wait for its reduce-scatter; OptimState::step on the shard (splat_adam_step_range: the
      element's group learning rate, fp64 moments, optimizer.cpp:29-68) — runs while later
      buckets are still being reduced
      all-gather of the updated parameter shard -> every replica's bucket b (only buckets holding
      a group the optimiser steps: the others are unchanged on every replica)
  renormalise the rotations (optimizer.cpp:69; after the gather, since a shard may cut a row)

Bytes on the wire per rank are those of an all-reduce (2 (G-1)/G x 4 x 59N); the optimiser
reads and writes only 1/G of the moments.  Each rank keeps only its shards of m and v current
(the rest of its moment buffers stays as it was); `gather_moments` assembles them for the
rare densify / prune events that remap rows.

Collectives go through torch.distributed (NCCL on GPUs; gloo stages CUDA tensors through host
memory, for the CPU / single-GPU tests).  The native C-ABI has the same exchange over its own
NCCL communicator (splat_comm_init / splat_train_step) for C++ callers.
"""
from __future__ import annotations

import ctypes as C
from typing import Callable, Optional

from . import capi

ALIGN = 4  # floats: shard boundaries stay 16-byte aligned (float4 traffic in the Adam kernel)


def padded_len(n: int, world: int, buckets: int) -> int:
    """Packed length 59 n rounded up to a multiple of world * buckets * ALIGN."""
    a = world * buckets * ALIGN
    return max(a, (59 * n + a - 1) // a * a)


class ShardedExchange:
    def __init__(self, n: int, world: int, rank: int, group=None, buckets: int = 4,
                 adam_range: Optional[Callable] = None, quat_normalize: Optional[Callable] = None):
        """adam_range(params_flat, grad_shard, m_flat, v_flat, n, begin, count, cfg, step, mask)
        and quat_normalize(rotations, n) default to the native kernels on the current context."""
        self.n, self.world, self.rank, self.group = int(n), int(world), int(rank), group
        self.buckets = max(1, int(buckets))
        self.flat_len = padded_len(self.n, self.world, self.buckets)
        self.bucket_len = self.flat_len // self.buckets
        self.shard_len = self.bucket_len // self.world
        self._adam_range = adam_range
        self._quat_normalize = quat_normalize
        self._shard = None
        self.events = None  # bench: list of (start, end) CUDA event pairs around each exchange

    def _stepped(self, group_mask: int):
        """Packed ranges [lo, hi) of the groups the optimiser steps (only these change)."""
        n = self.n
        spans = ((capi.GROUP_CENTERS, 0, 3 * n), (capi.GROUP_SCALES, 3 * n, 6 * n),
                 (capi.GROUP_ROTATIONS, 6 * n, 10 * n), (capi.GROUP_OPACITY, 10 * n, 11 * n),
                 (capi.GROUP_SH, 11 * n, 59 * n))
        return [(lo, hi) for bit, lo, hi in spans if group_mask & bit]

    def ranges(self):
        """(bucket begin, shard begin) in the packed buffer for every bucket; the shard is this
        rank's `shard_len` floats of the bucket."""
        return [(b * self.bucket_len, b * self.bucket_len + self.rank * self.shard_len) for b in range(self.buckets)]

    def _native_adam(self, ctx):
        def run(params, shard, m, v, n, begin, count, cfg, step, mask):
            ctx.check(ctx.lib.splat_adam_step_range(ctx.h, params.data_ptr(), shard.data_ptr(), m.data_ptr(),
                                                    v.data_ptr(), n, begin, count, C.byref(cfg), step, mask))
        return run

    def _native_quat(self, ctx):
        def run(rotations, n):
            ctx.check(ctx.lib.splat_quat_normalize(ctx.h, rotations.data_ptr(), n))
        return run

    def step(self, params_flat, grads_flat, m_flat, v_flat, cfg: capi.AdamConfig, step: int, group_mask: int,
             ctx=None) -> None:
        """One optimiser step of the replicas from their summed-over-own-views gradients.
        params_flat / grads_flat / m_flat / v_flat: packed buffers of at least flat_len floats
        (torch tensors on one device).  `step` = OptimState's count before this step."""
        import torch
        import torch.distributed as dist
        for t in (params_flat, grads_flat, m_flat, v_flat):
            if t.numel() < self.flat_len:
                raise ValueError("ShardedExchange: buffer shorter than the padded packed length")
        adam = self._adam_range or self._native_adam(ctx)
        quat = self._quat_normalize or self._native_quat(ctx)
        stage = grads_flat.is_cuda and dist.get_backend(self.group) != "nccl"
        if self._shard is None or self._shard.device != grads_flat.device:
            self._shard = torch.empty(self.buckets * self.shard_len, dtype=torch.float32, device=grads_flat.device)
        ev = None
        if self.events is not None and grads_flat.is_cuda:
            ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            ev[0].record()
        B, S, s = self.bucket_len, self.shard_len, self.shard_len
        rs = []
        for b, (b0, _) in enumerate(self.ranges()):
            out = self._shard[b * s:(b + 1) * s]
            src = grads_flat[b0:b0 + B]
            if stage:  # gloo: host copies of the CUDA buffers
                out_h, src_h = torch.empty(s, dtype=torch.float32), src.cpu()
                dist.reduce_scatter_tensor(out_h, src_h, group=self.group)
                out.copy_(out_h)
                rs.append(None)
            else:
                rs.append(dist.reduce_scatter_tensor(out, src, group=self.group, async_op=True))
        ag = []
        stepped = self._stepped(group_mask)
        for b, (b0, s0) in enumerate(self.ranges()):
            if rs[b] is not None:
                rs[b].wait()
            adam(params_flat, self._shard[b * s:(b + 1) * s], m_flat, v_flat, self.n, s0, S, cfg, step, group_mask)
            if not any(lo < b0 + B and b0 < hi for lo, hi in stepped):
                continue  # no stepped parameter in this bucket: every replica already holds it
            dst = params_flat[b0:b0 + B]
            mine = params_flat[s0:s0 + S]
            if stage:
                dst_h = torch.empty(B, dtype=torch.float32)
                dist.all_gather_into_tensor(dst_h, mine.cpu(), group=self.group)
                dst.copy_(dst_h)
            else:
                ag.append(dist.all_gather_into_tensor(dst, mine.clone(), group=self.group, async_op=True))
        for w in ag:
            w.wait()
        if group_mask & capi.GROUP_ROTATIONS:
            n = self.n
            quat(params_flat[6 * n:10 * n], n)
        if ev is not None:
            ev[1].record()
            self.events.append(ev)

    def gather_moments(self, m_flat, v_flat) -> None:
        """All-gather every rank's moment shards so each replica holds the full m and v."""
        import torch
        import torch.distributed as dist
        stage = m_flat.is_cuda and dist.get_backend(self.group) != "nccl"
        for buf in (m_flat, v_flat):
            for b0, s0 in self.ranges():
                dst, mine = buf[b0:b0 + self.bucket_len], buf[s0:s0 + self.shard_len]
                if stage:
                    dst_h = torch.empty(self.bucket_len, dtype=torch.float32)
                    dist.all_gather_into_tensor(dst_h, mine.cpu(), group=self.group)
                    dst.copy_(dst_h)
                else:
                    dist.all_gather_into_tensor(dst, mine.clone(), group=self.group)
