"""View-parallel training step across ranks with the gloo backend on CPU:
each rank computes the gradients of its views (the CPU oracle stands in for the per-view CUDA
work, which needs a GPU) into the padded packed 59N buffer, and the product's exchange
(paper_2411_12788_b200/exchange.py: bucketed reduce-scatter -> Adam on this rank's shards ->
all-gather -> quaternion renorm; the oracle's restatement of splat_adam_step_range stands in for
the kernel) steps the replicas.  The result must equal an all-reduce followed by the full
OptimState::step bit for bit, equal one process training all views within float-sum tolerance,
and stay identical across ranks."""
import os
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]
N_GAUSS, RING, V, STEPS = 600, 8, 2, 2


def _scene():
    from paper_2411_12788_b200 import scenes
    s = scenes.make_gaussians(N_GAUSS, seed=3, log_scale_mean=np.log(0.04))
    cams = [scenes.ring_camera(k, RING, width=48, height=32) for k in range(RING)]
    return s, cams


def _view_grads(oracle, s, cam, target):
    r = oracle.render(s, cam)
    _, dc = oracle.l1_loss(r["color"], target)
    return oracle.render_backward(s, cam, dc)


def _train(rank, world, out_q, port, mode="exchange", buckets=3, mask=31):
    sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
    from oracle_lib import OracleLib
    from paper_2411_12788_b200 import scenes
    from paper_2411_12788_b200.capi import AdamConfig, GROUP_ALL
    from paper_2411_12788_b200.exchange import ShardedExchange
    from paper_2411_12788_b200.scenes import GaussianSet
    from paper_2411_12788_b200.trainer import pack_grads, unpack_grads, views_for
    if world > 1:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
    oracle = OracleLib("oracle", "B")
    s, cams = _scene()
    targets = [oracle.render(scenes.perturbed(s), c)["color"] for c in cams]
    n = N_GAUSS
    cfg = AdamConfig()
    ex = ShardedExchange(n, world, rank, buckets=buckets,
                         adam_range=lambda p, g, m_, v_, n_, b, c, cf, st, mk: oracle.adam_step_range(
                             p.numpy(), g.numpy(), m_.numpy(), v_.numpy(), n_, b, c, cf, st, mk),
                         quat_normalize=lambda r, n_: oracle.quat_normalize(r.numpy(), n_))
    L = ex.flat_len
    params = torch.zeros(L)
    params[:59 * n] = torch.from_numpy(pack_grads(dict(d_centers=s.centers, d_log_scales=s.log_scales,
                                                       d_rotations=s.rotations, d_opacity_logits=s.opacity_logits,
                                                       d_sh=s.sh)))
    m, v = torch.zeros(L), torch.zeros(L)
    t = 0
    for step in range(STEPS):
        cur = unpack_grads(params[:59 * n].numpy().copy(), n)
        s = GaussianSet(cur["d_centers"], cur["d_log_scales"], cur["d_rotations"], cur["d_opacity_logits"],
                        cur["d_sh"])
        idx = views_for(step, rank, world, V * 2 // world, RING)  # same global batch for any world
        flat = np.zeros(59 * n, np.float32)
        for i in idx:
            flat += pack_grads(_view_grads(oracle, s, cams[i], targets[i]))
        grads = torch.zeros(L)
        grads[:59 * n] = torch.from_numpy(flat)
        if mode == "exchange":
            ex.step(params, grads, m, v, cfg, t, mask)
            t += 1
        else:  # all-reduce + the full OptimState::step on every rank
            if world > 1:
                dist.all_reduce(grads, op=dist.ReduceOp.SUM)
            s2, m2, v2, t = oracle.adam_step(s, unpack_grads(grads[:59 * n].numpy(), n), m[:59 * n].numpy(),
                                             v[:59 * n].numpy(), cfg, t, mask)
            params[:59 * n] = torch.from_numpy(pack_grads(dict(d_centers=s2.centers, d_log_scales=s2.log_scales,
                                                               d_rotations=s2.rotations,
                                                               d_opacity_logits=s2.opacity_logits, d_sh=s2.sh)))
            m[:59 * n], v[:59 * n] = torch.from_numpy(m2), torch.from_numpy(v2)
    out_q.put((rank, params[:59 * n].numpy().copy()))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def _run(world, port, mode="exchange", buckets=3, mask=31):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_train, args=(r, world, q, port, mode, buckets, mask)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(res, key=lambda x: x[0])


def test_views_partition_covers_ring_once_per_epoch():
    from paper_2411_12788_b200.trainer import views_for
    for world in (1, 2, 4, 8):
        seen = [i for step in range(RING // (world * 1)) for r in range(world) for i in views_for(step, r, world, 1, RING)]
        assert sorted(seen) == list(range(RING))


@pytest.mark.timeout(600)
def test_two_rank_gloo_exchange_matches_allreduce_and_single_process():
    single = _run(1, 29611, mode="allreduce")
    two = _run(2, 29612, mode="exchange", buckets=3)
    two_ar = _run(2, 29613, mode="allreduce")
    # ranks agree bit for bit (the gather hands every replica the same parameters)
    assert np.array_equal(two[0][1], two[1][1])
    # reduce-scatter + Adam on shards + all-gather + renorm == all-reduce + the full step, bitwise
    assert np.array_equal(two[0][1], two_ar[0][1])
    # and one process summing all views, within the float-sum order difference
    assert np.allclose(two[0][1], single[0][1], rtol=0, atol=1e-6)


@pytest.mark.timeout(600)
def test_two_rank_exchange_means_only_skips_unchanged_buckets():
    """Adam on the means only (config 1): buckets without a stepped group are not all-gathered,
    and the result still equals all-reduce + the masked full step bit for bit."""
    from paper_2411_12788_b200.capi import GROUP_CENTERS
    two = _run(2, 29614, mode="exchange", buckets=5, mask=GROUP_CENTERS)
    two_ar = _run(2, 29615, mode="allreduce", mask=GROUP_CENTERS)
    assert np.array_equal(two[0][1], two[1][1])
    assert np.array_equal(two[0][1], two_ar[0][1])


def test_exchange_ranges_partition_the_padded_buffer():
    from paper_2411_12788_b200.exchange import ShardedExchange, padded_len
    for n, world, buckets in ((1, 2, 1), (600, 2, 3), (1001, 8, 4), (3_000_000, 8, 4), (7, 3, 5)):
        L = padded_len(n, world, buckets)
        assert L >= 59 * n and L % (world * buckets * 4) == 0
        covered = np.zeros(L, np.int32)
        for r in range(world):
            ex = ShardedExchange(n, world, r, buckets=buckets)
            for b0, s0 in ex.ranges():
                assert b0 <= s0 and s0 + ex.shard_len <= b0 + ex.bucket_len and s0 % 4 == 0
                covered[s0:s0 + ex.shard_len] += 1
        assert (covered == 1).all()
