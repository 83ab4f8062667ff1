"""View-parallel config-3 (importance / visibility) and config-2 (depth unprojection) passes across
ranks with the gloo backend on CPU (paper_2411_12788_b200/multiview.py).  The per-view work is the
CPU oracle standing in for the CUDA view (which needs a GPU); the partition and the collectives are
the product code.  With 2 ranks the results must equal the single-process pass: bitmasks, argmax
counts, max blend weights and point indices exactly, the fp64 importance sums to 1e-12."""
import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]
N_GAUSS, N_VIEWS, THRESH = 500, 5, 1e-3


def _scene():
    from paper_2411_12788_b200 import scenes
    s = scenes.make_gaussians(N_GAUSS, seed=5, log_scale_mean=np.log(0.04))
    cams = [scenes.ring_camera(k, N_VIEWS, width=40, height=28) for k in range(N_VIEWS)]
    return s, cams


def _pack_bits(b):
    words = (b.size + 31) // 32
    pad = np.zeros(words * 32, bool)
    pad[: b.size] = b
    w = (pad.reshape(words, 32).astype(np.uint64) << np.arange(32, dtype=np.uint64)).sum(1)
    return w.astype(np.uint32).view(np.int32)


def _run_pass(world, rank):
    sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
    from oracle_lib import OracleLib
    from paper_2411_12788_b200 import multiview as MV
    oracle = OracleLib("oracle", "B")
    s, cams = _scene()

    def imp_fn(k, mask_row, accum, counts, max_all):
        r = oracle.render(s, cams[k])
        mask_row.copy_(torch.from_numpy(_pack_bits(r["max_weight"] > THRESH)))
        accum += torch.from_numpy(r["importance"].astype(np.float64))
        counts += torch.from_numpy(r["max_pixel_count"].astype(np.int64))
        torch.maximum(max_all, torch.from_numpy(r["max_weight"]), out=max_all)

    def pts_fn(k):
        r = oracle.render(s, cams[k])
        p, x = oracle.unproject(cams[k], r["max_contributor"], r["alpha"], r["depth"], rule=1, alpha_threshold=0.5,
                                view_index=k, stride=2, seed=3)
        return torch.from_numpy(np.ascontiguousarray(p, np.float32)), torch.from_numpy(x.astype(np.int32))

    masks, accum, counts, mx = MV.importance_views(imp_fn, N_VIEWS, s.n, "cpu")
    pts, views, pix = MV.points_views(pts_fn, N_VIEWS, "cpu")
    return [t.numpy().copy() for t in (masks, accum, counts, mx, pts, views, pix)]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, _run_pass(world, rank)))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_view_blocks_partition_views():
    from paper_2411_12788_b200.multiview import view_block
    for v in (1, 5, 8, 200, 256):
        for w in (1, 2, 3, 4, 8):
            got = [k for r in range(w) for k in view_block(v, r, w)]
            assert got == list(range(v))


def test_two_ranks_match_single_process():
    single = _run_pass(1, 0)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    names = ("masks", "accum", "counts", "max_weight", "points", "views", "pixels")
    for rank in (0, 1):
        for name, a, b in zip(names, res[rank], single):
            if name == "accum":
                assert np.allclose(a, b, rtol=1e-12, atol=0), name
            else:
                assert a.shape == b.shape and np.array_equal(a.view(np.uint8), b.view(np.uint8)), f"rank {rank} {name}"
    assert single[4].shape[0] > 0 and single[0].any()
