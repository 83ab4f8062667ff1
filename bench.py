#!/usr/bin/env python3
"""bench.py — fwd+bwd training views/s of the Mini-Splatting2 rasterizer hot path on B200.

Workload (BASELINE.json configs[1], the config the metric is quoted on): 1,000,000 Gaussians
(config-0 distributions, seed 0), SH degree 3, 1237x822 ring views (fov 70 deg, radius 3R,
height 0.5R), L1 loss against targets rendered from the same set with means + N(0, 0.01^2).
One step = per rank `--views` ring views of: preprocess -> (depth, tile) radix sorts -> blend
forward -> fused L1 -> blend backward -> per-Gaussian chain (all 59 gradients), then Adam on means
(lr 1.6e-4); with N > 1 ranks the full 59N-float gradient is exchanged (NCCL reduce-scatter ->
Adam on this rank's shards -> all-gather of the parameters, exchange.py).

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
Multi-GPU: python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "fwd+bwd views/s (1M Gaussians, 1237x822, SH3) at 1/2/4/8 B200 vs CPU ref"
UNIT = "views/s"
RING = 64
REASONS = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--profile-steps", type=int, default=20,
                    help="extra steps after the timed region, with per-kernel CUDA events (breakdown/roofline)")
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", type=int, choices=(1, 2, 3, 4), default=1,
                    help="1: the metric's workload (default); 2: the depth + unprojection pass (3 M Gaussians, "
                         "64 views); 3: the importance / visibility pass (700 K Gaussians, 200 views); 4: BASELINE "
                         "config 4, 3 M Gaussians, 8 views per rank from 256 ring views, the 59N gradient exchange, "
                         "Adam on every group")
    ap.add_argument("--views", type=int, default=None, help="ring views per rank per step (default 1, config 4: 8)")
    ap.add_argument("--gaussians", type=int, default=None, help="default 1 M (config 4: 3 M)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-threads", type=int, default=0)
    ap.add_argument("--comm", choices=("torch", "native"), default="torch",
                    help="N > 1 exchange: torch.distributed NCCL collectives (exchange.py) or the library's own "
                         "NCCL communicator inside splat_train_step")
    ap.add_argument("--buckets", type=int, default=8, help="exchange buckets (reduce-scatter / Adam pipelining)")
    a = ap.parse_args()
    if a.views is None:
        a.views = {4: 8, 2: 64, 3: 200}.get(a.config, 1)
    if a.gaussians is None:
        a.gaussians = {4: 3_000_000, 2: 3_000_000, 3: 700_000}.get(a.config, 1_000_000)
    if a.config in (2, 3) and "--steps" not in sys.argv:
        a.steps, a.warmup, a.profile_steps = 5, 3, 1
    return a


METRIC4 = "fwd+bwd views/s (3M Gaussians, 1237x822, SH3, 8 views/GPU, all-param Adam) at 1/2/4/8 B200"


def workload_config(args, world):
    if args.config == 4:
        return {"workload": "cfg4: 3M Gaussians SH3, 8 ring views per rank per step from 256, 1237x822, L1 vs "
                            "perturbed-means target, fwd+bwd summed over views, 59N-float gradient all-reduce, "
                            "Adam on all parameter groups",
                "gaussians": args.gaussians, "width": 1237, "height": 822, "views_per_rank_per_step": args.views,
                "ring_views": 256, "n_ranks": world,
                "allreduce": "59N gradient floats (fp32) when N > 1: NCCL reduce-scatter -> sharded Adam -> all-gather",
                "l2": "inputs larger than L2; views rotate each step", "scene_seed": 0}
    return {"workload": "cfg1: 1M Gaussians SH3, 1237x822 ring views, L1 vs perturbed-means target, "
                        "fwd+bwd (59 grads) + Adam(means, lr 1.6e-4)",
            "gaussians": args.gaussians, "width": 1237, "height": 822, "views_per_rank_per_step": args.views,
            "ring_views": RING, "n_ranks": world,
            "allreduce": "59N gradient floats (fp32) when N > 1: NCCL reduce-scatter -> sharded Adam -> all-gather",
            "l2": "inputs larger than L2 (236 MB parameters + 59N-float gradients and Adam moments, ~100 MB of per-view records and lists); views rotate each step",
            "scene_seed": 0}


# ---------------------------------------------------------------------------------------------
# CPU reference (oracle/_ref, the reference's own sources; test infrastructure, never the product)
# ---------------------------------------------------------------------------------------------
def _ref_lib():
    lib_path = ROOT / "oracle" / "_ref" / "libsplat_ref_libm.so"
    kind = "reference"
    if not lib_path.exists():
        return None, None
    from paper_2411_12788_b200.capi import AdamConfig, Camera, Gaussians, RasterConfig
    lib = C.CDLL(str(lib_path))
    lib.ref_scene_create.restype = C.c_void_p
    lib.ref_scene_create.argtypes = [C.POINTER(Gaussians), C.POINTER(AdamConfig)]
    lib.ref_scene_destroy.argtypes = [C.c_void_p]
    lib.ref_train_view.restype = C.c_int
    lib.ref_train_view.argtypes = [C.c_void_p, C.POINTER(Camera), C.POINTER(RasterConfig),
                                   C.POINTER(C.c_float), C.POINTER(C.c_float)]
    return lib, kind


class CpuReference:
    """The reference's own render -> l1_loss -> render_backward -> OptimState::step (means) on
    `threads` host threads (oracle/_ref, compiled in place from the reference's sources), each
    training one config-1 ring view per round on its own copy of the scene."""

    def __init__(self, n_gaussians, threads):
        from paper_2411_12788_b200 import scenes
        from paper_2411_12788_b200.capi import AdamConfig, Gaussians, RasterConfig
        self.lib, self.kind = _ref_lib()
        if self.lib is None:
            raise RuntimeError("oracle/_ref/libsplat_ref_libm.so not built")
        s = scenes.make_gaussians(n_gaussians, seed=0)
        self.arrs = [np.ascontiguousarray(a, np.float32) for a in (s.centers, s.log_scales, s.rotations,
                                                                   s.opacity_logits, s.sh)]
        fp = C.POINTER(C.c_float)
        g = Gaussians(*[a.ctypes.data_as(fp) for a in self.arrs], s.n, 3)
        adam = AdamConfig()
        self.cfg = RasterConfig()
        self.threads = threads
        self.cams = [scenes.ring_camera(k, RING) for k in range(threads)]
        # targets: a cheap deterministic stand-in image per view (the target render is not part of
        # the step); value range matches a render.
        rng = np.random.default_rng(0)
        self.tgt = [np.ascontiguousarray(rng.uniform(0, 1, size=(822, 1237, 3)).astype(np.float32))
                    for _ in range(threads)]
        self.handles = [self.lib.ref_scene_create(C.byref(g), C.byref(adam)) for _ in range(threads)]
        if not all(self.handles):
            self.close()
            raise RuntimeError("reference scene allocation failed")

    def round(self):
        """One view per thread, all threads in parallel; returns the wall seconds."""
        fp = C.POINTER(C.c_float)
        errors = []

        def work(i):
            loss = C.c_float()
            rc = self.lib.ref_train_view(self.handles[i], C.byref(self.cams[i]), C.byref(self.cfg),
                                         self.tgt[i].ctypes.data_as(fp), C.byref(loss))
            if rc:
                errors.append(rc)

        th = [threading.Thread(target=work, args=(i,)) for i in range(self.threads)]
        t0 = time.perf_counter()
        for t in th:
            t.start()
        for t in th:
            t.join()
        wall = time.perf_counter() - t0
        if errors:
            raise RuntimeError(f"reference train_view failed: {errors[:3]}")
        return wall

    def close(self):
        for hnd in self.handles:
            if hnd:
                self.lib.ref_scene_destroy(hnd)
        self.handles = []


def cpu_threads_default(args, cap):
    return args.cpu_threads or max(1, min(os.cpu_count() or 1, cap))


def cpu_views_per_s(n_gaussians, threads, rounds=1):
    """Bounded CPU-baseline sample: `rounds` rounds of one view per thread."""
    ref = CpuReference(n_gaussians, threads)
    try:
        wall = sum(ref.round() for _ in range(rounds))
    finally:
        ref.close()
    return {"value": threads * rounds / wall, "unit": UNIT, "cores": threads, "kind": ref.kind,
            "sample": f"{threads} threads x {rounds} config-1 ring view(s) each through the reference's own "
                      f"render<float> -> l1_loss -> render_backward<float> -> OptimState::step (means), "
                      f"{wall:.1f} s wall", "seconds": wall, "asymmetry": REF_ASYMMETRY}


REF_BUDGET_S = 150.0  # whole reference arm: warm-up + timed rounds
# stated in both arms' cpu_baseline: what the reference does differently per view
REF_ASYMMETRY = ("targets are seeded uniform noise (the perturbed-set render is not part of the step; the L1 "
                 "gradient has the same cost); OptimState::step runs over every group with the non-means "
                 "gradients zero (the reference has no group mask: about 0.4 s of its ~5.8 s per view, measured "
                 "with ref_adam_steps at 1 M), while the GPU arm steps the means group only")


def run_reference_arm(args):
    """The reference's own CPU implementation of the path (oracle/_ref) on the host cores, same
    metric/config as our arm.  Each step is one round of one config-1 view per host thread (a
    bounded sample of the workload); the number of timed steps is capped so the whole arm ends
    within REF_BUDGET_S, and the line reports the steps actually timed."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    threads = cpu_threads_default(args, 64)
    lib, _ = _ref_lib()
    if lib is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libsplat_ref_libm.so not built"}))
        return
    t_start = time.perf_counter()
    ref = CpuReference(args.gaussians, threads)
    try:
        first = ref.round() if args.warmup > 0 else None  # one untimed warm-up round bounds the rest
        per = first if first else 6.0
        steps = max(1, min(args.steps, int((REF_BUDGET_S - (time.perf_counter() - t_start)) / per)))
        t_total = sum(ref.round() for _ in range(steps))
    finally:
        ref.close()
    views = threads * steps
    value = views / t_total
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": steps,
            "warmup": 1 if args.warmup > 0 else 0, "steps_requested": args.steps, "warmup_requested": args.warmup,
            "ms_per_step": 1000 * t_total / steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded, BASELINE cfg1 shapes)",
            "config": workload_config(args, world), "impl": "reference",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                             "sample": f"{threads} threads x 1 config-1 view per step, {steps} timed step(s) "
                                       f"(capped to a {REF_BUDGET_S:.0f} s arm); the reference's own C++ "
                                       f"compiled in place, glibc expf",
                             "asymmetry": REF_ASYMMETRY},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


# ---------------------------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clock / throttle-reason sampling (every 50 ms) around the timed region.

    start() waits for the first sample so the sampler is live before the timed region; stop()
    summarises the samples taken inside [t0, t1] (monotonic seconds, the timed region), falling
    back to the samples nearest to it when the region is shorter than the sampling period."""

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self, wait_s=5.0):
        q = "clocks.sm,clocks.max.sm,power.draw," + ",".join(f"clocks_event_reasons.{r}" for r in REASONS)
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.device}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
            return
        t_end = time.monotonic() + wait_s
        while not self.lines and time.monotonic() < t_end:
            time.sleep(0.01)

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append((time.monotonic(), ln.strip()))

    def stop(self, t0, t1):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.06)  # one more period so the sample covering t1 arrives
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        parsed = []
        for ts, ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 3 + len(REASONS):
                continue
            try:
                parsed.append((ts, float(parts[0]), float(parts[1]),
                               {r for r, v in zip(REASONS, parts[3:]) if v.lower().startswith("active")}))
            except ValueError:
                continue
        inside = [p for p in parsed if t0 <= p[0] <= t1 + 0.05]
        sel = inside or sorted(parsed, key=lambda p: min(abs(p[0] - t0), abs(p[0] - t1)))[:2]
        if not sel:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        reasons = set().union(*(p[3] for p in sel))
        return {"sm_mhz": float(np.median([p[1] for p in sel])), "sm_max_mhz": sel[-1][2], "reasons": sorted(reasons),
                "samples": len(sel), "samples_in_timed_region": len(inside)}


def ncu_summary(kernel):
    """The committed ncu --set full summary of `kernel` (profiles/ncu_summary.json), if any."""
    p = ROOT / "profiles" / "ncu_summary.json"
    try:
        return json.loads(p.read_text())["kernels"].get(kernel)
    except Exception:
        return None


def algorithmic_bytes(kernel, n, n_surv, pairs, hw):
    """Compulsory HBM bytes per launch (SURVEY.md §8d terms)."""
    if kernel == "blend_backward":
        # sorted ids 4P + projected records 48 B/Gaussian + per-pixel T, last, colour, target (32 B)
        # + 2D gradient accumulators 48 B/Gaussian
        return 4 * pairs + 48 * n_surv + 32 * hw + 48 * n_surv
    if kernel == "blend_forward":
        return 4 * pairs + 48 * n_surv + 20 * hw  # ids + records + colour 12, T 4, last 4
    if kernel == "chain_compact":
        return 16 * n + 236 * n + 4 * n  # commit counts read, every gradient row zeroed, touched list
    if kernel == "chain":
        return None  # touched Gaussians only: ~650 B each (params, rec, grad2d, gradients)
    if kernel == "preprocess":
        return 236 * n + 48 * n + 12 * n
    return None


def run_ours(args):
    import torch
    import torch.distributed as dist

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    else:
        torch.cuda.set_device(0)
    device = torch.cuda.current_device()

    from paper_2411_12788_b200 import capi, scenes
    from paper_2411_12788_b200.rasterizer import Context, DeviceGaussians, render
    from paper_2411_12788_b200.trainer import ViewTrainer

    ctx = Context.default(device)
    s = scenes.make_gaussians(args.gaussians, seed=0)
    ds = DeviceGaussians.from_host(s, device)
    dt = DeviceGaussians.from_host(scenes.perturbed(s), device)
    ring = 256 if args.config == 4 else RING
    cams = [scenes.ring_camera(k, ring) for k in range(ring)]
    targets = [render(dt, cam, want_depth=False, ctx=ctx).color.clone() for cam in cams]
    del dt
    gmask = capi.GROUP_ALL if args.config == 4 else capi.GROUP_CENTERS
    trainer = ViewTrainer(ds, capi.AdamConfig(), group_mask=gmask, ctx=ctx, max_views=max(args.views, 1),
                          buckets=args.buckets, native_comm=(world > 1 and args.comm == "native"))
    V = args.views

    from paper_2411_12788_b200.trainer import views_for as _views_for

    def views_for(step):
        idx = _views_for(step, rank, world, V, ring)
        return [cams[i] for i in idx], [targets[i] for i in idx], idx

    stream = torch.cuda.current_stream()
    clocks = ClockSampler(device)
    clocks.start()
    for st in range(args.warmup):
        c, t, _ = views_for(st)
        trainer.step(c, t)
    torch.cuda.synchronize()

    # ---- device-timed region -----------------------------------------------------------------
    lib = ctx.lib
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = ctx.launches()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_wall0 = time.monotonic()
    ev0.record(stream)
    pairs, survivors = [], []
    for st in range(args.warmup, args.warmup + args.steps):
        c, t, _ = views_for(st)
        trainer.step(c, t)
    ev1.record(stream)
    torch.cuda.synchronize()
    t_wall1 = time.monotonic()
    if world > 1:
        dist.barrier()
    launches = ctx.launches() - launches0
    clk = clocks.stop(t_wall0, t_wall1)
    ms = ev0.elapsed_time(ev1)

    # ---- per-kernel breakdown: a separate profiled pass (CUDA events around every launch) ------
    lib.splat_profile_enable(ctx.h, 1)
    p_steps = max(1, args.profile_steps)
    if trainer.exchange is not None:
        trainer.exchange.events = []
    for st in range(args.warmup + args.steps, args.warmup + args.steps + p_steps):
        c, t, _ = views_for(st)
        trainer.step(c, t)
        pairs += trainer.pairs_last_step  # (host queries outside the timed region)
        survivors += trainer.survivors_last_step
    torch.cuda.synchronize()
    names = C.create_string_buffer(4096)
    tot = (C.c_double * 64)()
    cnt = (C.c_int64 * 64)()
    nk = C.c_int()
    ctx.check(lib.splat_profile_read(ctx.h, names, 4096, tot, cnt, 64, C.byref(nk)))
    lib.splat_profile_enable(ctx.h, 0)
    kern = {nm: (tot[i], cnt[i]) for i, nm in enumerate(names.value.decode().split("\n")[: nk.value])}
    allreduce = None
    if trainer.exchange is not None and trainer.exchange.events:
        ex = trainer.exchange
        ar_ms = float(np.mean([a.elapsed_time(b) for a, b in ex.events]))
        nbytes = 59 * trainer.params.n * 4
        allreduce = {"bytes": nbytes, "ms": ar_ms, "algbw_gbs": nbytes / (ar_ms * 1e6),
                     "busbw_gbs": 2 * (world - 1) / world * nbytes / (ar_ms * 1e6), "buckets": ex.buckets,
                     "note": "whole exchange of the 59N-float packed gradient: bucketed NCCL reduce-scatter -> "
                             "Adam on this rank's shards -> all-gather of the parameters -> quaternion renorm "
                             "(CUDA events on the compute stream, profiled pass)"}
        ex.events = None
    if world > 1:
        t_ms = torch.tensor([ms], device=f"cuda:{device}", dtype=torch.float64)
        dist.all_reduce(t_ms, op=dist.ReduceOp.MAX)
        ms = float(t_ms.item())
    total_views = world * V * args.steps
    value = total_views / (ms / 1000.0)

    # ---- V / C of one ring view (traverse_pixel visits and commits; a measurement pass) -----------
    vc = None
    if rank == 0 and args.config in (1, 4):
        from paper_2411_12788_b200.rasterizer import render, traversal_counts
        render(trainer.params, cams[0], ctx=ctx, want_depth=False)
        vc = traversal_counts(ctx)
        torch.cuda.synchronize()

    # ---- e2e through the public API with host buffers -------------------------------------------
    e2e = None
    if not args.no_e2e:
        host_t = [targets[i].cpu().pin_memory() for i in range(min(ring, 8 * V))]
        for st in range(2):
            c, _, idx = views_for(st)
            trainer.step_host(c, [host_t[i % len(host_t)] for i in idx])
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for st in range(args.steps):
            c, _, idx = views_for(st)
            trainer.step_host(c, [host_t[i % len(host_t)] for i in idx])
        e1.record(stream)
        torch.cuda.synchronize()
        ems = e0.elapsed_time(e1)
        if world > 1:
            t_ms = torch.tensor([ems], device=f"cuda:{device}", dtype=torch.float64)
            dist.all_reduce(t_ms, op=dist.ReduceOp.MAX)
            ems = float(t_ms.item())
        e2e = {"value": total_views / (ems / 1000.0), "unit": UNIT,
               "h2d_bytes_per_step": int(V * 822 * 1237 * 3 * 4), "d2h_bytes_per_step": int(V * 4),
               "path": "ViewTrainer.step_host: pinned host target -> device copy, C-ABI render/backward_l1/adam, "
                       "loss read back each step"}

    # ---- roofline of the dominant kernel (CUDA events around every launch, timed region) ----------
    peaks_path = ROOT / "MEASURED_PEAKS.json"
    peak, peak_src = 6537.6, "MEASURED_PEAKS.json hbm_gbs (fallback if absent)"
    if peaks_path.exists():
        try:
            peak = float(json.loads(peaks_path.read_text())["hbm_gbs"])
            peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)"
        except Exception:
            pass
    dom = max(kern.items(), key=lambda kv: kv[1][0])[0] if kern else None
    n_views = len(pairs)
    hw = 1237 * 822
    n = args.gaussians
    avg_pairs = float(np.mean(pairs)) if pairs else 0.0
    n_surv = float(np.mean(survivors)) if survivors else n
    roof = None
    if dom:
        ab = algorithmic_bytes(dom, n, n_surv, avg_pairs, hw)
        avg_ms = kern[dom][0] / max(kern[dom][1], 1)
        if ab:
            achieved = ab / (avg_ms / 1000.0) / 1e9
            roof = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                    "frac": achieved / peak, "traffic": None, "algorithmic_bytes_per_launch": ab,
                    "avg_launch_ms": avg_ms, "peak_source": peak_src,
                    "note": "blend kernels are issue-bound (FP32/SFU/LSU on staged records), not HBM-bound"}
            ncu = ncu_summary(dom)
            if ncu:
                roof["traffic"] = ncu.get("dram_bytes_per_launch")
                roof["ncu"] = ncu
    # FP32 peak: SMs x 128 lanes x 2 flop x the SM clock under load (nvidia-smi median in the timed
    # region), and at the maximum clock
    sms = torch.cuda.get_device_properties(device).multi_processor_count
    clk_mhz = (clk or {}).get("sm_mhz") or 1965.0
    fp32_peak = sms * 128 * 2 * clk_mhz * 1e6 / 1e12  # TFLOP/s
    if roof and vc and dom in ("blend_backward", "blend_forward"):
        V, Cc = vc
        fl = (15.0 * V + 45.0 * Cc) if dom == "blend_backward" else (15.0 * V + 12.0 * Cc)
        tf = fl / (roof["avg_launch_ms"] / 1000.0) / 1e12
        roof.update({"flops_per_launch": fl, "achieved_tflops": tf, "fp32_peak_tflops": fp32_peak,
                     "fp32_frac": tf / fp32_peak, "frac_max": max(roof["frac"], tf / fp32_peak),
                     "flops_model": "SURVEY.md 8d: backward 15 V + 45 C, forward 15 V + 12 C (V, C measured)"})
    # whole-step roofline (SURVEY.md §8d compulsory traffic: 1020 N + 12 P + 60 HW bytes per view at
    # config 1, Adam on means; FP32 work 600 N + 15 V + 12 C (fwd) + 15 V + 45 C (bwd) + 900 N (chain)),
    # max(bytes / HBM peak, flops / FP32 peak) / measured time
    step_roof = None
    if args.config == 1 and n_views:
        bpv = 1020.0 * n + 12.0 * avg_pairs + 60.0 * hw
        ach = bpv * value / world / 1e9  # per GPU
        step_roof = {"bytes_per_view": bpv, "achieved_gbs_per_gpu": ach, "peak": peak, "frac": ach / peak,
                     "note": "SURVEY.md 8d algorithmic bytes of the whole view (fwd + bwd + Adam on means)"}
        if vc:
            V, Cc = vc
            fpv = 1500.0 * n + 30.0 * V + 57.0 * Cc
            t_view = world / value  # s per view per GPU
            step_roof.update({"visits_per_view": V, "commits_per_view": Cc, "flops_per_view": fpv,
                              "achieved_tflops_per_gpu": fpv / t_view / 1e12, "fp32_peak_tflops": fp32_peak,
                              "fp32_frac": fpv / t_view / 1e12 / fp32_peak,
                              "frac_max": max(bpv / (peak * 1e9), fpv / (fp32_peak * 1e12)) / t_view})
    breakdown = {k: {"ms_per_step": v[0] / p_steps, "launches_per_step": v[1] / p_steps,
                     "share": v[0] / max(sum(x[0] for x in kern.values()), 1e-9)} for k, v in kern.items()}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and args.config == 1:
        threads = cpu_threads_default(args, 16)
        try:
            cpu = cpu_views_per_s(args.gaussians, threads, 1)
            if cpu:
                cpu.pop("seconds", None)
        except Exception as e:  # reported, not fatal
            cpu = {"value": None, "unit": UNIT, "cores": threads, "kind": "reference", "sample": f"failed: {e}"}

    if rank == 0:
        line = {"metric": METRIC4 if args.config == 4 else METRIC, "value": value, "unit": UNIT, "n_gpus": world,
                "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f32",
                "data": f"synthetic (seeded, BASELINE cfg{args.config} shapes)",
                "config": workload_config(args, world), "e2e": e2e, "gpu_launches": int(launches),
                "roofline": roof, "step_roofline": step_roof, "cpu_baseline": cpu, "clocks": clk,
                "pairs_per_view": avg_pairs, "survivors_per_view": n_surv,
                "visits_per_view": vc[0] if vc else None, "commits_per_view": vc[1] if vc else None,
                "kernel_breakdown": breakdown}
        if allreduce:
            line["allreduce"] = allreduce
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


# ---------------------------------------------------------------------------------------------
# configs 2 and 3: the two per-view passes (depth + unprojection, importance / visibility)
# ---------------------------------------------------------------------------------------------
PASS_METRIC = {2: "depth+unproject views/s (3M Gaussians, 1237x822, 64 ring views, alpha>0.5, stride 4)",
               3: "importance+visibility views/s (700K Gaussians, 1237x822, 200 ring views)"}


def pass_config(args, world):
    if args.config == 2:
        return {"workload": "cfg2: depth render + unprojection of every pixel with alpha > 0.5 and (view*HW + pixel) "
                            "% 4 == 0 over 64 ring views (aggressive densification's depth pass)",
                "gaussians": args.gaussians, "log_scale_mean": "ln 0.005", "width": 1237, "height": 822,
                "views_per_step": args.views, "n_ranks": world, "scene_seed": 0,
                "l2": "inputs larger than L2 (708 MB parameters); 64 distinct views per step"}
    return {"workload": "cfg3: accumulate_importance per view -> per-view visibility bitmask (max blend weight > "
                        "1e-3), fp64 global importance, argmax counts, over 200 ring views",
            "gaussians": args.gaussians, "width": 1237, "height": 822, "views_per_step": args.views,
            "n_ranks": world, "scene_seed": 0,
            "l2": "inputs larger than L2 (165 MB parameters); 200 distinct views per step"}


def cpu_pass_views_per_s(args, threads):
    """The reference's own render<float> (cfg 2: colour, alpha, depth, argmax; the unprojection loop
    over the pixels is not included) or accumulate_importance<float> (cfg 3), one ring view per host
    thread, all threads in parallel."""
    from paper_2411_12788_b200 import scenes
    from paper_2411_12788_b200.capi import Camera, Gaussians, RasterConfig
    lib = C.CDLL(str(ROOT / "oracle" / "_ref" / "libsplat_ref_libm.so"))
    ls = np.log(0.005) if args.config == 2 else np.log(0.02)
    s = scenes.make_gaussians(args.gaussians, seed=0, log_scale_mean=ls)
    arrs = [np.ascontiguousarray(a, np.float32) for a in (s.centers, s.log_scales, s.rotations, s.opacity_logits, s.sh)]
    fp = C.POINTER(C.c_float)
    g = Gaussians(*[a.ctypes.data_as(fp) for a in arrs], s.n, 3)
    cfg = RasterConfig()
    cams = [scenes.ring_camera(k, args.views) for k in range(threads)]
    hw = 1237 * 822
    errors = []

    def work(i):
        if args.config == 2:
            col = np.empty(hw * 3, np.float32)
            a = np.empty(hw, np.float32)
            d = np.empty(hw, np.float32)
            t = np.empty(hw, np.float32)
            mc = np.empty(hw, np.int32)
            bg = (C.c_float * 3)(0, 0, 0)
            rc = lib.ref_render(C.byref(g), C.byref(cams[i]), C.byref(cfg), None, bg, col.ctypes.data_as(fp),
                                a.ctypes.data_as(fp), d.ctypes.data_as(fp), t.ctypes.data_as(fp),
                                mc.ctypes.data_as(C.POINTER(C.c_int32)), None, None, None, None)
        else:
            imp = np.empty(s.n, np.float32)
            mw = np.empty(s.n, np.float32)
            mp = np.empty(s.n, np.int32)
            rc = lib.ref_accumulate_importance(C.byref(g), C.byref(cams[i]), C.byref(cfg), None, imp.ctypes.data_as(fp),
                                               mw.ctypes.data_as(fp), mp.ctypes.data_as(C.POINTER(C.c_int32)))
        if rc:
            errors.append(rc)

    th = [threading.Thread(target=work, args=(i,)) for i in range(threads)]
    t0 = time.perf_counter()
    for t in th:
        t.start()
    for t in th:
        t.join()
    wall = time.perf_counter() - t0
    if errors:
        raise RuntimeError(f"reference pass failed: {errors[:3]}")
    what = "render<float>" if args.config == 2 else "accumulate_importance<float>"
    return {"value": threads / wall, "unit": UNIT, "cores": threads, "kind": "reference",
            "sample": f"{threads} threads x 1 cfg{args.config} ring view each through the reference's own {what}, "
                      f"{wall:.1f} s wall"}


def run_pass(args):
    """Configs 2 / 3: one step = the whole multi-view pass (views partitioned across ranks, results
    gathered in view order)."""
    import torch
    import torch.distributed as dist
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    else:
        torch.cuda.set_device(0)
    device = torch.cuda.current_device()
    from paper_2411_12788_b200 import capi, multiview as MV, scenes
    from paper_2411_12788_b200.rasterizer import Context, DeviceGaussians
    ctx = Context.default(device)
    ls = np.log(0.005) if args.config == 2 else np.log(0.02)
    s = scenes.make_gaussians(args.gaussians, seed=0, log_scale_mean=ls)
    ds = DeviceGaussians.from_host(s, device)
    cams = [scenes.ring_camera(k, args.views) for k in range(args.views)]

    def one_pass(set_):
        if args.config == 2:
            return MV.depth_points_views(set_, cams, rule=capi.DEPTH_RULE_ALPHA, alpha_threshold=0.5, stride=4,
                                         seed=0, ctx=ctx)
        return MV.visibility_pass_views(set_, cams, threshold=1e-3, ctx=ctx)

    stream = torch.cuda.current_stream()
    clocks = ClockSampler(device)
    clocks.start()
    for _ in range(args.warmup):
        out = one_pass(ds)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches0 = ctx.launches()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_wall0 = time.monotonic()
    ev0.record(stream)
    for _ in range(args.steps):
        out = one_pass(ds)
    ev1.record(stream)
    torch.cuda.synchronize()
    t_wall1 = time.monotonic()
    launches = ctx.launches() - launches0
    clk = clocks.stop(t_wall0, t_wall1)
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        t_ms = torch.tensor([ms], device=f"cuda:{device}", dtype=torch.float64)
        dist.all_reduce(t_ms, op=dist.ReduceOp.MAX)
        ms = float(t_ms.item())
    value = args.views * args.steps / (ms / 1000.0)
    n_points = int(out[0].shape[0]) if args.config == 2 else None

    # per-kernel breakdown (a profiled pass) and the per-view pair counts
    ctx.lib.splat_profile_enable(ctx.h, 1)
    one_pass(ds)
    torch.cuda.synchronize()
    names = C.create_string_buffer(4096)
    tot = (C.c_double * 64)()
    cnt = (C.c_int64 * 64)()
    nk = C.c_int()
    ctx.check(ctx.lib.splat_profile_read(ctx.h, names, 4096, tot, cnt, 64, C.byref(nk)))
    ctx.lib.splat_profile_enable(ctx.h, 0)
    kern = {nm: (tot[i], cnt[i]) for i, nm in enumerate(names.value.decode().split("\n")[: nk.value])}
    ns_, np_ = C.c_int64(), C.c_int64()
    pairs = []
    for cam in cams[:: max(1, args.views // 8)]:
        if args.config == 2:
            from paper_2411_12788_b200.rasterizer import render
            render(ds, cam, ctx=ctx, want_depth=True)
        else:
            MV.visibility_pass_views(ds, [cam], ctx=ctx)
        ctx.lib.splat_forward_counts(ctx.h, C.byref(ns_), C.byref(np_), None, None)
        pairs.append(np_.value)
    avg_pairs = float(np.mean(pairs))

    # e2e: the Gaussian set from pinned host memory, the pass, the results read back to the host
    host_flat = ds.flat.cpu().pin_memory()
    ds2 = DeviceGaussians(s.n, 3, device)
    h2d = host_flat.numel() * 4
    d2h = 0

    pinned = {}

    def e2e_pass():
        ds2.flat.copy_(host_flat, non_blocking=True)
        res = one_pass(ds2)
        out = []
        for k, r in enumerate(res):  # read back into pinned host buffers (reused across passes)
            h = pinned.get(k)
            if h is None or h.shape != r.shape or h.dtype != r.dtype:
                h = pinned[k] = torch.empty(r.shape, dtype=r.dtype, pin_memory=True)
            h.copy_(r, non_blocking=True)
            out.append(h)
        torch.cuda.current_stream().synchronize()
        return out

    for _ in range(2):
        res = e2e_pass()
    d2h = sum(r.numel() * r.element_size() for r in res)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        e2e_pass()
    e1.record(stream)
    torch.cuda.synchronize()
    ems = e0.elapsed_time(e1)
    if world > 1:
        t_ms = torch.tensor([ems], device=f"cuda:{device}", dtype=torch.float64)
        dist.all_reduce(t_ms, op=dist.ReduceOp.MAX)
        ems = float(t_ms.item())
    e2e = {"value": args.views * args.steps / (ems / 1000.0), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
           "d2h_bytes_per_step": int(d2h),
           "path": "Gaussian set from pinned host memory -> device, the multiview pass through the C-ABI, "
                   + ("points / views / pixels" if args.config == 2 else "bitmasks / fp64 importance / counts")
                   + " read back to the host"}

    peak, peak_src = 6453.1, "fallback"
    try:
        peak = float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"])
        peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        pass
    dom = max(kern.items(), key=lambda kv: kv[1][0])[0] if kern else None
    roof = None
    if dom:
        avg_ms = kern[dom][0] / max(kern[dom][1], 1)
        hw = 1237 * 822
        n = args.gaussians
        # ids 4 P + records 48 B per Gaussian + outputs: cfg 2 colour / alpha / depth / argmax per
        # pixel (24 B); cfg 3 the importance report (sum, max weight, argmax count: 12 B per Gaussian)
        out_b = 24 * hw if args.config == 2 else 12 * n
        ab = {"blend_forward": 4 * avg_pairs + 48 * n + out_b, "preprocess": 236 * n + 48 * n + 12 * n}.get(dom)
        if ab:
            achieved = ab / (avg_ms / 1000.0) / 1e9
            roof = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                    "frac": achieved / peak, "traffic": None, "algorithmic_bytes_per_launch": ab,
                    "avg_launch_ms": avg_ms, "peak_source": peak_src}
        else:
            roof = {"kernel": dom, "avg_launch_ms": avg_ms, "note": "no algorithmic-bytes model for this kernel"}
    breakdown = {k: {"ms_per_step": v[0], "launches_per_step": v[1],
                     "share": v[0] / max(sum(x[0] for x in kern.values()), 1e-9)} for k, v in kern.items()}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = cpu_threads_default(args, 16)
        try:
            cpu = cpu_pass_views_per_s(args, threads)
        except Exception as e:
            cpu = {"value": None, "unit": UNIT, "cores": threads, "kind": "reference", "sample": f"failed: {e}"}
    if rank == 0:
        line = {"metric": PASS_METRIC[args.config], "value": value, "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f32",
                "data": f"synthetic (seeded, BASELINE cfg{args.config} shapes)", "config": pass_config(args, world),
                "e2e": e2e, "gpu_launches": int(launches), "roofline": roof, "cpu_baseline": cpu, "clocks": clk,
                "pairs_per_view": avg_pairs, "kernel_breakdown": breakdown}
        if n_points is not None:
            line["points_per_step"] = n_points
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference_arm(args)
    elif args.config in (2, 3):
        run_pass(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
