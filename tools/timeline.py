#!/usr/bin/env python3
"""GPU timeline of config-1 training steps (CUPTI kernel records through torch.profiler): per kernel
start offset, duration and the idle gap before it, to find launch gaps and serialisation.

    python tools/timeline.py [steps] [warmup]      (prints one table per profiled step)
"""
import json
import sys
import tempfile
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2411_12788_b200 import capi, scenes  # noqa: E402
from paper_2411_12788_b200.rasterizer import Context, DeviceGaussians, render  # noqa: E402
from paper_2411_12788_b200.trainer import ViewTrainer  # noqa: E402


def main(steps: int = 3, warmup: int = 5, host: bool = False):
    torch.cuda.set_device(0)
    ctx = Context.default(0)
    s = scenes.make_gaussians(1_000_000, seed=0)
    ds = DeviceGaussians.from_host(s, 0)
    dt = DeviceGaussians.from_host(scenes.perturbed(s), 0)
    cams = [scenes.ring_camera(k, 64) for k in range(warmup + steps)]
    targets = [render(dt, c, want_depth=False, ctx=ctx).color.clone() for c in cams]
    del dt
    host_t = [t.cpu().pin_memory() for t in targets]
    tr = ViewTrainer(ds, capi.AdamConfig(), group_mask=capi.GROUP_CENTERS, ctx=ctx)
    step = (lambda k: tr.step_host([cams[k]], [host_t[k]])) if host else (lambda k: tr.step([cams[k]], [targets[k]]))
    for k in range(warmup):
        step(k)
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        for k in range(warmup, warmup + steps):
            step(k)
            torch.cuda.synchronize()
    path = Path(tempfile.mkdtemp()) / "trace.json"
    prof.export_chrome_trace(str(path))
    ev = json.load(open(path))["traceEvents"]
    ks = sorted([e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")], key=lambda e: e["ts"])
    if "--api" in sys.argv:  # host-side runtime calls between the last two preprocess launches
        api = sorted([e for e in ev if e.get("cat") == "cuda_runtime"], key=lambda e: e["ts"])
        pre = [e for e in api if "Launch" in e["name"] or "Memcpy" in e["name"] or "Memset" in e["name"]
               or "Synchronize" in e["name"] or "Event" in e["name"]]
        t0 = pre[len(pre) // 2]["ts"] if pre else 0
        for e in pre[len(pre) // 2: len(pre) // 2 + 60]:
            print(f"API {e['ts'] - t0:9.1f} {e['dur']:8.1f}  {e['name']}")
        # host time between the end of one step's final synchronisation and the next step's
        # first runtime call (Python + ctypes overhead of the public API)
        syncs = [e for e in api if "Synchronize" in e["name"]]
        gaps = []
        for a in syncs:
            end = a["ts"] + a["dur"]
            nxt = [e for e in api if e["ts"] >= end and "Synchronize" not in e["name"]]
            if nxt:
                gaps.append(nxt[0]["ts"] - end)
        if gaps:
            print("inter-step host gaps (us):", [round(g, 1) for g in gaps])
    # split into steps at the preprocess kernel
    cur, all_steps = [], []
    for e in ks:
        if "preprocess" in e["name"] and cur:
            all_steps.append(cur)
            cur = []
        cur.append(e)
    all_steps.append(cur)
    for si, st in enumerate(all_steps):
        t0 = st[0]["ts"]
        end = t0
        busy = 0.0
        print(f"--- step {si}: {len(st)} records")
        for e in st:
            gap = e["ts"] - end
            nm = e["name"].replace("void ", "").replace("splat_b200::", "").replace("(anonymous namespace)::", "")
            nm = nm.split("(")[0][:40]
            print(f"{e['ts'] - t0:9.1f} {e['dur']:8.1f} gap {gap:7.1f}  s{e.get('args', {}).get('stream', '?')}  {nm}")
            end = max(end, e["ts"] + e["dur"])
            busy += e["dur"]
        print(f"step span {end - t0:.1f} us, kernel+copy busy {busy:.1f} us")


if __name__ == "__main__":
    a = sys.argv[1:]
    main(int(a[0]) if a else 3, int(a[1]) if len(a) > 1 else 5, "--host" in a)
