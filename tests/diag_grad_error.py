"""Diagnostic (GPU): gradient error triangle GPU / reference float / reference fp64 per block."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
from oracle_lib import OracleLib  # noqa: E402
from paper_2411_12788_b200 import rasterizer as R, scenes  # noqa: E402
from paper_2411_12788_b200.capi import RasterConfig  # noqa: E402


def metrics(a, b):
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64); sc = np.abs(b).max()
    out = {f"el{f:g}": (np.abs(a - b) / np.maximum(np.abs(b), f * sc)).max() for f in (1e-2, 1e-3)}
    out["norm"] = np.linalg.norm(a - b) / np.linalg.norm(b)
    out["max/max"] = np.abs(a - b).max() / sc
    return out


def main():
    o = OracleLib("oracle", "B")
    r = OracleLib("ref", "B")
    cases = {"smoke": (scenes.make_gaussians(2000, seed=0), scenes.fov_camera(128, 96, 60.0, (0, 0, -3))),
             "cfg0": (scenes.make_gaussians(20000, seed=0), scenes.config0_camera())}
    for name, (s, cam) in cases.items():
        want = o.render(s, cam)
        tgt = o.render(scenes.perturbed(s), cam)["color"]
        _, dc = o.l1_loss(want["color"], tgt)
        g32 = o.render_backward(s, cam, dc)
        g64 = r.render_backward_f64(s, cam, dc)
        gg = R.render_backward(s, cam, RasterConfig(), dc)
        print(name)
        for k in g64:
            print(f"  {k:18s} gpu-ref32", {kk: f"{v:.2e}" for kk, v in metrics(gg[k], g32[k]).items()})
            print(f"  {'':18s} gpu-ref64", {kk: f"{v:.2e}" for kk, v in metrics(gg[k], g64[k]).items()})
            print(f"  {'':18s} r32-ref64", {kk: f"{v:.2e}" for kk, v in metrics(g32[k], g64[k]).items()})


if __name__ == "__main__":
    main()
