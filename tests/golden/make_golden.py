#!/usr/bin/env python3
"""Generate tests/golden/*.npz from the REFERENCE's own code (oracle/_ref, built in place from
/root/reference/proj/src against oracle/compat/Eigen by oracle/Makefile).

Run in the build container (where /root/reference exists):  python tests/golden/make_golden.py
The fixtures pin the C restatement (oracle/splat_oracle.c) and, through it, the CUDA path, on
machines without the reference sources (e.g. the GPU box).

Each fixture stores the inputs (Gaussians, camera, raster config, background, d_color, mask) and
the reference outputs in both exp modes:
  mode B (splat_expf, the exp the CUDA path uses): expected bit-exact;
  mode A (glibc expf, the reference as shipped): for information / tolerance checks.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]

from oracle_lib import OracleLib  # noqa: E402
from paper_2411_12788_b200 import scenes  # noqa: E402
from paper_2411_12788_b200.capi import RasterConfig  # noqa: E402

OUT = Path(__file__).resolve().parent


def cam_to_arrays(cam):
    return dict(cam_wh=np.array([cam.width, cam.height], np.int32),
                cam_intr=np.array([cam.fx, cam.fy, cam.cx, cam.cy, cam.znear, cam.zfar], np.float32),
                cam_R=np.array(cam.rotation[:], np.float32), cam_t=np.array(cam.translation[:], np.float32))


def cfg_to_array(cfg):
    return np.array([cfg.tile_size, cfg.apply_thresholds, cfg.transmittance_min, cfg.contribution_min,
                     cfg.alpha_max, cfg.lowpass, cfg.radius_sigmas], np.float64)


def fixture(name, s, cam, cfg, bg=(0.0, 0.0, 0.0), mask=None, seed=0):
    refB, refA = OracleLib("ref", "B"), OracleLib("ref", "A")
    rng = np.random.default_rng(seed)
    d_color = rng.uniform(-1, 1, size=(cam.height, cam.width, 3)).astype(np.float32) / (3 * cam.width * cam.height)
    data = dict(centers=s.centers, log_scales=s.log_scales, rotations=s.rotations, opacity_logits=s.opacity_logits,
                sh=s.sh, sh_degree=np.int32(s.active_sh_degree), bg=np.array(bg, np.float32),
                cfg=cfg_to_array(cfg), d_color=d_color, **cam_to_arrays(cam))
    if mask is not None:
        data["mask"] = np.asarray(mask, np.uint8)
    rA = refA.render(s, cam, cfg, mask=mask, bg=bg)  # mode A: images only (information)
    for k in ("color", "alpha", "max_contributor"):
        data[f"A_{k}"] = rA[k]
    for tag, lib in (("B", refB),):
        r = lib.render(s, cam, cfg, mask=mask, bg=bg)
        for k in ("color", "alpha", "depth", "transmittance", "max_contributor", "importance", "max_weight",
                  "max_pixel_count"):
            data[f"{tag}_{k}"] = r[k]
        t = lib.tiles(s, cam, cfg, mask=mask)
        data[f"{tag}_ranges"] = t["ranges"]
        data[f"{tag}_lists"] = t["gaussian"]
        p = lib.project(s, cam, cfg, mask=mask)
        data[f"{tag}_order"] = p["order"]
        data[f"{tag}_rect"] = p["rect"]
        g = lib.render_backward(s, cam, d_color, cfg, mask=mask, bg=bg)
        for k, v in g.items():
            data[f"{tag}_{k}"] = v
    np.savez_compressed(OUT / f"{name}.npz", **data)
    print(f"wrote {name}.npz ({(OUT / f'{name}.npz').stat().st_size / 1e3:.0f} kB)")


def main():
    s = scenes.make_gaussians(2000, seed=7)
    fixture("cfg0_small", s, scenes.fov_camera(128, 96, 60.0, (0.0, 0.0, -3.0)), RasterConfig(), seed=1)
    s2 = scenes.make_gaussians(400, seed=11, log_scale_mean=np.log(0.05), sh_degree=2)
    fixture("tile32_bg", s2, scenes.fov_camera(50, 38, 60.0, (0.3, -0.2, -3.0)), RasterConfig(tile_size=32),
            bg=(0.25, 0.5, 0.75), seed=2)
    s3 = scenes.make_gaussians(60, seed=13, log_scale_mean=np.log(0.08), sh_degree=3)
    fixture("exact_mode", s3, scenes.fov_camera(32, 32, 60.0, (0.0, 0.5, -3.0)), RasterConfig(apply_thresholds=0),
            seed=3)
    s4 = scenes.make_gaussians(800, seed=17, log_scale_mean=np.log(0.05), sh_degree=1)
    mask = (np.random.default_rng(5).uniform(size=800) < 0.6).astype(np.uint8)
    fixture("masked", s4, scenes.fov_camera(64, 48, 60.0, (-0.4, 0.2, -3.0)), RasterConfig(), mask=mask, seed=4)


if __name__ == "__main__":
    main()
