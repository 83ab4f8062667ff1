"""Seeded synthetic inputs for the BASELINE configs.

The paper measures on Mip-NeRF360 / Tanks&Temples / Deep Blending; none of that
data is available here, so seeded synthetic scenes with the BASELINE.json distributions and the
datasets' 1/4-resolution image shape (1237x822) stand in for them.  Pinned choices (Appendix B):

  * RNG: numpy ``Generator(PCG64(seed))``; every array is drawn in a fixed order (below).
  * Means: uniform in the radius-R ball by rejection from U(-R, R)^3, batch-wise.
  * log-scales: i.i.d. N(log_scale_mean, 0.5) per axis.
  * rotations: normalise(N(0, I4)) stored (w, x, y, z).
  * opacity logits: N(0, 1.5)  (opacity = sigmoid of it).
  * SH (coefficient-major [k*3+c]): DC ~ N(0, 0.5), the other 45 values ~ N(0, 0.05); degree 3.
  * Cameras: ``look_at`` (camera.hpp:84-96) toward the origin with world up (0, 1, 0);
    fx = fy = (W/2) / tan(fov/2) with fov HORIZONTAL; cx = W/2, cy = H/2; znear 0.01.
  * Ring views k of K: position (r cos 2pi k/K, h, r sin 2pi k/K), r = 3R, h = 0.5R.
  * Targets: a render of the same set with means + N(0, 0.01^2) (computed by the caller).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .capi import Camera, RasterConfig


@dataclass
class GaussianSet:
    """GaussianSetT<float> (gaussian_set.hpp:60-135) as contiguous float32 host arrays."""

    centers: np.ndarray            # [n, 3]
    log_scales: np.ndarray         # [n, 3]
    rotations: np.ndarray          # [n, 4] (w, x, y, z)
    opacity_logits: np.ndarray     # [n]
    sh: np.ndarray                 # [n, 48] coefficient-major
    active_sh_degree: int = 3

    @property
    def n(self) -> int:
        return int(self.centers.shape[0])

    def check_consistent(self) -> None:
        """GaussianSetT::check_consistent (gaussian_set.hpp:87-93)."""
        n = self.centers.shape[0]
        if (self.centers.shape != (n, 3) or self.log_scales.shape != (n, 3)
                or self.rotations.shape != (n, 4) or self.opacity_logits.shape != (n,)
                or self.sh.shape != (n, 48)):
            raise ValueError("GaussianSet parallel arrays out of sync")

    def select(self, keep) -> "GaussianSet":
        """GaussianSetT::select (gaussian_set.hpp:96-110)."""
        keep = np.asarray(keep, dtype=np.int64)
        return GaussianSet(self.centers[keep].copy(), self.log_scales[keep].copy(),
                           self.rotations[keep].copy(), self.opacity_logits[keep].copy(),
                           self.sh[keep].copy(), self.active_sh_degree)

    def copy(self) -> "GaussianSet":
        return GaussianSet(self.centers.copy(), self.log_scales.copy(), self.rotations.copy(),
                           self.opacity_logits.copy(), self.sh.copy(), self.active_sh_degree)

    @staticmethod
    def empty(n: int = 0, sh_degree: int = 3) -> "GaussianSet":
        """GaussianSetT::resize defaults: zero centers/scales/logits/SH, identity rotation."""
        rot = np.zeros((n, 4), np.float32)
        rot[:, 0] = 1.0
        return GaussianSet(np.zeros((n, 3), np.float32), np.zeros((n, 3), np.float32), rot,
                           np.zeros(n, np.float32), np.zeros((n, 48), np.float32), sh_degree)


def make_gaussians(n: int, seed: int = 0, radius: float = 1.0,
                   log_scale_mean: float = math.log(0.02), log_scale_std: float = 0.5,
                   sh_degree: int = 3) -> GaussianSet:
    """Config-0 distributions (BASELINE.json configs[0]) for n Gaussians."""
    rng = np.random.Generator(np.random.PCG64(seed))
    pts = np.empty((0, 3), np.float64)
    while pts.shape[0] < n:
        need = n - pts.shape[0]
        cand = rng.uniform(-radius, radius, size=(max(1024, int(need * 2.0)), 3))
        cand = cand[np.einsum("ij,ij->i", cand, cand) <= radius * radius]
        pts = np.concatenate([pts, cand[:need]], axis=0)
    centers = pts.astype(np.float32)
    log_scales = rng.normal(log_scale_mean, log_scale_std, size=(n, 3)).astype(np.float32)
    q = rng.normal(0.0, 1.0, size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    rotations = q.astype(np.float32)
    opacity_logits = rng.normal(0.0, 1.5, size=n).astype(np.float32)
    sh = np.empty((n, 48), np.float32)
    sh[:, :3] = rng.normal(0.0, 0.5, size=(n, 3))
    sh[:, 3:] = rng.normal(0.0, 0.05, size=(n, 45))
    return GaussianSet(centers, log_scales, rotations, opacity_logits, sh, sh_degree)


def perturbed(set_: GaussianSet, sigma: float = 0.01, seed: int = 1) -> GaussianSet:
    """Same set with means + N(0, sigma^2): the target scene of configs 0, 1, 4."""
    rng = np.random.Generator(np.random.PCG64(seed))
    out = set_.copy()
    out.centers = (set_.centers.astype(np.float64)
                   + rng.normal(0.0, sigma, size=set_.centers.shape)).astype(np.float32)
    return out


def look_at(position, target=(0.0, 0.0, 0.0), world_up=(0.0, 1.0, 0.0)):
    """camera.hpp:84-96 (y down, z forward), evaluated in float32."""
    f32 = np.float32
    position = np.asarray(position, f32)
    target = np.asarray(target, f32)
    up = np.asarray(world_up, f32)

    def normalized(v):
        n = np.sqrt(f32(np.dot(v, v)))
        return (v / n).astype(f32) if n > 0 else v

    forward = normalized(target - position)
    right = np.cross(forward, up).astype(f32)
    if np.sqrt(np.dot(right, right)) < 1e-8:
        right = np.cross(forward, np.array([1, 0, 0], f32)).astype(f32)
    right = normalized(right)
    down = normalized(np.cross(forward, right).astype(f32))
    rot = np.stack([right, down, forward]).astype(f32)
    trans = (-(rot @ position)).astype(f32)
    return rot, trans


def make_camera(width: int, height: int, fx: float, fy: float, cx: float, cy: float,
                position, target=(0.0, 0.0, 0.0), znear: float = 0.01,
                zfar: float = 100.0) -> Camera:
    rot, trans = look_at(position, target)
    cam = Camera()
    cam.width, cam.height = int(width), int(height)
    cam.fx, cam.fy, cam.cx, cam.cy = float(fx), float(fy), float(cx), float(cy)
    for i in range(9):
        cam.rotation[i] = float(rot.reshape(-1)[i])
    for i in range(3):
        cam.translation[i] = float(trans[i])
    cam.znear, cam.zfar = float(np.float32(znear)), float(zfar)
    return cam


def fov_camera(width: int, height: int, fov_deg: float, position, target=(0.0, 0.0, 0.0)) -> Camera:
    f = (width / 2.0) / math.tan(math.radians(fov_deg) / 2.0)
    return make_camera(width, height, f, f, width / 2.0, height / 2.0, position, target)


def ring_camera(k: int, count: int, width: int = 1237, height: int = 822, fov_deg: float = 70.0,
                radius: float = 3.0, y: float = 0.5) -> Camera:
    """Config 1-4 ring view k of count (BASELINE.json configs[1..4])."""
    th = 2.0 * math.pi * k / count
    return fov_camera(width, height, fov_deg, (radius * math.cos(th), y, radius * math.sin(th)))


def front_camera(width: int, height: int, dist: float = 4.0) -> Camera:
    """test_utils.hpp:13-27: on the -z axis at `dist`, fx = fy = width."""
    return make_camera(width, height, width, width, width / 2.0, height / 2.0, (0.0, 0.0, -dist))


def config0_camera() -> Camera:
    """Config 0: 256x256, fov 60 deg, at distance 3R looking at the origin."""
    return fov_camera(256, 256, 60.0, (0.0, 0.0, -3.0))


def camera_center(cam: Camera) -> np.ndarray:
    r = np.array(cam.rotation[:], np.float32).reshape(3, 3)
    t = np.array(cam.translation[:], np.float32)
    return (-(r.T @ t)).astype(np.float32)


@dataclass
class Config:
    """One BASELINE.json config."""

    name: str
    n: int
    log_scale_mean: float = math.log(0.02)
    views: int = 1
    width: int = 1237
    height: int = 822
    seed: int = 0
    extra: dict = field(default_factory=dict)


CONFIGS = {
    "cfg0": Config("cfg0", 20_000, width=256, height=256),
    "cfg1": Config("cfg1", 1_000_000),
    "cfg2": Config("cfg2", 3_000_000, log_scale_mean=math.log(0.005), views=64),
    "cfg3": Config("cfg3", 700_000, views=200),
    "cfg4": Config("cfg4", 3_000_000, views=256),
}


def default_raster_config(**kw) -> RasterConfig:
    return RasterConfig(**kw)


def grid_gaussians(count: int, seed: int = 0, extent: float = 1.5, log_scale: float = math.log(0.01)) -> GaussianSet:
    """`count` small, non-overlapping Gaussians on a square grid in the z = 0 plane (test scenes whose
    visible / max-contributor count is exactly `count` from `fov_camera(..., (0, 0, -3))`)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    side = int(math.ceil(math.sqrt(count)))
    u = np.linspace(-extent, extent, side)
    gx, gy = np.meshgrid(u, u)
    s = GaussianSet.empty(count)
    s.centers[:, 0] = gx.ravel()[:count]
    s.centers[:, 1] = gy.ravel()[:count]
    s.log_scales[:] = np.float32(log_scale)
    s.opacity_logits[:] = rng.uniform(-2.0, 3.0, count).astype(np.float32)
    s.sh[:, :3] = rng.normal(0.0, 0.5, (count, 3)).astype(np.float32)
    return s
