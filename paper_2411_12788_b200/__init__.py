"""B200-native Mini-Splatting2 rasterizer hot path (sm_100a CUDA behind a C-ABI)."""
from .capi import AdamConfig, Camera, RasterConfig  # noqa: F401
from .scenes import GaussianSet, make_gaussians  # noqa: F401
