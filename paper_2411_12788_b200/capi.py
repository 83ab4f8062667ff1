"""ctypes mirror of include/splat_b200.h (the C-ABI boundary) and the product library loader.

The product library ``paper_2411_12788_b200/lib/libsplat_b200.so`` holds the sm_100a kernels and
the C++ host pipeline behind the C-ABI.  There is no CPU fallback: if the library is missing,
``load_library()`` raises.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
LIB_DIR = PKG_DIR / "lib"
LIB_PATH = LIB_DIR / "libsplat_b200.so"

SH_VALUES = 48
GRAD_FLOATS = 59

SPLAT_OK = 0
SPLAT_ERR_INVALID_ARGUMENT = 1
SPLAT_ERR_LOGIC = 2
SPLAT_ERR_RUNTIME = 3
SPLAT_ERR_CUDA = 4
SPLAT_ERR_OUT_OF_MEMORY = 5
SPLAT_ERR_NO_FORWARD_STATE = 6
SPLAT_ERR_NCCL = 7

GROUP_CENTERS = 1
GROUP_SCALES = 2
GROUP_ROTATIONS = 4
GROUP_OPACITY = 8
GROUP_SH = 16
GROUP_ALL = 31

DEPTH_RULE_ARGMAX = 0
DEPTH_RULE_ALPHA = 1

fp = C.POINTER(C.c_float)
ip = C.POINTER(C.c_int32)
u8p = C.POINTER(C.c_uint8)

# identify_critical criteria (include/splat_b200.h SPLAT_CRITERION_*, densify.hpp:15)
CRITERION_RANDOM, CRITERION_OPACITY, CRITERION_ACCUM_WEIGHT, CRITERION_MAX_WEIGHT = 0, 1, 2, 3


class Camera(C.Structure):
    """splat_camera — CameraT<float> (camera.hpp:12-22); rotation row-major world->camera."""

    _fields_ = [
        ("width", C.c_int32),
        ("height", C.c_int32),
        ("fx", C.c_float),
        ("fy", C.c_float),
        ("cx", C.c_float),
        ("cy", C.c_float),
        ("rotation", C.c_float * 9),
        ("translation", C.c_float * 3),
        ("znear", C.c_float),
        ("zfar", C.c_float),
    ]


class RasterConfig(C.Structure):
    """splat_raster_config — RasterConfig (rasterizer.hpp:17-25) with the reference defaults."""

    _fields_ = [
        ("tile_size", C.c_int32),
        ("apply_thresholds", C.c_int32),
        ("transmittance_min", C.c_double),
        ("contribution_min", C.c_double),
        ("alpha_max", C.c_double),
        ("lowpass", C.c_double),
        ("radius_sigmas", C.c_double),
    ]

    def __init__(self, **kw):
        super().__init__()
        self.tile_size = 16
        self.apply_thresholds = 1
        self.transmittance_min = 1e-4
        self.contribution_min = 1.0 / 255
        self.alpha_max = 0.99
        self.lowpass = 0.3
        self.radius_sigmas = 3.0
        for k, v in kw.items():
            setattr(self, k, v)


class Gaussians(C.Structure):
    """splat_gaussians — GaussianSetT<float> as plain pointers."""

    _fields_ = [
        ("centers", fp),
        ("log_scales", fp),
        ("rotations", fp),
        ("opacity_logits", fp),
        ("sh", fp),
        ("n", C.c_int32),
        ("active_sh_degree", C.c_int32),
    ]


class RenderOutputs(C.Structure):
    _fields_ = [
        ("color", fp),
        ("alpha", fp),
        ("depth", fp),
        ("transmittance", fp),
        ("max_contributor", ip),
    ]


class ImportanceOutputs(C.Structure):
    _fields_ = [("importance", fp), ("max_weight", fp), ("max_pixel_count", ip)]


class Projected(C.Structure):
    """splat_projected — ProjectedGaussian<float> (rasterizer.hpp:27-41)."""

    _fields_ = [
        ("mean2d", C.c_float * 2),
        ("cov2d", C.c_float * 3),
        ("conic", C.c_float * 3),
        ("depth_mean", C.c_float),
        ("radius", C.c_int32),
        ("index", C.c_int32),
        ("opacity", C.c_float),
        ("color", C.c_float * 3),
        ("x0", C.c_int32), ("x1", C.c_int32), ("y0", C.c_int32), ("y1", C.c_int32),
        ("center_world", C.c_float * 3),
        ("cov_world_inv", C.c_float * 9),
        ("cov_degenerate", C.c_int32),
    ]


class ParamGrads(C.Structure):
    _fields_ = [
        ("d_centers", fp),
        ("d_log_scales", fp),
        ("d_rotations", fp),
        ("d_opacity_logits", fp),
        ("d_sh", fp),
        ("grad2d_accum", fp),
        ("grad2d_count", ip),
    ]


class AdamConfig(C.Structure):
    """splat_adam_config — AdamConfig + LrSchedule (optimizer.hpp:12-32), reference defaults."""

    _fields_ = [
        ("beta1", C.c_double),
        ("beta2", C.c_double),
        ("eps", C.c_double),
        ("lr_init", C.c_double),
        ("lr_final", C.c_double),
        ("max_steps", C.c_int32),
        ("_pad", C.c_int32),
        ("scene_extent", C.c_double),
        ("lr_sh_dc", C.c_double),
        ("lr_sh_rest", C.c_double),
        ("lr_opacity", C.c_double),
        ("lr_scale", C.c_double),
        ("lr_rotation", C.c_double),
    ]

    def __init__(self, **kw):
        super().__init__()
        self.beta1, self.beta2, self.eps = 0.9, 0.999, 1e-15
        self.lr_init, self.lr_final, self.max_steps = 1.6e-4, 1.6e-6, 18000
        self.scene_extent = 1.0
        self.lr_sh_dc = 2.5e-3
        self.lr_sh_rest = 2.5e-3 / 20.0
        self.lr_opacity = 5e-2
        self.lr_scale = 5e-3
        self.lr_rotation = 1e-3
        for k, v in kw.items():
            setattr(self, k, v)


class ParamsMut(C.Structure):
    _fields_ = [
        ("centers", fp),
        ("log_scales", fp),
        ("rotations", fp),
        ("opacity_logits", fp),
        ("sh", fp),
        ("n", C.c_int32),
        ("active_sh_degree", C.c_int32),
    ]


class AdamMoments(C.Structure):
    _fields_ = [
        ("m_centers", fp), ("v_centers", fp),
        ("m_log_scales", fp), ("v_log_scales", fp),
        ("m_rotations", fp), ("v_rotations", fp),
        ("m_opacity", fp), ("v_opacity", fp),
        ("m_sh", fp), ("v_sh", fp),
    ]


def as_fp(addr) -> "C._Pointer":
    """Cast an integer address (device or host) or None to float*."""
    return C.cast(C.c_void_p(addr), fp) if addr else fp()


def as_ip(addr):
    return C.cast(C.c_void_p(addr), ip) if addr else ip()


def as_u8p(addr):
    return C.cast(C.c_void_p(addr), u8p) if addr else u8p()


_EXPORTS = {
    # name: (restype, argtypes)
    "splat_ctx_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    "splat_ctx_destroy": (C.c_int, [C.c_void_p]),
    "splat_ctx_set_stream": (C.c_int, [C.c_void_p, C.c_void_p]),
    "splat_sync": (C.c_int, [C.c_void_p]),
    "splat_last_error": (C.c_char_p, [C.c_void_p]),
    "splat_kernel_launches": (C.c_int64, [C.c_void_p]),
    "splat_profile_enable": (C.c_int, [C.c_void_p, C.c_int]),
    "splat_profile_read": (C.c_int, [C.c_void_p, C.c_char_p, C.c_int, C.POINTER(C.c_double),
                                     C.POINTER(C.c_int64), C.c_int, C.POINTER(C.c_int)]),
    "splat_render": (C.c_int, [C.c_void_p, C.POINTER(Gaussians), C.POINTER(Camera),
                               C.POINTER(RasterConfig), u8p, C.POINTER(C.c_float),
                               C.POINTER(RenderOutputs), C.POINTER(ImportanceOutputs)]),
    "splat_accumulate_importance": (C.c_int, [C.c_void_p, C.POINTER(Gaussians), C.POINTER(Camera),
                                              C.POINTER(RasterConfig), u8p,
                                              C.POINTER(ImportanceOutputs)]),
    "splat_render_backward": (C.c_int, [C.c_void_p, C.POINTER(Gaussians), C.POINTER(Camera),
                                        C.POINTER(RasterConfig), fp, u8p, C.POINTER(C.c_float),
                                        C.POINTER(ParamGrads), C.c_int, C.c_int]),
    "splat_l1_loss": (C.c_int, [C.c_void_p, fp, fp, C.c_int64, fp, fp]),
    "splat_render_backward_l1": (C.c_int, [C.c_void_p, C.POINTER(Gaussians), C.POINTER(Camera),
                                           C.POINTER(RasterConfig), fp, u8p, C.POINTER(C.c_float),
                                           C.POINTER(ParamGrads), C.c_int, fp]),
    "splat_adam_step": (C.c_int, [C.c_void_p, C.POINTER(ParamsMut), C.POINTER(ParamGrads),
                                  C.POINTER(AdamMoments), C.POINTER(AdamConfig),
                                  C.POINTER(C.c_int32), C.c_uint32]),
    "splat_depth_unproject": (C.c_int, [C.c_void_p, C.POINTER(Camera), C.c_int, C.c_float,
                                        C.c_int64, C.c_int32, C.c_int64, fp, ip, C.c_int64, ip]),
    "splat_visibility_update": (C.c_int, [C.c_void_p, C.POINTER(ImportanceOutputs), C.c_int32, C.c_float,
                                          C.c_void_p, C.c_void_p, C.c_void_p]),
    "splat_visibility_update_max": (C.c_int, [C.c_void_p, C.POINTER(ImportanceOutputs), C.c_int32, C.c_float,
                                              C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "splat_visibility_pass": (C.c_int, [C.c_void_p, C.POINTER(Gaussians), C.POINTER(Camera), C.c_int32,
                                        C.POINTER(RasterConfig), C.c_float, C.c_void_p, C.c_int64, C.c_void_p,
                                        C.c_void_p, C.c_void_p]),
    "splat_depth_points": (C.c_int, [C.c_void_p, C.POINTER(Gaussians), C.POINTER(Camera), C.c_int32,
                                     C.POINTER(RasterConfig), C.c_int, C.c_float, C.c_int64, C.c_int32, C.c_int64,
                                     C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]),
    "splat_quantile_threshold": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_double,
                                           C.POINTER(C.c_float), C.POINTER(C.c_int32)]),
    "splat_quantile_threshold_f64": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_double,
                                               C.POINTER(C.c_double), C.POINTER(C.c_int32)]),
    "splat_visibility_mask": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_double, C.c_void_p]),
    "splat_identify_critical": (C.c_int, [C.c_void_p, C.POINTER(Gaussians), C.c_void_p, C.c_void_p, C.c_void_p,
                                          C.c_int, C.c_double, C.c_void_p, C.c_void_p, C.POINTER(C.c_int32)]),
    "splat_aggressive_clone": (C.c_int, [C.c_void_p, C.POINTER(ParamsMut), C.c_int64, C.c_void_p, C.c_void_p,
                                         C.POINTER(C.c_int32)]),
    "splat_importance_prune": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_double, C.c_void_p,
                                         C.POINTER(C.c_int32)]),
    "splat_gather_rows": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_int32, C.c_void_p]),
    "splat_adam_step_range": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32,
                                        C.c_int64, C.c_int64, C.POINTER(AdamConfig), C.c_int32, C.c_uint32]),
    "splat_quat_normalize": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32]),
    "splat_comm_unique_id": (C.c_int, [C.c_void_p]),
    "splat_comm_init": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_int32]),
    "splat_comm_destroy": (C.c_int, [C.c_void_p]),
    "splat_exchange_len": (C.c_int64, [C.c_int32, C.c_int32, C.c_int32]),
    "splat_exchange_step": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32,
                                      C.c_int64, C.POINTER(AdamConfig), C.POINTER(C.c_int32), C.c_uint32]),
    "splat_allreduce": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_int32]),
    "splat_rng_create": (C.c_int, [C.c_uint32, C.POINTER(C.c_void_p)]),
    "splat_rng_destroy": (None, [C.c_void_p]),
    "splat_rng_get_state": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint32)]),
    "splat_rng_set_state": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint32)]),
    "splat_random_scores": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_int]),
    "splat_pool_sample": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p]),
    "splat_importance_sample": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_uint64, C.c_void_p,
                                          C.POINTER(C.c_int32)]),
    "splat_vanilla_clone_split": (C.c_int, [C.c_void_p, C.POINTER(Gaussians), C.c_void_p, C.c_void_p, C.c_float,
                                            C.c_float, C.c_float, C.c_void_p, C.POINTER(ParamsMut), C.c_int64,
                                            C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                            C.POINTER(C.c_int32)]),
    "splat_ssim": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_void_p,
                             C.c_void_p]),
    "splat_photometric_loss": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                                         C.c_float, C.c_void_p, C.c_void_p]),
    "splat_render_backward_photometric": (C.c_int, [C.c_void_p, C.POINTER(Gaussians), C.POINTER(Camera),
                                                    C.POINTER(RasterConfig), fp, u8p, C.POINTER(C.c_float),
                                                    C.POINTER(ParamGrads), C.c_int, C.c_float, fp]),
    "splat_third_neighbor_distances": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_float, C.c_void_p]),
    "splat_reinit_gaussians": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_float,
                                         C.POINTER(ParamsMut)]),
    "splat_train_step": (C.c_int, [C.c_void_p, C.POINTER(ParamsMut), C.POINTER(ParamGrads), C.POINTER(AdamMoments),
                                   C.POINTER(AdamConfig), C.POINTER(C.c_int32), C.c_uint32, C.c_void_p, C.c_int32,
                                   C.c_void_p, C.c_int, C.POINTER(RasterConfig), C.POINTER(C.c_float), C.c_float,
                                   C.c_void_p, C.c_void_p]),
    "splat_sort_pairs": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64,
                                   C.c_int, C.c_int, C.POINTER(C.c_int)]),
    "splat_exclusive_scan": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]),
    "splat_forward_counts": (C.c_int, [C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                       C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "splat_project": (C.c_int, [C.c_void_p, C.POINTER(Gaussians), C.POINTER(Camera), C.POINTER(RasterConfig), u8p,
                                C.c_void_p, C.c_int64, C.POINTER(C.c_int32)]),
    "splat_traversal_counts": (C.c_int, [C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "splat_project_debug": (C.c_int, [C.c_void_p, ip, ip, fp, u8p, fp, fp, fp, fp]),
    "splat_tiles_debug": (C.c_int, [C.c_void_p, ip, ip, ip, ip]),
}

EXPORTED_SYMBOLS = tuple(_EXPORTS)

_lib = None


def load_library(path: os.PathLike | str | None = None) -> C.CDLL:
    """Load libsplat_b200.so and declare every C-ABI entry point. Raises if it is missing."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    # SPLAT_B200_LIB selects an alternative build of the same library (tuning experiments)
    p = Path(path) if path else Path(os.environ.get("SPLAT_B200_LIB", LIB_PATH))
    if not p.exists():
        raise RuntimeError(
            f"{p} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback for the CUDA path)")
    lib = C.CDLL(str(p))
    for name, (res, args) in _EXPORTS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib
