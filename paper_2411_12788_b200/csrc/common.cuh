// common.cuh — shared device-side definitions for the sm_100a rasterizer kernels.
//
// Bit-exactness contract: everything that decides an integer output
// (pixel rects, tile keys, per-tile lists, gates, argmax) or a forward image value is computed
// with correctly rounded, non-contracted IEEE operations in the reference's operation order
// (as fixed by oracle/compat/Eigen/Dense), and with the shared splat_expf.  forward.cu is
// compiled with --fmad=false; the per-sample gate below uses explicit _rn intrinsics so the
// backward (compiled with FMA contraction on) replays the forward's alphas bit for bit.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "splat_expf.h"

namespace splat_b200 {

constexpr int kBlock = 256;  // threads per tile CTA (16 x 16 pixels)

// Projected Gaussian record, 48 B (3 x float4), indexed by Gaussian id:
//   r0 = (mean2d.x, mean2d.y, conic0, conic1)
//   r1 = (conic2, opacity, rect x0 | x1 << 16, rect y0 | y1 << 16)
//   r2 = (color.r, color.g, color.b, depth)
struct __align__(16) ProjRec {
    float4 r0, r1, r2;
};

// Auxiliary record for depth rendering (rasterizer.cpp:278-281): world center, symmetric
// inverse 3D covariance (or identity-flagged degenerate), 48 B.
//   a0 = (cx, cy, cz, degenerate ? 1 : 0), a1 = (i00, i01, i02, i11), a2 = (i12, i22, 0, 0)
struct __align__(16) AuxRec {
    float4 a0, a1, a2;
};

// Camera + raster constants passed by value to kernels.
struct CamParams {
    int width, height;
    float fx, fy, cx, cy;
    float R[9];
    float t[3];
    float center[3];  // -(R^T t), computed on the host in the reference's order
    float znear;
    int tile_size, tiles_x, tiles_y;
    int apply_thresholds;
    float lowpass, radius_sigmas, alpha_max, contribution_min, transmittance_min;
    float log_cond_limit;  // float(log(1e12))
};

__device__ __forceinline__ uint32_t pack_range(int lo, int hi) {
    return (uint32_t)lo | ((uint32_t)hi << 16);
}
__device__ __forceinline__ int range_lo(float f) { return (int)(__float_as_uint(f) & 0xffffu); }
__device__ __forceinline__ int range_hi(float f) { return (int)(__float_as_uint(f) >> 16); }

// Per-sample gate of traverse_pixel (rasterizer.hpp:125-143), shared by the forward and the
// backward so both see identical alphas.  Returns false when the sample is skipped (outside
// the rect, power > 0, or alpha below the contribution floor).  The T-break test is left to
// the caller (it needs T).  All arithmetic is explicitly rounded: no FMA contraction.
__device__ __forceinline__ bool gate_sample(const float4& r0, const float4& r1, int px, int py,
                                            float x, float y, int thresholds, float alpha_max,
                                            float contribution_min, float& alpha, float& g2d,
                                            bool& clamped, float& dx, float& dy) {
    const float rx = r1.z, ry = r1.w;
    if (px < range_lo(rx) || px >= range_hi(rx) || py < range_lo(ry) || py >= range_hi(ry))
        return false;
    dx = __fsub_rn(r0.x, x);
    dy = __fsub_rn(r0.y, y);
    // power = -0.5 * (c0 dx dx + c2 dy dy) - c1 dx dy
    const float a = __fmul_rn(__fmul_rn(r0.z, dx), dx);
    const float b = __fmul_rn(__fmul_rn(r1.x, dy), dy);
    const float m = __fmul_rn(-0.5f, __fadd_rn(a, b));
    const float power = __fsub_rn(m, __fmul_rn(__fmul_rn(r0.w, dx), dy));
    if (power > 0.0f) return false;
    g2d = splat_expf(power);
    alpha = __fmul_rn(r1.y, g2d);
    clamped = false;
    if (thresholds) {
        if (alpha > alpha_max) {
            alpha = alpha_max;
            clamped = true;
        }
        if (alpha < contribution_min) return false;
    }
    return true;
}

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm volatile("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

}  // namespace splat_b200
