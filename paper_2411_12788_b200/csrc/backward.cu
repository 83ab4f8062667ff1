// backward.cu — blend backward (K9), per-Gaussian 2D->3D chain (K10), L1 loss (K8) and Adam (K11).
//
// Gradients are compared against the oracle within tolerance (1e-4 relative, SURVEY.md §8
// Appendix C): summation order over pixels differs (warp/CTA reductions + atomics) and the
// backward reconstructs T_before = T_after / (1 - alpha) instead of storing per-sample T.
// The gates themselves are replayed bit-exactly (gate_sample uses explicit _rn intrinsics), so
// the set of committed samples is identical to the forward's.  FMA contraction is allowed here.
#include <cstdint>

#include "common.cuh"
#include "internal.h"

namespace splat_b200 {

namespace {

constexpr int kGradSlots = 10;   // 9 gradient values + touched count per staged Gaussian
constexpr int kGradStride = 10;  // smem row stride (floats): conflict-free lane->value scatter

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Transpose-reduce of 10 per-lane values across the warp in 12 shuffles (instead of 50):
// every level exchanges the half a lane does not keep.  On return, lane l holds the warp total
// of value index *which, or *which = -1 when l holds padding / a duplicate.
__device__ __forceinline__ float warp_transpose_reduce10(const float v[10], int lane, int* which) {
    const bool a = lane & 16, b = lane & 8, c = lane & 4, d = lane & 2;
    float u[6];
#pragma unroll
    for (int i = 0; i < 5; ++i) {
        const float send = a ? v[i] : v[5 + i];
        const float keep = a ? v[5 + i] : v[i];
        u[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
    u[5] = 0.0f;
    float w[4];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const float send = b ? u[i] : u[3 + i];
        const float keep = b ? u[3 + i] : u[i];
        w[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
    w[3] = 0.0f;
    float x[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const float send = c ? w[i] : w[2 + i];
        const float keep = c ? w[2 + i] : w[i];
        x[i] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
    }
    const float send = d ? x[0] : x[1];
    float y = (d ? x[1] : x[0]) + __shfl_xor_sync(0xffffffffu, send, 2);
    y += __shfl_xor_sync(0xffffffffu, y, 1);
    const int oc = (c ? 2 : 0) + (d ? 1 : 0);
    const int local = (b ? 3 : 0) + oc;
    const bool valid = !(lane & 1) && local < 5 && oc < 3;
    *which = valid ? (a ? 5 : 0) + local : -1;
    return y;
}

// Blend backward (gradients.cpp:73-123): per pixel, walk the tile list back to front from the
// pixel's last committed sample, re-evaluating the forward gates; b = colour behind the sample
// (normalised), exactly the reference recursion; T_before = T_after / (1 - alpha).
// Per staged Gaussian the 9 per-pixel contributions (d_mean2d 2, d_conic 3 (01 = 10),
// d_opacity, d_colour 3) are warp-reduced, accumulated in shared memory, and flushed to the
// per-Gaussian accumulator with three float4 atomics per (CTA, Gaussian).
// With target != nullptr, dL/dC = sign(C - target)/n (l1_loss, loss.cpp:63-76) is fused in and
// the CTA's L1 partial sum is written to loss_partials[block].
__global__ void __launch_bounds__(256) blend_backward_kernel(CamParams cp, const uint32_t* __restrict__ ranges,
                                                            const uint32_t* __restrict__ pair_gauss,
                                                            const ProjRec* __restrict__ rec,
                                                            const float* __restrict__ t_final,
                                                            const int32_t* __restrict__ last_index, float bg0,
                                                            float bg1, float bg2, const float* __restrict__ d_color,
                                                            const float* __restrict__ color,
                                                            const float* __restrict__ target, float inv_n,
                                                            float* __restrict__ loss_partials,
                                                            float4* __restrict__ grad2d) {
    __shared__ float4 s_r0[kBlock], s_r1[kBlock], s_r2[kBlock];
    __shared__ uint32_t s_gid[kBlock];
    __shared__ float s_g[kBlock * kGradStride];
    __shared__ float s_red[kBlock / 32];
    __shared__ int s_maxlast[kBlock / 32];
    const int nthreads = blockDim.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nwarps = nthreads >> 5;
    const int ts = cp.tile_size;
    const int bw = ts < 16 ? ts : 16;
    const int tile = blockIdx.x;
    const int tx = tile % cp.tiles_x, ty = tile / cp.tiles_x;
    const int subs = ts / bw;
    const int sx = blockIdx.y % subs, sy = blockIdx.y / subs;
    const int px = tx * ts + sx * bw + tid % bw;
    const int py = ty * ts + sy * bw + tid / bw;
    const bool inside = px < cp.width && py < cp.height;
    const size_t pix = inside ? (size_t)py * cp.width + px : 0;

    float dL0 = 0.f, dL1 = 0.f, dL2 = 0.f;
    if (inside) {
        if (target) {
            float l = 0.0f;
            float* dl[3] = {&dL0, &dL1, &dL2};
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const float dd = color[3 * pix + c] - target[3 * pix + c];
                l += fabsf(dd);
                *dl[c] = dd > 0.0f ? inv_n : (dd < 0.0f ? -inv_n : 0.0f);
            }
            if (loss_partials) {
                const float ws = warp_sum(l);
                if (lane == 0) s_red[warp] = ws;
            }
        } else {
            dL0 = d_color[3 * pix];
            dL1 = d_color[3 * pix + 1];
            dL2 = d_color[3 * pix + 2];
        }
    } else if (target && loss_partials) {
        const float ws = warp_sum(0.0f);
        if (lane == 0) s_red[warp] = ws;
    }
    const int my_last = inside ? last_index[pix] : -1;
    const int wl = __reduce_max_sync(0xffffffffu, (unsigned)(my_last + 1)) - 1;
    if (lane == 0) s_maxlast[warp] = wl;
    __syncthreads();
    if (target && loss_partials && tid == 0) {
        float s = 0.0f;
        for (int w = 0; w < nwarps; ++w) s += s_red[w];
        loss_partials[blockIdx.y * gridDim.x + blockIdx.x] = s;
    }
    int block_last = -1;
    for (int w = 0; w < nwarps; ++w) block_last = max(block_last, s_maxlast[w]);
    const uint32_t start = ranges[2 * tile];
    if (block_last < (int)start) return;  // nothing committed in this block

    const int thr = cp.apply_thresholds;
    const float amax_c = cp.alpha_max, cmin = cp.contribution_min;
    const float x = (float)px + 0.5f, y = (float)py + 0.5f;
    float T = inside ? t_final[pix] : 1.0f;
    float b0 = bg0, b1 = bg1, b2 = bg2;

    for (int hi = block_last + 1; hi > (int)start; hi -= nthreads) {
        const int lo = max((int)start, hi - nthreads);
        const int cnt = hi - lo;
        if (tid < cnt) {
            const uint32_t gid = pair_gauss[hi - 1 - tid];
            const ProjRec rr = rec[gid];
            s_r0[tid] = rr.r0;
            s_r1[tid] = rr.r1;
            s_r2[tid] = rr.r2;
            s_gid[tid] = gid;
#pragma unroll
            for (int k = 0; k < kGradSlots; ++k) s_g[tid * kGradStride + k] = 0.0f;
        }
        __syncthreads();
        // samples above this warp's last commit are skipped by the whole warp
        const int jstart = max(0, hi - 1 - wl);
        for (int j = jstart; j < cnt; ++j) {
            const int idx = hi - 1 - j;
            float v[10];
#pragma unroll
            for (int k = 0; k < 10; ++k) v[k] = 0.0f;
            bool committed = false;
            if (idx <= my_last) {
                float alpha, g2d, dx, dy;
                bool clamped;
                const float4 r0 = s_r0[j], r1 = s_r1[j];
                if (gate_sample(r0, r1, px, py, x, y, thr, amax_c, cmin, alpha, g2d, clamped, dx, dy)) {
                    committed = true;
                    const float4 r2 = s_r2[j];
                    const float one_m_a = 1.0f - alpha;
                    const float t_before = T / one_m_a;
                    const float w = t_before * alpha;
                    v[6] = w * dL0;
                    v[7] = w * dL1;
                    v[8] = w * dL2;
                    const float da = t_before * (dL0 * (r2.x - b0) + dL1 * (r2.y - b1) + dL2 * (r2.z - b2));
                    if (!clamped) {
                        v[5] = da * g2d;
                        const float dpower = da * r1.y * g2d;
                        v[0] = dpower * (-(r0.z * dx + r0.w * dy));
                        v[1] = dpower * (-(r1.x * dy + r0.w * dx));
                        const float hp = -0.5f * dpower;
                        v[2] = hp * dx * dx;
                        v[3] = hp * dx * dy;
                        v[4] = hp * dy * dy;
                    }
                    v[9] = 1.0f;
                    b0 = alpha * r2.x + one_m_a * b0;
                    b1 = alpha * r2.y + one_m_a * b1;
                    b2 = alpha * r2.z + one_m_a * b2;
                    T = t_before;
                }
            }
            if (__any_sync(0xffffffffu, committed)) {
                int which;
                const float s = warp_transpose_reduce10(v, lane, &which);
                if (which >= 0 && s != 0.0f) atomicAdd(&s_g[j * kGradStride + which], s);
            }
        }
        __syncthreads();
        if (tid < cnt && s_g[tid * kGradStride + 9] > 0.0f) {
            const float* gs = &s_g[tid * kGradStride];
            float4* dst = grad2d + 3 * (size_t)s_gid[tid];
            atomicAdd(dst + 0, make_float4(gs[0], gs[1], gs[2], gs[3]));
            atomicAdd(dst + 1, make_float4(gs[4], gs[5], gs[6], gs[7]));
            atomicAdd(dst + 2, make_float4(gs[8], gs[9], 0.0f, 0.0f));
        }
        __syncthreads();
    }
}

__device__ __forceinline__ void sh_basis_all(float x, float y, float z, int degree, float bs[16]) {
#pragma unroll
    for (int i = 0; i < 16; ++i) bs[i] = 0.0f;
    bs[0] = (float)0.28209479177387814;
    if (degree < 1) return;
    const float c1 = (float)0.4886025119029199;
    bs[1] = -c1 * y;
    bs[2] = c1 * z;
    bs[3] = -c1 * x;
    if (degree < 2) return;
    const float xx = x * x, yy = y * y, zz = z * z;
    bs[4] = (float)1.0925484305920792 * x * y;
    bs[5] = (float)-1.0925484305920792 * y * z;
    bs[6] = (float)0.31539156525252005 * (2.0f * zz - xx - yy);
    bs[7] = (float)-1.0925484305920792 * x * z;
    bs[8] = (float)0.5462742152960396 * (xx - yy);
    if (degree < 3) return;
    bs[9] = (float)-0.5900435899266435 * y * (3.0f * xx - yy);
    bs[10] = (float)2.890611442640554 * x * y * z;
    bs[11] = (float)-0.4570457994644658 * y * (4.0f * zz - xx - yy);
    bs[12] = (float)0.3731763325901154 * z * (2.0f * zz - 3.0f * xx - 3.0f * yy);
    bs[13] = (float)-0.4570457994644658 * x * (4.0f * zz - xx - yy);
    bs[14] = (float)1.445305721320277 * z * (xx - yy);
    bs[15] = (float)-0.5900435899266435 * x * (xx - 3.0f * yy);
}

// sh_basis_grad (sh.hpp:55-79) contracted with coef[k]: returns sum_k coef[k] * d basis_k / d dir.
__device__ __forceinline__ void sh_dir_grad(float x, float y, float z, int degree, const float coef[16], float g[3]) {
    g[0] = g[1] = g[2] = 0.0f;
    if (degree < 1) return;
    const float c1 = (float)0.4886025119029199;
    g[1] += -c1 * coef[1];
    g[2] += c1 * coef[2];
    g[0] += -c1 * coef[3];
    if (degree < 2) return;
    const float xx = x * x, yy = y * y, zz = z * z;
    const float C20 = (float)1.0925484305920792, C21 = (float)-1.0925484305920792, C22 = (float)0.31539156525252005,
                C23 = (float)-1.0925484305920792, C24 = (float)0.5462742152960396;
    g[0] += coef[4] * C20 * y;  g[1] += coef[4] * C20 * x;
    g[1] += coef[5] * C21 * z;  g[2] += coef[5] * C21 * y;
    g[0] += coef[6] * C22 * (-2.0f * x); g[1] += coef[6] * C22 * (-2.0f * y); g[2] += coef[6] * C22 * (4.0f * z);
    g[0] += coef[7] * C23 * z;  g[2] += coef[7] * C23 * x;
    g[0] += coef[8] * C24 * (2.0f * x); g[1] += coef[8] * C24 * (-2.0f * y);
    if (degree < 3) return;
    const float C30 = (float)-0.5900435899266435, C31 = (float)2.890611442640554, C32 = (float)-0.4570457994644658,
                C33 = (float)0.3731763325901154, C34 = (float)-0.4570457994644658, C35 = (float)1.445305721320277,
                C36 = (float)-0.5900435899266435;
    g[0] += coef[9] * C30 * (6.0f * x * y); g[1] += coef[9] * C30 * (3.0f * xx - 3.0f * yy);
    g[0] += coef[10] * C31 * (y * z); g[1] += coef[10] * C31 * (x * z); g[2] += coef[10] * C31 * (x * y);
    g[0] += coef[11] * C32 * (-2.0f * x * y); g[1] += coef[11] * C32 * (4.0f * zz - xx - 3.0f * yy);
    g[2] += coef[11] * C32 * (8.0f * y * z);
    g[0] += coef[12] * C33 * (-6.0f * x * z); g[1] += coef[12] * C33 * (-6.0f * y * z);
    g[2] += coef[12] * C33 * (6.0f * zz - 3.0f * xx - 3.0f * yy);
    g[0] += coef[13] * C34 * (4.0f * zz - 3.0f * xx - yy); g[1] += coef[13] * C34 * (-2.0f * x * y);
    g[2] += coef[13] * C34 * (8.0f * x * z);
    g[0] += coef[14] * C35 * (2.0f * x * z); g[1] += coef[14] * C35 * (-2.0f * y * z); g[2] += coef[14] * C35 * (xx - yy);
    g[0] += coef[15] * C36 * (3.0f * xx - 3.0f * yy); g[1] += coef[15] * C36 * (-6.0f * x * y);
}

// Per-Gaussian geometric chain (gradients.cpp:127-220).  Untouched Gaussians get exact zeros
// (or nothing when accumulating).  The 2D accumulator is re-zeroed as it is consumed.
template <bool VEC>
__global__ void __launch_bounds__(128) chain_kernel(GaussianPtrs g, CamParams cp, float4* __restrict__ grad2d,
                                                   const ProjRec* __restrict__ rec, splat_param_grads out,
                                                   int accumulate) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= g.n) return;
    const float4 g0 = grad2d[3 * (size_t)i], g1 = grad2d[3 * (size_t)i + 1], g2 = grad2d[3 * (size_t)i + 2];
    const bool touched = g2.y > 0.0f;
    if (!touched) {
        if (!accumulate) {
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                out.d_centers[3 * (size_t)i + k] = 0.0f;
                out.d_log_scales[3 * (size_t)i + k] = 0.0f;
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) out.d_rotations[4 * (size_t)i + k] = 0.0f;
            out.d_opacity_logits[i] = 0.0f;
            if (VEC) {
                float4* d4 = reinterpret_cast<float4*>(out.d_sh + 48 * (size_t)i);
#pragma unroll
                for (int k = 0; k < 12; ++k) d4[k] = make_float4(0.f, 0.f, 0.f, 0.f);
            } else {
                for (int k = 0; k < 48; ++k) out.d_sh[48 * (size_t)i + k] = 0.0f;
            }
            if (out.grad2d_accum) out.grad2d_accum[i] = 0.0f;
            if (out.grad2d_count) out.grad2d_count[i] = 0;
        }
        return;
    }
    const float4 zero4 = make_float4(0.f, 0.f, 0.f, 0.f);
    grad2d[3 * (size_t)i] = zero4;
    grad2d[3 * (size_t)i + 1] = zero4;
    grad2d[3 * (size_t)i + 2] = zero4;

    const float dmx = g0.x, dmy = g0.y, dq00 = g0.z, dq01 = g0.w, dq11 = g1.x, dopac = g1.y;
    const float dcol[3] = {g1.z, g1.w, g2.x};
    const ProjRec pr = rec[i];
    const float k0 = pr.r0.z, k1 = pr.r0.w, k2 = pr.r1.x, opacity = pr.r1.y;

    // dV = -Q dQ Q  (conic = inverse(cov2d)), dQ symmetric with off-diagonal dq01
    const float n00 = -(k0 * dq00 + k1 * dq01), n01 = -(k0 * dq01 + k1 * dq11);
    const float n10 = -(k1 * dq00 + k2 * dq01), n11 = -(k1 * dq01 + k2 * dq11);
    const float dV00 = n00 * k0 + n01 * k1, dV01 = n00 * k1 + n01 * k2;
    const float dV10 = n10 * k0 + n11 * k1, dV11 = n10 * k1 + n11 * k2;

    const float px = g.centers[3 * (size_t)i], py = g.centers[3 * (size_t)i + 1], pz = g.centers[3 * (size_t)i + 2];
    const float* R = cp.R;
    const float pc0 = R[0] * px + R[1] * py + R[2] * pz + cp.t[0];
    const float pc1 = R[3] * px + R[4] * py + R[5] * pz + cp.t[1];
    const float z = R[6] * px + R[7] * py + R[8] * pz + cp.t[2];
    const float iz = 1.0f / z, iz2 = iz * iz;
    const float J00 = cp.fx * iz, J02 = -cp.fx * pc0 * iz2, J11 = cp.fy * iz, J12 = -cp.fy * pc1 * iz2;
    float M[6];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        M[c] = J00 * R[c] + J02 * R[6 + c];
        M[3 + c] = J11 * R[3 + c] + J12 * R[6 + c];
    }
    // covariance
    float qw = g.rotations[4 * (size_t)i], qx = g.rotations[4 * (size_t)i + 1], qy = g.rotations[4 * (size_t)i + 2],
          qz = g.rotations[4 * (size_t)i + 3];
    const float qn = sqrtf(qw * qw + qx * qx + qy * qy + qz * qz);
    float qh[4];
    if (!(qn > 0.0f)) {
        qh[0] = 1.0f; qh[1] = qh[2] = qh[3] = 0.0f;
    } else {
        qh[0] = qw / qn; qh[1] = qx / qn; qh[2] = qy / qn; qh[3] = qz / qn;
    }
    const float w_ = qh[0], x_ = qh[1], y_ = qh[2], z_ = qh[3];
    float Rq[9];
    Rq[0] = 1.0f - 2.0f * (y_ * y_ + z_ * z_);
    Rq[1] = 2.0f * (x_ * y_ - w_ * z_);
    Rq[2] = 2.0f * (x_ * z_ + w_ * y_);
    Rq[3] = 2.0f * (x_ * y_ + w_ * z_);
    Rq[4] = 1.0f - 2.0f * (x_ * x_ + z_ * z_);
    Rq[5] = 2.0f * (y_ * z_ - w_ * x_);
    Rq[6] = 2.0f * (x_ * z_ - w_ * y_);
    Rq[7] = 2.0f * (y_ * z_ + w_ * x_);
    Rq[8] = 1.0f - 2.0f * (x_ * x_ + y_ * y_);
    const float sc[3] = {splat_expf(g.log_scales[3 * (size_t)i]), splat_expf(g.log_scales[3 * (size_t)i + 1]),
                         splat_expf(g.log_scales[3 * (size_t)i + 2])};
    float M3[9], C[9];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) M3[r * 3 + c] = Rq[r * 3 + c] * sc[c];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c)
            C[r * 3 + c] = M3[r * 3] * M3[c * 3] + M3[r * 3 + 1] * M3[c * 3 + 1] + M3[r * 3 + 2] * M3[c * 3 + 2];
    // d_cov3d = M^T dV M
    float D[9];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
        const float p0 = M[r] * dV00 + M[3 + r] * dV10;
        const float p1 = M[r] * dV01 + M[3 + r] * dV11;
#pragma unroll
        for (int c = 0; c < 3; ++c) D[r * 3 + c] = p0 * M[c] + p1 * M[3 + c];
    }
    // dM = 2 dV M cov3d ; dJ = dM R^T
    float E[6], F[6];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        E[c] = 2.0f * (dV00 * M[c] + dV01 * M[3 + c]);
        E[3 + c] = 2.0f * (dV10 * M[c] + dV11 * M[3 + c]);
    }
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c)
            F[r * 3 + c] = E[r * 3] * C[c] + E[r * 3 + 1] * C[3 + c] + E[r * 3 + 2] * C[6 + c];
    float dJ[6];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c)
            dJ[r * 3 + c] = F[r * 3] * R[c * 3] + F[r * 3 + 1] * R[c * 3 + 1] + F[r * 3 + 2] * R[c * 3 + 2];
    float dp0 = dJ[2] * (-cp.fx * iz2);
    float dp1 = dJ[5] * (-cp.fy * iz2);
    float dp2 = dJ[0] * (-cp.fx * iz2) + dJ[2] * (2.0f * cp.fx * pc0 * iz2 * iz) + dJ[4] * (-cp.fy * iz2) +
                dJ[5] * (2.0f * cp.fy * pc1 * iz2 * iz);
    dp0 += dmx * cp.fx * iz;
    dp1 += dmy * cp.fy * iz;
    dp2 += dmx * (-cp.fx * pc0 * iz2) + dmy * (-cp.fy * pc1 * iz2);
    float dc0 = R[0] * dp0 + R[3] * dp1 + R[6] * dp2;
    float dc1 = R[1] * dp0 + R[4] * dp1 + R[7] * dp2;
    float dc2 = R[2] * dp0 + R[5] * dp1 + R[8] * dp2;
    // scales / rotation: dM3 = 2 D M3, dR = dM3 diag(s)
    float G[9];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c)
            G[r * 3 + c] = 2.0f * (D[r * 3] * M3[c] + D[r * 3 + 1] * M3[3 + c] + D[r * 3 + 2] * M3[6 + c]);
    float dls[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) dls[k] = (Rq[k] * G[k] + Rq[3 + k] * G[3 + k] + Rq[6 + k] * G[6 + k]) * sc[k];
    float H[9];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) H[r * 3 + c] = G[r * 3 + c] * sc[c];
    // d q_hat = sum(dR .* dR/dq_k), quat_rotation_jacobians (gradients.cpp:25-41)
    float dqh[4];
    dqh[0] = 2.0f * (-z_ * H[1] + y_ * H[2] + z_ * H[3] - x_ * H[5] - y_ * H[6] + x_ * H[7]);
    dqh[1] = 2.0f * (y_ * H[1] + z_ * H[2] + y_ * H[3] - 2.0f * x_ * H[4] - w_ * H[5] + z_ * H[6] + w_ * H[7] -
                     2.0f * x_ * H[8]);
    dqh[2] = 2.0f * (-2.0f * y_ * H[0] + x_ * H[1] + w_ * H[2] + x_ * H[3] + z_ * H[5] - w_ * H[6] + z_ * H[7] -
                     2.0f * y_ * H[8]);
    dqh[3] = 2.0f * (-2.0f * z_ * H[0] - w_ * H[1] + x_ * H[2] + w_ * H[3] - 2.0f * z_ * H[4] + y_ * H[5] +
                     x_ * H[6] + y_ * H[7]);
    float drot[4] = {0.f, 0.f, 0.f, 0.f};
    if (qn > 1e-12f) {
        const float qd = qh[0] * dqh[0] + qh[1] * dqh[1] + qh[2] * dqh[2] + qh[3] * dqh[3];
        const float iq = 1.0f / qn;
#pragma unroll
        for (int k = 0; k < 4; ++k) drot[k] = (dqh[k] - qh[k] * qd) * iq;
    }
    const float dlogit = dopac * opacity * (1.0f - opacity);
    // SH (gradients.cpp:192-219)
    const float u0 = px - cp.center[0], u1 = py - cp.center[1], u2 = pz - cp.center[2];
    const float len = sqrtf(u0 * u0 + u1 * u1 + u2 * u2);
    const float il = 1.0f / len;
    const float d0 = u0 * il, d1 = u1 * il, d2 = u2 * il;
    const int deg = g.sh_degree;
    const int nco = (deg + 1) * (deg + 1);
    float bs[16];
    sh_basis_all(d0, d1, d2, deg, bs);
    float shv[48];
    if (VEC) {
        const float4* s4 = reinterpret_cast<const float4*>(g.sh + 48 * (size_t)i);
#pragma unroll
        for (int k = 0; k < 12; ++k) {
            const float4 vv = s4[k];
            shv[4 * k] = vv.x; shv[4 * k + 1] = vv.y; shv[4 * k + 2] = vv.z; shv[4 * k + 3] = vv.w;
        }
    } else {
#pragma unroll
        for (int k = 0; k < 48; ++k) shv[k] = g.sh[48 * (size_t)i + k];
    }
    float rgb[3] = {0.5f, 0.5f, 0.5f};
#pragma unroll
    for (int k = 0; k < 16; ++k)
        if (k < nco) {
            rgb[0] += bs[k] * shv[3 * k];
            rgb[1] += bs[k] * shv[3 * k + 1];
            rgb[2] += bs[k] * shv[3 * k + 2];
        }
    float dc[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) dc[c] = rgb[c] < 0.0f ? 0.0f : dcol[c];
    float dsh[48];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        const bool on = k < nco;
        dsh[3 * k] = on ? bs[k] * dc[0] : 0.0f;
        dsh[3 * k + 1] = on ? bs[k] * dc[1] : 0.0f;
        dsh[3 * k + 2] = on ? bs[k] * dc[2] : 0.0f;
    }
    if (deg > 0) {
        float coef[16];
#pragma unroll
        for (int k = 0; k < 16; ++k)
            coef[k] = (k >= 1 && k < nco) ? dc[0] * shv[3 * k] + dc[1] * shv[3 * k + 1] + dc[2] * shv[3 * k + 2] : 0.0f;
        float gd[3];
        sh_dir_grad(d0, d1, d2, deg, coef, gd);
        const float dd = d0 * gd[0] + d1 * gd[1] + d2 * gd[2];
        dc0 += (gd[0] - d0 * dd) * il;
        dc1 += (gd[1] - d1 * dd) * il;
        dc2 += (gd[2] - d2 * dd) * il;
    }
    const float dmn = sqrtf(dmx * dmx + dmy * dmy);
    const size_t i3 = 3 * (size_t)i, i4 = 4 * (size_t)i;
    if (accumulate) {
        out.d_centers[i3] += dc0; out.d_centers[i3 + 1] += dc1; out.d_centers[i3 + 2] += dc2;
#pragma unroll
        for (int k = 0; k < 3; ++k) out.d_log_scales[i3 + k] += dls[k];
#pragma unroll
        for (int k = 0; k < 4; ++k) out.d_rotations[i4 + k] += drot[k];
        out.d_opacity_logits[i] += dlogit;
        if (VEC) {
            float4* d4 = reinterpret_cast<float4*>(out.d_sh + 48 * (size_t)i);
#pragma unroll
            for (int k = 0; k < 12; ++k) {
                float4 o = d4[k];
                o.x += dsh[4 * k]; o.y += dsh[4 * k + 1]; o.z += dsh[4 * k + 2]; o.w += dsh[4 * k + 3];
                d4[k] = o;
            }
        } else {
            for (int k = 0; k < 48; ++k) out.d_sh[48 * (size_t)i + k] += dsh[k];
        }
        if (out.grad2d_accum) out.grad2d_accum[i] += dmn;
        if (out.grad2d_count) out.grad2d_count[i] += 1;
    } else {
        out.d_centers[i3] = dc0; out.d_centers[i3 + 1] = dc1; out.d_centers[i3 + 2] = dc2;
#pragma unroll
        for (int k = 0; k < 3; ++k) out.d_log_scales[i3 + k] = dls[k];
#pragma unroll
        for (int k = 0; k < 4; ++k) out.d_rotations[i4 + k] = drot[k];
        out.d_opacity_logits[i] = dlogit;
        if (VEC) {
            float4* d4 = reinterpret_cast<float4*>(out.d_sh + 48 * (size_t)i);
#pragma unroll
            for (int k = 0; k < 12; ++k) d4[k] = make_float4(dsh[4 * k], dsh[4 * k + 1], dsh[4 * k + 2], dsh[4 * k + 3]);
        } else {
            for (int k = 0; k < 48; ++k) out.d_sh[48 * (size_t)i + k] = dsh[k];
        }
        if (out.grad2d_accum) out.grad2d_accum[i] = dmn;
        if (out.grad2d_count) out.grad2d_count[i] = 1;
    }
}

constexpr int kL1Threads = 256;
constexpr int kL1Items = 8;

__global__ void __launch_bounds__(kL1Threads) l1_kernel(const float* __restrict__ a, const float* __restrict__ b,
                                                      int64_t n, float* __restrict__ grad,
                                                      float* __restrict__ partials) {
    __shared__ float s_red[kL1Threads / 32];
    const float inv_n = 1.0f / (float)n;
    float l = 0.0f;
    const int64_t base = (int64_t)blockIdx.x * kL1Threads * kL1Items;
#pragma unroll
    for (int k = 0; k < kL1Items; ++k) {
        const int64_t i = base + (int64_t)k * kL1Threads + threadIdx.x;
        if (i < n) {
            const float d = a[i] - b[i];
            l += fabsf(d);
            if (grad) grad[i] = d > 0.0f ? inv_n : (d < 0.0f ? -inv_n : 0.0f);
        }
    }
    l = warp_sum(l);
    if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = l;
    __syncthreads();
    if (threadIdx.x == 0) {
        float s = 0.0f;
        for (int w = 0; w < kL1Threads / 32; ++w) s += s_red[w];
        partials[blockIdx.x] = s;
    }
}

// Deterministic final sum (fixed order, fp64 accumulation).
__global__ void loss_reduce_kernel(const float* __restrict__ partials, int n, float inv_n, float* __restrict__ loss) {
    __shared__ double s[256];
    double acc = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) acc += (double)partials[i];
    s[threadIdx.x] = acc;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) s[threadIdx.x] += s[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) *loss = (float)s[0] * inv_n;
}

// adam_delta (optimizer.cpp:29-36) with every fp64 operation explicitly rounded (no DFMA), so
// the update is bit-identical to the reference's.
__global__ void adam_kernel(float* __restrict__ param, const float* __restrict__ grad, float* __restrict__ m,
                            float* __restrict__ v, int64_t count, double lr, double lr_alt, int sh_layout,
                            double b1, double omb1, double b2, double omb2, double eps, double bias1, double bias2) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const double g = (double)grad[i];
    const float mf = (float)__dadd_rn(__dmul_rn(b1, (double)m[i]), __dmul_rn(omb1, g));
    const float vf = (float)__dadd_rn(__dmul_rn(b2, (double)v[i]), __dmul_rn(__dmul_rn(omb2, g), g));
    m[i] = mf;
    v[i] = vf;
    const double m_hat = __ddiv_rn((double)mf, bias1);
    const double v_hat = __ddiv_rn((double)vf, bias2);
    const double l = (sh_layout && (i % 48) >= 3) ? lr_alt : lr;
    const float delta = (float)__ddiv_rn(__dmul_rn(l, m_hat), __dadd_rn(__dsqrt_rn(v_hat), eps));
    param[i] = __fsub_rn(param[i], delta);
}

// normalized_quat (gaussian_set.hpp:15-20) in place, optimizer.cpp:69
__global__ void quat_normalize_kernel(float* __restrict__ q, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float* p = q + 4 * (size_t)i;
    const float w = p[0], x = p[1], y = p[2], z = p[3];
    const float s = __fadd_rn(__fadd_rn(__fmul_rn(w, w), __fmul_rn(x, x)), __fadd_rn(__fmul_rn(y, y), __fmul_rn(z, z)));
    const float nn = __fsqrt_rn(s);
    if (!(nn > 0.0f)) {
        p[0] = 1.0f; p[1] = p[2] = p[3] = 0.0f;
        return;
    }
    p[0] = __fdiv_rn(w, nn); p[1] = __fdiv_rn(x, nn); p[2] = __fdiv_rn(y, nn); p[3] = __fdiv_rn(z, nn);
}

inline unsigned blocks_for(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

}  // namespace

cudaError_t launch_blend_backward(LaunchCtx& lc, const CamParams& cp, const uint32_t* ranges,
                                  const uint32_t* pair_gauss, const ProjRec* rec, const float* t_final,
                                  const int32_t* last_index, const float bg[3], const float* d_color,
                                  const float* color, const float* target, float* loss_partials, float* grad2d) {
    const int ts = cp.tile_size;
    const int bw = ts < 16 ? ts : 16;
    const int subs = ts / bw;
    dim3 grid((unsigned)(cp.tiles_x * cp.tiles_y), (unsigned)(subs * subs));
    const float inv_n = 1.0f / (float)(3 * (int64_t)cp.width * cp.height);
    {
        LaunchScope ls_(lc, "blend_backward");
        blend_backward_kernel<<<grid, bw * bw, 0, lc.stream>>>(cp, ranges, pair_gauss, rec, t_final, last_index, bg[0],
                                                          bg[1], bg[2], d_color, color, target, inv_n, loss_partials,
                                                          reinterpret_cast<float4*>(grad2d));
    }
    lc.count++;
    return cudaGetLastError();
}

cudaError_t launch_loss_reduce(LaunchCtx& lc, const float* partials, int n, float inv_n, float* loss) {
    {
        LaunchScope ls_(lc, "loss_reduce");
        loss_reduce_kernel<<<1, 256, 0, lc.stream>>>(partials, n, inv_n, loss);
    }
    lc.count++;
    return cudaGetLastError();
}

cudaError_t launch_chain(LaunchCtx& lc, const GaussianPtrs& g, const CamParams& cp, float* grad2d, const ProjRec* rec,
                         const splat_param_grads& out, int accumulate) {
    if (g.n == 0) return cudaSuccess;
    const bool vec = ((reinterpret_cast<uintptr_t>(g.sh) | reinterpret_cast<uintptr_t>(out.d_sh)) & 15u) == 0;
    if (vec)
        {
            LaunchScope ls_(lc, "chain");
            chain_kernel<true><<<blocks_for(g.n, 128), 128, 0, lc.stream>>>(g, cp, reinterpret_cast<float4*>(grad2d), rec,
                                                                       out, accumulate);
        }
    else
        {
            LaunchScope ls_(lc, "chain");
            chain_kernel<false><<<blocks_for(g.n, 128), 128, 0, lc.stream>>>(g, cp, reinterpret_cast<float4*>(grad2d),
                                                                        rec, out, accumulate);
        }
    lc.count++;
    return cudaGetLastError();
}

int l1_partials_count(int64_t n) { return (int)((n + kL1Threads * kL1Items - 1) / (kL1Threads * kL1Items)); }

cudaError_t launch_l1(LaunchCtx& lc, const float* a, const float* b, int64_t n, float* grad, float* partials,
                      int n_partials) {
    if (n == 0) return cudaSuccess;
    l1_kernel<<<n_partials, kL1Threads, 0, lc.stream>>>(a, b, n, grad, partials);
    lc.count++;
    return cudaGetLastError();
}

cudaError_t launch_adam(LaunchCtx& lc, const AdamGroupArgs& a, double beta1, double beta2, double eps, double bias1,
                        double bias2) {
    if (a.count == 0) return cudaSuccess;
    {
        LaunchScope ls_(lc, "adam");
        adam_kernel<<<blocks_for(a.count, 256), 256, 0, lc.stream>>>(a.param, a.grad, a.m, a.v, a.count, a.lr, a.lr_alt,
                                                                a.sh_layout, beta1, 1.0 - beta1, beta2, 1.0 - beta2,
                                                                eps, bias1, bias2);
    }
    lc.count++;
    return cudaGetLastError();
}

cudaError_t launch_quat_normalize(LaunchCtx& lc, float* rotations, int n) {
    if (n == 0) return cudaSuccess;
    {
        LaunchScope ls_(lc, "quat_normalize");
        quat_normalize_kernel<<<blocks_for(n, 256), 256, 0, lc.stream>>>(rotations, n);
    }
    lc.count++;
    return cudaGetLastError();
}

}  // namespace splat_b200
