// chain.cu — per-Gaussian 2D -> 3D gradient chain (K10, gradients.cpp:127-220).
//
// Compiled with --fmad=false and written in the reference's operation order (the order fixed by
// oracle/compat/Eigen/Dense: halving reductions, left-associative products), so that for equal
// 2D inputs (d_mean2d, d_conic, d_opacity, d_colour) it produces the reference's float results bit
// for bit.  The only GPU-vs-reference gradient difference left is then the summation order of the
// per-pixel contributions in blend_backward.  One thread per Gaussian; ~1 kFLOP each (3% of a
// step), so exactness here is free.
#include <cstdint>

#include "common.cuh"
#include "internal.h"

namespace splat_b200 {

namespace {

__device__ __forceinline__ float dot3(float a0, float a1, float a2, float b0, float b1, float b2) {
    return a0 * b0 + (a1 * b1 + a2 * b2);
}

// sh_basis (sh.hpp:27-51)
__device__ __forceinline__ void sh_basis_all(float x, float y, float z, int degree, float b[16]) {
#pragma unroll
    for (int i = 0; i < 16; ++i) b[i] = 0.0f;
    b[0] = (float)0.28209479177387814;
    if (degree < 1) return;
    const float c1 = (float)0.4886025119029199;
    b[1] = -c1 * y;
    b[2] = c1 * z;
    b[3] = -c1 * x;
    if (degree < 2) return;
    const float xx = x * x, yy = y * y, zz = z * z;
    b[4] = (float)1.0925484305920792 * x * y;
    b[5] = (float)-1.0925484305920792 * y * z;
    b[6] = (float)0.31539156525252005 * (2.0f * zz - xx - yy);
    b[7] = (float)-1.0925484305920792 * x * z;
    b[8] = (float)0.5462742152960396 * (xx - yy);
    if (degree < 3) return;
    b[9] = (float)-0.5900435899266435 * y * (3.0f * xx - yy);
    b[10] = (float)2.890611442640554 * x * y * z;
    b[11] = (float)-0.4570457994644658 * y * (4.0f * zz - xx - yy);
    b[12] = (float)0.3731763325901154 * z * (2.0f * zz - 3.0f * xx - 3.0f * yy);
    b[13] = (float)-0.4570457994644658 * x * (4.0f * zz - xx - yy);
    b[14] = (float)1.445305721320277 * z * (xx - yy);
    b[15] = (float)-0.5900435899266435 * x * (xx - 3.0f * yy);
}

// sh_basis_grad (sh.hpp:55-79): g[k] = d basis_k / d dir
__device__ __forceinline__ void sh_basis_grad_all(float x, float y, float z, int degree, float g[16][3]) {
#pragma unroll
    for (int k = 0; k < 16; ++k) g[k][0] = g[k][1] = g[k][2] = 0.0f;
    if (degree < 1) return;
    const float c1 = (float)0.4886025119029199;
    g[1][1] = -c1;
    g[2][2] = c1;
    g[3][0] = -c1;
    if (degree < 2) return;
    const float xx = x * x, yy = y * y, zz = z * z;
#define SET3(k, C, a, b, c) { const float cc_ = (float)(C); g[k][0] = cc_ * (a); g[k][1] = cc_ * (b); g[k][2] = cc_ * (c); }
    SET3(4, 1.0925484305920792, y, x, 0.0f)
    SET3(5, -1.0925484305920792, 0.0f, z, y)
    SET3(6, 0.31539156525252005, -2.0f * x, -2.0f * y, 4.0f * z)
    SET3(7, -1.0925484305920792, z, 0.0f, x)
    SET3(8, 0.5462742152960396, 2.0f * x, -2.0f * y, 0.0f)
    if (degree < 3) return;
    SET3(9, -0.5900435899266435, 6.0f * x * y, 3.0f * xx - 3.0f * yy, 0.0f)
    SET3(10, 2.890611442640554, y * z, x * z, x * y)
    SET3(11, -0.4570457994644658, -2.0f * x * y, 4.0f * zz - xx - 3.0f * yy, 8.0f * y * z)
    SET3(12, 0.3731763325901154, -6.0f * x * z, -6.0f * y * z, 6.0f * zz - 3.0f * xx - 3.0f * yy)
    SET3(13, -0.4570457994644658, 4.0f * zz - 3.0f * xx - yy, -2.0f * x * y, 8.0f * x * z)
    SET3(14, 1.445305721320277, 2.0f * x * z, -2.0f * y * z, xx - yy)
    SET3(15, -0.5900435899266435, 3.0f * xx - 3.0f * yy, -6.0f * x * y, 0.0f)
#undef SET3
}

constexpr int kChainThreads = 128;
constexpr int kShRow = 13;  // float4 per staged SH row (12 + 1 pad: conflict-free LDS/STS.128)

// One Gaussian.  With VEC, its SH row is read from and its SH gradient row written to s_sh (the
// caller copies rows in and out); untouched Gaussians leave a zero gradient row.
template <bool VEC>
__device__ __forceinline__ void chain_one(GaussianPtrs g, CamParams cp, float4* __restrict__ grad2d,
                                          const ProjRec* __restrict__ rec, splat_param_grads out, int accumulate,
                                          int i, float4* s_sh, int row) {
    if (i >= g.n) return;
    // accumulator (blend_backward, moment form): g0 = (S0, Sx, Sy), g1 = (Sxx, Sxy, Syy) with
    // s = dL/dalpha g per sample, g2 = (d colour, number of committed (warp, pixel) samples)
    const float4 g0 = grad2d[kG2Stride * (size_t)i], g1 = grad2d[kG2Stride * (size_t)i + 1], g2 = grad2d[kG2Stride * (size_t)i + 2];
    const float cnt = g2.w;
    const size_t i3 = 3 * (size_t)i, i4 = 4 * (size_t)i, i48 = 48 * (size_t)i;
    // the per-Gaussian inputs, loaded before the touched test so every load is in flight at once
    const ProjRec pr = rec[i];
    const float p0 = g.centers[i3], p1 = g.centers[i3 + 1], p2 = g.centers[i3 + 2];
    const float qraw[4] = {g.rotations[i4], g.rotations[i4 + 1], g.rotations[i4 + 2], g.rotations[i4 + 3]};
    const float ls[3] = {g.log_scales[i3], g.log_scales[i3 + 1], g.log_scales[i3 + 2]};
    const bool touched = cnt > 0.0f;
    if (!touched) {
        if (!accumulate) {
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                out.d_centers[i3 + k] = 0.0f;
                out.d_log_scales[i3 + k] = 0.0f;
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) out.d_rotations[i4 + k] = 0.0f;
            out.d_opacity_logits[i] = 0.0f;
            if (!VEC)
                for (int k = 0; k < 48; ++k) out.d_sh[i48 + k] = 0.0f;
            if (out.grad2d_accum) out.grad2d_accum[i] = 0.0f;
            if (out.grad2d_count) out.grad2d_count[i] = 0;
        }
        if (VEC) {  // zero gradient row (copied out / added by the caller)
#pragma unroll
            for (int k = 0; k < 12; ++k) s_sh[row * kShRow + k] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        return;
    }
    const float4 zero4 = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int k = 0; k < 3; ++k) grad2d[kG2Stride * (size_t)i + k] = zero4;

    const float k0 = pr.r0.z, k1 = pr.r0.w, k2 = pr.r1.x, opacity = pr.r1.y;
    // moments -> 2D gradients (backward.cu commit_sample): dmean = -o (conic (Sx, Sy)),
    // dconic = -o/2 (Sxx, Sxy, Syy), dopacity = S0
    const float dm0 = -opacity * (k0 * g0.y + k1 * g0.z);
    const float dm1 = -opacity * (k2 * g0.z + k1 * g0.y);
    const float hq = -0.5f * opacity;
    const float dQ[4] = {hq * g1.x, hq * g1.y, hq * g1.y, hq * g1.z};  // row-major (00, 01, 10, 11); 01 == 10
    const float dopac = g0.x;
    const float dcol[3] = {g2.x, g2.y, g2.z};

    const float gaccum = sqrtf(dm0 * dm0 + dm1 * dm1);
    // dV = (-Q) dQ Q
    const float Qn[4] = {-k0, -k1, -k1, -k2};
    const float Q[4] = {k0, k1, k1, k2};
    float N[4], dV[4];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int c = 0; c < 2; ++c) N[r * 2 + c] = Qn[r * 2] * dQ[c] + Qn[r * 2 + 1] * dQ[2 + c];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int c = 0; c < 2; ++c) dV[r * 2 + c] = N[r * 2] * Q[c] + N[r * 2 + 1] * Q[2 + c];

    const float* Rc = cp.R;
    const float fx = cp.fx, fy = cp.fy;
    const float pc0 = dot3(Rc[0], Rc[1], Rc[2], p0, p1, p2) + cp.t[0];
    const float pc1 = dot3(Rc[3], Rc[4], Rc[5], p0, p1, p2) + cp.t[1];
    const float z = dot3(Rc[6], Rc[7], Rc[8], p0, p1, p2) + cp.t[2];
    const float J[6] = {fx / z, 0.0f, -fx * pc0 / (z * z), 0.0f, fy / z, -fy * pc1 / (z * z)};
    float Mm[6];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) Mm[r * 3 + c] = dot3(J[r * 3], J[r * 3 + 1], J[r * 3 + 2], Rc[c], Rc[3 + c], Rc[6 + c]);
    // covariance_from_params
    float Rq0[9];
    rotation_from_quat(qraw, Rq0);
    const float sc[3] = {splat_expf(ls[0]), splat_expf(ls[1]), splat_expf(ls[2])};
    float m3[9], C[9];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) m3[r * 3 + c] = Rq0[r * 3 + c] * sc[c];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = r; c < 3; ++c) {
            const float v = dot3(m3[r * 3], m3[r * 3 + 1], m3[r * 3 + 2], m3[c * 3], m3[c * 3 + 1], m3[c * 3 + 2]);
            C[r * 3 + c] = v;
            C[c * 3 + r] = v;
        }
    // d_cov3d = M^T dV M
    float P[6], D[9];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 2; ++c) P[r * 2 + c] = Mm[0 * 3 + r] * dV[0 * 2 + c] + Mm[1 * 3 + r] * dV[1 * 2 + c];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) D[r * 3 + c] = P[r * 2] * Mm[0 * 3 + c] + P[r * 2 + 1] * Mm[1 * 3 + c];
    // dM = 2 dV M cov3d ; dJ = dM R^T
    float dV2[4], E[6], F[6], dJ[6];
#pragma unroll
    for (int k = 0; k < 4; ++k) dV2[k] = 2.0f * dV[k];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) E[r * 3 + c] = dV2[r * 2] * Mm[0 * 3 + c] + dV2[r * 2 + 1] * Mm[1 * 3 + c];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) F[r * 3 + c] = dot3(E[r * 3], E[r * 3 + 1], E[r * 3 + 2], C[c], C[3 + c], C[6 + c]);
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c)
            dJ[r * 3 + c] = dot3(F[r * 3], F[r * 3 + 1], F[r * 3 + 2], Rc[c * 3], Rc[c * 3 + 1], Rc[c * 3 + 2]);
    float dp[3] = {0.0f, 0.0f, 0.0f};
    dp[0] += dJ[2] * (-fx / (z * z));
    dp[1] += dJ[5] * (-fy / (z * z));
    dp[2] += dJ[0] * (-fx / (z * z)) + dJ[2] * (2.0f * fx * pc0 / (z * z * z)) + dJ[4] * (-fy / (z * z)) +
             dJ[5] * (2.0f * fy * pc1 / (z * z * z));
    dp[0] += dm0 * fx / z;
    dp[1] += dm1 * fy / z;
    dp[2] += dm0 * (-fx * pc0 / (z * z)) + dm1 * (-fy * pc1 / (z * z));
    float dcen[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) dcen[k] = dot3(Rc[k], Rc[3 + k], Rc[6 + k], dp[0], dp[1], dp[2]);
    // M3 = R(q_hat) diag(s); note rotation_from_quat normalises q_hat again (gradients.cpp:173-174)
    float qh[4], Rq[9], M3[9], D2[9], G[9], H[9];
    normalized_quat(qraw[0], qraw[1], qraw[2], qraw[3], qh);
    rotation_from_quat(qh, Rq);
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) M3[r * 3 + c] = Rq[r * 3 + c] * sc[c];
#pragma unroll
    for (int k = 0; k < 9; ++k) D2[k] = 2.0f * D[k];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c)
            G[r * 3 + c] = dot3(D2[r * 3], D2[r * 3 + 1], D2[r * 3 + 2], M3[c], M3[3 + c], M3[6 + c]);
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) H[r * 3 + c] = G[r * 3 + c] * sc[c];
    float dls[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) dls[k] = dot3(Rq[k], Rq[3 + k], Rq[6 + k], G[k], G[3 + k], G[6 + k]) * sc[k];
    const float w_ = qh[0], x_ = qh[1], y_ = qh[2], z_ = qh[3];
    const float dRq[4][9] = {{0.0f, -z_, y_, z_, 0.0f, -x_, -y_, x_, 0.0f},
                             {0.0f, y_, z_, y_, -2.0f * x_, -w_, z_, w_, -2.0f * x_},
                             {-2.0f * y_, x_, w_, x_, 0.0f, z_, -w_, z_, -2.0f * y_},
                             {-2.0f * z_, -w_, x_, w_, -2.0f * z_, y_, x_, y_, 0.0f}};
    float dqh[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        float e[9];  // column-major element order of H .* (2 dR/dq_k)
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
            for (int r = 0; r < 3; ++r) e[c * 3 + r] = H[r * 3 + c] * (dRq[k][r * 3 + c] * 2.0f);
        dqh[k] = ((e[0] + e[1]) + (e[2] + e[3])) + ((e[4] + e[5]) + (e[6] + (e[7] + e[8])));
    }
    float drot[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    const float qn = sqrtf((qraw[0] * qraw[0] + qraw[1] * qraw[1]) + (qraw[2] * qraw[2] + qraw[3] * qraw[3]));
    const bool rot_ok = qn > 1e-12f;
    if (rot_ok) {
        const float qd = (qh[0] * dqh[0] + qh[1] * dqh[1]) + (qh[2] * dqh[2] + qh[3] * dqh[3]);
#pragma unroll
        for (int k = 0; k < 4; ++k) drot[k] = (dqh[k] - qh[k] * qd) / qn;
    }
    const float dlogit = dopac * opacity * (1.0f - opacity);
    // SH (gradients.cpp:192-219)
    const float u0 = p0 - cp.center[0], u1 = p1 - cp.center[1], u2 = p2 - cp.center[2];
    const float len = sqrtf(dot3(u0, u1, u2, u0, u1, u2));
    const float dir0 = u0 / len, dir1 = u1 / len, dir2 = u2 / len;
    const int deg = g.sh_degree;
    const int nco = (deg + 1) * (deg + 1);
    float basis[16];
    sh_basis_all(dir0, dir1, dir2, deg, basis);
    // SH coefficient j = 3 k + c, streamed from the staged shared-memory row a float4 at a time
    // (conflict-free LDS.128 on the padded rows) in j order — the per-channel summation order of
    // the reference — instead of 48 registers held across the SH section
    const float4* s4 = VEC ? &s_sh[row * kShRow] : nullptr;
    auto sh_quad = [&](int q) -> float4 {
        if (VEC) return s4[q];
        return make_float4(g.sh[i48 + 4 * q], g.sh[i48 + 4 * q + 1], g.sh[i48 + 4 * q + 2], g.sh[i48 + 4 * q + 3]);
    };
    float rgb[3] = {0.5f, 0.5f, 0.5f};
#pragma unroll
    for (int q = 0; q < 12; ++q) {
        const float4 v4 = sh_quad(q);
        const float vv[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int j = 4 * q + e, k = j / 3, c = j % 3;
            if (k < nco) rgb[c] = rgb[c] + basis[k] * vv[e];
        }
    }
    float dc[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) dc[c] = rgb[c] < 0.0f ? 0.0f : dcol[c];
    if (deg > 0) {
        float gb[16][3];
        sh_basis_grad_all(dir0, dir1, dir2, deg, gb);
        float dd[3] = {0.0f, 0.0f, 0.0f};
        float coef = 0.0f;
#pragma unroll
        for (int q = 0; q < 12; ++q) {
            const float4 v4 = sh_quad(q);
            const float vv[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int j = 4 * q + e, k = j / 3, c = j % 3;
                if (k < 1 || k >= nco) continue;
                coef = (c == 0 ? 0.0f : coef) + dc[c] * vv[e];
                if (c == 2) {
                    dd[0] = dd[0] + gb[k][0] * coef;
                    dd[1] = dd[1] + gb[k][1] * coef;
                    dd[2] = dd[2] + gb[k][2] * coef;
                }
            }
        }
        const float ddot = dot3(dir0, dir1, dir2, dd[0], dd[1], dd[2]);
        dcen[0] = dcen[0] + (dd[0] - dir0 * ddot) / len;
        dcen[1] = dcen[1] + (dd[1] - dir1 * ddot) / len;
        dcen[2] = dcen[2] + (dd[2] - dir2 * ddot) / len;
    }
    // write (fresh ParamGrads: 0 + x; accumulate: existing + x, ParamGrads::add)
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const float bc = accumulate ? out.d_centers[i3 + k] : 0.0f;
        const float bs = accumulate ? out.d_log_scales[i3 + k] : 0.0f;
        out.d_centers[i3 + k] = bc + dcen[k];
        out.d_log_scales[i3 + k] = bs + dls[k];
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const float br = accumulate ? out.d_rotations[i4 + k] : 0.0f;
        out.d_rotations[i4 + k] = br + drot[k];
    }
    out.d_opacity_logits[i] = (accumulate ? out.d_opacity_logits[i] : 0.0f) + dlogit;
    // d_sh = basis_k * dc (zero past the active degree), after the SH row's last read
#pragma unroll
    for (int q = 0; q < 12; ++q) {
        float d[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int j = 4 * q + e, k = j / 3, c = j % 3;
            d[e] = k < nco ? basis[k] * dc[c] : 0.0f;
        }
        if (VEC) {  // the fresh gradient row, over the staged SH row; the caller writes (or adds) it coalesced
            s_sh[row * kShRow + q] = make_float4(d[0], d[1], d[2], d[3]);
        } else {
#pragma unroll
            for (int e = 0; e < 4; ++e)
                out.d_sh[i48 + 4 * q + e] = (accumulate ? out.d_sh[i48 + 4 * q + e] : 0.0f) + d[e];
        }
    }
    if (out.grad2d_accum) out.grad2d_accum[i] = (accumulate ? out.grad2d_accum[i] : 0.0f) + gaccum;
    if (out.grad2d_count) out.grad2d_count[i] = (accumulate ? out.grad2d_count[i] : 0) + 1;
}

// Plain one-thread-per-Gaussian chain (SH pointers not 16-byte aligned).
__global__ void __launch_bounds__(kChainThreads) chain_kernel(GaussianPtrs g, CamParams cp, float4* __restrict__ grad2d,
                                                             const ProjRec* __restrict__ rec, splat_param_grads out,
                                                             int accumulate) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    chain_one<false>(g, cp, grad2d, rec, out, accumulate, i, nullptr, 0);
}

// Zero count floats from p, cooperatively by one warp (float4 stores when p is 16-byte aligned).
__device__ __forceinline__ void zero_span_warp(float* p, int count, int lane) {
    int head = 0;
    if ((reinterpret_cast<uintptr_t>(p) & 15u) == 0) {
        const int n4 = count >> 2;
        float4* p4 = reinterpret_cast<float4*>(p);
        for (int q = lane; q < n4; q += 32) p4[q] = make_float4(0.f, 0.f, 0.f, 0.f);
        head = n4 << 2;
    }
    for (int q = head + lane; q < count; q += 32) p[q] = 0.0f;
}

// Only Gaussians some pixel committed ("touched": a fraction of the survivors) need the chain.
// Pass 1 lists them (warp-aggregated append; list order is irrelevant, every Gaussian's chain is
// independent) and, for a fresh gradient, writes the zero gradients of all others with
// coalesced stores.  Pass 2 runs the chain on the list with every lane busy; each thread stages
// its own 192-byte SH row in shared memory with float4 loads and writes its gradient row back
// the same way.
constexpr int kCompactItems = 4;  // Gaussians per thread in chain_compact (four commit-count loads in flight)

__global__ void __launch_bounds__(256) chain_compact_kernel(const float4* __restrict__ grad2d, int n,
                                                            splat_param_grads out, int zero_untouched,
                                                            uint32_t* __restrict__ list, uint32_t* __restrict__ count,
                                                            uint32_t* __restrict__ count_next) {
    // one list append (atomic) per CTA: a single counter takes ~1 ns per atomic, so per-warp
    // appends would serialise ~n/32 of them.  The CTA's 1024 rows are listed in index order.
    __shared__ uint32_t s_wc[kCompactItems * 8];
    __shared__ uint32_t s_base;
    pdl_trigger();  // chain_touched (PDL) may be scheduled
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int base = blockIdx.x * (256 * kCompactItems);
    bool touched[kCompactItems];
#pragma unroll
    for (int k = 0; k < kCompactItems; ++k) {
        const int i = base + k * 256 + threadIdx.x;
        touched[k] = i < n && grad2d[kG2Stride * (size_t)i + 2].w > 0.0f;
    }
    unsigned m[kCompactItems];
#pragma unroll
    for (int k = 0; k < kCompactItems; ++k) {
        m[k] = __ballot_sync(0xffffffffu, touched[k]);
        if (lane == 0) s_wc[k * 8 + warp] = __popc(m[k]);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t tot = 0;
        for (int w = 0; w < kCompactItems * 8; ++w) {
            const uint32_t c = s_wc[w];
            s_wc[w] = tot;
            tot += c;
        }
        s_base = tot ? atomicAdd(count, tot) : 0u;
        // the other slot was consumed by the previous view's chain (stream order): zero it for the
        // next view, so no memset precedes this kernel
        if (blockIdx.x == 0) *count_next = 0u;
    }
    __syncthreads();
    const unsigned lt = lanemask_lt();
#pragma unroll
    for (int k = 0; k < kCompactItems; ++k)
        if (touched[k]) list[s_base + s_wc[k * 8 + warp] + __popc(m[k] & lt)] = (uint32_t)(base + k * 256 + threadIdx.x);
    if (!zero_untouched) return;  // accumulating, or the rows are already zero
    // Every gradient of the warp's rows is zeroed here (touched ones are overwritten by pass 2):
    // each array's span for the warp's 32 rows is contiguous, so the warp writes it with float4
    // stores (full sectors only).
#pragma unroll 1
    for (int k = 0; k < kCompactItems; ++k) {
        const int w0 = base + k * 256 + warp * 32;
        const int rows = min(32, n - w0);
        if (rows <= 0) return;
        zero_span_warp(out.d_centers + 3 * (size_t)w0, 3 * rows, lane);
        zero_span_warp(out.d_log_scales + 3 * (size_t)w0, 3 * rows, lane);
        zero_span_warp(out.d_rotations + 4 * (size_t)w0, 4 * rows, lane);
        zero_span_warp(out.d_opacity_logits + (size_t)w0, rows, lane);
        zero_span_warp(out.d_sh + 48 * (size_t)w0, 48 * rows, lane);
        if (out.grad2d_accum) zero_span_warp(out.grad2d_accum + (size_t)w0, rows, lane);
        if (out.grad2d_count && lane < rows) out.grad2d_count[w0 + lane] = 0;
    }
}

__global__ void __launch_bounds__(kChainThreads) chain_touched_kernel(GaussianPtrs g, CamParams cp,
                                                                     float4* __restrict__ grad2d,
                                                                     const ProjRec* __restrict__ rec,
                                                                     splat_param_grads out, int accumulate,
                                                                     const uint32_t* __restrict__ list,
                                                                     const uint32_t* __restrict__ count) {
    __shared__ float4 s_sh[kChainThreads * kShRow];
    pdl_wait();
    pdl_trigger();
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (int)*count) return;
    const int i = (int)list[t];
    const int row = threadIdx.x;
    const float4* src = reinterpret_cast<const float4*>(g.sh + 48 * (size_t)i);
#pragma unroll
    for (int k = 0; k < 12; ++k) s_sh[row * kShRow + k] = __ldg(src + k);
    chain_one<true>(g, cp, grad2d, rec, out, accumulate, i, s_sh, row);
    float4* dst = reinterpret_cast<float4*>(out.d_sh + 48 * (size_t)i);
#pragma unroll
    for (int k = 0; k < 12; ++k) {
        const float4 d = s_sh[row * kShRow + k];
        if (accumulate) {
            float4 o = dst[k];
            o.x = o.x + d.x; o.y = o.y + d.y; o.z = o.z + d.z; o.w = o.w + d.w;
            dst[k] = o;
        } else {
            dst[k] = d;
        }
    }
}

inline unsigned blocks_for(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

}  // namespace

cudaError_t launch_chain(LaunchCtx& lc, const GaussianPtrs& g, const CamParams& cp, float* grad2d, const ProjRec* rec,
                         const splat_param_grads& out, int accumulate, int n_surv, uint32_t* list,
                         bool prezeroed) {
    if (g.n == 0) return cudaSuccess;
    const bool vec = ((reinterpret_cast<uintptr_t>(g.sh) | reinterpret_cast<uintptr_t>(out.d_sh)) & 15u) == 0;
    float4* g2 = reinterpret_cast<float4*>(grad2d);
    if (!vec) {
        LaunchScope ls(lc, "chain");
        chain_kernel<<<blocks_for(g.n, kChainThreads), kChainThreads, 0, lc.stream>>>(g, cp, g2, rec, out, accumulate);
        lc.count++;
        return cudaGetLastError();
    }
    // touched-list length: two slots (work_counters[4 + parity]) used alternately, each zeroed by the
    // compact kernel of the call before its next use (zero at rest initially)
    uint32_t* count = reinterpret_cast<uint32_t*>(lc.work_counters + 4 + lc.chain_parity);
    uint32_t* count_next = reinterpret_cast<uint32_t*>(lc.work_counters + 5 - lc.chain_parity);
    lc.chain_parity ^= 1;
    {
        LaunchScope ls(lc, "chain_compact");
        chain_compact_kernel<<<blocks_for(g.n, 256 * kCompactItems), 256, 0, lc.stream>>>(g2, g.n, out, !accumulate && !prezeroed,
                                                                          list, count, count_next);
        lc.count++;
    }
    if (n_surv > 0) {
        LaunchScope ls(lc, "chain");
        const cudaError_t e = launch_pdl(lc.stream, chain_touched_kernel, dim3(blocks_for(n_surv, kChainThreads)),
                                         dim3(kChainThreads), 0, g, cp, g2, rec, out, accumulate,
                                         (const uint32_t*)list, (const uint32_t*)count);
        if (e != cudaSuccess) return e;
        lc.count++;
    }
    return cudaGetLastError();
}

}  // namespace splat_b200
