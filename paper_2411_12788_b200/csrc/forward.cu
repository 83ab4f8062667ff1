// forward.cu — preprocess, tile-pair emission, tile ranges, per-tile blend forward (+ importance,
// argmax depth) and depth unprojection.  Compiled with --fmad=false: every float expression is
// evaluated with separately rounded operations in the order written, which is the reference's
// order (oracle/compat/Eigen/Dense), so integer outputs and forward images are bit-exact
// against the oracle.
#include <cstdint>

#include "common.cuh"
#include "internal.h"

namespace splat_b200 {
#ifdef SPLAT_STATS
// Instrumented builds only (tools/stats_build.sh): forward traversal counters, read with
// splat_debug_stats.
__device__ unsigned long long g_stats[12];
#endif

namespace {

__device__ __forceinline__ float dot3(float a0, float a1, float a2, float b0, float b1, float b2) {
    return a0 * b0 + (a1 * b1 + a2 * b2);  // Eigen 3.4 unrolled redux: x0 + (x1 + x2)
}

// sh_basis (sh.hpp:27-51)
__device__ __forceinline__ void sh_basis16(float x, float y, float z, int degree, float b[16]);

// sh_to_color (sh.hpp:84-100) with the 48 coefficients fetched a float4 at a time by quad(q)
// (coefficient j = 3 k + c), accumulated in j order — per channel, the reference's k order.
template <typename Quad>
__device__ __forceinline__ void sh_color_stream(Quad quad, float x, float y, float z, int degree, float rgb[3]) {
    float b[16];
    sh_basis16(x, y, z, degree, b);
    rgb[0] = rgb[1] = rgb[2] = 0.5f;
    const int n = (degree + 1) * (degree + 1);
#pragma unroll
    for (int q = 0; q < 12; ++q) {
        const float4 v4 = quad(q);
        const float vv[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int j = 4 * q + e, k = j / 3, c = j % 3;
            if (k < n) rgb[c] = rgb[c] + b[k] * vv[e];
        }
    }
#pragma unroll
    for (int c = 0; c < 3; ++c)
        if (rgb[c] < 0.0f) rgb[c] = 0.0f;
}

__device__ __forceinline__ void sh_basis16(float x, float y, float z, int degree, float b[16]) {
#pragma unroll
    for (int i = 0; i < 16; ++i) b[i] = 0.0f;
    b[0] = (float)(0.28209479177387814);
    if (degree >= 1) {
        const float c1 = (float)(0.4886025119029199);
        b[1] = -c1 * y;
        b[2] = c1 * z;
        b[3] = -c1 * x;
    }
    const float xx = x * x, yy = y * y, zz = z * z;
    if (degree >= 2) {
        b[4] = (float)(1.0925484305920792) * x * y;
        b[5] = (float)(-1.0925484305920792) * y * z;
        b[6] = (float)(0.31539156525252005) * (2.0f * zz - xx - yy);
        b[7] = (float)(-1.0925484305920792) * x * z;
        b[8] = (float)(0.5462742152960396) * (xx - yy);
    }
    if (degree >= 3) {
        b[9] = (float)(-0.5900435899266435) * y * (3.0f * xx - yy);
        b[10] = (float)(2.890611442640554) * x * y * z;
        b[11] = (float)(-0.4570457994644658) * y * (4.0f * zz - xx - yy);
        b[12] = (float)(0.3731763325901154) * z * (2.0f * zz - 3.0f * xx - 3.0f * yy);
        b[13] = (float)(-0.4570457994644658) * x * (4.0f * zz - xx - yy);
        b[14] = (float)(1.445305721320277) * z * (xx - yy);
        b[15] = (float)(-0.5900435899266435) * x * (xx - 3.0f * yy);
    }
}

__device__ __forceinline__ float std_max(float a, float b) { return (a < b) ? b : a; }
__device__ __forceinline__ float std_min(float a, float b) { return (b < a) ? b : a; }

constexpr int kPreThreads = 128;
constexpr int kShRow = 13;  // float4 per staged SH row (12 + 1 pad: conflict-free LDS.128)

// project<T> body for one Gaussian (rasterizer.cpp:24-82).  With VEC_SH the block first copies its
// Gaussians' 192-byte SH rows into shared memory with coalesced float4 loads.
template <bool VEC_SH>
__global__ void __launch_bounds__(kPreThreads) preprocess_kernel(GaussianPtrs g, CamParams cp, const uint8_t* __restrict__ mask,
                                                        ProjRec* __restrict__ rec, AuxRec* __restrict__ aux,
                                                        uint32_t* __restrict__ keys, uint32_t* __restrict__ vals,
                                                        uint32_t* __restrict__ tile_counts,
                                                        uint32_t* __restrict__ n_surv, float* __restrict__ depth_out,
                                                        uint2* __restrict__ rect_ref, float4* __restrict__ proj_dbg) {
    __shared__ float4 s_sh[VEC_SH ? kPreThreads * kShRow : 1];
    pdl_wait();
    pdl_trigger();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (VEC_SH) {
        // the block's SH rows stream into shared memory (cp.async, coalesced) while the geometry
        // below runs; the colour waits for them after the projection
        const int base = blockIdx.x * kPreThreads;
        const int cnt = min(kPreThreads, g.n - base);
        const float4* src = reinterpret_cast<const float4*>(g.sh + 48 * (size_t)base);
        const uint32_t dst0 = (uint32_t)__cvta_generic_to_shared(s_sh);
        for (int q = threadIdx.x; q < cnt * 12; q += kPreThreads)
            cp_async16(dst0 + 16u * (uint32_t)((q / 12) * kShRow + q % 12), src + q);
        cp_async_commit();
    }
    bool want_rgb = false;
    float u0 = 0.f, u1 = 0.f, u2 = 0.f;
    bool alive = i < g.n;
    if (alive && mask && !mask[i]) alive = false;
    float px = 0.f, py = 0.f, pz = 0.f, zc = 0.f;
    float pc0 = 0.f, pc1 = 0.f;
    // every parameter load issued up front (independent of the culls) so their latencies overlap
    float ls0 = 0.f, ls1 = 0.f, ls2 = 0.f, qw = 0.f, qx = 0.f, qy = 0.f, qz = 0.f, ologit = 0.f;
    if (i < g.n) {
        px = __ldg(&g.centers[3 * i]);
        py = __ldg(&g.centers[3 * i + 1]);
        pz = __ldg(&g.centers[3 * i + 2]);
        ls0 = __ldg(&g.log_scales[3 * i]);
        ls1 = __ldg(&g.log_scales[3 * i + 1]);
        ls2 = __ldg(&g.log_scales[3 * i + 2]);
        if ((reinterpret_cast<uintptr_t>(g.rotations) & 15u) == 0) {
            const float4 q4 = __ldg(reinterpret_cast<const float4*>(g.rotations) + i);
            qw = q4.x; qx = q4.y; qy = q4.z; qz = q4.w;
        } else {
            qw = __ldg(&g.rotations[4 * i]);
            qx = __ldg(&g.rotations[4 * i + 1]);
            qy = __ldg(&g.rotations[4 * i + 2]);
            qz = __ldg(&g.rotations[4 * i + 3]);
        }
        ologit = __ldg(&g.opacity_logits[i]);
    }
    if (alive) {
        pc0 = dot3(cp.R[0], cp.R[1], cp.R[2], px, py, pz) + cp.t[0];
        pc1 = dot3(cp.R[3], cp.R[4], cp.R[5], px, py, pz) + cp.t[1];
        zc = dot3(cp.R[6], cp.R[7], cp.R[8], px, py, pz) + cp.t[2];
        if (zc <= cp.znear) alive = false;
    }
    ProjRec r;
    AuxRec a;
    uint2 ref_rect = make_uint2(0u, 0u);
    uint32_t count = 0, tiles = 0;
    if (alive) {
        const float z = zc;
        const float m0 = cp.fx * pc0 / z + cp.cx;
        const float m1 = cp.fy * pc1 / z + cp.cy;
        // covariance_from_params (gaussian_set.hpp:41-55)
        const float qn = sqrtf((qw * qw + qx * qx) + (qy * qy + qz * qz));
        if (!(qn > 0.0f)) {
            qw = 1.0f; qx = qy = qz = 0.0f;
        } else {
            qw = qw / qn; qx = qx / qn; qy = qy / qn; qz = qz / qn;
        }
        float Rq[9];
        Rq[0] = 1.0f - 2.0f * (qy * qy + qz * qz);
        Rq[1] = 2.0f * (qx * qy - qw * qz);
        Rq[2] = 2.0f * (qx * qz + qw * qy);
        Rq[3] = 2.0f * (qx * qy + qw * qz);
        Rq[4] = 1.0f - 2.0f * (qx * qx + qz * qz);
        Rq[5] = 2.0f * (qy * qz - qw * qx);
        Rq[6] = 2.0f * (qx * qz - qw * qy);
        Rq[7] = 2.0f * (qy * qz + qw * qx);
        Rq[8] = 1.0f - 2.0f * (qx * qx + qy * qy);
        const float s0 = splat_expf(ls0), s1 = splat_expf(ls1), s2 = splat_expf(ls2);
        float Mq[9];
#pragma unroll
        for (int rr = 0; rr < 3; ++rr) {
            Mq[rr * 3 + 0] = Rq[rr * 3 + 0] * s0;
            Mq[rr * 3 + 1] = Rq[rr * 3 + 1] * s1;
            Mq[rr * 3 + 2] = Rq[rr * 3 + 2] * s2;
        }
        float C[9];
#pragma unroll
        for (int rr = 0; rr < 3; ++rr)
#pragma unroll
            for (int cc = rr; cc < 3; ++cc) {
                const float v = dot3(Mq[rr * 3], Mq[rr * 3 + 1], Mq[rr * 3 + 2], Mq[cc * 3], Mq[cc * 3 + 1],
                                     Mq[cc * 3 + 2]);
                C[rr * 3 + cc] = v;
                C[cc * 3 + rr] = v;
            }
        // EWA: cov2d = (J R) cov3d (J R)^T + lowpass I
        const float J00 = cp.fx / z, J02 = -cp.fx * pc0 / (z * z);
        const float J11 = cp.fy / z, J12 = -cp.fy * pc1 / (z * z);
        const float J[6] = {J00, 0.0f, J02, 0.0f, J11, J12};
        float M[6], A[6];
#pragma unroll
        for (int rr = 0; rr < 2; ++rr)
#pragma unroll
            for (int cc = 0; cc < 3; ++cc)
                M[rr * 3 + cc] = dot3(J[rr * 3], J[rr * 3 + 1], J[rr * 3 + 2], cp.R[cc], cp.R[3 + cc], cp.R[6 + cc]);
#pragma unroll
        for (int rr = 0; rr < 2; ++rr)
#pragma unroll
            for (int cc = 0; cc < 3; ++cc)
                A[rr * 3 + cc] = dot3(M[rr * 3], M[rr * 3 + 1], M[rr * 3 + 2], C[cc], C[3 + cc], C[6 + cc]);
        const float V00 = dot3(A[0], A[1], A[2], M[0], M[1], M[2]);
        const float V01 = dot3(A[0], A[1], A[2], M[3], M[4], M[5]);
        const float V11 = dot3(A[3], A[4], A[5], M[3], M[4], M[5]);
        const float c0 = V00 + cp.lowpass, c1 = V01, c2 = V11 + cp.lowpass;
        const float det = c0 * c2 - c1 * c1;
        if (!(det > 0.0f)) {
            alive = false;
        } else {
            const float inv_det = 1.0f / det;
            const float k0 = c2 * inv_det, k1 = -c1 * inv_det, k2 = c0 * inv_det;
            int x0, x1, y0, y1;
            int radius = max(cp.width, cp.height);  // exact mode (rasterizer.cpp:53-56)
            if (!cp.apply_thresholds) {
                x0 = 0; x1 = cp.width; y0 = 0; y1 = cp.height;
            } else {
                const float mid = 0.5f * (c0 + c2);
                const float lmax = mid + sqrtf(std_max(mid * mid - det, 0.0f));
                radius = (int)ceilf(cp.radius_sigmas * sqrtf(lmax));
                const float rf = (float)radius;
                x0 = max(0, (int)ceilf(m0 - rf - 0.5f));
                x1 = min(cp.width, (int)floorf(m0 + rf - 0.5f) + 1);
                y0 = max(0, (int)ceilf(m1 - rf - 0.5f));
                y1 = min(cp.height, (int)floorf(m1 + rf - 0.5f) + 1);
                if (x0 >= x1 || y0 >= y1) alive = false;
            }
            if (alive) {
                const float opacity = 1.0f / (1.0f + splat_expf(-ologit));
                // view_dir = (p - cam_center).normalized(); the SH colour follows after the barrier
                u0 = px - cp.center[0];
                u1 = py - cp.center[1];
                u2 = pz - cp.center[2];
                const float zz = dot3(u0, u1, u2, u0, u1, u2);
                if (zz > 0.0f) {
                    const float nn = sqrtf(zz);
                    u0 = u0 / nn; u1 = u1 / nn; u2 = u2 / nn;
                }
                want_rgb = true;
                const int ts = cp.tile_size;
                const int tx0 = x0 / ts, tx1 = (x1 - 1) / ts, ty0 = y0 / ts, ty1 = (y1 - 1) / ts;
                tiles = (uint32_t)((tx1 - tx0 + 1) * (ty1 - ty0 + 1));
                count = (uint32_t)((tx1 / 4 - tx0 / 4 + 1) * (ty1 / 4 - ty0 / 4 + 1));  // supertiles
                r.r0 = make_float4(m0, m1, k0, k1);
                r.r1 = make_float4(k2, opacity, __uint_as_float(pack_range(x0, x1)),
                                   __uint_as_float(pack_range(y0, y1)));
                // cut = ln(cmin / opacity) - 1e-3: below it alpha cannot reach the floor
                const float cut = cp.apply_thresholds ? logf(cp.contribution_min / opacity) - 1e-3f : -INFINITY;
                // Effective rect for blending: the reference rect intersected with the bounding box
                // of the ellipse power >= cut, i.e. |dx| <= sqrt(-2 cut cov2d_xx) (the conic is the
                // inverse of cov2d); 1e-4 relative + 0.01 px of slack cover every rounding.
                int ex0 = x0, ex1 = x1, ey0 = y0, ey1 = y1;
                if (cp.apply_thresholds) {
                    if (!(cut < 0.0f)) {
                        ex1 = ex0;
                        ey1 = ey0;
                    } else {
                        const float Q = -2.0f * cut;
                        const float rx = sqrtf(Q * c0) * 1.0001f + 0.01f;
                        const float ry = sqrtf(Q * c2) * 1.0001f + 0.01f;
                        ex0 = max(x0, (int)ceilf(m0 - rx - 0.5f));
                        ex1 = min(x1, (int)floorf(m0 + rx - 0.5f) + 1);
                        ey0 = max(y0, (int)ceilf(m1 - ry - 0.5f));
                        ey1 = min(y1, (int)floorf(m1 + ry - 0.5f) + 1);
                        if (ex1 < ex0) ex1 = ex0;
                        if (ey1 < ey0) ey1 = ey0;
                    }
                }
                r.r0 = make_float4(m0, m1, k0, k1);
                r.r1 = make_float4(k2, opacity, __uint_as_float(pack_range(ex0, ex1)),
                                   __uint_as_float(pack_range(ey0, ey1)));
                r.r2 = make_float4(0.f, 0.f, 0.f, cut);  // colour filled in after the SH barrier
                ref_rect = make_uint2(pack_range(x0, x1), pack_range(y0, y1));
                if (proj_dbg) proj_dbg[i] = make_float4(c0, c1, c2, __int_as_float(radius));  // splat_project
                if (aux) {
                    const float smax = std_max(std_max(ls0, ls1), ls2);
                    const float smin = std_min(std_min(ls0, ls1), ls2);
                    const bool degenerate = 2.0f * (smax - smin) > cp.log_cond_limit;
                    a.a0 = make_float4(px, py, pz, degenerate ? 1.0f : 0.0f);
                    if (degenerate) {
                        a.a1 = make_float4(1.0f, 0.0f, 0.0f, 1.0f);
                        a.a2 = make_float4(0.0f, 1.0f, 0.0f, 0.0f);
                    } else {
                        // Eigen cofactor inverse (compat/Eigen/Dense)
#define CM(r_, c_) C[(r_) * 3 + (c_)]
#define COF(i_, j_) (CM(((i_) + 1) % 3, ((j_) + 1) % 3) * CM(((i_) + 2) % 3, ((j_) + 2) % 3) - \
                     CM(((i_) + 1) % 3, ((j_) + 2) % 3) * CM(((i_) + 2) % 3, ((j_) + 1) % 3))
                        const float f00 = COF(0, 0), f10 = COF(1, 0), f20 = COF(2, 0);
                        const float dt = f00 * CM(0, 0) + (f10 * CM(1, 0) + f20 * CM(2, 0));
                        const float inv = 1.0f / dt;
                        const float i00 = f00 * inv, i01 = f10 * inv, i02 = f20 * inv;
                        const float i11 = COF(1, 1) * inv, i12 = COF(2, 1) * inv, i22 = COF(2, 2) * inv;
#undef COF
#undef CM
                        a.a1 = make_float4(i00, i01, i02, i11);
                        a.a2 = make_float4(i12, i22, 0.0f, 0.0f);
                    }
                }
            }
        }
    }
    if (VEC_SH) {
        cp_async_wait_all();
        __syncthreads();
    }
    if (want_rgb && alive) {  // sh_to_color (rasterizer.cpp:75)
        float rgb[3];
        const float4* s4 = &s_sh[threadIdx.x * kShRow];
        const float* shg = g.sh + 48 * (size_t)i;
        sh_color_stream(
            [&](int q) -> float4 {
                if (VEC_SH) return s4[q];
                return make_float4(__ldg(shg + 4 * q), __ldg(shg + 4 * q + 1), __ldg(shg + 4 * q + 2),
                                   __ldg(shg + 4 * q + 3));
            },
            u0, u1, u2, g.sh_degree, rgb);
        r.r2.x = rgb[0];
        r.r2.y = rgb[1];
        r.r2.z = rgb[2];
    }
    if (i < g.n) {
        keys[i] = alive ? __float_as_uint(zc) : 0xffffffffu;
        vals[i] = (uint32_t)i;
        tile_counts[i] = alive ? count : 0u;
        depth_out[i] = alive ? zc : 0.0f;
        rect_ref[i] = ref_rect;
        if (alive) {
            rec[i] = r;
            if (aux) aux[i] = a;
        }
    }
    __shared__ uint32_t s_pairs[8], s_st[8];
    uint32_t wp = tiles, ws = alive ? count : 0u;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        wp += __shfl_xor_sync(0xffffffffu, wp, o);
        ws += __shfl_xor_sync(0xffffffffu, ws, o);
    }
    if ((threadIdx.x & 31) == 0) {
        s_pairs[threadIdx.x >> 5] = wp;
        s_st[threadIdx.x >> 5] = ws;
    }
    const int block_alive = __syncthreads_count(alive);
    if (threadIdx.x == 0 && block_alive) {
        uint32_t bp = 0, bs = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            bp += s_pairs[w];
            bs += s_st[w];
        }
        atomicAdd(n_surv, (uint32_t)block_alive);
        atomicAdd(n_surv + 1, bs);
        atomicAdd(n_surv + 2, bp);
    }
}

// [survivors, Ps, P] straight to the host's mapped pinned memory, and the device counters back to
// zero for the next view: a one-warp kernel instead of a memset + a copy-engine transfer (a bulk
// H2D in flight queues copy-engine work behind it).
__global__ void publish_counts_kernel(uint32_t* __restrict__ n_surv, uint32_t* host_counts,
                                      uint32_t* __restrict__ cls_cnt, uint32_t* __restrict__ tcls_cnt) {
    pdl_wait();
    if (threadIdx.x < 3) {
        const uint32_t c = n_surv[threadIdx.x];
        n_surv[threadIdx.x] = 0u;
        reinterpret_cast<volatile uint32_t*>(host_counts)[threadIdx.x] = c;
    }
    // the work-order classes of the view about to be binned and blended (BinningArgs::tcls,
    // FwdOutputs::cls_cnt)
    for (int k = threadIdx.x; k < kCostClasses; k += 32) {
        if (cls_cnt) cls_cnt[k] = 0u;
        if (tcls_cnt) tcls_cnt[k] = 0u;
    }
    // no system fence: the host reads after synchronising with this kernel's completion, which
    // makes its writes to mapped memory visible (a fence here costs ~3 us on the critical path)
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Per-tile front-to-back blend (rasterizer.cpp:124-169 + traverse_pixel rasterizer.hpp:116-147).
// One CTA per BW x BW pixel block (BW = min(tile, 16)); a tile of size 16k is covered by k*k
// CTAs sharing its list (blockIdx.y).  The tile list is walked in batches of blockDim.x entries;
// each batch is culled to the Gaussians that can reach the alpha floor inside the block and
// staged in shared memory, and all threads walk it in the same order (broadcast reads).
// ARG: track each pixel's max-weight sample (max_contributor, depth, importance counts); off in
// training, where only colour, T and the last committed position are consumed.
template <bool REPORT, bool THR, int BW, int BH, bool ARG = true>
__device__ __forceinline__ void blend_forward_block(int bid, CamParams cp, const uint32_t* __restrict__ ranges,
                                                           const uint32_t* __restrict__ pair_gauss,
                                                           const ProjRec* __restrict__ rec,
                                                           const AuxRec* __restrict__ aux, float bg0, float bg1,
                                                           float bg2, FwdOutputs out) {
    // list entries staged per thread and batch (StagePipe ITEMS)
    constexpr int ITEMS = 1;  // (2 per thread measured slower: 306 vs 298 us at config 1)
    constexpr int CAP = BW * BH * ITEMS;
    __shared__ StageSmem<CAP> sm;
    __shared__ StageRaw<CAP> raw;
    __shared__ float s_imp[REPORT ? CAP : 1];
    __shared__ uint32_t s_maxw[REPORT ? CAP : 1];
    const int nthreads = blockDim.x;  // (a compile-time BW * BH here measured slower: 261 -> 283 us)
    const int tid = threadIdx.x;
    const int ts = cp.tile_size;
    constexpr int bw = BW;
    // sub-blocks of one tile are adjacent in the grid, so the tile's list and records are
    // re-read from L2 while still hot
    const int subs_x = ts / BW, nsub = subs_x * (ts / BH);
    const int tile = bid / nsub, sub = bid - tile * nsub;
    const int tx = tile % cp.tiles_x, ty = tile / cp.tiles_x;
    const int sx = sub % subs_x, sy = sub / subs_x;
    const int bx0 = tx * ts + sx * BW, by0 = ty * ts + sy * BH;
    const int bx1 = min(bx0 + BW, cp.width), by1 = min(by0 + BH, cp.height);
    // pixel of this thread: warps own compact patches (8 x 4 for 16 x 16 blocks, 8 x 4 for 8 x 8)
    const int lx = ((tid >> 5) & ((bw >> 3) - 1)) * 8 + (tid & 7);
    const int ly = ((tid >> 5) / (bw >> 3)) * 4 + ((tid & 31) >> 3);
    const int px = bx0 + lx;
    const int py = by0 + ly;
    const bool inside = px < cp.width && py < cp.height;
    const uint32_t start = ranges[2 * tile];
    __shared__ ListTail s_tail;
    uint32_t end;
    const int split = list_tail_setup(out.tails, out.st_list, out.st_cover, tile, cp.tiles_x, ranges[2 * tile + 1], end,
                                      &s_tail, tid == 0, []() { __syncthreads(); });
    const float amax_c = cp.alpha_max, cmin = cp.contribution_min, tmin = cp.transmittance_min;
    const float x = (float)px + 0.5f, y = (float)py + 0.5f;
    // this pixel's bits in the staged masks, and this warp's rows (32 / bw rows per warp)
    const uint32_t mybits = (1u << lx) | (1u << (16 + ly));
    // this warp's columns and rows in the staged masks: skip an entry when either misses
    const uint32_t wcols = 0xffu << (lx & ~7), wrows = 0xfu << (16 + (ly & ~3));

    const uint32_t a_r0 = smem_base(sm.r0), a_r1 = smem_base(sm.r1), a_r2 = smem_base(sm.r2);
    const uint32_t a_gid = smem_base(sm.gid), a_idx = smem_base(sm.idx);
    float T = 1.0f, acc0 = 0.0f, acc1 = 0.0f, acc2 = 0.0f, wmax = 0.0f;
    int32_t amax_gid = -1, last = -1;
    int run = 0;  // entries staged so far (position in the block list)
    bool done = !inside;
    if (REPORT)
        for (int q = tid; q < CAP; q += nthreads) {
            s_imp[q] = 0.0f;
            s_maxw[q] = 0u;
        }
    if (bx0 < bx1 && by0 < by1 && start < end) {
        auto pos = [&](int b, int t) -> int {
            const uint32_t i = start + (uint32_t)b * (uint32_t)CAP + (uint32_t)t;
            return i < end ? (int)i : -1;
        };
        StagePipe<CAP, decltype(pos), true, ITEMS> pipe(pos, pair_gauss, rec, &raw, split, &s_tail);
        pipe.start();
        const int nb = (int)((end - start + (uint32_t)CAP - 1u) / (uint32_t)CAP);
        for (int b = 0; b < nb; ++b) {
            const int cnt = pipe.stage(b, !done, bx0, bx1, by0, by1, sm);
            if (cnt < 0) break;
            if (!REPORT && out.blist && run + cnt <= kBlockList)
                for (int q = tid; q < cnt; q += nthreads) {
                    out.blist[(size_t)bid * kBlockList + run + q] = sm.gid[q];
                    out.bidx[(size_t)bid * kBlockList + run + q] = (uint32_t)sm.idx[q];
                }
#ifdef SPLAT_STATS
            {
                const unsigned wa = __ballot_sync(0xffffffffu, !done);
                const int act = __syncthreads_count(!done);
                if ((tid & 31) == 0 && wa) atomicAdd(&g_stats[7], 1ull);          // warps with work
                if (tid == 0) {
                    atomicAdd(&g_stats[8], (unsigned long long)((act + 31) / 32));  // warps needed
                    atomicAdd(&g_stats[9], (unsigned long long)act);                  // active pixels
                    atomicAdd(&g_stats[10], 1ull);                                    // CTA batches
                }
            }
            if (tid == 0) {
                atomicAdd(&g_stats[4], (unsigned long long)cnt);
                atomicAdd(&g_stats[6], (unsigned long long)min((uint32_t)CAP, end - start - (uint32_t)b * CAP));
            }
#endif
            if (!REPORT) {
                // Two staged entries per iteration: independent branch-free gates, then the
                // per-pixel recursion commits them in list order.
                for (int j = 0; j < cnt && !done; j += 2) {
                    const bool has_b = j + 1 < cnt;
                    const uint32_t jb = has_b ? (uint32_t)(j + 1) : (uint32_t)j;
                    const float4 r1a = lds_f4(a_r1 + 16u * j);
                    const float4 r1b = lds_f4(a_r1 + 16u * jb);
                    const uint32_t ma = __float_as_uint(r1a.z), mb = __float_as_uint(r1b.z);
                    const bool wa = (ma & wrows) && (ma & wcols);  // warp-uniform: rect meets the patch
                    const bool wb = has_b && (mb & wrows) && (mb & wcols);
                    if (!wa && !wb) continue;
                    const float4 r0a = lds_f4(a_r0 + 16u * j), r0b = lds_f4(a_r0 + 16u * jb);
                    float alpha_a, alpha_b, g2d, dx, dy;
                    bool clamped;
                    const bool ga = gate_sample_nb<THR>(r0a, r1a, mybits, x, y, amax_c, cmin, alpha_a, g2d, clamped, dx,
                                                        dy) && wa;
                    const bool gb = gate_sample_nb<THR>(r0b, r1b, mybits, x, y, amax_c, cmin, alpha_b, g2d, clamped, dx,
                                                        dy) && wb;
#ifdef SPLAT_STATS
                    {
                        auto patch_ok = [&](const float4& r0, const float4& r1, uint32_t msk) {
                            const uint32_t cols = msk & wcols & 0xffffu, rows = (msk & wrows) >> 16;
                            if (!cols || !rows) return false;
                            const int X0 = __ffs(cols) - 1, X1 = 32 - __clz(cols);
                            const int Y0 = __ffs(rows) - 1, Y1 = 32 - __clz(rows);
                            return quad_box_reaches(r0, r1.x, r1.w, bx0 + X0, bx0 + X1, by0 + Y0, by0 + Y1);
                        };
                        const bool pa = wa && patch_ok(r0a, r1a, ma), pb = wb && patch_ok(r0b, r1b, mb);
                        const unsigned am = __activemask();
                        const bool anya = __any_sync(am, ga), anyb = __any_sync(am, gb);
                        if ((tid & 31) == __ffs(am) - 1) {
                            atomicAdd(&g_stats[0], (unsigned long long)(wa + wb));
                            atomicAdd(&g_stats[1], (unsigned long long)((wa && !pa) + (wb && !pb)));
                            atomicAdd(&g_stats[2], (unsigned long long)(anya + anyb));
                            atomicAdd(&g_stats[3], (unsigned long long)((pa && !anya) + (pb && !anyb)));
                            atomicAdd(&g_stats[5], (unsigned long long)__popc(am));
                        }
                    }
#endif
                    {  // branch-free commits of a then b (b only when a did not end the pixel)
                        const float na = T * (1.0f - alpha_a);
                        const bool sa = THR && ga && na < tmin;
                        const bool ca = ga && !sa;
                        const float wa_ = T * alpha_a;
                        const float4 r2a = lds_f4(a_r2 + 16u * j);
                        const float a0 = acc0 + wa_ * r2a.x, a1 = acc1 + wa_ * r2a.y, a2 = acc2 + wa_ * r2a.z;
                        acc0 = ca ? a0 : acc0;
                        acc1 = ca ? a1 : acc1;
                        acc2 = ca ? a2 : acc2;
                        if (ARG && ca && wa_ > wmax) {
                            wmax = wa_;
                            amax_gid = (int32_t)lds_u32(a_gid + 4u * j);
                        }
                        const int32_t ia = (int32_t)lds_u32(a_idx + 4u * j);
                        last = ca ? ia : last;
                        T = ca ? na : T;
                        const bool gb2 = gb && !sa;
                        const float nb = T * (1.0f - alpha_b);
                        const bool sb = THR && gb2 && nb < tmin;
                        const bool cb = gb2 && !sb;
                        const float wb_ = T * alpha_b;
                        const float4 r2b = lds_f4(a_r2 + 16u * jb);
                        const float b0 = acc0 + wb_ * r2b.x, b1 = acc1 + wb_ * r2b.y, b2 = acc2 + wb_ * r2b.z;
                        acc0 = cb ? b0 : acc0;
                        acc1 = cb ? b1 : acc1;
                        acc2 = cb ? b2 : acc2;
                        if (ARG && cb && wb_ > wmax) {
                            wmax = wb_;
                            amax_gid = (int32_t)lds_u32(a_gid + 4u * jb);
                        }
                        const int32_t ib = (int32_t)lds_u32(a_idx + 4u * jb);
                        last = cb ? ib : last;
                        T = cb ? nb : T;
                        if (sa || sb) {
                            done = true;
                            break;
                        }
                    }
                }
            } else {
                // accumulate_importance (rasterizer.cpp:184-193): the training loop's branch-free
                // pair form; each entry's per-warp weight sum and maximum go to shared memory
                // (combining the CTA's two warps), then one global atomic pair per entry and batch.
                const int lane = tid & 31;
                for (int j = 0; j < cnt; j += 2) {
                    if (__all_sync(0xffffffffu, done)) break;
                    const bool has_b = j + 1 < cnt;
                    const uint32_t jb = has_b ? (uint32_t)(j + 1) : (uint32_t)j;
                    const float4 r1a = lds_f4(a_r1 + 16u * j);
                    const float4 r1b = lds_f4(a_r1 + 16u * jb);
                    const uint32_t ma = __float_as_uint(r1a.z), mb = __float_as_uint(r1b.z);
                    const bool wa = (ma & wrows) && (ma & wcols);  // warp-uniform: rect meets the patch
                    const bool wb = has_b && (mb & wrows) && (mb & wcols);
                    if (!wa && !wb) continue;
                    const float4 r0a = lds_f4(a_r0 + 16u * j), r0b = lds_f4(a_r0 + 16u * jb);
                    float alpha_a, alpha_b, g2d, dx, dy;
                    bool clamped;
                    const bool ga = gate_sample_nb<THR>(r0a, r1a, mybits, x, y, amax_c, cmin, alpha_a, g2d, clamped, dx,
                                                        dy) && wa && !done;
                    const bool gb = gate_sample_nb<THR>(r0b, r1b, mybits, x, y, amax_c, cmin, alpha_b, g2d, clamped, dx,
                                                        dy) && wb && !done;
                    const float na = T * (1.0f - alpha_a);
                    const bool sa = THR && ga && na < tmin;
                    const bool ca = ga && !sa;
                    const float wa_ = ca ? T * alpha_a : 0.0f;
                    {
                        const float4 r2a = lds_f4(a_r2 + 16u * j);
                        acc0 = ca ? acc0 + wa_ * r2a.x : acc0;
                        acc1 = ca ? acc1 + wa_ * r2a.y : acc1;
                        acc2 = ca ? acc2 + wa_ * r2a.z : acc2;
                    }
                    if (ARG && ca && wa_ > wmax) {
                        wmax = wa_;
                        amax_gid = (int32_t)lds_u32(a_gid + 4u * j);
                    }
                    T = ca ? na : T;
                    const bool gb2 = gb && !sa;
                    const float nb = T * (1.0f - alpha_b);
                    const bool sb = THR && gb2 && nb < tmin;
                    const bool cb = gb2 && !sb;
                    const float wb_ = cb ? T * alpha_b : 0.0f;
                    {
                        const float4 r2b = lds_f4(a_r2 + 16u * jb);
                        acc0 = cb ? acc0 + wb_ * r2b.x : acc0;
                        acc1 = cb ? acc1 + wb_ * r2b.y : acc1;
                        acc2 = cb ? acc2 + wb_ * r2b.z : acc2;
                    }
                    if (ARG && cb && wb_ > wmax) {
                        wmax = wb_;
                        amax_gid = (int32_t)lds_u32(a_gid + 4u * jb);
                    }
                    T = cb ? nb : T;
                    done = done || sa || sb;
                    // weights are >= 0: their float bits order like the values (max over the warp)
                    if (__any_sync(0xffffffffu, ca)) {
                        const float sum = warp_sum(wa_);
                        const uint32_t mx = __reduce_max_sync(0xffffffffu, __float_as_uint(wa_));
                        if (lane == 0) {
                            atomicAdd(&s_imp[j], sum);
                            atomicMax(&s_maxw[j], mx);
                        }
                    }
                    if (__any_sync(0xffffffffu, cb)) {
                        const float sum = warp_sum(wb_);
                        const uint32_t mx = __reduce_max_sync(0xffffffffu, __float_as_uint(wb_));
                        if (lane == 0) {
                            atomicAdd(&s_imp[jb], sum);
                            atomicMax(&s_maxw[jb], mx);
                        }
                    }
                }
                __syncthreads();
                for (int q = tid; q < cnt; q += nthreads)
                    if (s_maxw[q] != 0u) {
                        const uint32_t gid = sm.gid[q];
                        atomicAdd(&out.importance[gid], s_imp[q]);
                        atomicMax(reinterpret_cast<uint32_t*>(&out.max_weight[gid]), s_maxw[q]);
                        s_imp[q] = 0.0f;
                        s_maxw[q] = 0u;
                    }
            }
            // the next stage() starts with a barrier: staged entries stay until every warp is done
            run += cnt;
            // the walk reached the list's tail (past the materialised prefix): tell the host,
            // which materialises longer prefixes from the next view on
            if (tid == 0 && out.tail_note && start + (uint32_t)(b + 1) * (uint32_t)CAP > (uint32_t)split)
                *reinterpret_cast<volatile uint32_t*>(out.tail_note) = 1u;
        }
        pipe.finish();
    }
    if (!REPORT && out.bcount && tid == 0) out.bcount[bid] = run;
    if (!REPORT && out.cls_cnt && tid == 0) {  // the backward's work order: heaviest blocks first
        const int c = kCostClasses - 1 - min(kCostClasses - 1, run >> 4);
        out.cls_list[(size_t)c * out.n_blocks + atomicAdd(&out.cls_cnt[c], 1u)] = (uint32_t)bid;
    }
    if (!inside) return;
    const size_t pix = (size_t)py * cp.width + px;
    if (REPORT && amax_gid >= 0) atomicAdd(&out.max_pixel_count[amax_gid], 1);
    if (out.color) {
        out.color[3 * pix + 0] = acc0 + T * bg0;
        out.color[3 * pix + 1] = acc1 + T * bg1;
        out.color[3 * pix + 2] = acc2 + T * bg2;
    }
    if (out.alpha) out.alpha[pix] = 1.0f - T;
    if (out.transmittance) out.transmittance[pix] = T;
    if (out.max_contributor) out.max_contributor[pix] = amax_gid;
    if (out.t_final) out.t_final[pix] = T;
    if (out.last_index) out.last_index[pix] = last;
    if (out.depth) {
        float d = 0.0f;
        if (amax_gid >= 0) {
            // cam.ray_direction (camera.hpp:32-36) and depth_along_ray (rasterizer.hpp:87-96)
            float d0 = ((float)px + 0.5f - cp.cx) / cp.fx;
            float d1 = ((float)py + 0.5f - cp.cy) / cp.fy;
            float d2 = 1.0f;
            const float z2 = dot3(d0, d1, d2, d0, d1, d2);
            if (z2 > 0.0f) {
                const float nn = sqrtf(z2);
                d0 = d0 / nn; d1 = d1 / nn; d2 = d2 / nn;
            }
            const float w0 = dot3(cp.R[0], cp.R[3], cp.R[6], d0, d1, d2);
            const float w1 = dot3(cp.R[1], cp.R[4], cp.R[7], d0, d1, d2);
            const float w2 = dot3(cp.R[2], cp.R[5], cp.R[8], d0, d1, d2);
            const AuxRec ax = aux[amax_gid];
            const float r0 = ax.a0.x - cp.center[0], r1 = ax.a0.y - cp.center[1], r2 = ax.a0.z - cp.center[2];
            if (ax.a0.w != 0.0f) {
                d = dot3(r0, r1, r2, w0, w1, w2);
            } else {
                const float i00 = ax.a1.x, i01 = ax.a1.y, i02 = ax.a1.z, i11 = ax.a1.w, i12 = ax.a2.x,
                            i22 = ax.a2.y;
                const float cd0 = dot3(i00, i01, i02, w0, w1, w2);
                const float cd1 = dot3(i01, i11, i12, w0, w1, w2);
                const float cd2 = dot3(i02, i12, i22, w0, w1, w2);
                const float denom = dot3(w0, w1, w2, cd0, cd1, cd2);
                const float t = dot3(r0, r1, r2, cd0, cd1, cd2) / denom;
                d = (!(t > 0.0f) || !isfinite(t)) ? dot3(r0, r1, r2, w0, w1, w2) : t;
            }
        }
        out.depth[pix] = d;
    }
}

template <bool REPORT, bool THR, int BW, int BH, bool ARG>
__global__ void __launch_bounds__(BW * BH) blend_forward_kernel(CamParams cp, const uint32_t* __restrict__ ranges,
                                                           const uint32_t* __restrict__ pair_gauss,
                                                           const ProjRec* __restrict__ rec,
                                                           const AuxRec* __restrict__ aux, float bg0, float bg1,
                                                           float bg2, FwdOutputs out) {
    blend_forward_block<REPORT, THR, BW, BH, ARG>((int)blockIdx.x, cp, ranges, pair_gauss, rec, aux, bg0, bg1, bg2, out);
}

// Persistent variant: one wave of CTAs pulls pixel blocks from a work counter (no CTA launch /
// retire gaps between blocks, occupancy stays at the register limit through the whole kernel).
template <bool REPORT, bool THR, int BW, int BH, bool ARG>
__global__ void __launch_bounds__(BW * BH) blend_forward_persistent(CamParams cp, const uint32_t* __restrict__ ranges,
                                                           const uint32_t* __restrict__ pair_gauss,
                                                           const ProjRec* __restrict__ rec,
                                                           const AuxRec* __restrict__ aux, float bg0, float bg1,
                                                           float bg2, FwdOutputs out, int nblocks, int* __restrict__ counter,
                                                           const uint32_t* __restrict__ tcls) {
    __shared__ int s_bid;
    __shared__ uint32_t s_excl[kCostClasses + 1];
    pdl_wait();
    // Work order: binning filed every tile under a list-length class (longest first); the k-th
    // pull is sub-block k % nsub of the (k / nsub)-th tile in that order (a tile's sub-blocks stay
    // adjacent, so their list reads hit L2).  Without classes: raster order.
    const int nsub = (cp.tile_size / BW) * (cp.tile_size / BH);
    const int ntiles = cp.tiles_x * cp.tiles_y;
    if (tcls && threadIdx.x < 32) {
        const int lane = threadIdx.x;
        const uint32_t c0 = tcls[2 * lane], c1 = tcls[2 * lane + 1];
        uint32_t incl = c0 + c1;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += u;
        }
        s_excl[2 * lane] = incl - c0 - c1;
        s_excl[2 * lane + 1] = incl - c1;
        if (lane == 31) s_excl[kCostClasses] = incl;
    }
    for (;;) {
        __syncthreads();  // the previous block's shared-memory reads are done
        if (threadIdx.x == 0) {
            int b = pull_work(counter, nblocks);
            if (tcls && b < nblocks) {
                const uint32_t ti = (uint32_t)(b / nsub);
                int lo = 0, hi = kCostClasses - 1;  // last class whose start <= ti
                while (lo < hi) {
                    const int mid = (lo + hi + 1) >> 1;
                    if (s_excl[mid] <= ti) lo = mid;
                    else hi = mid - 1;
                }
                const uint32_t t = tcls[kCostClasses + (size_t)lo * ntiles + (ti - s_excl[lo])];
                b = (int)t * nsub + b % nsub;
            }
            s_bid = b;
        }
        __syncthreads();
        const int b = s_bid;
        if (b >= nblocks) break;
        blend_forward_block<REPORT, THR, BW, BH, ARG>(b, cp, ranges, pair_gauss, rec, aux, bg0, bg1, bg2, out);
    }
}

// Traversal statistics of the reference's traverse_pixel (rasterizer.hpp:116-147) over the forward's
// per-tile lists, per pixel and plain (one thread per pixel, no culls): V = list entries visited
// (the breaking sample included), C = samples committed.  A measurement kernel (bench / tests),
// not on the training path; gates in the reference's operation order (this file: --fmad=false).
__global__ void traversal_counts_kernel(CamParams cp, const uint32_t* __restrict__ ranges,
                                        const uint32_t* __restrict__ pair_gauss, const ProjRec* __restrict__ rec,
                                        const uint2* __restrict__ rect_ref, unsigned long long* __restrict__ out) {
    const int64_t pix = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long v = 0, c = 0;
    if (pix < (int64_t)cp.width * cp.height) {
        const int px = (int)(pix % cp.width), py = (int)(pix / cp.width);
        const int tile = (py / cp.tile_size) * cp.tiles_x + px / cp.tile_size;
        const uint32_t start = ranges[2 * tile], end = ranges[2 * tile + 1];
        const float x = (float)px + 0.5f, y = (float)py + 0.5f;
        float T = 1.0f;
        for (uint32_t k = start; k < end; ++k) {
            const uint32_t gid = pair_gauss[k];
            ++v;
            const uint2 rr = rect_ref[gid];
            if (px < (int)(rr.x & 0xffffu) || px >= (int)(rr.x >> 16) || py < (int)(rr.y & 0xffffu) ||
                py >= (int)(rr.y >> 16))
                continue;
            const ProjRec r = rec[gid];
            const float dx = r.r0.x - x, dy = r.r0.y - y;
            const float power = -0.5f * (r.r0.z * dx * dx + r.r1.x * dy * dy) - r.r0.w * dx * dy;
            if (power > 0.0f) continue;
            float a = r.r1.y * splat_expf(power);
            if (cp.apply_thresholds) {
                if (a > cp.alpha_max) a = cp.alpha_max;
                if (a < cp.contribution_min) continue;
            }
            const float next = T * (1.0f - a);
            if (cp.apply_thresholds && next < cp.transmittance_min) break;
            ++c;
            T = next;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        v += __shfl_xor_sync(0xffffffffu, v, o);
        c += __shfl_xor_sync(0xffffffffu, c, o);
    }
    if ((threadIdx.x & 31) == 0 && (v || c)) {
        atomicAdd(out, v);
        atomicAdd(out + 1, c);
    }
}

__global__ void unproject_flags_kernel(int width, int height, const int32_t* __restrict__ max_contributor,
                                       const float* __restrict__ alpha, int rule, float thr, int64_t view_index,
                                       int32_t stride, int64_t seed, uint32_t* __restrict__ flags) {
    const int64_t pix = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t hw = (int64_t)width * height;
    if (pix >= hw) return;
    const bool valid = rule == SPLAT_DEPTH_RULE_ALPHA ? (alpha[pix] > thr) : (max_contributor[pix] >= 0);
    const int64_t key = view_index * hw + pix + seed;
    const int64_t m = ((key % stride) + stride) % stride;
    flags[pix] = (valid && m == 0) ? 1u : 0u;
}

// append: the view's points go after the *count points already written (the multi-view pass),
// and view_out (nullable) gets the view index of each point.
__global__ void unproject_write_kernel(CamParams cp, const uint32_t* __restrict__ flags,
                                       const uint32_t* __restrict__ offsets, const float* __restrict__ depth,
                                       float* __restrict__ points, int32_t* __restrict__ pixel, int64_t capacity,
                                       const int32_t* __restrict__ base, int32_t* __restrict__ view_out,
                                       int32_t view_index) {
    const int64_t pix = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t hw = (int64_t)cp.width * cp.height;
    if (pix >= hw || !flags[pix]) return;
    const int64_t o = offsets[pix] + (base ? (int64_t)*base : 0);
    if (o >= capacity) return;
    const int px = (int)(pix % cp.width), py = (int)(pix / cp.width);
    float d0 = ((float)px + 0.5f - cp.cx) / cp.fx;
    float d1 = ((float)py + 0.5f - cp.cy) / cp.fy;
    float d2 = 1.0f;
    const float z2 = dot3(d0, d1, d2, d0, d1, d2);
    if (z2 > 0.0f) {
        const float nn = sqrtf(z2);
        d0 = d0 / nn; d1 = d1 / nn; d2 = d2 / nn;
    }
    const float w0 = dot3(cp.R[0], cp.R[3], cp.R[6], d0, d1, d2);
    const float w1 = dot3(cp.R[1], cp.R[4], cp.R[7], d0, d1, d2);
    const float w2 = dot3(cp.R[2], cp.R[5], cp.R[8], d0, d1, d2);
    const float d = depth[pix];
    points[3 * o + 0] = cp.center[0] + d * w0;
    points[3 * o + 1] = cp.center[1] + d * w1;
    points[3 * o + 2] = cp.center[2] + d * w2;
    pixel[o] = (int32_t)pix;
    if (view_out) view_out[o] = view_index;
}

__global__ void count_from_scan_kernel(const uint32_t* __restrict__ offsets, const uint32_t* __restrict__ flags,
                                       int64_t hw, int32_t* __restrict__ count, bool append) {
    *count = (append ? *count : 0) + (int32_t)(offsets[hw - 1] + flags[hw - 1]);
}

inline unsigned blocks_for(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

}  // namespace

cudaError_t launch_preprocess(LaunchCtx& lc, const GaussianPtrs& g, const CamParams& cp, const uint8_t* mask,
                              ProjRec* rec, AuxRec* aux, uint32_t* keys, uint32_t* vals, uint32_t* tile_counts,
                              uint32_t* n_survivors_dev, float* depth_out, uint2* rect_ref,
                              uint32_t* host_counts, float4* proj_dbg, uint32_t* cls_cnt, uint32_t* tcls_cnt) {
    if (g.n == 0) return cudaSuccess;
    const bool vec = (reinterpret_cast<uintptr_t>(g.sh) & 15u) == 0;
    if (vec)
        {
            LaunchScope ls_(lc, "preprocess");
            preprocess_kernel<true><<<blocks_for(g.n, kPreThreads), kPreThreads, 0, lc.stream>>>(g, cp, mask, rec, aux, keys, vals,
                                                                             tile_counts, n_survivors_dev, depth_out, rect_ref, proj_dbg);
        }
    else
        {
            LaunchScope ls_(lc, "preprocess");
            preprocess_kernel<false><<<blocks_for(g.n, kPreThreads), kPreThreads, 0, lc.stream>>>(g, cp, mask, rec, aux, keys, vals,
                                                                              tile_counts, n_survivors_dev, depth_out, rect_ref, proj_dbg);
        }
    lc.count++;
    if (host_counts) {
        const cudaError_t e = launch_pdl(lc.stream, publish_counts_kernel, dim3(1), dim3(32), 0, n_survivors_dev,
                                         host_counts, cls_cnt, tcls_cnt);
        if (e != cudaSuccess) return e;
        lc.count++;
    }
    return cudaGetLastError();
}

cudaError_t launch_publish_counts(cudaStream_t s, uint32_t* n_survivors_dev, uint32_t* host_counts, uint32_t* cls_cnt,
                                  uint32_t* tcls_cnt) {
    publish_counts_kernel<<<1, 32, 0, s>>>(n_survivors_dev, host_counts, cls_cnt, tcls_cnt);
    return cudaGetLastError();
}

cudaError_t launch_blend_forward(LaunchCtx& lc, const CamParams& cp, const uint32_t* ranges,
                                 const uint32_t* pair_gauss, const ProjRec* rec, const AuxRec* aux, const float bg[3],
                                 const FwdOutputs& out, const uint32_t* tcls) {
    const int ts = cp.tile_size;
    const unsigned grid = (unsigned)(cp.tiles_x * cp.tiles_y * (ts / cp.block_w) * (ts / cp.block_h));
    LaunchScope ls_(lc, "blend_forward");
#define BLEND_FWD_SHAPE(R, T, W, H, A)                                                                           \
    do {                                                                                                         \
        if (lc.persistent_blend && lc.work_counters) {                                                           \
            static int per_sm = 0;                                                                               \
            if (!per_sm) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, blend_forward_persistent<R, T, W, H, A>, \
                                                                      W * H, 0);                                 \
            const unsigned pg = (unsigned)(lc.num_sms * (per_sm > 0 ? per_sm : 1));                             \
            launch_pdl(lc.stream, blend_forward_persistent<R, T, W, H, A>, dim3(pg < grid ? pg : grid), dim3(W * H), \
                       0, cp, ranges, pair_gauss, rec, aux, bg[0], bg[1], bg[2], out, (int)grid, lc.work_counters,   \
                       tcls);                                                                                    \
        } else {                                                                                                 \
            blend_forward_kernel<R, T, W, H, A><<<grid, W * H, 0, lc.stream>>>(cp, ranges, pair_gauss, rec, aux, \
                                                                              bg[0], bg[1], bg[2], out);         \
        }                                                                                                        \
    } while (0)
#define BLEND_FWD(R, T, A)                                                     \
    do {                                                                       \
        if (cp.block_w == 16) BLEND_FWD_SHAPE(R, T, 16, 16, A);                \
        else if (cp.block_h == 8) BLEND_FWD_SHAPE(R, T, 8, 8, A);              \
        else BLEND_FWD_SHAPE(R, T, 8, 4, A);                                   \
    } while (0)
    const bool arg = out.max_contributor || out.depth;
    if (out.importance) {
        if (cp.apply_thresholds) BLEND_FWD(true, true, true);
        else BLEND_FWD(true, false, true);
    } else if (arg) {
        if (cp.apply_thresholds) BLEND_FWD(false, true, true);
        else BLEND_FWD(false, false, true);
    } else {
        if (cp.apply_thresholds) BLEND_FWD(false, true, false);
        else BLEND_FWD(false, false, false);
    }
#undef BLEND_FWD_SHAPE
#undef BLEND_FWD
    lc.count++;
    return cudaGetLastError();
}

cudaError_t launch_unproject(LaunchCtx& lc, const CamParams& cp, const int32_t* max_contributor, const float* alpha,
                             const float* depth, int rule, float alpha_threshold, int64_t view_index, int32_t stride,
                             int64_t seed, float* points, int32_t* pixel, int64_t capacity, int32_t* count_dev,
                             uint32_t* flags, uint32_t* offsets, uint32_t* scan_tmp, bool append,
                             int32_t* view_out) {
    const int64_t hw = (int64_t)cp.width * cp.height;
    {
        LaunchScope ls_(lc, "unproject_flags");
        unproject_flags_kernel<<<blocks_for(hw, 256), 256, 0, lc.stream>>>(cp.width, cp.height, max_contributor, alpha,
                                                                       rule, alpha_threshold, view_index, stride,
                                                                       seed, flags);
    }
    lc.count++;
    cudaError_t e = exclusive_scan_u32(lc, flags, offsets, (uint64_t)hw, scan_tmp, nullptr);
    if (e != cudaSuccess) return e;
    {
        LaunchScope ls_(lc, "unproject_write");
        unproject_write_kernel<<<blocks_for(hw, 256), 256, 0, lc.stream>>>(cp, flags, offsets, depth, points, pixel,
                                                                       capacity, append ? count_dev : nullptr,
                                                                       view_out, (int32_t)view_index);
    }
    {
        LaunchScope ls_(lc, "count_from_scan");
        count_from_scan_kernel<<<1, 1, 0, lc.stream>>>(offsets, flags, hw, count_dev, append);
    }
    lc.count += 2;
    return cudaGetLastError();
}

cudaError_t launch_traversal_counts(LaunchCtx& lc, const CamParams& cp, const uint32_t* ranges,
                                    const uint32_t* pair_gauss, const ProjRec* rec, const uint2* rect_ref,
                                    unsigned long long* out) {
    const int64_t hw = (int64_t)cp.width * cp.height;
    if (hw == 0) return cudaSuccess;
    traversal_counts_kernel<<<(unsigned)((hw + 255) / 256), 256, 0, lc.stream>>>(cp, ranges, pair_gauss, rec, rect_ref,
                                                                                 out);
    lc.count++;
    return cudaGetLastError();
}

}  // namespace splat_b200

// Instrumented builds: copy (and with reset != 0, zero) the forward traversal counters.
extern "C" int splat_debug_stats(unsigned long long* out, int reset) {
#ifdef SPLAT_STATS
    cudaError_t e = cudaDeviceSynchronize();
    if (e == cudaSuccess) e = cudaMemcpyFromSymbol(out, splat_b200::g_stats, sizeof(unsigned long long) * 12);
    if (e != cudaSuccess) return 100 + (int)e;
    if (reset) {
        unsigned long long z[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
        cudaMemcpyToSymbol(splat_b200::g_stats, z, sizeof(z));
    }
    return 0;
#else
    (void)out;
    (void)reset;
    return -1;
#endif
}
