// ssim.cu — SSIM and the photometric loss on device (loss.cpp:10-153).
//
// mean SSIM over an H x W x C image pair with the reference's 11-tap Gaussian window (sigma 1.5,
// normalised in float, gaussian_kernel loss.cpp:13-22 — computed on the host with the shared
// splat_expf and passed in), separable "same" blur with zero padding realised by skipping
// out-of-image taps exactly like blur() (loss.cpp:26-53), and the analytic gradient
// (loss.cpp:105-131: three maps blurred a second time).  Compiled with --fmad=false and written in
// the reference's operation order, so every per-pixel value (SSIM map, the t1..t3 maps, the
// gradient) is bit-identical to the reference's; only the image-wide means are summed in a
// different order (per-CTA fp64 partials instead of one sequential float sum).
//
// Tiling: one CTA per (32 x 8 pixel tile, channel).  The tile plus a 5-pixel halo of the inputs is
// staged in shared memory, the horizontal pass writes (8 + 10) x 32 partial rows for each blurred
// quantity, the vertical pass gives each thread its pixel.  HBM-bound: a, b read once per pass,
// t1..t3 written once and read once, the gradient written once.
#include <cstdint>

#include "common.cuh"
#include "internal.h"

namespace splat_b200 {

namespace {

constexpr int kHalf = 5;           // 11-tap window
constexpr int kTW = 32, kTH = 8;   // output tile
constexpr int kSW = kTW + 2 * kHalf, kSH = kTH + 2 * kHalf;

struct SsimWindow {
    float k[11];
};

// Stage NQ input maps (channel c of H x W x C images) for the tile [x0, x0+32) x [y0, y0+8) plus
// halo; out-of-image entries are never read by the passes (taps are skipped), so they stay 0.
template <int NQ>
__device__ __forceinline__ void stage_inputs(const float* const* src, int w, int h, int ch, int c, int x0, int y0,
                                             float (*s_in)[kSH][kSW]) {
    for (int i = threadIdx.x; i < kSH * kSW; i += blockDim.x) {
        const int r = i / kSW, q = i - r * kSW;
        const int y = y0 - kHalf + r, x = x0 - kHalf + q;
        const bool in = x >= 0 && x < w && y >= 0 && y < h;
        const size_t off = in ? ((size_t)y * w + x) * ch + c : 0;
#pragma unroll
        for (int k = 0; k < NQ; ++k) s_in[k][r][q] = in ? src[k][off] : 0.0f;
    }
}

// Horizontal pass of blur() for staged row r (image row y0 - 5 + r) and output column x0 + q.
__device__ __forceinline__ float hblur(const float (*row)[kSW], int q, int x, int w, const SsimWindow& win) {
    float acc = 0.0f;
#pragma unroll
    for (int k = -kHalf; k <= kHalf; ++k) {
        const int xx = x + k;
        if (xx >= 0 && xx < w) acc = __fadd_rn(acc, __fmul_rn(win.k[k + kHalf], (*row)[q + kHalf + k]));
    }
    return acc;
}

// Vertical pass for the thread's pixel from the horizontal results s_h[quantity][row][col].
__device__ __forceinline__ float vblur(const float (*col)[kTW], int r, int q, int y, int h, const SsimWindow& win) {
    float acc = 0.0f;
#pragma unroll
    for (int k = -kHalf; k <= kHalf; ++k) {
        const int yy = y + k;
        if (yy >= 0 && yy < h) acc = __fadd_rn(acc, __fmul_rn(win.k[k + kHalf], col[r + kHalf + k][q]));
    }
    return acc;
}

// Pass 1: the SSIM map (loss.cpp:97-107) + its CTA partial sum, the L1 partial sum, and (GRAD)
// the maps t1..t3 (loss.cpp:108-117).
template <bool GRAD>
__global__ void __launch_bounds__(kTW * kTH) ssim_fwd_kernel(const float* __restrict__ a, const float* __restrict__ b,
                                                            int w, int h, int ch, SsimWindow win, float inv_n,
                                                            float* __restrict__ t1, float* __restrict__ t2,
                                                            float* __restrict__ t3, double* __restrict__ partials) {
    __shared__ float s_in[2][kSH][kSW];
    __shared__ float s_h[5][kSH][kTW];
    __shared__ double s_red[2][kTW * kTH / 32];
    const int c = blockIdx.z;
    const int x0 = blockIdx.x * kTW, y0 = blockIdx.y * kTH;
    const float* srcs[2] = {a, b};
    stage_inputs<2>(srcs, w, h, ch, c, x0, y0, s_in);
    __syncthreads();
    // horizontal pass of a, b, a*a, b*b, a*b (the products formed per tap input, loss.cpp:86-90)
    for (int i = threadIdx.x; i < kSH * kTW; i += blockDim.x) {
        const int r = i / kTW, q = i - r * kTW;
        const int x = x0 + q;
        float acc[5] = {0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int k = -kHalf; k <= kHalf; ++k) {
            const int xx = x + k;
            if (xx >= 0 && xx < w) {
                const float va = s_in[0][r][q + kHalf + k], vb = s_in[1][r][q + kHalf + k];
                const float wk = win.k[k + kHalf];
                acc[0] = __fadd_rn(acc[0], __fmul_rn(wk, va));
                acc[1] = __fadd_rn(acc[1], __fmul_rn(wk, vb));
                acc[2] = __fadd_rn(acc[2], __fmul_rn(wk, __fmul_rn(va, va)));
                acc[3] = __fadd_rn(acc[3], __fmul_rn(wk, __fmul_rn(vb, vb)));
                acc[4] = __fadd_rn(acc[4], __fmul_rn(wk, __fmul_rn(va, vb)));
            }
        }
#pragma unroll
        for (int k = 0; k < 5; ++k) s_h[k][r][q] = acc[k];
    }
    __syncthreads();
    const int q = threadIdx.x % kTW, r = threadIdx.x / kTW;
    const int x = x0 + q, y = y0 + r;
    double s_part = 0.0, l_part = 0.0;
    if (x < w && y < h) {
        float m[5];
#pragma unroll
        for (int k = 0; k < 5; ++k) m[k] = vblur(s_h[k], r, q, y, h, win);
        const float c1 = (float)(0.01 * 0.01), c2 = (float)(0.03 * 0.03);
        const float ma = m[0], mb = m[1];
        const float va = __fsub_rn(m[2], __fmul_rn(ma, ma));
        const float vb = __fsub_rn(m[3], __fmul_rn(mb, mb));
        const float cov = __fsub_rn(m[4], __fmul_rn(ma, mb));
        const float a1 = __fadd_rn(__fmul_rn(__fmul_rn(2.0f, ma), mb), c1);
        const float a2 = __fadd_rn(__fmul_rn(2.0f, cov), c2);
        const float b1 = __fadd_rn(__fadd_rn(__fmul_rn(ma, ma), __fmul_rn(mb, mb)), c1);
        const float b2 = __fadd_rn(__fadd_rn(va, vb), c2);
        const float sv = __fdiv_rn(__fmul_rn(a1, a2), __fmul_rn(b1, b2));
        s_part = (double)sv;
        const size_t o = ((size_t)y * w + x) * ch + c;
        const float av = s_in[0][r + kHalf][q + kHalf], bv = s_in[1][r + kHalf][q + kHalf];
        l_part = (double)fabsf(__fsub_rn(av, bv));
        if (GRAD) {
            const float ds_dmu = __fdiv_rn(
                __fmul_rn(2.0f, __fsub_rn(__fmul_rn(__fmul_rn(mb, a2), b1), __fmul_rn(__fmul_rn(ma, a1), a2))),
                __fmul_rn(__fmul_rn(b1, b1), b2));
            const float ds_dva = __fdiv_rn(__fmul_rn(-a1, a2), __fmul_rn(__fmul_rn(b1, b2), b2));
            const float ds_dcov = __fdiv_rn(__fmul_rn(2.0f, a1), __fmul_rn(b1, b2));
            t1[o] = __fmul_rn(inv_n, __fsub_rn(__fsub_rn(ds_dmu, __fmul_rn(__fmul_rn(2.0f, ma), ds_dva)),
                                               __fmul_rn(mb, ds_dcov)));
            t2[o] = __fmul_rn(inv_n, ds_dva);
            t3[o] = __fmul_rn(inv_n, ds_dcov);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        s_part += __shfl_xor_sync(0xffffffffu, s_part, o);
        l_part += __shfl_xor_sync(0xffffffffu, l_part, o);
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) {
        s_red[0][warp] = s_part;
        s_red[1][warp] = l_part;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double ss = 0.0, ll = 0.0;
        for (int k = 0; k < kTW * kTH / 32; ++k) {
            ss += s_red[0][k];
            ll += s_red[1][k];
        }
        const size_t blk = ((size_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
        partials[2 * blk] = ss;
        partials[2 * blk + 1] = ll;
    }
}

// Pass 2: g1..g3 = blur(t1..t3), grad_ssim = g1 + 2 a g2 + b g3 (loss.cpp:120-130); with
// lambda >= 0 the photometric gradient (loss.cpp:140-144): (1 - lambda) g_l1 - lambda grad_ssim,
// g_l1 = sign(a - b) / n (loss.cpp:70-73).
__global__ void __launch_bounds__(kTW * kTH) ssim_bwd_kernel(const float* __restrict__ a, const float* __restrict__ b,
                                                            const float* __restrict__ t1, const float* __restrict__ t2,
                                                            const float* __restrict__ t3, int w, int h, int ch,
                                                            SsimWindow win, float lambda, float inv_n,
                                                            float* __restrict__ grad) {
    __shared__ float s_in[3][kSH][kSW];
    __shared__ float s_h[3][kSH][kTW];
    const int c = blockIdx.z;
    const int x0 = blockIdx.x * kTW, y0 = blockIdx.y * kTH;
    const float* srcs[3] = {t1, t2, t3};
    stage_inputs<3>(srcs, w, h, ch, c, x0, y0, s_in);
    __syncthreads();
    for (int i = threadIdx.x; i < kSH * kTW; i += blockDim.x) {
        const int r = i / kTW, q = i - r * kTW;
#pragma unroll
        for (int k = 0; k < 3; ++k) s_h[k][r][q] = hblur(&s_in[k][r], q, x0 + q, w, win);
    }
    __syncthreads();
    const int q = threadIdx.x % kTW, r = threadIdx.x / kTW;
    const int x = x0 + q, y = y0 + r;
    if (x >= w || y >= h) return;
    const float g1 = vblur(s_h[0], r, q, y, h, win);
    const float g2 = vblur(s_h[1], r, q, y, h, win);
    const float g3 = vblur(s_h[2], r, q, y, h, win);
    const size_t o = ((size_t)y * w + x) * ch + c;
    const float av = a[o], bv = b[o];
    const float gs = __fadd_rn(__fadd_rn(g1, __fmul_rn(__fmul_rn(2.0f, av), g2)), __fmul_rn(bv, g3));
    if (lambda < 0.0f) {
        grad[o] = gs;
        return;
    }
    const float d = __fsub_rn(av, bv);
    const float gl1 = d > 0.0f ? inv_n : (d < 0.0f ? -inv_n : 0.0f);
    grad[o] = __fsub_rn(__fmul_rn(__fsub_rn(1.0f, lambda), gl1), __fmul_rn(lambda, gs));
}

// Final means: ssim = sum / n, l1 = sum / n; value = ssim (lambda < 0) or the photometric loss
// (1 - lambda) l1 + lambda (1 - ssim) (loss.cpp:146).
__global__ void ssim_finish_kernel(const double* __restrict__ partials, int nblocks, double n, float lambda,
                                   float* __restrict__ out) {
    __shared__ double s[2][32];
    double ss = 0.0, ll = 0.0;
    for (int i = threadIdx.x; i < nblocks; i += blockDim.x) {
        ss += partials[2 * i];
        ll += partials[2 * i + 1];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        ss += __shfl_xor_sync(0xffffffffu, ss, o);
        ll += __shfl_xor_sync(0xffffffffu, ll, o);
    }
    if ((threadIdx.x & 31) == 0) {
        s[0][threadIdx.x >> 5] = ss;
        s[1][threadIdx.x >> 5] = ll;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0, l = 0.0;
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k) {
            a += s[0][k];
            l += s[1][k];
        }
        const float ssim = (float)(a / n), l1 = (float)(l / n);
        out[0] = lambda < 0.0f ? ssim : __fadd_rn(__fmul_rn(__fsub_rn(1.0f, lambda), l1),
                                                   __fmul_rn(lambda, __fsub_rn(1.0f, ssim)));
    }
}

SsimWindow make_window() {
    // gaussian_kernel (loss.cpp:13-22) in float with the shared exp, sequential sum
    SsimWindow win;
    float sum = 0.0f;
    for (int i = 0; i < 11; ++i) {
        const float d = (float)(i - 5);
        win.k[i] = splat_expf(-d * d / (float)(2 * 1.5 * 1.5));
        sum += win.k[i];
    }
    for (int i = 0; i < 11; ++i) win.k[i] /= sum;
    return win;
}

}  // namespace

size_t ssim_partials_count(int w, int h, int ch) {
    return (size_t)((w + kTW - 1) / kTW) * ((h + kTH - 1) / kTH) * ch;
}

// value_dev: mean SSIM (lambda < 0) or the photometric loss.  grad (nullable): d value / d a.
// tmp: 3 w h ch floats (t1..t3) when grad is requested; partials: 2 ssim_partials_count doubles.
cudaError_t launch_ssim(LaunchCtx& lc, const float* a, const float* b, int w, int h, int ch, float lambda,
                        float* grad, float* value_dev, float* tmp, double* partials) {
    if (w <= 0 || h <= 0 || ch <= 0) return cudaErrorInvalidValue;
    const SsimWindow win = make_window();
    const size_t n = (size_t)w * h * ch;
    const float inv_n = 1.0f / (float)n;
    const dim3 grid((w + kTW - 1) / kTW, (h + kTH - 1) / kTH, ch);
    float *t1 = tmp, *t2 = tmp ? tmp + n : nullptr, *t3 = tmp ? tmp + 2 * n : nullptr;
    {
        LaunchScope s(lc, "ssim_fwd");
        if (grad)
            ssim_fwd_kernel<true><<<grid, kTW * kTH, 0, lc.stream>>>(a, b, w, h, ch, win, inv_n, t1, t2, t3, partials);
        else
            ssim_fwd_kernel<false><<<grid, kTW * kTH, 0, lc.stream>>>(a, b, w, h, ch, win, inv_n, nullptr, nullptr,
                                                                      nullptr, partials);
        lc.count++;
    }
    if (grad) {
        LaunchScope s(lc, "ssim_bwd");
        ssim_bwd_kernel<<<grid, kTW * kTH, 0, lc.stream>>>(a, b, t1, t2, t3, w, h, ch, win, lambda, inv_n, grad);
        lc.count++;
    }
    if (value_dev) {
        LaunchScope s(lc, "ssim_finish");
        ssim_finish_kernel<<<1, 1024, 0, lc.stream>>>(partials, (int)ssim_partials_count(w, h, ch), (double)n, lambda,
                                                      value_dev);
        lc.count++;
    }
    return cudaGetLastError();
}

}  // namespace splat_b200
