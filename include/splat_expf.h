/*
 * splat_expf.h — the one exponential shared by the CUDA kernels and the CPU oracle.
 *
 * The reference evaluates std::exp(float) at three places that decide integer outputs
 * (pixel rects, tile lists, gates, argmax): log-scale -> scale (gaussian_set.hpp:44, 84),
 * sigmoid (types.hpp:58-60) and the 2D Gaussian falloff (rasterizer.hpp:131).  glibc's
 * expf and CUDA's expf round differently in a few ulps, which flips a handful of
 * rects/gates per million Gaussians.  "Mode B" parity therefore routes all
 * three through this function on both sides: range reduction with fmaf, a degree-7
 * polynomial evaluated with fmaf, and an exact two-step 2^k scaling.  Every step is a
 * correctly-rounded IEEE operation, so gcc (libm fmaf) and nvcc (__fmaf_rn) produce the
 * same bits.  Accuracy: <= 1 ulp against the correctly rounded exp on [-103, 88.7].
 *
 * Plain C99 so the oracle (gcc) and the kernels (nvcc, host and device) share it.
 */
#ifndef SPLAT_EXPF_H
#define SPLAT_EXPF_H

#include <math.h>
#include <stdint.h>
#include <string.h>

#if defined(__CUDACC__)
#define SPLAT_HD __host__ __device__ __forceinline__
#else
#define SPLAT_HD static inline
#endif

SPLAT_HD float splat_bits_to_float(uint32_t u) {
#if defined(__CUDA_ARCH__)
    return __uint_as_float(u);
#else
    float f;
    memcpy(&f, &u, 4);
    return f;
#endif
}

SPLAT_HD float splat_fma(float a, float b, float c) {
#if defined(__CUDA_ARCH__)
    return __fmaf_rn(a, b, c);
#else
    return fmaf(a, b, c);
#endif
}

SPLAT_HD float splat_mul(float a, float b) {
#if defined(__CUDA_ARCH__)
    return __fmul_rn(a, b);
#else
    return a * b;
#endif
}

SPLAT_HD float splat_expf(float x) {
    if (x != x) return x;                         /* NaN */
    if (x > 88.72283935546875f) return splat_bits_to_float(0x7f800000u); /* +inf */
    if (x < -103.97208404541015625f) return 0.0f; /* below half the smallest subnormal */
    /* k = nearest integer to x / ln 2; r = x - k ln2 in two exact-ish pieces */
    const float kf = rintf(splat_mul(x, 1.44269502162933349609375f));
    float r = splat_fma(kf, -0.693145751953125f, x);          /* ln2_hi, 16 bits: exact */
    r = splat_fma(kf, -1.428606765330187045037746429443359375e-06f, r); /* ln2_lo */
    /* exp(r), |r| <= 0.3467: Taylor to degree 7 (truncation < 5e-9 relative) */
    float p = 1.98412698412698412698e-4f;         /* 1/5040 */
    p = splat_fma(p, r, 1.38888888888888888889e-3f);  /* 1/720 */
    p = splat_fma(p, r, 8.33333333333333333333e-3f);  /* 1/120 */
    p = splat_fma(p, r, 4.16666666666666666667e-2f);  /* 1/24 */
    p = splat_fma(p, r, 1.66666666666666666667e-1f);  /* 1/6 */
    p = splat_fma(p, r, 0.5f);
    p = splat_fma(p, r, 1.0f);
    p = splat_fma(p, r, 1.0f);
    /* scale by 2^k = 2^k1 * 2^k2 with both halves in the normal range: the first product
     * is exact, the second rounds once (also into the subnormal range). */
    const int k = (int)kf;
    const int k1 = k / 2;
    const int k2 = k - k1;
    const float s1 = splat_bits_to_float((uint32_t)(k1 + 127) << 23);
    const float s2 = splat_bits_to_float((uint32_t)(k2 + 127) << 23);
    return splat_mul(splat_mul(p, s1), s2);
}

/* splat_expf without the special cases, for arguments whose k = rint(x / ln2) lies in
 * [-126, 127] (x in [-87.3, 88.0]): there 2^k is a normal float, so p * 2^k is the exact value
 * rounded once — the same single rounding the two-step scaling of splat_expf performs — and the
 * result is bit-identical to splat_expf (checked exhaustively over [-87.3, 0] by
 * tests/test_expf.py).  The blend kernels use it after the `power >= cut` test, which confines
 * the argument to [ln(cmin) - 1e-3, 0]. */
SPLAT_HD float splat_expf_core(float x) {
    const float kf = rintf(splat_mul(x, 1.44269502162933349609375f));
    float r = splat_fma(kf, -0.693145751953125f, x);
    r = splat_fma(kf, -1.428606765330187045037746429443359375e-06f, r);
    float p = 1.98412698412698412698e-4f;
    p = splat_fma(p, r, 1.38888888888888888889e-3f);
    p = splat_fma(p, r, 8.33333333333333333333e-3f);
    p = splat_fma(p, r, 4.16666666666666666667e-2f);
    p = splat_fma(p, r, 1.66666666666666666667e-1f);
    p = splat_fma(p, r, 0.5f);
    p = splat_fma(p, r, 1.0f);
    p = splat_fma(p, r, 1.0f);
    return splat_mul(p, splat_bits_to_float((uint32_t)((int)kf + 127) << 23));
}

#endif /* SPLAT_EXPF_H */
