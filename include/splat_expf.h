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
    /* rint(x / ln2) by the 1.5 * 2^23 shifter: in the core's domain |x / ln2| < 2^22, so the
     * sum lands in [2^23, 2^24) (ulp 1) and rounds x / ln2 to the nearest integer, ties to even,
     * exactly as rintf; the shifter's low mantissa bits are that integer k.  Two adds and an
     * integer subtract instead of a round and a float-to-int conversion (the XU pipe). */
    const float t = splat_mul(x, 1.44269502162933349609375f);
    const float sh = splat_fma(1.0f, t, 12582912.0f);   /* t + 1.5 * 2^23, rounded once */
    const float kf = splat_fma(1.0f, sh, -12582912.0f); /* exact */
    uint32_t shb;
#if defined(__CUDA_ARCH__)
    shb = __float_as_uint(sh);
#else
    memcpy(&shb, &sh, 4);
#endif
    const int k = (int)(shb - 0x4B400000u);
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
    return splat_mul(p, splat_bits_to_float((uint32_t)(k + 127) << 23));
}

/* splat_expf_core with the final scaling as an exponent add: for k >= -125 (x >= -86.6) p * 2^k
 * is a normal float, so the product is exact and equals p's bits plus k << 23 — one integer
 * multiply-add instead of building 2^k and a multiply.  Bit-identical to splat_expf on
 * [-86.6, 0] (tests/test_expf.py); the gates use it on [ln(cmin) - 1e-3, 0]. */
SPLAT_HD float splat_expf_gate(float x) {
    const float t = splat_mul(x, 1.44269502162933349609375f);
    const float sh = splat_fma(1.0f, t, 12582912.0f);
    const float kf = splat_fma(1.0f, sh, -12582912.0f);
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
    uint32_t shb, pb;
#if defined(__CUDA_ARCH__)
    shb = __float_as_uint(sh);
    pb = __float_as_uint(p);
#else
    memcpy(&shb, &sh, 4);
    memcpy(&pb, &p, 4);
#endif
    return splat_bits_to_float(pb + ((shb - 0x4B400000u) << 23));
}

SPLAT_HD float splat_add(float a, float b) {
#if defined(__CUDA_ARCH__)
    return __fadd_rn(a, b);
#else
    return a + b;
#endif
}

SPLAT_HD float splat_sub(float a, float b) {
#if defined(__CUDA_ARCH__)
    return __fsub_rn(a, b);
#else
    return a - b;
#endif
}

SPLAT_HD float splat_div(float a, float b) {
#if defined(__CUDA_ARCH__)
    return __fdiv_rn(a, b);
#else
    return a / b;
#endif
}

SPLAT_HD uint32_t splat_float_to_bits(float f) {
#if defined(__CUDA_ARCH__)
    return __float_as_uint(f);
#else
    uint32_t u;
    memcpy(&u, &f, 4);
    return u;
#endif
}

/* The one natural logarithm shared by the CUDA kernels and the mode-B oracle (the reference
 * calls std::log(float) in aggressive_clone and logit, densify.cpp:116-121, types.hpp:63-65).
 * The classic fdlibm/FreeBSD logf scheme: x = 2^k (1 + f) with 1 + f in [sqrt(2)/2, sqrt(2)),
 * s = f / (2 + f), log(1 + f) = f - (f^2/2 - s (f^2/2 + R(s^2))) with the published minimax
 * coefficients, and k ln2 split hi/lo.  Only correctly rounded +, -, *, / (no contraction), so
 * gcc and nvcc agree bit for bit.  Accuracy: < 1 ulp (tests/test_expf.py). */
SPLAT_HD float splat_logf(float x) {
    const float ln2_hi = 6.9313812256e-01f, ln2_lo = 9.0580006145e-06f;
    const float Lg1 = 6.6666662693e-01f, Lg2 = 4.0000972152e-01f, Lg3 = 2.8498786688e-01f,
                Lg4 = 2.4279078841e-01f;
    uint32_t ix = splat_float_to_bits(x);
    int k = 0;
    if (ix < 0x00800000u || (ix >> 31)) {          /* x < 2^-126 (subnormal or 0) or negative */
        if ((ix & 0x7fffffffu) == 0) return splat_bits_to_float(0xff800000u); /* -inf */
        if (ix >> 31) return splat_bits_to_float(0x7fc00000u);                 /* NaN */
        k -= 25;
        x = splat_mul(x, 33554432.0f);            /* 2^25: exact */
        ix = splat_float_to_bits(x);
    } else if (ix >= 0x7f800000u) {
        return x;                                  /* +inf or NaN */
    } else if (ix == 0x3f800000u) {
        return 0.0f;
    }
    k += (int)(ix >> 23) - 127;
    ix &= 0x007fffffu;
    const uint32_t i = (ix + (0x95f64u << 3)) & 0x800000u;   /* mantissa above sqrt(2): halve */
    x = splat_bits_to_float(ix | (i ^ 0x3f800000u));
    k += (int)(i >> 23);
    const float f = splat_sub(x, 1.0f);
    const float s = splat_div(f, splat_add(2.0f, f));
    const float dk = (float)k;
    const float z = splat_mul(s, s);
    const float w = splat_mul(z, z);
    const float t1 = splat_mul(w, splat_add(Lg2, splat_mul(w, Lg4)));
    const float t2 = splat_mul(z, splat_add(Lg1, splat_mul(w, Lg3)));
    const float R = splat_add(t2, t1);
    const float hfsq = splat_mul(splat_mul(0.5f, f), f);
    /* dk*ln2_hi - ((hfsq - (s*(hfsq+R) + dk*ln2_lo)) - f) */
    const float inner = splat_add(splat_mul(s, splat_add(hfsq, R)), splat_mul(dk, ln2_lo));
    return splat_sub(splat_mul(dk, ln2_hi), splat_sub(splat_sub(hfsq, inner), f));
}

#endif /* SPLAT_EXPF_H */
