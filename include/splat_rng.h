/* splat_rng.h — the reference's random draws, restated in C so the library's host code draws
 * exactly the sequences the reference does (shared with the CPU oracle).
 *
 * The reference draws with libstdc++ (GCC 13) engines and distributions:
 *   identify_critical Random criterion  std::uniform_real_distribution<double> on std::mt19937&
 *                                        (densify.cpp:78-80)
 *   vanilla_clone_split                 std::normal_distribution<float>(0, 1) on std::mt19937&
 *                                        (densify.cpp:141, 154)
 *   depth_reinitialize                  std::uniform_int_distribution<int> partial Fisher-Yates on
 *                                        std::mt19937& (densify.cpp:227-235)
 *   importance_sample                   std::mt19937_64(seed), std::uniform_real_distribution<double>
 *                                        + uniform_int_distribution<int> filler (simplify.cpp:44-84)
 * The engines are fully specified by the C++ standard ([rand.eng.mers]); the distributions follow
 * libstdc++'s published algorithms (bits/random.tcc generate_canonical with one or two engine
 * words, bits/uniform_int_dist.h Lemire's nearly-divisionless downscaling with a 2x-wide
 * product, the Marsaglia polar method with one saved value for normal_distribution).  Pinned
 * bit for bit against the reference's own draws in tests/test_rng_oracle.py.
 *
 * The normal draws take their log from SPLAT_RNG_LOGF (default splat_logf, the shared < 1 ulp
 * logf the oracle's mode B substitutes for glibc's; define it as logf for mode A).
 */
#ifndef SPLAT_RNG_H
#define SPLAT_RNG_H

#include <math.h>
#include <stdint.h>

#include "splat_expf.h"

#ifndef SPLAT_RNG_LOGF
#define SPLAT_RNG_LOGF splat_logf
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* std::mt19937 (w=32, n=624, m=397, r=31): state words + libstdc++'s index _M_p. */
typedef struct splat_mt19937 {
    uint32_t x[624];
    uint32_t p;
} splat_mt19937;

/* std::mt19937_64 (w=64, n=312, m=156, r=31). */
typedef struct splat_mt19937_64 {
    uint64_t x[312];
    uint32_t p;
} splat_mt19937_64;

static inline void splat_mt19937_seed(splat_mt19937* g, uint32_t s) {
    g->x[0] = s;
    for (uint32_t i = 1; i < 624; ++i) g->x[i] = 1812433253u * (g->x[i - 1] ^ (g->x[i - 1] >> 30)) + i;
    g->p = 624;
}

static inline uint32_t splat_mt19937_next(splat_mt19937* g) {
    if (g->p >= 624) {
        for (int k = 0; k < 624; ++k) {
            const uint32_t y = (g->x[k] & 0x80000000u) | (g->x[(k + 1) % 624] & 0x7fffffffu);
            g->x[k] = g->x[(k + 397) % 624] ^ (y >> 1) ^ ((y & 1u) ? 0x9908b0dfu : 0u);
        }
        g->p = 0;
    }
    uint32_t z = g->x[g->p++];
    z ^= z >> 11;
    z ^= (z << 7) & 0x9d2c5680u;
    z ^= (z << 15) & 0xefc60000u;
    z ^= z >> 18;
    return z;
}

static inline void splat_mt19937_64_seed(splat_mt19937_64* g, uint64_t s) {
    g->x[0] = s;
    for (uint64_t i = 1; i < 312; ++i)
        g->x[i] = 6364136223846793005ull * (g->x[i - 1] ^ (g->x[i - 1] >> 62)) + i;
    g->p = 312;
}

static inline uint64_t splat_mt19937_64_next(splat_mt19937_64* g) {
    if (g->p >= 312) {
        for (int k = 0; k < 312; ++k) {
            const uint64_t y = (g->x[k] & 0xffffffff80000000ull) | (g->x[(k + 1) % 312] & 0x7fffffffull);
            g->x[k] = g->x[(k + 156) % 312] ^ (y >> 1) ^ ((y & 1ull) ? 0xb5026f5aa96619e9ull : 0ull);
        }
        g->p = 0;
    }
    uint64_t z = g->x[g->p++];
    z ^= (z >> 29) & 0x5555555555555555ull;
    z ^= (z << 17) & 0x71d67fffeda60000ull;
    z ^= (z << 37) & 0xfff7eee000000000ull;
    z ^= z >> 43;
    return z;
}

/* uniform_real_distribution<double>(0, 1) on mt19937_64: generate_canonical<double, 53> takes one
 * 64-bit word, sum = double(x), divided by 2^64; a result of 1 becomes nextafter(1, 0). */
static inline double splat_canonical_f64_64(splat_mt19937_64* g) {
    double r = (double)splat_mt19937_64_next(g) / 18446744073709551616.0;
    if (r >= 1.0) r = nextafter(1.0, 0.0);
    return r;
}

/* uniform_real_distribution<double>(0, 1) on mt19937: two 32-bit words, sum = x0 + x1 * 2^32
 * (rounded once), divided by 2^64. */
static inline double splat_canonical_f64_32(splat_mt19937* g) {
    const double lo = (double)splat_mt19937_next(g);
    const double hi = (double)splat_mt19937_next(g);
    double r = (lo + hi * 4294967296.0) / 18446744073709551616.0;
    if (r >= 1.0) r = nextafter(1.0, 0.0);
    return r;
}

/* generate_canonical<float, 24> on mt19937 (normal_distribution<float>'s adaptor). */
static inline float splat_canonical_f32_32(splat_mt19937* g) {
    float r = (float)splat_mt19937_next(g) / 4294967296.0f;
    if (r >= 1.0f) r = nextafterf(1.0f, 0.0f);
    return r;
}

/* uniform_int_distribution<int>(a, b) on mt19937_64: 128-bit nearly-divisionless downscaling. */
static inline int32_t splat_uniform_int_64(splat_mt19937_64* g, int32_t a, int32_t b) {
    const uint64_t range = (uint64_t)(int64_t)b - (uint64_t)(int64_t)a + 1u;
    unsigned __int128 prod = (unsigned __int128)splat_mt19937_64_next(g) * range;
    uint64_t low = (uint64_t)prod;
    if (low < range) {
        const uint64_t threshold = (0u - range) % range;
        while (low < threshold) {
            prod = (unsigned __int128)splat_mt19937_64_next(g) * range;
            low = (uint64_t)prod;
        }
    }
    return (int32_t)((uint64_t)(prod >> 64) + (uint64_t)(int64_t)a);
}

/* uniform_int_distribution<int>(a, b) on mt19937: 64-bit nearly-divisionless downscaling. */
static inline int32_t splat_uniform_int_32(splat_mt19937* g, int32_t a, int32_t b) {
    const uint32_t range = (uint32_t)((uint64_t)(int64_t)b - (uint64_t)(int64_t)a + 1u);
    uint64_t prod = (uint64_t)splat_mt19937_next(g) * range;
    uint32_t low = (uint32_t)prod;
    if (low < range) {
        const uint32_t threshold = (0u - range) % range;
        while (low < threshold) {
            prod = (uint64_t)splat_mt19937_next(g) * range;
            low = (uint32_t)prod;
        }
    }
    return (int32_t)((uint64_t)(prod >> 32) + (uint64_t)(int64_t)a);
}

/* std::normal_distribution<float>: Marsaglia polar method, one value saved between calls. */
typedef struct splat_normal_f32 {
    float saved;
    int has_saved;
} splat_normal_f32;

static inline float splat_normal_f32_next(splat_normal_f32* d, splat_mt19937* g, float mean, float stddev) {
    float ret;
    if (d->has_saved) {
        d->has_saved = 0;
        ret = d->saved;
    } else {
        float x, y, r2;
        do {
            x = (float)((double)(2.0f * splat_canonical_f32_32(g)) - 1.0);
            y = (float)((double)(2.0f * splat_canonical_f32_32(g)) - 1.0);
            r2 = x * x + y * y;
        } while ((double)r2 > 1.0 || (double)r2 == 0.0);
        const float mult = sqrtf(-2.0f * SPLAT_RNG_LOGF(r2) / r2);
        d->saved = x * mult;
        d->has_saved = 1;
        ret = y * mult;
    }
    return ret * stddev + mean;
}

/* depth_reinitialize's partial Fisher-Yates (densify.cpp:227-235): idx[0, pool) <- identity, then
 * for r < take: swap(idx[r], idx[uniform_int(r, pool - 1)]).  idx needs pool entries. */
static inline void splat_partial_fisher_yates(splat_mt19937* g, int32_t* idx, int32_t pool, int32_t take) {
    for (int32_t i = 0; i < pool; ++i) idx[i] = i;
    for (int32_t r = 0; r < take; ++r) {
        const int32_t j = splat_uniform_int_32(g, r, pool - 1);
        const int32_t t = idx[r];
        idx[r] = idx[j];
        idx[j] = t;
    }
}

#ifdef __cplusplus
}
#endif

#endif /* SPLAT_RNG_H */
