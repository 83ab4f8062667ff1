// sort.cu — single-pass exclusive scan and Onesweep-style stable LSD radix sort (hand-written,
// sm_100a).
//
// Replaces the reference's std::sort of ProjectedGaussian by (depth_mean, index)
// (rasterizer.cpp:85-88).  The N depth keys (IEEE bits of depth_mean > 0, monotone as uint32;
// culled Gaussians carry 0xFFFFFFFF) are sorted stably with the Gaussian ids as values, in index
// order, which yields exactly the reference's (depth, index) order; the same sort orders the
// (supertile, Gaussian) pairs of binning.cu.
//
// Scan: one kernel.  Tiles of 4096 items take their tile id from an atomic counter (so every
// predecessor is already running: forward progress without relying on block scheduling order),
// publish their aggregate, then look back over predecessors' (flag, value) words (decoupled
// look-back) for the exclusive prefix.
//
// Radix sort: one histogram kernel computes the digit histograms of every pass in a single read
// of the keys; then each pass is one kernel: tiles rank their keys per warp with __match_any_sync
// (stable), publish per-digit tile counts, look back per digit (one thread per digit) for the
// tile's global digit offsets, and scatter.  2 + passes launches per sort instead of 5 per pass.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include <cooperative_groups.h>
#include <cstdint>

#include "common.cuh"
#include "internal.h"

namespace splat_b200 {

namespace {

constexpr int kThreads = 256;
constexpr int kItems = 16;
constexpr int kTile = kThreads * kItems;  // 4096 (scan)
constexpr int kWarps = kThreads / 32;
constexpr int kSortItems = 8;
constexpr int kSortTile = kThreads * kSortItems;  // 2048 (radix passes: more CTAs, fewer registers)

// 64-bit look-back words: bits 62-63 flag (1 aggregate, 2 inclusive prefix), low bits value.
constexpr uint64_t kFlagAgg = 1ull << 62;
constexpr uint64_t kFlagInc = 2ull << 62;
constexpr uint64_t kValMask = (1ull << 62) - 1;

// 32-bit look-back words for the per-digit radix status: bits 30-31 flag, low 30 bits value.
constexpr uint32_t kFlagAgg32 = 1u << 30;
constexpr uint32_t kFlagInc32 = 2u << 30;
constexpr uint32_t kValMask32 = (1u << 30) - 1;

__device__ __forceinline__ void st_relaxed64(uint64_t* p, uint64_t v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_relaxed64(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed32(uint32_t* p, uint32_t v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_relaxed32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
    }
    return v;
}

// Block-wide exclusive scan of one value per thread (kThreads threads); *total gets the sum.
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* total, uint32_t* s_warp) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t inc = warp_incl_scan(v, lane);
    if (lane == 31) s_warp[warp] = inc;
    __syncthreads();
    uint32_t off = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
        const uint32_t c = s_warp[w];
        off += w < warp ? c : 0u;
        tot += c;
    }
    *total = tot;
    __syncthreads();
    return off + inc - v;
}

// ---- single-pass scan -------------------------------------------------------------------------
// tmp layout (u64 words): [0] tile counter, [1 + t] look-back word of tile t, [1 + ntiles] done
// count.  RESET: tmp is zero at rest (no memset before the launch): the last tile to finish its
// look-back re-zeroes the counter, the look-back words and the done count.
template <bool GATHER, bool RESET = false>
__global__ void __launch_bounds__(kThreads) scan_lookback_kernel(const uint32_t* __restrict__ in,
                                                                const uint32_t* __restrict__ idx,
                                                                uint32_t* __restrict__ out, uint64_t n,
                                                                uint64_t* __restrict__ tmp,
                                                                uint32_t* __restrict__ total_out) {
    // padded by one word per 32 (spad): a thread's kItems consecutive elements, read and written
    // across the warp, would otherwise fall 16 lanes to a bank
    __shared__ uint32_t s_data[kTile + kTile / 32];
    auto spad = [](int li) { return li + (li >> 5); };
    __shared__ uint32_t s_warp[kWarps];
    __shared__ uint64_t s_tile, s_prefix;
    pdl_wait();
    pdl_trigger();
    if (threadIdx.x == 0) s_tile = atomicAdd(reinterpret_cast<unsigned long long*>(tmp), 1ull);
    __syncthreads();
    const uint64_t tile = s_tile;
    const uint64_t base = tile * kTile;
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
        const int li = k * kThreads + threadIdx.x;
        const uint64_t i = base + li;
        s_data[spad(li)] = i < n ? (GATHER ? in[idx[i]] : in[i]) : 0u;
    }
    __syncthreads();
    uint32_t local[kItems];
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
        local[k] = s;
        s += s_data[spad(threadIdx.x * kItems + k)];
    }
    uint32_t agg;
    const uint32_t ex = block_exclusive_scan(s, &agg, s_warp);
    uint64_t* status = tmp + 1;
    if (threadIdx.x < 32) {  // warp-cooperative look-back: 32 predecessors per round trip
        const int lane = threadIdx.x;
        uint64_t prefix = 0;
        if (tile == 0) {
            if (lane == 0) st_relaxed64(&status[0], kFlagInc | agg);
        } else {
            if (lane == 0) st_relaxed64(&status[tile], kFlagAgg | agg);
            int64_t hi_p = (int64_t)tile - 1;
            while (true) {
                const int64_t p = hi_p - lane;
                const uint64_t w = p >= 0 ? ld_relaxed64(&status[p]) : kFlagInc;
                if (__any_sync(0xffffffffu, (w >> 62) == 0)) continue;
                const unsigned inc = __ballot_sync(0xffffffffu, (w >> 62) == 2);
                const int first_inc = inc ? __ffs(inc) - 1 : 32;  // nearest inclusive predecessor
                uint64_t v = lane <= first_inc ? (w & kValMask) : 0ull;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                prefix += v;
                if (inc) break;
                hi_p -= 32;
            }
            if (lane == 0) st_relaxed64(&status[tile], kFlagInc | (prefix + agg));
        }
        const uint64_t ntiles = (n + kTile - 1) / kTile;
        if (lane == 0) {
            s_prefix = prefix;
            if (total_out && tile == ntiles - 1) *total_out = (uint32_t)(prefix + agg);
        }
        if (RESET) {
            unsigned long long last = 0;
            if (lane == 0) {
                __threadfence();
                last = atomicAdd(reinterpret_cast<unsigned long long*>(status + ntiles), 1ull) == ntiles - 1;
            }
            if (__shfl_sync(0xffffffffu, last, 0)) {  // every tile is past its look-back
                __threadfence();
                for (uint64_t q = lane; q < ntiles + 2; q += 32) tmp[q] = 0ull;
            }
        }
    }
    __syncthreads();
    const uint32_t off = (uint32_t)s_prefix + ex;
#pragma unroll
    for (int k = 0; k < kItems; ++k) s_data[spad(threadIdx.x * kItems + k)] = off + local[k];
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
        const int li = k * kThreads + threadIdx.x;
        const uint64_t i = base + li;
        if (i < n) out[i] = s_data[spad(li)];
    }
}

// ---- radix sort -------------------------------------------------------------------------------
// Digit histograms of all passes (passes x 256 bins, digit width `bits`) in one read.
__global__ void __launch_bounds__(kThreads) radix_histogram_kernel(const uint32_t* __restrict__ keys, uint64_t n,
                                                                  int begin_bit, int bits, int passes,
                                                                  uint32_t* __restrict__ hist) {
    __shared__ uint32_t s_hist[4][512];
    for (int i = threadIdx.x; i < 4 * 512; i += kThreads) (&s_hist[0][0])[i] = 0u;
    __syncthreads();
    const uint32_t mask = (1u << bits) - 1u;
    for (uint64_t i = (uint64_t)blockIdx.x * kThreads + threadIdx.x; i < n; i += (uint64_t)gridDim.x * kThreads) {
        const uint32_t k = keys[i];
        for (int p = 0; p < passes; ++p) atomicAdd(&s_hist[p][(k >> (begin_bit + p * bits)) & mask], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < passes * 512; i += kThreads) {
        const uint32_t v = (&s_hist[0][0])[i];
        if (v) atomicAdd(&hist[i], v);
    }
}

// One stable pass.  status: [ntiles][BINS] look-back words (zeroed); counter: tile id counter.
template <int BITS>
__global__ void __launch_bounds__(kThreads) radix_onesweep_kernel(
    const uint32_t* __restrict__ keys_in, const uint32_t* __restrict__ vals_in, uint32_t* __restrict__ keys_out,
    uint32_t* __restrict__ vals_out, uint32_t n, int shift, const uint32_t* __restrict__ hist,
    uint32_t* __restrict__ status, uint32_t* __restrict__ counter) {
    constexpr int BINS = 1 << BITS;
    constexpr int PER_WARP = kSortTile / kWarps;  // consecutive keys per warp
    __shared__ uint32_t s_cnt[kWarps][BINS];
    __shared__ uint32_t s_glob[BINS];
    __shared__ uint32_t s_warp[kWarps];
    __shared__ uint32_t s_tile;
    // A pass whose digit is the same for every key (one histogram bin holds all n keys, e.g. the
    // exponent byte of depths within one binade) is the identity permutation: copy.
    bool trivial = false;
    for (int d = threadIdx.x; d < BINS; d += kThreads) trivial |= hist[d] == n;
    if (__syncthreads_or(trivial)) {
        const uint64_t base = (uint64_t)blockIdx.x * kSortTile;
        for (int r = threadIdx.x; r < kSortTile; r += kThreads) {
            const uint64_t i = base + r;
            if (i < n) {
                keys_out[i] = keys_in[i];
                vals_out[i] = vals_in[i];
            }
        }
        return;
    }
    for (int i = threadIdx.x; i < kWarps * BINS; i += kThreads) (&s_cnt[0][0])[i] = 0u;
    if (threadIdx.x == 0) s_tile = atomicAdd(counter, 1u);
    {  // global exclusive digit offsets of this pass (BINS <= 2 * kThreads)
        uint32_t tot0, tot1;
        const uint32_t v0 = threadIdx.x < BINS ? hist[threadIdx.x] : 0u;
        const uint32_t ex0 = block_exclusive_scan(v0, &tot0, s_warp);
        if (threadIdx.x < BINS) s_glob[threadIdx.x] = ex0;
        if (BINS > kThreads) {
            const uint32_t v1 = threadIdx.x + kThreads < BINS ? hist[threadIdx.x + kThreads] : 0u;
            const uint32_t ex1 = block_exclusive_scan(v1, &tot1, s_warp);
            if (threadIdx.x + kThreads < BINS) s_glob[threadIdx.x + kThreads] = tot0 + ex1;
        }
    }
    const uint32_t tile = s_tile;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t wbase = (uint64_t)tile * kSortTile + (uint64_t)warp * PER_WARP;
    uint32_t k[kSortItems], v[kSortItems];
#pragma unroll
    for (int r = 0; r < kSortItems; ++r) {
        const uint64_t i = wbase + (uint64_t)r * 32 + lane;
        k[r] = i < n ? keys_in[i] : 0u;
        v[r] = i < n ? vals_in[i] : 0u;
    }
    __syncthreads();
    const unsigned lt = lanemask_lt();
    uint32_t rank[kSortItems];
#pragma unroll
    for (int r = 0; r < kSortItems; ++r) {
        const uint64_t i = wbase + (uint64_t)r * 32 + lane;
        const bool valid = i < n;
        const uint32_t d = (k[r] >> shift) & (BINS - 1);
        const uint32_t label = valid ? d : (0x80000000u | (uint32_t)lane);
        const unsigned peers = __match_any_sync(0xffffffffu, label);
        const uint32_t old = valid ? s_cnt[warp][d] : 0u;
        __syncwarp();
        if (valid && (peers & lt) == 0u) s_cnt[warp][d] = old + __popc(peers);
        __syncwarp();
        rank[r] = old + __popc(peers & lt);
    }
    __syncthreads();
    for (int d = threadIdx.x; d < BINS; d += kThreads) {
        uint32_t c = 0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) c += s_cnt[w][d];
        uint32_t* st = status + (uint64_t)tile * BINS + d;
        uint32_t prefix = 0;
        if (tile == 0) {
            st_relaxed32(st, kFlagInc32 | c);
        } else {
            st_relaxed32(st, kFlagAgg32 | c);
            // windowed look-back: kWin predecessors per round trip instead of one
            constexpr int kWin = 16;
            int64_t hi_p = (int64_t)tile - 1;
            while (true) {
                uint32_t w[kWin];
#pragma unroll
                for (int q = 0; q < kWin; ++q) {
                    const int64_t p = hi_p - q;
                    w[q] = p >= 0 ? ld_relaxed32(status + (uint64_t)p * BINS + d) : kFlagInc32;
                }
                bool ready = true;
#pragma unroll
                for (int q = 0; q < kWin; ++q) ready &= (w[q] >> 30) != 0;
                if (!ready) continue;
                uint32_t acc = 0;
                bool done = false;
#pragma unroll
                for (int q = 0; q < kWin; ++q) {
                    if (!done) {
                        acc += w[q] & kValMask32;
                        done = (w[q] >> 30) == 2;
                    }
                }
                prefix += acc;
                if (done) break;
                hi_p -= kWin;
            }
            st_relaxed32(st, kFlagInc32 | (prefix + c));
        }
        uint32_t run = s_glob[d] + prefix;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            const uint32_t cw = s_cnt[w][d];
            s_cnt[w][d] = run;
            run += cw;
        }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kSortItems; ++r) {
        const uint64_t i = wbase + (uint64_t)r * 32 + lane;
        if (i < n) {
            const uint32_t d = (k[r] >> shift) & (BINS - 1);
            const uint32_t pos = s_cnt[warp][d] + rank[r];
            keys_out[pos] = k[r];
            vals_out[pos] = v[r];
        }
    }
}

// Reduce-then-scan variant of one pass, for passes with many tiles (the Onesweep look-back chain
// grows with the tile count): per-tile digit counts (digit-major), the single-pass scan over that
// matrix, then the same stable ranking + scatter with the scanned offsets.
template <int BITS>
__global__ void __launch_bounds__(kThreads) radix_tile_counts_kernel(const uint32_t* __restrict__ keys, uint32_t n,
                                                                    int shift, uint32_t* __restrict__ counts,
                                                                    uint32_t ntiles) {
    constexpr int BINS = 1 << BITS;
    __shared__ uint32_t s_hist[kWarps][BINS];
    for (int i = threadIdx.x; i < kWarps * BINS; i += kThreads) (&s_hist[0][0])[i] = 0u;
    __syncthreads();
    const int warp = threadIdx.x >> 5;
    const uint64_t base = (uint64_t)blockIdx.x * kSortTile;
#pragma unroll
    for (int r = 0; r < kSortItems; ++r) {
        const uint64_t i = base + (uint64_t)r * kThreads + threadIdx.x;
        if (i < n) atomicAdd(&s_hist[warp][(keys[i] >> shift) & (BINS - 1)], 1u);
    }
    __syncthreads();
    for (int d = threadIdx.x; d < BINS; d += kThreads) {
        uint32_t c = 0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) c += s_hist[w][d];
        counts[(uint64_t)d * ntiles + blockIdx.x] = c;
    }
}

template <int BITS>
__global__ void __launch_bounds__(kThreads) radix_scatter_kernel(
    const uint32_t* __restrict__ keys_in, const uint32_t* __restrict__ vals_in, uint32_t* __restrict__ keys_out,
    uint32_t* __restrict__ vals_out, uint32_t n, int shift, const uint32_t* __restrict__ offs, uint32_t ntiles) {
    constexpr int BINS = 1 << BITS;
    constexpr int PER_WARP = kSortTile / kWarps;
    __shared__ uint32_t s_cnt[kWarps][BINS];
    for (int i = threadIdx.x; i < kWarps * BINS; i += kThreads) (&s_cnt[0][0])[i] = 0u;
    const uint32_t tile = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t wbase = (uint64_t)tile * kSortTile + (uint64_t)warp * PER_WARP;
    uint32_t k[kSortItems], v[kSortItems];
#pragma unroll
    for (int r = 0; r < kSortItems; ++r) {
        const uint64_t i = wbase + (uint64_t)r * 32 + lane;
        k[r] = i < n ? keys_in[i] : 0u;
        v[r] = i < n ? vals_in[i] : 0u;
    }
    __syncthreads();
    const unsigned lt = lanemask_lt();
    uint32_t rank[kSortItems];
#pragma unroll
    for (int r = 0; r < kSortItems; ++r) {
        const uint64_t i = wbase + (uint64_t)r * 32 + lane;
        const bool valid = i < n;
        const uint32_t d = (k[r] >> shift) & (BINS - 1);
        const uint32_t label = valid ? d : (0x80000000u | (uint32_t)lane);
        const unsigned peers = __match_any_sync(0xffffffffu, label);
        const uint32_t old = valid ? s_cnt[warp][d] : 0u;
        __syncwarp();
        if (valid && (peers & lt) == 0u) s_cnt[warp][d] = old + __popc(peers);
        __syncwarp();
        rank[r] = old + __popc(peers & lt);
    }
    __syncthreads();
    for (int d = threadIdx.x; d < BINS; d += kThreads) {
        uint32_t run = offs[(uint64_t)d * ntiles + tile];
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            const uint32_t cw = s_cnt[w][d];
            s_cnt[w][d] = run;
            run += cw;
        }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kSortItems; ++r) {
        const uint64_t i = wbase + (uint64_t)r * 32 + lane;
        if (i < n) {
            const uint32_t d = (k[r] >> shift) & (BINS - 1);
            const uint32_t pos = s_cnt[warp][d] + rank[r];
            keys_out[pos] = k[r];
            vals_out[pos] = v[r];
        }
    }
}

// Above this many tiles the Onesweep look-back chain costs more than a reduce-then-scan pass.
static uint32_t onesweep_max_tiles() {
    static uint32_t v = [] {
        const char* e = std::getenv("SPLAT_ONESWEEP_MAX");
        return e ? (uint32_t)std::strtoul(e, nullptr, 10) : 640u;
    }();
    return v;
}

template <int BITS>
void launch_onesweep(LaunchCtx& lc, const uint32_t* ki, const uint32_t* vi, uint32_t* ko, uint32_t* vo, uint32_t n,
                     int shift, const uint32_t* hist, uint32_t* status, uint32_t* counter, uint32_t* scan_tmp) {
    const uint32_t ntiles = (n + kSortTile - 1) / kSortTile;
    if (ntiles <= onesweep_max_tiles()) {
        radix_onesweep_kernel<BITS><<<ntiles, kThreads, 0, lc.stream>>>(ki, vi, ko, vo, n, shift, hist, status, counter);
        return;
    }
    uint32_t* counts = status;  // [BINS][ntiles] fits in the pass's status area
    radix_tile_counts_kernel<BITS><<<ntiles, kThreads, 0, lc.stream>>>(ki, n, shift, counts, ntiles);
    exclusive_scan_u32(lc, counts, counts, (uint64_t)ntiles << BITS, scan_tmp, nullptr);
    radix_scatter_kernel<BITS><<<ntiles, kThreads, 0, lc.stream>>>(ki, vi, ko, vo, n, shift, counts, ntiles);
    lc.count += 2;
}

// ---- cooperative whole-sort kernel ---------------------------------------------------------
// For N up to (resident CTAs) x 4096 keys the whole LSD sort runs as ONE cooperative kernel: each
// CTA owns one 4096-key tile for the whole sort, so a pass is rank -> publish per-digit tile
// counts -> grid barrier -> 256 CTAs scan one digit row each -> grid barrier -> scatter -> grid
// barrier, with no look-back chain (the Onesweep look-back serialises ~tiles/16 round trips when
// every tile runs in the same wave).  The first phase histograms all four byte digits; passes
// whose digit is the same for every key are skipped, and the buffer chain is routed through a
// third buffer so the result always lands in (keys1, vals1).
namespace cg = cooperative_groups;
#ifdef SPLAT_SORT_STAMPS  // phase timestamps of CTA 0 printed at exit (tools/variant_build.py experiments)
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define STAMP(i) \
    if (blockIdx.x == 0 && threadIdx.x == 0) stamps[i] = gtimer()
#else
#define STAMP(i)
#endif
constexpr int kCoopItems = 16;
constexpr int kCoopTile = kThreads * kCoopItems;
constexpr int kCoopMaxTpc = 6;  // tiles per CTA (up to 148 x 6 x 4096 = 3.6 M keys in one wave)
constexpr size_t coop_dyn_smem(int tpc) { return (size_t)tpc * (2 * kCoopTile + 256) * 4; }  // 4096 (245 CTAs at N = 1 M: fewer to barrier)

// Multi-tile form: CTA b owns tiles b, b + grid, ... (tpc of them); each tile's keys are held in
// its own dynamic shared-memory slot between the rank phase and the scatter, so the three grid
// barriers per pass are shared by all of the CTA's tiles.
// TPC = 1: one tile per CTA, its slot in static shared memory; TPC = 0: `tpc` tiles per CTA in
// dynamic shared memory.
template <int TPC>
__global__ void __launch_bounds__(kThreads, 2) radix_coop_kernel(uint32_t* __restrict__ k0, uint32_t* __restrict__ v0,
                                                              uint32_t* __restrict__ k1, uint32_t* __restrict__ v1,
                                                              uint32_t* __restrict__ k2, uint32_t* __restrict__ v2,
                                                              uint32_t n, uint32_t* __restrict__ hist,
                                                              uint32_t* __restrict__ counts, int tpc_rt,
                                                              uint32_t* key_range) {
    const int tpc = TPC > 0 ? TPC : tpc_rt;
    cg::grid_group grid = cg::this_grid();
    pdl_trigger();  // st_count (PDL) may be scheduled on the SM slots left free
#ifdef SPLAT_SORT_STAMPS
    unsigned long long stamps[32];
    int ns = 0;
#endif
    STAMP(0);
    constexpr int kChains = 2;  // independent rank-counter chains per warp
    constexpr int kVW = kChains * kWarps;  // virtual warps
    __shared__ __align__(16) uint16_t s_cnt[kVW][256];
    __shared__ uint32_t s_gh[4][256];
    __shared__ uint32_t s_warp[kWarps];
    __shared__ uint32_t s_delta[256];
    // per owned tile: its keys / values in local (digit, original position) order (the scatter then
    // writes each digit's run of the tile to consecutive global positions) and the local start of
    // each digit
    extern __shared__ __align__(16) uint32_t s_dyn[];
    __shared__ __align__(16) uint32_t s_static[TPC == 1 ? 2 * kCoopTile + 256 : 1];
    uint32_t* const s_slots = TPC == 1 ? s_static : s_dyn;
    const uint32_t ntiles = (n + kCoopTile - 1) / kCoopTile;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    auto slot_k = [&](int q) { return s_slots + (size_t)q * (2 * kCoopTile + 256); };
    auto slot_v = [&](int q) { return s_slots + (size_t)q * (2 * kCoopTile + 256) + kCoopTile; };
    auto slot_ls = [&](int q) { return s_slots + (size_t)q * (2 * kCoopTile + 256) + 2 * kCoopTile; };
    auto tile_of = [&](int q) { return blockIdx.x + (uint32_t)q * gridDim.x; };
    uint32_t k[kCoopItems], v[kCoopItems];
    // The depth sort (key_range given): phase 0 only reduces the survivors' key range
    // [max(~key), max(key)] (keys other than 0xFFFFFFFF); the executed passes follow from it and
    // each pass's histogram is summed from the tiles' digit counts in its rank phase — no
    // histogram atomics per key.  Culled keys (0xFFFFFFFF) become kmax + 1, so they still sort
    // after every survivor when the passes above the range's common prefix are skipped.
    const bool ranged = key_range != nullptr;
    uint32_t kmax1 = 0;
    int passes[4], m = 0;
    if (ranged) {
        uint32_t kmx = 0, knm = 0;
        // (owned tiles in reverse, so tile 0's keys stay in registers for the first pass)
        for (int q = tpc - 1; q >= 0; --q) {
            const uint32_t wbase = tile_of(q) * kCoopTile + warp * (kCoopTile / kWarps);
#pragma unroll
            for (int r = 0; r < kCoopItems; ++r) {
                const uint32_t i = wbase + r * 32 + lane;
                k[r] = i < n ? k0[i] : 0xffffffffu;
                if (q == 0) v[r] = i < n ? v0[i] : 0u;
                if (k[r] != 0xffffffffu) {
                    kmx = max(kmx, k[r]);
                    knm = max(knm, ~k[r]);
                }
            }
        }
        kmx = __reduce_max_sync(0xffffffffu, kmx);
        knm = __reduce_max_sync(0xffffffffu, knm);
        if (lane == 0) {
            s_warp[warp] = kmx;
            s_delta[warp] = knm;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int w = 1; w < kWarps; ++w) {
                kmx = max(kmx, s_warp[w]);
                knm = max(knm, s_delta[w]);
            }
            if (kmx | knm) {
                atomicMax(key_range, knm);
                atomicMax(key_range + 1, kmx);
            }
        }
        STAMP(1);
        grid.sync();
        STAMP(2);
        const uint32_t r0 = *reinterpret_cast<volatile uint32_t*>(key_range);
        const uint32_t r1 = *reinterpret_cast<volatile uint32_t*>(key_range + 1);
        if (r0 | r1) {  // (no survivors: nothing to order)
            const uint32_t kmin = ~r0;
            kmax1 = r1 + 1u;
            for (int p = 0; p < 4; ++p)
                if ((kmin >> (8 * p)) != (kmax1 >> (8 * p))) passes[m++] = p;
#pragma unroll
            for (int r = 0; r < kCoopItems; ++r)  // tile 0, in registers
                if (k[r] == 0xffffffffu) k[r] = kmax1;
        }
    } else {
    // phase 0: digit histograms of all four bytes
    for (int i = threadIdx.x; i < 4 * 256; i += kThreads) (&s_gh[0][0])[i] = 0u;
    __syncthreads();
    // (owned tiles in reverse, so tile 0's keys stay in registers for the first pass)
    for (int q = tpc - 1; q >= 0; --q) {
        const uint32_t wbase = tile_of(q) * kCoopTile + warp * (kCoopTile / kWarps);
#pragma unroll
        for (int r = 0; r < kCoopItems; ++r) {
            const uint32_t i = wbase + r * 32 + lane;
            k[r] = i < n ? k0[i] : 0u;
            if (q == 0) v[r] = i < n ? v0[i] : 0u;
            if (i < n)
#pragma unroll
                for (int p = 0; p < 4; ++p) atomicAdd(&s_gh[p][(k[r] >> (8 * p)) & 255u], 1u);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 4 * 256; i += kThreads)
        if ((&s_gh[0][0])[i]) atomicAdd(&hist[i], (&s_gh[0][0])[i]);
    STAMP(1);
    grid.sync();
    STAMP(2);
    for (int i = threadIdx.x; i < 4 * 256; i += kThreads) (&s_gh[0][0])[i] = hist[i];
    __syncthreads();
    // executed passes (uniform over the grid) and the buffer chain 0 -> ... -> 1 (alternating
    // 1 / 2 backwards from the last pass)
    for (int p = 0; p < 4; ++p) {
        bool trivial = false;
        for (int d = threadIdx.x; d < 256; d += kThreads) trivial |= s_gh[p][d] == n;
        if (!__syncthreads_or(trivial)) passes[m++] = p;
    }
    }
    uint32_t* kb[3] = {k0, k1, k2};
    uint32_t* vb[3] = {v0, v1, v2};
    if (m == 0) {  // nothing to reorder: copy to the result buffers
        for (int q = 0; q < tpc; ++q)
            for (uint32_t i = tile_of(q) * kCoopTile + threadIdx.x; i < min(n, (tile_of(q) + 1) * kCoopTile);
                 i += kThreads) {
                k1[i] = k0[i];
                v1[i] = v0[i];
            }
        grid.sync();  // every CTA has read hist / the key range
        if (blockIdx.x == 0)
            for (int i = threadIdx.x; i < 4 * 256; i += kThreads) hist[i] = 0u;  // zero at rest
        if (ranged && blockIdx.x == 0 && threadIdx.x < 2) key_range[threadIdx.x] = 0u;  // zero at rest
        return;
    }
    int src = 0;
    const unsigned lt = lanemask_lt();
    for (int j = 0; j < m; ++j) {
        const int dst = ((m - 1 - j) & 1) ? 2 : 1;
        const int shift = 8 * passes[j];
        for (int q = 0; q < tpc; ++q) {
            const uint32_t tile = tile_of(q);
            if (tile >= ntiles) break;  // the last CTAs own one tile fewer (CTA-uniform)
            const uint32_t wbase = tile * kCoopTile + warp * (kCoopTile / kWarps);
            if (j > 0 || q > 0) {  // tile 0 of the first pass is still in registers
#pragma unroll
                for (int r = 0; r < kCoopItems; ++r) {
                    const uint32_t i = wbase + r * 32 + lane;
                    k[r] = i < n ? kb[src][i] : 0u;
                    v[r] = i < n ? vb[src][i] : 0u;
                    if (ranged && j == 0 && k[r] == 0xffffffffu) k[r] = kmax1;
                }
            }
            for (int i = threadIdx.x; i < kVW * 256 / 2; i += kThreads) reinterpret_cast<uint32_t*>(&s_cnt[0][0])[i] = 0u;
            __syncthreads();
            // Stable ranks per virtual warp: warp w's rows are cut into kChains consecutive groups,
            // group h being virtual warp kChains w + h (key order), so each warp runs kChains
            // independent counter chains.  Lanes with equal digits are found with 8 ballots
            // (faster than __match_any_sync).
            constexpr int kRows = kCoopItems / kChains;
            uint32_t rank[kCoopItems];
#pragma unroll
            for (int r = 0; r < kRows; ++r) {
                unsigned peers[kChains];
                uint32_t dd[kChains], old[kChains];
                bool valid[kChains];
#pragma unroll
                for (int h = 0; h < kChains; ++h) {
                    const int rr = r + h * kRows;
                    valid[h] = wbase + rr * 32 + lane < n;
                    dd[h] = (k[rr] >> shift) & 255u;
                    unsigned pm = __ballot_sync(0xffffffffu, valid[h]);
#pragma unroll
                    for (int b = 0; b < 8; ++b) {
                        const bool bit = (dd[h] >> b) & 1u;
                        const unsigned bal = __ballot_sync(0xffffffffu, bit);
                        pm &= bit ? bal : ~bal;
                    }
                    peers[h] = pm;
                    old[h] = valid[h] ? s_cnt[kChains * warp + h][dd[h]] : 0u;
                }
                __syncwarp();
#pragma unroll
                for (int h = 0; h < kChains; ++h)
                    if (valid[h] && (peers[h] & lt) == 0u)
                        s_cnt[kChains * warp + h][dd[h]] = (uint16_t)(old[h] + __popc(peers[h]));
                __syncwarp();
#pragma unroll
                for (int h = 0; h < kChains; ++h) rank[r + h * kRows] = old[h] + __popc(peers[h] & lt);
            }
            __syncthreads();
            // thread d: tile total of digit d (published digit-major), its local start L (exclusive
            // over digits) and the local start of every virtual warp's run of d (< 4096: 16 bits)
            {
                const int d = threadIdx.x;
                uint32_t c = 0;
#pragma unroll
                for (int w = 0; w < kVW; ++w) c += s_cnt[w][d];
                counts[(size_t)d * ntiles + tile] = c;
                if (ranged && c) atomicAdd(&hist[256 * passes[j] + d], c);  // the pass histogram
                uint32_t tot;
                const uint32_t ls = block_exclusive_scan(c, &tot, s_warp);
                slot_ls(q)[d] = ls;
                uint32_t run = ls;
#pragma unroll
                for (int w = 0; w < kVW; ++w) {
                    const uint32_t cw = s_cnt[w][d];
                    s_cnt[w][d] = (uint16_t)run;
                    run += cw;
                }
            }
            __syncthreads();
            uint32_t* sk = slot_k(q);
            uint32_t* sv = slot_v(q);
#pragma unroll
            for (int r = 0; r < kCoopItems; ++r)
                if (wbase + r * 32 + lane < n) {
                    const uint32_t lp = s_cnt[kChains * warp + r / (kCoopItems / kChains)][(k[r] >> shift) & 255u] + rank[r];
                    sk[lp] = k[r];
                    sv[lp] = v[r];
                }
            __syncthreads();  // s_cnt is reused by the next owned tile
        }
        STAMP(3 + 6 * j);
        grid.sync();
        STAMP(4 + 6 * j);
        // phase B: digit rows, exclusive over tiles, plus the digit's global base (the exclusive
        // scan of the pass histogram, in s_delta until phase C reuses it).  A warp per row (a
        // CTA per row cost two barriers per row: 256 rows on one CTA took 0.4 ms at 2 K keys);
        // with few tiles a thread per row.
        if (ranged) {
            s_gh[passes[j]][threadIdx.x] = hist[256 * passes[j] + threadIdx.x];
            __syncthreads();
        }
        {
            uint32_t tot;
            const uint32_t hb = block_exclusive_scan(s_gh[passes[j]][threadIdx.x], &tot, s_warp);
            s_delta[threadIdx.x] = hb;
            __syncthreads();
        }
        if (ntiles <= 32) {
            if (blockIdx.x == 0) {
                uint32_t* row = counts + (size_t)threadIdx.x * ntiles;
                uint32_t acc = s_delta[threadIdx.x];
                for (uint32_t t0 = 0; t0 < ntiles; t0 += 8) {
                    uint32_t x[8];
#pragma unroll
                    for (int qq = 0; qq < 8; ++qq) x[qq] = t0 + qq < ntiles ? row[t0 + qq] : 0u;
#pragma unroll
                    for (int qq = 0; qq < 8; ++qq) {
                        if (t0 + qq < ntiles) row[t0 + qq] = acc;
                        acc += x[qq];
                    }
                }
            }
        } else {
            for (uint32_t d = blockIdx.x * kWarps + warp; d < 256; d += gridDim.x * kWarps) {
                uint32_t* row = counts + (size_t)d * ntiles;
                uint32_t carry = s_delta[d];
                for (uint32_t t0 = 0; t0 < ntiles; t0 += 32 * 8) {
                    uint32_t x[8], sum = 0;
#pragma unroll
                    for (int qq = 0; qq < 8; ++qq) {
                        const uint32_t t = t0 + lane * 8 + qq;
                        x[qq] = t < ntiles ? row[t] : 0u;
                        sum += x[qq];
                    }
                    const uint32_t inc = warp_incl_scan(sum, lane);
                    uint32_t acc = carry + inc - sum;
#pragma unroll
                    for (int qq = 0; qq < 8; ++qq) {
                        const uint32_t t = t0 + lane * 8 + qq;
                        if (t < ntiles) row[t] = acc;
                        acc += x[qq];
                    }
                    carry += __shfl_sync(0xffffffffu, inc, 31);
                }
            }
        }
        STAMP(5 + 6 * j);
        grid.sync();
        STAMP(6 + 6 * j);
        // phase C: global position = tile's global offset of the digit + (local position - L)
        uint32_t* kd = kb[dst];
        uint32_t* vd = vb[dst];
        for (int q = 0; q < tpc; ++q) {
            const uint32_t tile = tile_of(q);
            if (tile >= ntiles) break;
            const uint32_t tbase = tile * kCoopTile;
            const uint32_t tcount = min(n - tbase, (uint32_t)kCoopTile);
            s_delta[threadIdx.x] = counts[(size_t)threadIdx.x * ntiles + tile] - slot_ls(q)[threadIdx.x];
            __syncthreads();
            const uint32_t* sk = slot_k(q);
            const uint32_t* sv = slot_v(q);
#pragma unroll 4
            for (uint32_t i = threadIdx.x; i < tcount; i += kThreads) {
                const uint32_t key = sk[i];
                const uint32_t pos = s_delta[(key >> shift) & 255u] + i;
                kd[pos] = key;
                vd[pos] = sv[i];
            }
            __syncthreads();  // s_delta is reused by the next owned tile
        }
        src = dst;
        STAMP(7 + 6 * j);
        // the next pass reads what every CTA scattered; after the last pass nothing in this kernel
        // does (hist / key_range were last read before this pass's phase-C barrier)
        if (j + 1 < m) grid.sync();
        STAMP(8 + 6 * j);
    }
    // hist was last read before the first pass's first grid barrier: re-zero it for the next sort
    // (the caller allocates it zeroed; no memset launch per sort)
    if (blockIdx.x == 0)
        for (int i = threadIdx.x; i < 4 * 256; i += kThreads) hist[i] = 0u;
    if (ranged && blockIdx.x == 0 && threadIdx.x < 2) key_range[threadIdx.x] = 0u;  // zero at rest
#ifdef SPLAT_SORT_STAMPS
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        ns = 3 + 6 * m;
        printf("SORTSTAMPS m=%d", m);
        for (int i = 1; i < ns; ++i) printf(" %llu", stamps[i] - stamps[i - 1]);
        printf("\n");
    }
#endif
}

}  // namespace

size_t scan_temp_words(uint64_t n) {
    const uint64_t nt = (n + kTile - 1) / kTile;
    return (size_t)(2 * (nt + 1) + 2);  // u64 counter + u64 status per tile, in 32-bit words
}

size_t radix_hist_words(uint64_t n, int bits) {
    (void)bits;
    const uint64_t nt = (n + kSortTile - 1) / kSortTile;
    return (size_t)(4 * 512 + 4 + 4 * nt * 512);  // hist [4][512] + counters [4] + status [4][nt][512]
}

cudaError_t exclusive_scan_u32(LaunchCtx& lc, const uint32_t* in, uint32_t* out, uint64_t n, uint32_t* tmp,
                               uint32_t* total_dev) {
    return exclusive_scan_gather_u32(lc, in, nullptr, out, n, tmp, total_dev);
}

cudaError_t exclusive_scan_u32_zeroed(LaunchCtx& lc, const uint32_t* in, uint32_t* out, uint64_t n, uint32_t* tmp) {
    if (n == 0) return cudaSuccess;
    const uint64_t nt = (n + kTile - 1) / kTile;
    LaunchScope s(lc, "scan");
    const cudaError_t e = launch_pdl(lc.stream, scan_lookback_kernel<false, true>, dim3((unsigned)nt), dim3(kThreads), 0,
                                     in, (const uint32_t*)nullptr, out, n, reinterpret_cast<uint64_t*>(tmp),
                                     (uint32_t*)nullptr);
    lc.count++;
    return e;
}

cudaError_t exclusive_scan_gather_u32(LaunchCtx& lc, const uint32_t* in, const uint32_t* idx, uint32_t* out,
                                      uint64_t n, uint32_t* tmp, uint32_t* total_dev) {
    if (n == 0) {
        if (total_dev) return cudaMemsetAsync(total_dev, 0, sizeof(uint32_t), lc.stream);
        return cudaSuccess;
    }
    const uint64_t nt = (n + kTile - 1) / kTile;
    cudaError_t e = cudaMemsetAsync(tmp, 0, 8 * (nt + 1), lc.stream);
    if (e != cudaSuccess) return e;
    LaunchScope s(lc, "scan");
    uint64_t* t64 = reinterpret_cast<uint64_t*>(tmp);
    if (idx)
        scan_lookback_kernel<true><<<(unsigned)nt, kThreads, 0, lc.stream>>>(in, idx, out, n, t64, total_dev);
    else
        scan_lookback_kernel<false><<<(unsigned)nt, kThreads, 0, lc.stream>>>(in, idx, out, n, t64, total_dev);
    lc.count++;
    return cudaGetLastError();
}

cudaError_t radix_sort_pairs(LaunchCtx& lc, uint32_t* keys, uint32_t* vals, uint32_t* keys_alt, uint32_t* vals_alt,
                             uint64_t n, int begin_bit, int end_bit, uint32_t* hist, uint32_t* scan_tmp,
                             bool* result_in_alt) {
    *result_in_alt = false;
    if (n == 0 || end_bit <= begin_bit) return cudaSuccess;
    const int total = end_bit - begin_bit;
    const int passes = total <= 9 ? 1 : (total + 7) / 8;  // one 9-bit pass for small key ranges
    const int bits = (total + passes - 1) / passes;       // balanced digits, <= 9
    const uint64_t nt = (n + kSortTile - 1) / kSortTile;
    uint32_t* counters = hist + 4 * 512;
    uint32_t* status = counters + 4;
    cudaError_t e = cudaMemsetAsync(hist, 0, 4 * (size_t)(4 * 512 + 4 + (size_t)passes * nt * 512), lc.stream);
    if (e != cudaSuccess) return e;
    {
        LaunchScope s(lc, "radix_histogram");
        const unsigned grid =
            (unsigned)std::min<uint64_t>((n + kThreads * 8 - 1) / (kThreads * 8), (uint64_t)lc.num_sms * 4);
        radix_histogram_kernel<<<grid, kThreads, 0, lc.stream>>>(keys, n, begin_bit, bits, passes, hist);
        lc.count++;
    }
    uint32_t *ki = keys, *vi = vals, *ko = keys_alt, *vo = vals_alt;
    for (int p = 0; p < passes; ++p) {
        const int shift = begin_bit + p * bits;
        const uint32_t* h = hist + 512 * p;
        uint32_t* st = status + (size_t)p * nt * 512;
        LaunchScope s(lc, "radix_onesweep");
        switch (bits) {
            case 1: launch_onesweep<1>(lc, ki, vi, ko, vo, (uint32_t)n, shift, h, st, counters + p, scan_tmp); break;
            case 2: launch_onesweep<2>(lc, ki, vi, ko, vo, (uint32_t)n, shift, h, st, counters + p, scan_tmp); break;
            case 3: launch_onesweep<3>(lc, ki, vi, ko, vo, (uint32_t)n, shift, h, st, counters + p, scan_tmp); break;
            case 4: launch_onesweep<4>(lc, ki, vi, ko, vo, (uint32_t)n, shift, h, st, counters + p, scan_tmp); break;
            case 5: launch_onesweep<5>(lc, ki, vi, ko, vo, (uint32_t)n, shift, h, st, counters + p, scan_tmp); break;
            case 6: launch_onesweep<6>(lc, ki, vi, ko, vo, (uint32_t)n, shift, h, st, counters + p, scan_tmp); break;
            case 7: launch_onesweep<7>(lc, ki, vi, ko, vo, (uint32_t)n, shift, h, st, counters + p, scan_tmp); break;
            case 8: launch_onesweep<8>(lc, ki, vi, ko, vo, (uint32_t)n, shift, h, st, counters + p, scan_tmp); break;
            default: launch_onesweep<9>(lc, ki, vi, ko, vo, (uint32_t)n, shift, h, st, counters + p, scan_tmp); break;
        }
        lc.count++;
        std::swap(ki, ko);
        std::swap(vi, vo);
        *result_in_alt = !*result_in_alt;
    }
    return cudaGetLastError();
}

size_t radix_coop_count_words(uint64_t n) {
    const uint64_t nt = (n + kCoopTile - 1) / kCoopTile;
    return (size_t)(4 * 256 + 256 * nt + 16);
}

// Whole 32-bit LSD sort of (keys, vals) as one cooperative kernel; the result always lands in
// (keys_alt, vals_alt).  Returns cudaErrorCooperativeLaunchTooLarge (nothing launched) when the
// tiles do not fit in one resident wave; the caller falls back to radix_sort_pairs.
cudaError_t radix_sort_coop(LaunchCtx& lc, uint32_t* keys, uint32_t* vals, uint32_t* keys_alt, uint32_t* vals_alt,
                            uint32_t* keys_tmp, uint32_t* vals_tmp, uint64_t n, uint32_t* work, uint32_t* key_range) {
    if (n == 0) return cudaSuccess;
    if (n >= (1ull << 31)) return cudaErrorCooperativeLaunchTooLarge;
    const uint64_t nt = (n + kCoopTile - 1) / kCoopTile;
    // tiles per CTA: the fewest that fit the tiles into one resident wave (each owned tile keeps
    // 33 KB of shared memory between its rank phase and its scatter; one tile: static memory)
    static int per_sm_of[kCoopMaxTpc + 1] = {};
    int tpc = 0, grid = 0;
    for (int t = 1; t <= kCoopMaxTpc; ++t) {
        const size_t smem = t == 1 ? 0 : coop_dyn_smem(t);
        if (!per_sm_of[t]) {
            cudaError_t e = cudaSuccess;
            if (t == 1) {
                e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_of[t], radix_coop_kernel<1>, kThreads, 0);
            } else {
                if (smem > 48 * 1024)
                    e = cudaFuncSetAttribute(radix_coop_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                if (e == cudaSuccess)
                    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_of[t], radix_coop_kernel<0>, kThreads, smem);
            }
            if (e != cudaSuccess) {
                cudaGetLastError();
                per_sm_of[t] = -1;
            }
        }
        if (per_sm_of[t] <= 0) continue;
        const uint64_t cap = (uint64_t)lc.num_sms * per_sm_of[t];
        if (cap * t >= nt) {
            tpc = t;
            grid = (int)((nt + t - 1) / t);
            break;
        }
    }
    if (!tpc) return cudaErrorCooperativeLaunchTooLarge;
    const size_t smem = tpc == 1 ? 0 : coop_dyn_smem(tpc);
    if (smem > 48 * 1024) cudaFuncSetAttribute(radix_coop_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    uint32_t* hist = work;  // zero at rest: allocated zeroed, re-zeroed by the kernel
    uint32_t* counts = work + 4 * 256;
    uint32_t nn = (uint32_t)n;
    void* args[] = {&keys, &vals, &keys_alt, &vals_alt, &keys_tmp, &vals_tmp, &nn, &hist, &counts, &tpc, &key_range};
    LaunchScope s(lc, "radix_sort");
    const void* fn = tpc == 1 ? (const void*)radix_coop_kernel<1> : (const void*)radix_coop_kernel<0>;
    const cudaError_t e = cudaLaunchCooperativeKernel(fn, dim3((unsigned)grid), dim3(kThreads), args, smem, lc.stream);
    lc.count++;
    return e;
}

}  // namespace splat_b200
