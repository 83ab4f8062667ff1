// sort.cu — device-wide exclusive scan and stable LSD radix sort (hand-written, sm_100a).
//
// Replaces the reference's std::sort of ProjectedGaussian by (depth_mean, index)
// (rasterizer.cpp:85-88) and the push_back binning of detail::bin_tiles
// (rasterizer.hpp:156-174).  The per-tile lists come out of two stable sorts:
//   1. the N depth keys (IEEE bits of depth_mean > 0, monotone as uint32; culled Gaussians
//      carry 0xFFFFFFFF) with Gaussian ids as values, in index order  -> (depth, index) order;
//   2. the P (tile id, Gaussian id) pairs, emitted in that depth order, by tile id only.
// Stability of both passes reproduces the reference lists exactly.
//
// Radix pass = upsweep (per-CTA digit histogram, digit-major) + exclusive scan of the histogram
// + downsweep (warp-synchronous stable ranking with __match_any_sync, scatter).  4096 keys per
// CTA (256 threads x 16), digits of up to 8 bits.
#include <cstdint>

#include "common.cuh"
#include "internal.h"

namespace splat_b200 {

namespace {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 16;
constexpr int kScanTile = kScanThreads * kScanItems;  // 4096

constexpr int kSortThreads = 256;
constexpr int kSortItems = 16;
constexpr int kSortTile = kSortThreads * kSortItems;  // 4096
constexpr int kSortWarps = kSortThreads / 32;

__device__ __forceinline__ uint32_t warp_inclusive_scan(uint32_t v, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
    }
    return v;
}

// Block-wide exclusive scan of one value per thread; returns the block total in *total.
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* total) {
    __shared__ uint32_t s_warp[kScanThreads / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t inc = warp_inclusive_scan(v, lane);
    if (lane == 31) s_warp[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = lane < kScanThreads / 32 ? s_warp[lane] : 0u;
        w = warp_inclusive_scan(w, lane);
        if (lane < kScanThreads / 32) s_warp[lane] = w;
    }
    __syncthreads();
    const uint32_t warp_off = warp > 0 ? s_warp[warp - 1] : 0u;
    *total = s_warp[kScanThreads / 32 - 1];
    __syncthreads();
    return warp_off + inc - v;
}

__global__ void __launch_bounds__(kScanThreads) scan_reduce_kernel(const uint32_t* __restrict__ in,
                                                                    uint32_t n,
                                                                    uint32_t* __restrict__ block_sums) {
    const uint64_t base = (uint64_t)blockIdx.x * kScanTile;
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const uint64_t i = base + (uint64_t)k * kScanThreads + threadIdx.x;
        if (i < n) s += in[i];
    }
    uint32_t total;
    block_exclusive_scan(s, &total);
    if (threadIdx.x == 0) block_sums[blockIdx.x] = total;
}

// Single CTA: exclusive scan of the block sums in place; writes the grand total.
__global__ void __launch_bounds__(kScanThreads) scan_sums_kernel(uint32_t* __restrict__ sums,
                                                                  uint32_t nblocks,
                                                                  uint32_t* __restrict__ total_out) {
    uint32_t carry = 0;
    for (uint32_t base = 0; base < nblocks; base += kScanThreads) {
        const uint32_t i = base + threadIdx.x;
        const uint32_t v = i < nblocks ? sums[i] : 0u;
        uint32_t total;
        const uint32_t ex = block_exclusive_scan(v, &total);
        if (i < nblocks) sums[i] = carry + ex;
        carry += total;
    }
    if (threadIdx.x == 0 && total_out) *total_out = carry;
}

// Each thread owns kScanItems consecutive elements (blocked arrangement) for a local serial
// scan, then a block scan of the thread totals.
__global__ void __launch_bounds__(kScanThreads) scan_down_kernel(const uint32_t* __restrict__ in,
                                                                  uint32_t* __restrict__ out, uint32_t n,
                                                                  const uint32_t* __restrict__ block_offs) {
    __shared__ uint32_t s_data[kScanTile];
    const uint64_t base = (uint64_t)blockIdx.x * kScanTile;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const int li = k * kScanThreads + threadIdx.x;
        const uint64_t i = base + li;
        s_data[li] = i < n ? in[i] : 0u;
    }
    __syncthreads();
    uint32_t local[kScanItems];
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        local[k] = s;
        s += s_data[threadIdx.x * kScanItems + k];
    }
    uint32_t total;
    const uint32_t ex = block_exclusive_scan(s, &total) + block_offs[blockIdx.x];
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) s_data[threadIdx.x * kScanItems + k] = ex + local[k];
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const int li = k * kScanThreads + threadIdx.x;
        const uint64_t i = base + li;
        if (i < n) out[i] = s_data[li];
    }
}

template <int BITS>
__global__ void __launch_bounds__(kSortThreads) radix_upsweep_kernel(const uint32_t* __restrict__ keys,
                                                                      uint32_t n, int shift,
                                                                      uint32_t* __restrict__ hist,
                                                                      uint32_t nblocks) {
    constexpr int BINS = 1 << BITS;
    __shared__ uint32_t s_hist[kSortWarps][BINS];
    for (int i = threadIdx.x; i < kSortWarps * BINS; i += kSortThreads) (&s_hist[0][0])[i] = 0u;
    __syncthreads();
    const int warp = threadIdx.x >> 5;
    const uint64_t base = (uint64_t)blockIdx.x * kSortTile;
#pragma unroll 4
    for (int k = 0; k < kSortItems; ++k) {
        const uint64_t i = base + (uint64_t)k * kSortThreads + threadIdx.x;
        if (i < n) atomicAdd(&s_hist[warp][(keys[i] >> shift) & (BINS - 1)], 1u);
    }
    __syncthreads();
    for (int d = threadIdx.x; d < BINS; d += kSortThreads) {
        uint32_t s = 0;
#pragma unroll
        for (int w = 0; w < kSortWarps; ++w) s += s_hist[w][d];
        hist[(uint64_t)d * nblocks + blockIdx.x] = s;
    }
}

template <int BITS>
__global__ void __launch_bounds__(kSortThreads) radix_downsweep_kernel(
    const uint32_t* __restrict__ keys_in, const uint32_t* __restrict__ vals_in,
    uint32_t* __restrict__ keys_out, uint32_t* __restrict__ vals_out, uint32_t n, int shift,
    const uint32_t* __restrict__ offs, uint32_t nblocks) {
    constexpr int BINS = 1 << BITS;
    constexpr int PER_WARP = kSortTile / kSortWarps;  // 512 consecutive keys per warp
    __shared__ uint32_t s_cnt[kSortWarps][BINS];
    for (int i = threadIdx.x; i < kSortWarps * BINS; i += kSortThreads) (&s_cnt[0][0])[i] = 0u;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t wbase = (uint64_t)blockIdx.x * kSortTile + (uint64_t)warp * PER_WARP;
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
        // invalid lanes get unique non-digit labels so they form singleton groups
        const uint32_t label = valid ? d : (0x80000000u | (uint32_t)lane);
        const unsigned peers = __match_any_sync(0xffffffffu, label);
        const uint32_t old = valid ? s_cnt[warp][d] : 0u;
        __syncwarp();
        if (valid && (peers & lt) == 0u) s_cnt[warp][d] = old + __popc(peers);
        __syncwarp();
        rank[r] = old + __popc(peers & lt);
    }
    __syncthreads();
    for (int d = threadIdx.x; d < BINS; d += kSortThreads) {
        uint32_t run = offs[(uint64_t)d * nblocks + blockIdx.x];
#pragma unroll
        for (int w = 0; w < kSortWarps; ++w) {
            const uint32_t c = s_cnt[w][d];
            s_cnt[w][d] = run;
            run += c;
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

template <int BITS>
cudaError_t radix_pass(LaunchCtx& lc, const uint32_t* ki, const uint32_t* vi, uint32_t* ko, uint32_t* vo,
                       uint32_t n, int shift, uint32_t* hist, uint32_t* scan_tmp) {
    const uint32_t nblocks = (n + kSortTile - 1) / kSortTile;
    constexpr uint32_t BINS = 1u << BITS;
    {
        LaunchScope ls_(lc, "radix_upsweep");
        radix_upsweep_kernel<BITS><<<nblocks, kSortThreads, 0, lc.stream>>>(ki, n, shift, hist, nblocks);
    }
    lc.count++;
    cudaError_t e = exclusive_scan_u32(lc, hist, hist, BINS * nblocks, scan_tmp, nullptr);
    if (e != cudaSuccess) return e;
    {
        LaunchScope ls_(lc, "radix_downsweep");
        radix_downsweep_kernel<BITS><<<nblocks, kSortThreads, 0, lc.stream>>>(ki, vi, ko, vo, n, shift, hist, nblocks);
    }
    lc.count++;
    return cudaGetLastError();
}

}  // namespace

size_t scan_temp_words(uint64_t n) {
    const uint64_t nb = (n + kScanTile - 1) / kScanTile;
    return (size_t)nb + 1;
}

size_t radix_hist_words(uint64_t n, int bits) {
    const uint64_t nb = (n + kSortTile - 1) / kSortTile;
    return (size_t)(nb << bits);
}

cudaError_t exclusive_scan_u32(LaunchCtx& lc, const uint32_t* in, uint32_t* out, uint64_t n,
                               uint32_t* tmp, uint32_t* total_dev) {
    if (n == 0) {
        if (total_dev) return cudaMemsetAsync(total_dev, 0, sizeof(uint32_t), lc.stream);
        return cudaSuccess;
    }
    const uint32_t nb = (uint32_t)((n + kScanTile - 1) / kScanTile);
    {
        LaunchScope ls_(lc, "scan_reduce");
        scan_reduce_kernel<<<nb, kScanThreads, 0, lc.stream>>>(in, (uint32_t)n, tmp);
    }
    {
        LaunchScope ls_(lc, "scan_sums");
        scan_sums_kernel<<<1, kScanThreads, 0, lc.stream>>>(tmp, nb, total_dev);
    }
    {
        LaunchScope ls_(lc, "scan_down");
        scan_down_kernel<<<nb, kScanThreads, 0, lc.stream>>>(in, out, (uint32_t)n, tmp);
    }
    lc.count += 3;
    return cudaGetLastError();
}

cudaError_t radix_sort_pairs(LaunchCtx& lc, uint32_t* keys, uint32_t* vals, uint32_t* keys_alt,
                             uint32_t* vals_alt, uint64_t n, int begin_bit, int end_bit, uint32_t* hist,
                             uint32_t* scan_tmp, bool* result_in_alt) {
    *result_in_alt = false;
    if (n == 0 || end_bit <= begin_bit) return cudaSuccess;
    uint32_t *ki = keys, *vi = vals, *ko = keys_alt, *vo = vals_alt;
    const int total = end_bit - begin_bit;
    const int passes = (total + 7) / 8;
    const int bits = (total + passes - 1) / passes;  // balanced digits, <= 8
    int shift = begin_bit;
    for (int p = 0; p < passes; ++p) {
        const int b = (shift + bits <= end_bit) ? bits : end_bit - shift;
        cudaError_t e;
        switch (b) {
            case 1: e = radix_pass<1>(lc, ki, vi, ko, vo, (uint32_t)n, shift, hist, scan_tmp); break;
            case 2: e = radix_pass<2>(lc, ki, vi, ko, vo, (uint32_t)n, shift, hist, scan_tmp); break;
            case 3: e = radix_pass<3>(lc, ki, vi, ko, vo, (uint32_t)n, shift, hist, scan_tmp); break;
            case 4: e = radix_pass<4>(lc, ki, vi, ko, vo, (uint32_t)n, shift, hist, scan_tmp); break;
            case 5: e = radix_pass<5>(lc, ki, vi, ko, vo, (uint32_t)n, shift, hist, scan_tmp); break;
            case 6: e = radix_pass<6>(lc, ki, vi, ko, vo, (uint32_t)n, shift, hist, scan_tmp); break;
            case 7: e = radix_pass<7>(lc, ki, vi, ko, vo, (uint32_t)n, shift, hist, scan_tmp); break;
            default: e = radix_pass<8>(lc, ki, vi, ko, vo, (uint32_t)n, shift, hist, scan_tmp); break;
        }
        if (e != cudaSuccess) return e;
        std::swap(ki, ko);
        std::swap(vi, vo);
        *result_in_alt = !*result_in_alt;
        shift += b;
    }
    return cudaSuccess;
}

}  // namespace splat_b200
