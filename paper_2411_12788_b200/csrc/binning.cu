// binning.cu — per-tile lists (detail::bin_tiles, rasterizer.hpp:156-174) built without sorting
// the P (tile, Gaussian) pairs.
//
// The reference pushes every depth-sorted Gaussian into each tile its pixel rect touches, so a
// tile's list is "the Gaussians covering it, in (depth, index) order".  A stable radix sort of P
// pairs by tile reproduces that but moves ~16 B x P x 2 passes.  Instead:
//   1-2. supertile lists (a supertile is 4 x 4 tiles, so Ps ~ P/6), stable in depth order, by a
//      chunked counting sort with no pair array and no radix pass: the depth-ordered survivors
//      are cut into chunks of kStChunk; one warp per chunk counts its entries per supertile
//      (st_chunk_kernel<false>), an exclusive scan over the counts laid out supertile-major /
//      chunk-minor gives every (supertile, chunk) its output offset, and the same warp re-walks
//      the chunk writing each Gaussian id at offset + (rank among the chunk's earlier entries of
//      that supertile), ranks from __match_any_sync over the flattened (Gaussian, supertile)
//      entries.  (Fallback for > kStMaxSmem supertiles: emit pairs + stable radix sort.)
//   3. split every supertile list into segments of kSeg entries; a count pass gives, per
//      (tile, segment), how many entries of the segment cover the tile; an exclusive scan of those
//      counts laid out tile-major / segment-minor gives every (tile, segment) its output offset;
//   4. an emit pass re-walks each segment in order and writes each Gaussian id into the lists of
//      the tiles it covers at offset + (rank among the segment's earlier entries covering that
//      tile), the rank coming from one warp ballot per tile of the supertile.
// Stability at every step makes each list exactly the reference's, and only P x 4 B are written.
#include <cstdint>

#include "common.cuh"
#include "internal.h"

namespace splat_b200 {

namespace {

constexpr int kST = 4;              // supertile side in tiles
constexpr int kSTT = kST * kST;     // tiles per supertile
constexpr int kSeg = 1024;          // entries per segment of a supertile list
constexpr int kBinThreads = 256;
constexpr int kStChunk = 128;       // depth-ordered survivors per chunk of the supertile pass
constexpr int kStMaxSmem = 6144;    // supertiles the chunked pass keeps in shared memory

struct TileRect {
    int tx0, tx1, ty0, ty1;  // inclusive tile range of a Gaussian's pixel rect
};

__device__ __forceinline__ TileRect tile_rect(uint2 r, int ts) {
    TileRect t;
    t.tx0 = (int)(r.x & 0xffffu) / ts;
    t.tx1 = ((int)(r.x >> 16) - 1) / ts;
    t.ty0 = (int)(r.y & 0xffffu) / ts;
    t.ty1 = ((int)(r.y >> 16) - 1) / ts;
    return t;
}

// (supertile, Gaussian) pairs in depth order: one thread per survivor.
__global__ void __launch_bounds__(256) emit_st_pairs_kernel(const uint32_t* __restrict__ order,
                                                           const uint32_t* __restrict__ offsets,
                                                           const uint2* __restrict__ rect_ref, int ts, int st_x,
                                                           int n_surv, uint32_t* __restrict__ st_key,
                                                           uint32_t* __restrict__ st_gauss) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n_surv) return;
    const uint32_t gid = order[r];
    uint32_t o = offsets[r];
    const TileRect t = tile_rect(rect_ref[gid], ts);
    for (int sy = t.ty0 / kST; sy <= t.ty1 / kST; ++sy)
        for (int sx = t.tx0 / kST; sx <= t.tx1 / kST; ++sx) {
            st_key[o] = (uint32_t)(sy * st_x + sx);
            st_gauss[o] = gid;
            ++o;
        }
}

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
    }
    return v;
}

// Supertile pass over one chunk of depth-ordered survivors, one warp per chunk.  The chunk's
// Gaussians are flattened, 32 at a time, into (Gaussian, supertile) entries in (depth, raster)
// order; every window of 32 entries is ranked per supertile with __match_any_sync, and a
// per-supertile running count in shared memory carries the rank across windows.
//   EMIT = false: cnt[st * nchunks + c] = entries of chunk c in supertile st.
//   EMIT = true:  cnt holds the exclusive scan of those counts; writes st_gauss[offset + rank].
template <bool EMIT>
__global__ void __launch_bounds__(32) st_chunk_kernel(const uint32_t* __restrict__ order,
                                                      const uint2* __restrict__ rect_ref, int n_surv, int ts,
                                                      int st_x, int n_st, int nchunks, uint32_t* __restrict__ cnt,
                                                      uint32_t* __restrict__ st_gauss) {
    extern __shared__ uint32_t s_run[];  // [n_st]
    const int c = blockIdx.x, lane = threadIdx.x;
    for (int st = lane; st < n_st; st += 32) s_run[st] = EMIT ? cnt[(size_t)st * nchunks + c] : 0u;
    if (!EMIT && c == 0 && lane == 0) cnt[(size_t)n_st * nchunks] = 0u;  // scan slot of the total
    __syncwarp();
    const int g0 = c * kStChunk, g1 = min(g0 + kStChunk, n_surv);
    const unsigned lt = lanemask_lt();
    // the whole chunk's ids and rects are loaded up front (two dependent round trips per chunk)
    constexpr int kPer = kStChunk / 32;
    uint32_t gids[kPer];
    uint2 rects[kPer];
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
        const int r = g0 + k * 32 + lane;
        gids[k] = r < g1 ? order[r] : 0u;
    }
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
        const int r = g0 + k * 32 + lane;
        rects[k] = r < g1 ? rect_ref[gids[k]] : make_uint2(0u, 0u);
    }
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
        const int r = g0 + k * 32 + lane;
        const uint32_t gid = gids[k];
        int sx0 = 0, sy0 = 0, w = 1, m = 0;
        if (r < g1) {
            const TileRect t = tile_rect(rects[k], ts);
            sx0 = t.tx0 / kST;
            sy0 = t.ty0 / kST;
            w = t.tx1 / kST - sx0 + 1;
            m = w * (t.ty1 / kST - sy0 + 1);
        }
        if (!EMIT) {  // counts are order-free: shared-memory atomics per entry
            for (int q = 0; q < m; ++q) atomicAdd(&s_run[(sy0 + q / w) * st_x + sx0 + q % w], 1u);
            continue;
        }
        if (!__any_sync(0xffffffffu, m > 0)) continue;
        const int inc = (int)warp_incl_scan((uint32_t)m, lane);
        const int off = inc - m;
        const int total = __shfl_sync(0xffffffffu, inc, 31);
        for (int e0 = 0; e0 < total; e0 += 32) {
            const int e = e0 + lane;
            const bool valid = e < total;
            int owner = 0;  // last lane whose entries start at or before e
#pragma unroll
            for (int step = 16; step > 0; step >>= 1)
                if (__shfl_sync(0xffffffffu, off, owner + step) <= e) owner += step;
            const int q = e - __shfl_sync(0xffffffffu, off, owner);
            const int ow = __shfl_sync(0xffffffffu, w, owner);
            const int st = (__shfl_sync(0xffffffffu, sy0, owner) + q / ow) * st_x + __shfl_sync(0xffffffffu, sx0, owner) +
                           q % ow;
            const uint32_t ogid = __shfl_sync(0xffffffffu, gid, owner);
            const unsigned grp = __match_any_sync(0xffffffffu, valid ? st : -1);
            const int leader = __ffs(grp) - 1;
            uint32_t base = 0;
            if (valid && lane == leader) {
                base = s_run[st];
                s_run[st] = base + (uint32_t)__popc(grp);
            }
            base = __shfl_sync(0xffffffffu, base, leader);
            if (valid) st_gauss[base + __popc(grp & lt)] = ogid;
            __syncwarp();
        }
    }
    if (!EMIT) {
        __syncwarp();
        for (int st = lane; st < n_st; st += 32) cnt[(size_t)st * nchunks + c] = s_run[st];
    }
}


// Block-wide exclusive scan of `n` values produced by `val(i)`, written to out[0..n] (out[n] =
// total).  One CTA of kBinThreads threads.
// Block-wide exclusive scan of `n` values produced by `val(i)`, written to out[0..n] (out[n] =
// total).  One CTA of T threads.
template <int T, typename F>
__device__ void cta_scan(int n, F val, uint32_t* __restrict__ out, uint32_t* s_warp) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint32_t carry = 0;
    for (int base = 0; base < n; base += T) {
        const int i = base + tid;
        const uint32_t v = i < n ? val(i) : 0u;
        const uint32_t inc = warp_incl_scan(v, lane);
        if (lane == 31) s_warp[warp] = inc;
        __syncthreads();
        uint32_t off = 0, tot = 0;
#pragma unroll 8
        for (int w = 0; w < T / 32; ++w) {
            const uint32_t c = s_warp[w];
            off += w < warp ? c : 0u;
            tot += c;
        }
        if (i < n) out[i] = carry + off + inc - v;
        carry += tot;
        __syncthreads();
    }
    if (tid == 0) out[n] = carry;
}

constexpr int kSetupThreads = 1024;
constexpr int kSetupSmemSt = 16384;  // supertiles whose segment counts fit shared memory

// One CTA: (chunked path) supertile ranges from the scanned (supertile, chunk) counts; segment
// counts per supertile; seg_start = their exclusive scan; seg_st[s] = supertile of segment s;
// tile_base[t] = first slot of tile t in the (tile, segment) count array.
__global__ void __launch_bounds__(kSetupThreads) seg_setup_kernel(const uint32_t* __restrict__ st_cnt, int nchunks,
                                                                 uint32_t* __restrict__ st_ranges, int n_st,
                                                                 int tiles_x, int tiles_y, int st_x,
                                                                 uint32_t* __restrict__ seg_start,
                                                                 uint32_t* __restrict__ seg_st,
                                                                 uint32_t* __restrict__ tile_base) {
    extern __shared__ uint32_t s_nseg[];  // [n_st] when n_st <= kSetupSmemSt
    __shared__ uint32_t s_warp[kSetupThreads / 32];
    const bool in_smem = n_st <= kSetupSmemSt;
    for (int st = threadIdx.x; st < n_st; st += kSetupThreads) {
        uint32_t lo, hi;
        if (st_cnt) {
            lo = st_cnt[(size_t)st * nchunks];
            hi = st_cnt[(size_t)(st + 1) * nchunks];
            st_ranges[2 * st] = lo;
            st_ranges[2 * st + 1] = hi;
        } else {
            lo = st_ranges[2 * st];
            hi = st_ranges[2 * st + 1];
        }
        if (in_smem) s_nseg[st] = (hi - lo + kSeg - 1) / kSeg;
    }
    __syncthreads();
    auto nseg = [&](int st) {
        if (in_smem) return s_nseg[st];
        return (st_ranges[2 * st + 1] - st_ranges[2 * st] + kSeg - 1) / kSeg;
    };
    cta_scan<kSetupThreads>(n_st, nseg, seg_start, s_warp);
    __syncthreads();
    for (int st = threadIdx.x; st < n_st; st += kSetupThreads)
        for (uint32_t q = seg_start[st]; q < seg_start[st + 1]; ++q) seg_st[q] = (uint32_t)st;
    cta_scan<kSetupThreads>(tiles_x * tiles_y,
                            [&](int t) {
                                const int tx = t % tiles_x, ty = t / tiles_x;
                                return nseg((ty / kST) * st_x + tx / kST);
                            },
                            tile_base, s_warp);
}

// Count (EMIT = false) or emit (EMIT = true) pass over one segment of one supertile list.  The
// segment is walked in chunks of kBinThreads entries; per local tile f, a warp ballot gives each
// entry its rank among the chunk's entries covering f.  Emitted ids are staged per tile in shared
// memory and written out as contiguous runs (coalesced), since a tile's entries of one chunk are
// consecutive in its list.
template <bool EMIT>
__global__ void __launch_bounds__(kBinThreads) bin_segments_kernel(
    const uint32_t* __restrict__ st_ranges, const uint32_t* __restrict__ seg_start, int n_st,
    const uint32_t* __restrict__ tile_base, const uint32_t* __restrict__ st_gauss, const uint2* __restrict__ rect_ref,
    int ts, int tiles_x, int tiles_y, int st_x, uint32_t* __restrict__ slots, uint32_t* __restrict__ pair_gauss) {
    constexpr int kWarpsB = kBinThreads / 32;
    __shared__ uint32_t s_wc[kWarpsB][kSTT];   // per-warp counts, then exclusive prefixes over warps
    __shared__ uint32_t s_tot[kSTT + 1];       // chunk totals per tile, then exclusive prefix over tiles
    __shared__ uint32_t s_run[kSTT];
    __shared__ uint32_t s_base[kSTT];
    __shared__ uint32_t s_out[EMIT ? kSTT * kBinThreads : 1];
    const int b = blockIdx.x;
    if (b >= (int)seg_start[n_st]) return;
    const int st = (int)seg_start[n_st + 1 + b];  // seg_st (seg_setup)
    const int seg = b - (int)seg_start[st];
    const uint32_t st_end = st_ranges[2 * st + 1];
    const uint32_t lo = st_ranges[2 * st] + (uint32_t)seg * kSeg;
    const uint32_t hi = min(lo + (uint32_t)kSeg, st_end);
    const int tx_base = (st % st_x) * kST, ty_base = (st / st_x) * kST;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid < kSTT) {
        s_run[tid] = 0;
        if (EMIT) {
            const int tx = tx_base + (tid % kST), ty = ty_base + (tid / kST);
            s_base[tid] = (tx < tiles_x && ty < tiles_y) ? slots[tile_base[ty * tiles_x + tx] + seg] : 0u;
        }
    }
    __syncthreads();
    const unsigned lt = lanemask_lt();
    for (uint32_t c = lo; c < hi; c += kBinThreads) {
        const uint32_t e = c + tid;
        uint32_t gid = 0, cover = 0;
        if (e < hi) {
            gid = st_gauss[e];
            const TileRect t = tile_rect(rect_ref[gid], ts);
            const int lx0 = max(t.tx0 - tx_base, 0), lx1 = min(t.tx1 - tx_base, kST - 1);
            const int ly0 = max(t.ty0 - ty_base, 0), ly1 = min(t.ty1 - ty_base, kST - 1);
            const uint32_t row = ((1u << (lx1 + 1)) - 1u) & ~((1u << lx0) - 1u);
            for (int ly = ly0; ly <= ly1; ++ly) cover |= row << (ly * kST);
        }
        uint32_t rank[kSTT];
#pragma unroll
        for (int f = 0; f < kSTT; ++f) {
            const unsigned m = __ballot_sync(0xffffffffu, (cover >> f) & 1u);
            rank[f] = __popc(m & lt);
            if (lane == 0) s_wc[warp][f] = __popc(m);
        }
        __syncthreads();
        if (tid < kSTT) {  // exclusive prefix over warps per tile; chunk total per tile
            uint32_t run = 0;
#pragma unroll
            for (int w = 0; w < kWarpsB; ++w) {
                const uint32_t cw = s_wc[w][tid];
                s_wc[w][tid] = run;
                run += cw;
            }
            s_tot[tid] = run;
        }
        __syncthreads();
        if (EMIT) {
            if (cover) {
#pragma unroll
                for (int f = 0; f < kSTT; ++f)
                    if ((cover >> f) & 1u) s_out[f * kBinThreads + s_wc[warp][f] + rank[f]] = gid;
            }
            __syncthreads();
            // tile f's entries of this chunk are consecutive in its list: warp w copies tiles w, w + 8
#pragma unroll
            for (int f = warp; f < kSTT; f += kWarpsB) {
                const uint32_t tot = s_tot[f];
                uint32_t* dst = pair_gauss + s_base[f] + s_run[f];
                for (uint32_t i = lane; i < tot; i += 32) dst[i] = s_out[f * kBinThreads + i];
            }
            __syncthreads();
            if (tid < kSTT) s_run[tid] += s_tot[tid];
        } else {
            if (tid < kSTT) s_run[tid] += s_tot[tid];
        }
        __syncthreads();
    }
    if (!EMIT && tid < kSTT) {
        const int tx = tx_base + (tid % kST), ty = ty_base + (tid / kST);
        if (tx < tiles_x && ty < tiles_y) slots[tile_base[ty * tiles_x + tx] + seg] = s_run[tid];
    }
}

// ranges[t] = [scanned[tile_base[t]], scanned[tile_base[t + 1]])
__global__ void ranges_from_slots_kernel(const uint32_t* __restrict__ scanned, const uint32_t* __restrict__ tile_base,
                                         int n_tiles, uint32_t* __restrict__ ranges) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n_tiles) return;
    ranges[2 * t] = scanned[tile_base[t]];
    ranges[2 * t + 1] = scanned[tile_base[t + 1]];
}

// supertile ranges over the st-sorted keys (lower bounds)
__global__ void key_ranges_kernel(const uint32_t* __restrict__ keys, uint32_t n, uint32_t* __restrict__ ranges,
                                  int n_keys) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n_keys) return;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const uint32_t key = (uint32_t)t + k;
        uint32_t lo = 0, hi = n;
        while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (keys[mid] < key) lo = mid + 1;
            else hi = mid;
        }
        ranges[2 * t + k] = lo;
    }
}

inline unsigned blocks_for(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

}  // namespace

int supertile_side() { return kST; }
size_t bin_segment_upper(uint64_t st_pairs, int n_st) { return (size_t)(st_pairs / kSeg + n_st + 1); }

bool st_chunked(int n_st) { return n_st <= kStMaxSmem; }
int st_chunks(int n_surv) { return n_surv > kStChunk ? (n_surv + kStChunk - 1) / kStChunk : 1; }
size_t st_chunk_words(int n_surv, int n_st) { return (size_t)n_st * st_chunks(n_surv) + 1; }

cudaError_t launch_binning(LaunchCtx& lc, const BinningArgs& a) {
    const int n_st = a.st_x * a.st_y;
    const int n_tiles = a.tiles_x * a.tiles_y;
    const uint32_t* gauss;
    cudaError_t e;
    if (st_chunked(n_st)) {
        const int nchunks = st_chunks(a.n_surv);
        const size_t smem = (size_t)n_st * 4;
        if (smem > 48 * 1024) {
            cudaFuncSetAttribute(st_chunk_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            cudaFuncSetAttribute(st_chunk_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        }
        {
            LaunchScope s(lc, "st_count");
            st_chunk_kernel<false><<<nchunks, 32, smem, lc.stream>>>(a.order, a.rect_ref, a.n_surv, a.tile_size, a.st_x,
                                                                     n_st, nchunks, a.st_cnt, nullptr);
            lc.count++;
        }
        e = exclusive_scan_u32(lc, a.st_cnt, a.st_cnt, (uint64_t)n_st * nchunks + 1, a.scan_tmp, nullptr);
        if (e != cudaSuccess) return e;
        {
            LaunchScope s(lc, "st_emit");
            st_chunk_kernel<true><<<nchunks, 32, smem, lc.stream>>>(a.order, a.rect_ref, a.n_surv, a.tile_size, a.st_x,
                                                                    n_st, nchunks, a.st_cnt, a.st_gauss[0]);
            lc.count++;
        }
        gauss = a.st_gauss[0];
    } else {
        if (a.n_surv > 0) {
            LaunchScope s(lc, "emit_st_pairs");
            emit_st_pairs_kernel<<<blocks_for(a.n_surv, 256), 256, 0, lc.stream>>>(
                a.order, a.st_offsets, a.rect_ref, a.tile_size, a.st_x, a.n_surv, a.st_key[0], a.st_gauss[0]);
            lc.count++;
        }
        bool alt = false;
        e = radix_sort_pairs(lc, a.st_key[0], a.st_gauss[0], a.st_key[1], a.st_gauss[1], a.st_pairs, 0, a.st_bits,
                             a.hist, a.scan_tmp, &alt);
        if (e != cudaSuccess) return e;
        const uint32_t* keys = a.st_key[alt ? 1 : 0];
        gauss = a.st_gauss[alt ? 1 : 0];
        {
            LaunchScope s(lc, "st_ranges");
            key_ranges_kernel<<<blocks_for(n_st, 256), 256, 0, lc.stream>>>(keys, (uint32_t)a.st_pairs, a.st_ranges,
                                                                           n_st);
            lc.count++;
        }
    }
    {
        LaunchScope s(lc, "seg_setup");
        const bool chunked = st_chunked(n_st);
        const size_t smem = n_st <= kSetupSmemSt ? (size_t)n_st * 4 : 0;
        if (smem > 48 * 1024)
            cudaFuncSetAttribute(seg_setup_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        seg_setup_kernel<<<1, kSetupThreads, smem, lc.stream>>>(chunked ? a.st_cnt : nullptr, st_chunks(a.n_surv),
                                                                a.st_ranges, n_st, a.tiles_x, a.tiles_y, a.st_x,
                                                                a.seg_start, a.seg_start + n_st + 1, a.tile_base);
        lc.count++;
    }
    const size_t segs = bin_segment_upper(a.st_pairs, n_st);
    const size_t n_slots = segs * kSTT + 1;
    e = cudaMemsetAsync(a.slots, 0, n_slots * 4, lc.stream);
    if (e != cudaSuccess) return e;
    {
        LaunchScope s(lc, "bin_count");
        bin_segments_kernel<false><<<(unsigned)segs, kBinThreads, 0, lc.stream>>>(
            a.st_ranges, a.seg_start, n_st, a.tile_base, gauss, a.rect_ref, a.tile_size, a.tiles_x, a.tiles_y, a.st_x,
            a.slots, nullptr);
        lc.count++;
    }
    e = exclusive_scan_u32(lc, a.slots, a.slots, n_slots, a.scan_tmp, nullptr);
    if (e != cudaSuccess) return e;
    {
        LaunchScope s(lc, "tile_ranges");
        ranges_from_slots_kernel<<<blocks_for(n_tiles, 256), 256, 0, lc.stream>>>(a.slots, a.tile_base, n_tiles,
                                                                                  a.ranges);
        lc.count++;
    }
    {
        LaunchScope s(lc, "bin_emit");
        bin_segments_kernel<true><<<(unsigned)segs, kBinThreads, 0, lc.stream>>>(
            a.st_ranges, a.seg_start, n_st, a.tile_base, gauss, a.rect_ref, a.tile_size, a.tiles_x, a.tiles_y, a.st_x,
            a.slots, a.pair_gauss);
        lc.count++;
    }
    return cudaGetLastError();
}

}  // namespace splat_b200
