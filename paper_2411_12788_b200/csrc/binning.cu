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
//   3. per-tile lists from the supertile lists: every supertile list entry carries its 16-bit
//      tile cover (written by step 2); the lists are cut into fixed-size pieces, a count pass
//      gives per (piece, tile) counts, and an emit pass ranks each entry per tile by warp ballots
//      + a scan over the piece's warps and writes contiguous runs.  No global scan: every tile
//      list of supertile s lives in a fixed-capacity slot (a tile's list is a sub-list of its
//      supertile's list, so L_s entries suffice): tile f of s starts at 16 lo_s + f L_s, and
//      ranges[t] = [start, start + count).
// Stability at every step makes each list exactly the reference's, and only P x 4 B are written
// (into a 16 Ps-entry capacity; the debug getter compacts the lists to CSR for the bit-exact checks).
#include <cstdint>

#include "common.cuh"
#include "internal.h"

namespace splat_b200 {

namespace {

constexpr int kST = 4;              // supertile side in tiles
constexpr int kSTT = kST * kST;     // tiles per supertile
constexpr int kL2Threads = 512;     // level-2 CTA: one per piece of a supertile list
constexpr int kStChunk = 96;        // depth-ordered survivors per warp of the supertile pass (96: 0.6 % faster
                                    // than 128, shorter emit warps, less wave tail; 64: the scan grows)
constexpr int kStWarps = 12;        // warps per supertile-count CTA (one count column per 1152 survivors;
                                    // 12: +0.3 % over 16, a smaller last wave of count CTAs)
constexpr int kEmitWarps = 1;       // warps per supertile-emit CTA (1: 60 us, 4 independent warps: 67 us)
constexpr int kStChunkCta = kStChunk * kStWarps;  // survivors per CTA chunk (one count column)
constexpr int kStMaxSmem = 3328;    // supertiles the chunked pass keeps in shared memory (x kStWarps rows)

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

// Same, for a power-of-two tile size (shift; rect bounds are >= 0 and x1 > x0 >= 0 on survivors).
__device__ __forceinline__ TileRect tile_rect_shift(uint2 r, int sh) {
    TileRect t;
    t.tx0 = (int)(r.x & 0xffffu) >> sh;
    t.tx1 = ((int)(r.x >> 16) - 1) >> sh;
    t.ty0 = (int)(r.y & 0xffffu) >> sh;
    t.ty1 = ((int)(r.y >> 16) - 1) >> sh;
    return t;
}

__device__ __forceinline__ TileRect tile_rect_any(uint2 r, int ts, int sh) {
    return sh >= 0 ? tile_rect_shift(r, sh) : tile_rect(r, ts);
}

// Tiles of supertile (sx, sy) that the inclusive tile rect covers, as 16 bits (bit 4 ly + lx).
__device__ __forceinline__ uint32_t cover16(int tx0, int tx1, int ty0, int ty1, int sx, int sy) {
    const int lx0 = max(tx0 - sx * kST, 0), lx1 = min(tx1 - sx * kST, kST - 1);
    const int ly0 = max(ty0 - sy * kST, 0), ly1 = min(ty1 - sy * kST, kST - 1);
    if (lx0 > lx1 || ly0 > ly1) return 0u;
    const uint32_t row = ((2u << lx1) - 1u) & ~((1u << lx0) - 1u);
    const uint32_t rows = ((2u << ly1) - 1u) & ~((1u << ly0) - 1u);
    // bit ly of rows -> nibble ly: multiplying the 4-bit row by sum 16^ly places one copy per row
    const uint32_t spread = (rows & 1u) | ((rows & 2u) << 3) | ((rows & 4u) << 6) | ((rows & 8u) << 9);
    return row * spread;
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

// st_cnt layout (chunked path): [cnt: n_st x nchunks (supertile-major), exclusive-scanned in
// place][total][per-warp prefix rows: nchunks x kStWarps x n_st]; cnt[st][0] is the start of
// supertile st's list.
// Supertile pass over one chunk of depth-ordered survivors: kStWarps warps per CTA, each owning
// kStChunk consecutive survivors of the CTA's chunk.  A warp flattens its Gaussians, 32 at a
// time, into (Gaussian, supertile) entries in (depth, raster) order; every window of 32 entries is
// ranked per supertile with __match_any_sync, and a per-(warp, supertile) running count in shared
// memory carries the rank across windows.
//   EMIT = false: each warp counts its entries per supertile; wpre[(c kStWarps + warp) n_st + st]
//                 gets the warp's exclusive prefix within the chunk (coalesced rows) and
//                 cnt[st nchunks + c] the CTA's total.
//   EMIT = true:  cnt holds the exclusive scan of the CTA counts (supertile-major); launched with
//                 kEmitWarps independent warps per CTA (one: more resident warps per SM were
//                 measured slower — the shuffle / shared-memory pipe, not latency, bounds it),
//                 each with base cnt[st nchunks + c] plus its wpre row; it writes
//                 st_gauss[base + rank].
template <bool EMIT>
__global__ void __launch_bounds__(EMIT ? 32 * kEmitWarps : 32 * kStWarps) st_chunk_kernel(const uint32_t* __restrict__ order,
                                                                 const uint2* __restrict__ rect_ref, int n_surv,
                                                                 int ts, int ts_shift, int st_x, int n_st, int nchunks,
                                                                 uint32_t* __restrict__ cnt,
                                                                 uint32_t* __restrict__ st_gauss,
                                                                 uint16_t* __restrict__ st_cover) {
    // count: kStWarps warps per CTA chunk, s_mem = [kStWarps][n_st] per-warp counts;
    // emit: kEmitWarps independent warps per CTA (global warp gw = warp `warp` of chunk c), each
    // with its own [n_st] running offsets in s_mem; no CTA barrier
    extern __shared__ uint32_t s_mem[];
    pdl_wait();
    pdl_trigger();
    const int lane = threadIdx.x & 31;
    const int gw = blockIdx.x * kEmitWarps + (threadIdx.x >> 5);
    const int c = EMIT ? gw / kStWarps : blockIdx.x;
    const int warp = EMIT ? gw % kStWarps : threadIdx.x >> 5;
    uint32_t* s_run = s_mem + (size_t)(threadIdx.x >> 5) * n_st;
    uint32_t* wcnt = cnt + (size_t)n_st * nchunks + 1;  // per-warp prefix rows
    if (EMIT) {
        const uint32_t* wpre = wcnt + ((size_t)c * kStWarps + warp) * n_st;
        for (int st = lane; st < n_st; st += 32) s_run[st] = cnt[(size_t)st * nchunks + c] + wpre[st];
    } else {
        for (int st = lane; st < n_st; st += 32) s_run[st] = 0u;
        if (c == 0 && threadIdx.x == 0) cnt[(size_t)n_st * nchunks] = 0u;  // scan slot of the total
    }
    const int g0 = c * kStChunkCta + warp * kStChunk, g1 = min(g0 + kStChunk, n_surv);
    const unsigned lt = lanemask_lt();
    // the warp's ids and rects are loaded up front (two dependent round trips)
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
    __syncwarp();
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
        const int r = g0 + k * 32 + lane;
        int sx0 = 0, sy0 = 0, w = 1, m = 0;
        uint32_t ptx = 0, pty = 0;  // (tx0 | tx1 << 16), (ty0 | ty1 << 16)
        if (r < g1) {
            const TileRect t = tile_rect_any(rects[k], ts, ts_shift);
            sx0 = t.tx0 / kST;
            sy0 = t.ty0 / kST;
            w = t.tx1 / kST - sx0 + 1;
            m = w * (t.ty1 / kST - sy0 + 1);
            ptx = (uint32_t)t.tx0 | ((uint32_t)t.tx1 << 16);
            pty = (uint32_t)t.ty0 | ((uint32_t)t.ty1 << 16);
        }
        if (!EMIT) {  // counts are order-free: shared-memory atomics per entry
            int x = 0, row = sy0 * st_x + sx0;
            for (int q = 0; q < m; ++q) {
                atomicAdd(&s_run[row + x], 1u);
                if (++x == w) {
                    x = 0;
                    row += st_x;
                }
            }
            continue;
        }
        if (!__any_sync(0xffffffffu, m > 0)) continue;
        const uint32_t gid = gids[k];
        const int inc = (int)warp_incl_scan((uint32_t)m, lane);
        const int off = inc - m;
        const int total = __shfl_sync(0xffffffffu, inc, 31);
        // The entry of lane `lane` in window e0: its owner (last lane whose entries start at or
        // before it, by binary search over the scanned offsets) and its supertile.  The owner's
        // tile rect is all it needs (the supertile rect follows from it).
        auto locate = [&](int e0, int& st, uint32_t& optx, uint32_t& opty, uint32_t& ogid, int& esx, int& esy) {
            const int e = e0 + lane;
            int owner = 0;
#pragma unroll
            for (int step = 16; step > 0; step >>= 1)
                if (__shfl_sync(0xffffffffu, off, owner + step) <= e) owner += step;
            const int q = e - __shfl_sync(0xffffffffu, off, owner);
            optx = __shfl_sync(0xffffffffu, ptx, owner);
            opty = __shfl_sync(0xffffffffu, pty, owner);
            ogid = __shfl_sync(0xffffffffu, gid, owner);
            const int osx0 = (int)(optx & 0xffffu) / kST, osy0 = (int)(opty & 0xffffu) / kST;
            const int ow = (int)(optx >> 16) / kST - osx0 + 1;
            // q / ow without an integer division: (q + 0.5) / ow is >= 0.5 / ow away from an
            // integer and the float error of (q + 0.5) * rcp(ow) is below (q + 0.5) 2^-21 / ow,
            // so truncation is exact for q < 2^20 (q < n_st here)
            const int qy = __float2int_rz(((float)q + 0.5f) * __fdividef(1.0f, (float)ow));
            esx = osx0 + (q - qy * ow);
            esy = osy0 + qy;
            st = esy * st_x + esx;
        };
        int st = 0, esx = 0, esy = 0;
        uint32_t optx = 0, opty = 0, ogid = 0;
        if (total > 0) locate(0, st, optx, opty, ogid, esx, esy);
        for (int e0 = 0; e0 < total; e0 += 32) {
            const bool valid = e0 + lane < total;
            const unsigned grp = __match_any_sync(0xffffffffu, valid ? st : -1);
            const int leader = __ffs(grp) - 1;
            uint32_t base = 0;
            if (valid && lane == leader) {
                base = s_run[st];
                s_run[st] = base + (uint32_t)__popc(grp);
            }
            // software pipelining: the next window's entries are located (shuffles only) while
            // this window's shared-memory update is in flight
            int st_n = 0, esx_n = 0, esy_n = 0;
            uint32_t optx_n = 0, opty_n = 0, ogid_n = 0;
            if (e0 + 32 < total) locate(e0 + 32, st_n, optx_n, opty_n, ogid_n, esx_n, esy_n);
            base = __shfl_sync(0xffffffffu, base, leader);
            if (valid) {
                const uint32_t o = base + __popc(grp & lt);
                st_gauss[o] = ogid;
                st_cover[o] = (uint16_t)cover16((int)(optx & 0xffffu), (int)(optx >> 16), (int)(opty & 0xffffu),
                                                (int)(opty >> 16), esx, esy);
            }
            __syncwarp();
            st = st_n;
            esx = esx_n;
            esy = esy_n;
            optx = optx_n;
            opty = opty_n;
            ogid = ogid_n;
        }
    }
    if (!EMIT) {
        // per supertile: the CTA total (scanned later) and each warp's exclusive prefix within the
        // chunk (coalesced rows: the emit warp then reads one row)
        __syncthreads();
        uint32_t* wpre = wcnt + (size_t)c * kStWarps * n_st;
        for (int st = threadIdx.x; st < n_st; st += blockDim.x) {
            uint32_t t = 0;
#pragma unroll
            for (int ww = 0; ww < kStWarps; ++ww) {
                const uint32_t x = s_mem[(size_t)ww * n_st + st];
                wpre[(size_t)ww * n_st + st] = t;
                t += x;
            }
            cnt[(size_t)st * nchunks + c] = t;
        }
    }
}


// ---- level 2 -----------------------------------------------------------------------------------
// Every supertile list is cut into pieces of kPiece entries.  Piece ids need no scan: supertile s
// owns ids [g(s), g(s+1)) with g(s) = floor(lo_s / kPiece) + s (strictly increasing, and its
// ceil(L_s / kPiece) pieces fit), so each piece CTA finds its supertile by a ballot search.  Each
// list entry carries its 16-bit tile cover (written by the level-1 emit), so level 2 reads only
// coalesced (id, cover) pairs:
//   bin_count: per piece, entries covering each of the 16 tiles (ballots);
//   bin_emit:  per piece, the tile offsets of its earlier pieces (<= a few dozen counts), the
//              ranks of its entries per tile from ballots + a scan over (slice, warp) in shared
//              memory, and one store instruction per (slice, warp, tile) writing a contiguous
//              run of the tile's list.
constexpr int kPiece = 2048;
constexpr int kPieceK = kPiece / kL2Threads;  // entries per thread

// lo_s: start of supertile s's list (s in [0, n_st]) in the concatenated supertile lists.
__device__ __forceinline__ uint32_t st_lo(const uint32_t* __restrict__ st_cnt, int nchunks,
                                          const uint32_t* __restrict__ st_ranges, int n_st, int s) {
    if (st_cnt) return st_cnt[(size_t)s * nchunks];
    return s < n_st ? st_ranges[2 * s] : st_ranges[2 * n_st - 1];
}

// The forward's work order: tile t filed under cost class 63 - min(63, list length / 512) (longest
// lists first), tcls = [64 counters (zeroed by publish_counts) | 64 x n_tiles lists].
__device__ __forceinline__ void file_tile(uint32_t* tcls, int n_tiles, int t, uint32_t len) {
    const int c = kCostClasses - 1 - (int)min((uint32_t)kCostClasses - 1u, len >> 9);
    tcls[kCostClasses + (size_t)c * n_tiles + atomicAdd(&tcls[c], 1u)] = (uint32_t)t;
}


// The 16 cover bits of a lane as four words of byte counters (byte j of word i = bit 4 i + j):
// each nibble is spread to bytes by one multiply (copies at bit offsets 0, 7, 14, 21 never
// overlap), so per-tile counts over a warp are four __reduce_add_sync instead of 16 ballots.
__device__ __forceinline__ void spread16(uint32_t c, uint32_t out[4]) {
#pragma unroll
    for (int i = 0; i < 4; ++i) out[i] = (((c >> (4 * i)) & 0xfu) * 0x00204081u) & 0x01010101u;
}
__device__ __forceinline__ uint32_t byte_of(const uint32_t w[4], int f) { return (w[f >> 2] >> (8 * (f & 3))) & 0xffu; }

struct PieceInfo {
    int st;
    uint32_t p, lo_s, hi_s, lo, hi;
};

// Piece id -> supertile without a map kernel: g(s) = floor(lo_s / kPiece) + s is strictly
// increasing, so the owner is the last s with g(s) <= id — found by warp 0 with ballots over 32
// candidates per round (two rounds up to 1024 supertiles) and shared with the CTA.  Returns false
// for the ids past a supertile's last piece; *empty_st gets the supertile when the id is the one
// id of an empty supertile (its tiles' ranges are written by bin_emit).
__device__ __forceinline__ bool piece_info(uint32_t id, const uint32_t* __restrict__ st_cnt, int nchunks,
                                           const uint32_t* __restrict__ st_ranges, int n_st, PieceInfo& pi,
                                           int* empty_st) {
    __shared__ int s_st;
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        int base = 0, span = n_st;
        while (true) {
            const int stride = span > 32 ? (span + 31) / 32 : 1;
            const int cand = base + lane * stride;
            const bool ok = lane * stride < span &&
                            st_lo(st_cnt, nchunks, st_ranges, n_st, cand) / kPiece + (uint32_t)cand <= id;
            const unsigned m = __ballot_sync(0xffffffffu, ok);
            base += (31 - __clz(m)) * stride;  // g(base) <= id always (g(0) = 0)
            if (stride == 1) break;
            span = min(stride, n_st - base);
        }
        if (lane == 0) s_st = base;
    }
    __syncthreads();
    const int st = s_st;
    pi.st = st;
    pi.lo_s = st_lo(st_cnt, nchunks, st_ranges, n_st, st);
    pi.hi_s = st_lo(st_cnt, nchunks, st_ranges, n_st, st + 1);
    pi.p = id - (pi.lo_s / kPiece + (uint32_t)st);
    const uint32_t np = (pi.hi_s - pi.lo_s + kPiece - 1) / kPiece;
    if (empty_st) *empty_st = (np == 0) ? st : -1;
    if (pi.p >= np) return false;
    pi.lo = pi.lo_s + pi.p * kPiece;
    pi.hi = min(pi.lo + (uint32_t)kPiece, pi.hi_s);
    return true;
}

// The ranges (empty) of an empty supertile's tiles, by its one bin_emit CTA.
__device__ __forceinline__ void empty_supertile(int st, uint32_t lo, int tiles_x, int tiles_y, int st_x,
                                                uint32_t* __restrict__ ranges, uint32_t* __restrict__ tcls,
                                                uint32_t* __restrict__ tails) {
    const int f = threadIdx.x;
    if (f >= kSTT) return;
    const int tx = (st % st_x) * kST + (f % kST), ty = (st / st_x) * kST + (f / kST);
    if (tx < tiles_x && ty < tiles_y) {
        const int t = ty * tiles_x + tx;
        ranges[2 * t] = kSTT * lo;
        ranges[2 * t + 1] = kSTT * lo;
        if (tails) {
            tails[2 * t] = 0u;
            tails[2 * t + 1] = 0u;
        }
        if (tcls) file_tile(tcls, tiles_x * tiles_y, t, 0u);
    }
}

__global__ void __launch_bounds__(kL2Threads) bin_count_kernel(const uint32_t* __restrict__ st_cnt, int nchunks,
                                                              const uint32_t* __restrict__ st_ranges, int n_st,
                                                              const uint16_t* __restrict__ st_cover,
                                                              uint32_t* __restrict__ piece_cnt) {
    __shared__ uint32_t s_cnt[kSTT];
    pdl_wait();
    pdl_trigger();
    PieceInfo pi;
    if (!piece_info(blockIdx.x, st_cnt, nchunks, st_ranges, n_st, pi, nullptr)) return;
    const int tid = threadIdx.x, lane = tid & 31;
    if (tid < kSTT) s_cnt[tid] = 0u;
    uint32_t cv[kPieceK];
#pragma unroll
    for (int k = 0; k < kPieceK; ++k) {
        const uint32_t e = pi.lo + k * kL2Threads + tid;
        cv[k] = e < pi.hi ? (uint32_t)st_cover[e] : 0u;
    }
    // lane f: this warp's entries covering tile f (byte counters: <= 32 kPieceK = 128 per byte)
    uint32_t acc[4] = {0u, 0u, 0u, 0u};
#pragma unroll
    for (int k = 0; k < kPieceK; ++k) {
        uint32_t sp[4];
        spread16(cv[k], sp);
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[i] += sp[i];
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[i] = __reduce_add_sync(0xffffffffu, acc[i]);
    static_assert(32 * kPieceK < 256, "byte counters");
    const uint32_t mine = byte_of(acc, lane & 15);
    __syncthreads();
    if (lane < kSTT && mine) atomicAdd(&s_cnt[lane], mine);
    __syncthreads();
    if (tid < kSTT) piece_cnt[(size_t)blockIdx.x * kSTT + tid] = s_cnt[tid];
}

__global__ void __launch_bounds__(kL2Threads, 2) bin_emit_kernel(
    const uint32_t* __restrict__ st_cnt, int nchunks, const uint32_t* __restrict__ st_ranges, int n_st,
    const uint32_t* __restrict__ piece_cnt, const uint32_t* __restrict__ st_gauss, const uint16_t* __restrict__ st_cover, int tiles_x, int tiles_y, int st_x,
    uint32_t* __restrict__ pair_gauss, uint32_t* __restrict__ ranges, uint32_t* __restrict__ tcls,
    uint32_t* __restrict__ tails, uint32_t kpre) {
    constexpr int kW = kL2Threads / 32;
    // (slice k, warp) entries covering tile f, then their list position; rows padded to 17 words so
    // the column scan below (lane reads rows 2 lane, 2 lane + 1) is 2-way instead of 32-way conflicted
    constexpr int kRow = kSTT + 1;
    __shared__ uint32_t s_c[kPieceK][kW][kRow];
    __shared__ uint32_t s_prefix[kSTT];
    __shared__ int s_open;  // tiles of the supertile whose list prefix is not complete yet
    pdl_wait();
    pdl_trigger();
    PieceInfo pi;
    int empty = -1;
    if (!piece_info(blockIdx.x, st_cnt, nchunks, st_ranges, n_st, pi, &empty)) {
        if (empty >= 0) empty_supertile(empty, pi.lo_s, tiles_x, tiles_y, st_x, ranges, tcls, tails);
        return;
    }
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t cap = pi.hi_s - pi.lo_s;  // capacity of every tile list of this supertile
    const bool last_piece = pi.hi == pi.hi_s;
    if (warp == 0) {  // counts of this supertile's earlier pieces
        // lane f + 16 h sums tile f's counts over the pieces q = h (mod 2), eight loads in flight
        const uint32_t id0 = pi.lo_s / kPiece + (uint32_t)pi.st;
        const int f = lane & (kSTT - 1), h = lane >> 4;
        uint32_t pre = 0;
        for (uint32_t q0 = (uint32_t)h; q0 < pi.p; q0 += 16) {
            uint32_t x[8];
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                const uint32_t q = q0 + 2u * r;
                x[r] = q < pi.p ? piece_cnt[(size_t)(id0 + q) * kSTT + f] : 0u;
            }
#pragma unroll
            for (int r = 0; r < 8; ++r) pre += x[r];
        }
        pre += __shfl_xor_sync(0xffffffffu, pre, 16);
        if (lane < kSTT) s_prefix[lane] = pre;
        const unsigned open = __ballot_sync(0xffffffffu, lane < kSTT && pre < kpre);
        if (lane == 0) s_open = (int)open;
        // every tile's prefix already complete: only the last piece has work (the tiles' ranges)
        if (!open && last_piece && lane < kSTT) {
            const int tx = (pi.st % st_x) * kST + (lane % kST), ty = (pi.st / st_x) * kST + (lane / kST);
            if (tx < tiles_x && ty < tiles_y) {
                const int t = ty * tiles_x + tx;
                const uint32_t list0 = (uint32_t)kSTT * pi.lo_s + (uint32_t)lane * cap;
                const uint32_t len = pre + piece_cnt[(size_t)blockIdx.x * kSTT + lane];
                ranges[2 * t] = list0;
                ranges[2 * t + 1] = list0 + kpre;
                if (tcls) file_tile(tcls, tiles_x * tiles_y, t, len);
            }
        }
    }
    __syncthreads();
    const unsigned open = (unsigned)s_open;
    if (!open) return;  // (pieces past every tile's prefix: no loads, no ballots)
    uint32_t gid[kPieceK], cv[kPieceK];
#pragma unroll
    for (int k = 0; k < kPieceK; ++k) {
        const uint32_t e = pi.lo + k * kL2Threads + tid;
        const bool ok = e < pi.hi;
        gid[k] = ok ? st_gauss[e] : 0u;
        cv[k] = ok ? (uint32_t)st_cover[e] : 0u;
    }
#pragma unroll
    for (int k = 0; k < kPieceK; ++k) {
        uint32_t sp[4];
        spread16(cv[k], sp);
#pragma unroll
        for (int i = 0; i < 4; ++i) sp[i] = __reduce_add_sync(0xffffffffu, sp[i]);
        if (lane < kSTT) s_c[k][warp][lane] = byte_of(sp, lane);
    }
    __syncthreads();
    {   // warp f: exclusive scan of tile f's counts over the 64 (slice, warp) positions in entry order
        static_assert(kPieceK * kW == 64 && kW == kSTT, "scan layout assumes 16 warps x 4 slices");
        const int f = warp;
        uint32_t* col = &s_c[0][0][0];
        const int q0 = 2 * lane, q1 = 2 * lane + 1;
        const uint32_t v0 = col[q0 * kRow + f], v1 = col[q1 * kRow + f];
        const uint32_t inc = warp_incl_scan(v0 + v1, lane);
        const uint32_t list0 = (uint32_t)kSTT * pi.lo_s + (uint32_t)f * cap;
        const uint32_t base = list0 + s_prefix[f];
        col[q0 * kRow + f] = base + inc - v0 - v1;
        col[q1 * kRow + f] = base + inc - v1;
        if (lane == 31 && last_piece) {  // last piece: the tile's range (materialised part)
            const int tx = (pi.st % st_x) * kST + (f % kST), ty = (pi.st / st_x) * kST + (f / kST);
            if (tx < tiles_x && ty < tiles_y) {
                const int t = ty * tiles_x + tx;
                const uint32_t len = base + inc - list0;
                ranges[2 * t] = list0;
                ranges[2 * t + 1] = list0 + min(len, kpre);
                if (tcls) file_tile(tcls, tiles_x * tiles_y, t, len);
                if (tails && len <= kpre) {  // complete list: no tail
                    tails[2 * t] = 0u;
                    tails[2 * t + 1] = 0u;
                }
            }
        }
    }
    __syncthreads();
    // Each tile's entries up to its prefix length kpre are written; the entry at rank kpre - 1
    // records where the tile's tail starts in the supertile list (StagePipe reads it from there).
    const unsigned lt = lanemask_lt();
    const int tx0 = (pi.st % st_x) * kST, ty0 = (pi.st / st_x) * kST;
#pragma unroll
    for (int f = 0; f < kSTT; ++f) {
        if (!((open >> f) & 1u)) continue;  // warp-uniform: this tile's prefix is complete
        const uint32_t list0 = (uint32_t)kSTT * pi.lo_s + (uint32_t)f * cap;
#pragma unroll
        for (int k = 0; k < kPieceK; ++k) {
            const bool on = (cv[k] >> f) & 1u;
            const unsigned m = __ballot_sync(0xffffffffu, on);
            const uint32_t rank = s_c[k][warp][f] + __popc(m & lt) - list0;
            if (on && rank < kpre) pair_gauss[list0 + rank] = gid[k];
            if (on && rank + 1u == kpre && tails) {
                const int tx = tx0 + (f % kST), ty = ty0 + (f / kST);
                if (tx < tiles_x && ty < tiles_y) {
                    const int t = ty * tiles_x + tx;
                    tails[2 * t] = pi.lo + k * kL2Threads + tid + 1u;
                    tails[2 * t + 1] = pi.hi_s;
                }
            }
        }
    }
}

// Fallback path (supertile lists from the pair sort): covers from the rects.
__global__ void st_cover_kernel(const uint32_t* __restrict__ st_key, const uint32_t* __restrict__ st_gauss,
                                const uint2* __restrict__ rect_ref, uint32_t n, int ts, int ts_shift, int st_x,
                                uint16_t* __restrict__ st_cover) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const TileRect t = tile_rect_any(rect_ref[st_gauss[i]], ts, ts_shift);
    const int st = (int)st_key[i];
    st_cover[i] = (uint16_t)cover16(t.tx0, t.tx1, t.ty0, t.ty1, st % st_x, st / st_x);
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
size_t bin_l2_pieces(uint64_t st_pairs, int n_st) { return (size_t)(st_pairs / kPiece + n_st); }
size_t bin_l2_words(uint64_t st_pairs, int n_st) { return bin_l2_pieces(st_pairs, n_st) * (1 + kSTT) + 1; }

bool st_chunked(int n_st) { return n_st <= kStMaxSmem; }
int st_chunks(int n_surv) { return n_surv > kStChunkCta ? (n_surv + kStChunkCta - 1) / kStChunkCta : 1; }
// CTA counts (scanned in place) + the total slot, then the per-warp count rows
size_t st_chunk_words(int n_surv, int n_st) { return (size_t)n_st * st_chunks(n_surv) * (1 + kStWarps) + 1; }

namespace {
// Level 2's emit: every tile's list up to kpre entries (0xffffffff: the whole list) and the
// supertile-list position of the rest (tails).
cudaError_t launch_bin_emit(LaunchCtx& lc, const BinningArgs& a, const uint32_t* gauss, uint32_t kpre,
                            uint32_t* tcls) {
    const int n_st = a.st_x * a.st_y;
    const uint32_t* cnt = st_chunked(n_st) ? a.st_cnt : nullptr;
    const int nch = st_chunks(a.n_surv);
    const uint32_t np = (uint32_t)bin_l2_pieces(a.st_pairs, n_st);
    if (np == 0) return cudaSuccess;
    LaunchScope s(lc, "bin_emit");
    const cudaError_t e = launch_pdl(lc.stream, bin_emit_kernel, dim3(np), dim3(kL2Threads), 0, cnt, nch,
                                     (const uint32_t*)a.st_ranges, n_st, (const uint32_t*)(a.l2_tmp + np), gauss, (const uint16_t*)a.st_cover, a.tiles_x,
                                     a.tiles_y, a.st_x, a.pair_gauss, a.ranges, tcls, a.tails, kpre);
    lc.count++;
    return e;
}
}  // namespace

cudaError_t launch_binning(LaunchCtx& lc, const BinningArgs& a) {
    const int n_st = a.st_x * a.st_y;
    const int n_tiles = a.tiles_x * a.tiles_y;
    const uint32_t* gauss;
    cudaError_t e;
    const int ts = a.tile_size;
    int ts_shift = -1;
    if ((ts & (ts - 1)) == 0) {
        ts_shift = 0;
        while ((1 << ts_shift) < ts) ++ts_shift;
    }
    if (st_chunked(n_st)) {
        const int nchunks = st_chunks(a.n_surv);
        const size_t smem_count = (size_t)n_st * 4 * kStWarps, smem_emit = (size_t)n_st * 4 * kEmitWarps;
        if (smem_count > 48 * 1024)
            cudaFuncSetAttribute(st_chunk_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_count);
        if (smem_emit > 48 * 1024)
            cudaFuncSetAttribute(st_chunk_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_emit);
        {
            LaunchScope s(lc, "st_count");
            e = launch_pdl(lc.stream, st_chunk_kernel<false>, dim3(nchunks), dim3(32 * kStWarps), smem_count, a.order,
                           a.rect_ref, a.n_surv, ts, ts_shift, a.st_x, n_st, nchunks, a.st_cnt, (uint32_t*)nullptr,
                           (uint16_t*)nullptr);
            if (e != cudaSuccess) return e;
            lc.count++;
        }
        e = exclusive_scan_u32_zeroed(lc, a.st_cnt, a.st_cnt, (uint64_t)n_st * nchunks + 1, a.st_scan_tmp);
        if (e != cudaSuccess) return e;
        {
            LaunchScope s(lc, "st_emit");
            e = launch_pdl(lc.stream, st_chunk_kernel<true>, dim3(nchunks * (kStWarps / kEmitWarps)), dim3(32 * kEmitWarps),
                           smem_emit, a.order,
                           a.rect_ref, a.n_surv, ts, ts_shift, a.st_x, n_st, nchunks, a.st_cnt, a.st_gauss[0],
                           a.st_cover);
            if (e != cudaSuccess) return e;
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
        if (a.st_pairs > 0) {
            LaunchScope s(lc, "st_cover");
            st_cover_kernel<<<blocks_for((int64_t)a.st_pairs, 256), 256, 0, lc.stream>>>(
                keys, gauss, a.rect_ref, (uint32_t)a.st_pairs, ts, ts_shift, a.st_x, a.st_cover);
            lc.count++;
        }
    }
    {
        const uint32_t* cnt = st_chunked(n_st) ? a.st_cnt : nullptr;
        const int nch = st_chunks(a.n_surv);
        const uint32_t np = (uint32_t)bin_l2_pieces(a.st_pairs, n_st);
        uint32_t* piece_cnt = a.l2_tmp + np;  // (the first np words: unused)
        if (np > 0) {
            {
                LaunchScope s(lc, "bin_count");
                e = launch_pdl(lc.stream, bin_count_kernel, dim3(np), dim3(kL2Threads), 0, cnt, nch,
                               (const uint32_t*)a.st_ranges, n_st,
                               (const uint16_t*)a.st_cover, piece_cnt);
                if (e != cudaSuccess) return e;
                lc.count++;
            }
            e = launch_bin_emit(lc, a, gauss, a.list_prefix, cnt ? a.tcls : nullptr);
            if (e != cudaSuccess) return e;
        }
    }
    if (a.st_list) *a.st_list = gauss;
    (void)n_tiles;
    return cudaGetLastError();
}

cudaError_t complete_tile_lists(LaunchCtx& lc, const BinningArgs& a, const uint32_t* st_list) {
    return launch_bin_emit(lc, a, st_list, 0xffffffffu, nullptr);
}

}  // namespace splat_b200
