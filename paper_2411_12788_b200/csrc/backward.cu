// backward.cu — blend backward (K9), per-Gaussian 2D->3D chain (K10), L1 loss (K8) and Adam (K11).
//
// Gradients are compared against the oracle within tolerance (1e-4 relative, SURVEY.md §8
// Appendix C): summation order over pixels differs (warp/CTA reductions + atomics) and the
// backward reconstructs T_before = T_after / (1 - alpha) instead of storing per-sample T.
// The gates themselves are replayed bit-exactly (gate_sample uses explicit _rn intrinsics), so
// the set of committed samples is identical to the forward's.  FMA contraction is allowed here.
#include <climits>
#include <cstdint>
#include <type_traits>

#include "common.cuh"
#include "internal.h"

namespace splat_b200 {
#ifdef SPLAT_STATS
__device__ unsigned long long g_bstats[8];
#endif

namespace {


__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Transpose reduction of 18 per-lane values (two entries x three groups of 3) across the warp
// in 24 shuffles (a butterfly would take 90).  Level 16: lanes keep their entry (bit 16 clear:
// a), send the other.  Level 8: lanes with bit 8 clear keep groups 0-1 and send group 2, their
// partners keep group 2 (6 shuffles: one direction carries 6 values, the other 3).  Level 4: the
// group-0/1 lanes split them, the group-2 lanes reduce theirs; levels 2 and 1 reduce the quad.  On
// return lanes 4q hold, in out[0..2], the warp totals of entry (lane >> 4), group
// (lane & 8 ? 2 : (lane >> 2) & 1) (lanes 12 and 28 duplicate 8 and 24).
__device__ __forceinline__ void warp_reduce18(const float v[18], int lane, float out[3]) {
    const bool a = lane & 16, b = lane & 8, c = lane & 4;
    float u[9], w[6];
#pragma unroll
    for (int i = 0; i < 9; ++i) {
        const float send = a ? v[i] : v[9 + i];
        const float keep = a ? v[9 + i] : v[i];
        u[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
#pragma unroll
    for (int i = 0; i < 6; ++i) {
        const float send = b ? u[i] : u[6 + i % 3];
        const float keep = b ? u[6 + i % 3] : u[i];
        w[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const float send = (b || c) ? w[i] : w[3 + i];
        const float keep = (!b && c) ? w[3 + i] : w[i];
        out[i] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
    }
#pragma unroll
    for (int o = 2; o > 0; o >>= 1)
#pragma unroll
        for (int i = 0; i < 3; ++i) out[i] += __shfl_xor_sync(0xffffffffu, out[i], o);
}

__device__ __forceinline__ void red_add_v4(float4* addr, float x, float y, float z, float w) {
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(x), "f"(y), "f"(z), "f"(w)
                 : "memory");
}

// One sample of the per-pixel back-to-front recursion (gradients.cpp:73-123) in moment form: with
// s = dL/dalpha * g (the opacity gradient of the sample), the pixel adds s, s dx, s dy, s dx^2,
// s dx dy, s dy^2 to vv[0..5]; the per-Gaussian factors (opacity, conic) are applied once per
// Gaussian by the chain (chain.cu), after the sums over all pixels:
//   d mean.x = -o (c0 Sx + c1 Sy), d mean.y = -o (c2 Sy + c1 Sx), d conic = -o/2 (Sxx, Sxy, Syy),
// which is sum(dpower * (-(c0 dx + c1 dy))), ... of the reference with dpower = o s.  vv[6..8] get
// the colour gradient w dL (commits are counted by the caller's ballots).  T_before = T_after / (1 - alpha).  The pixel
// carries B = dL . b, b the colour behind the sample (b = alpha c + (1 - alpha) b is linear in b),
// instead of three channels.  Branch-free: the kernels call it for every lane, and a sample the
// pixel does not commit (p false) contributes exactly nothing (alpha = G = 0: T unchanged, w = 0,
// B += 0) and is not counted — measured faster than a divergent branch (backward 484 -> 450 us).
template <bool ACC = true>  // false: the first sample into vv assigns (no zero-init, no 0 + x)
__device__ __forceinline__ void commit_sample(bool p, float* vv, float& T, float& B, float dL0, float dL1, float dL2,
                                              const float4& r2, float alpha, float g2d, bool clamped, float dx,
                                              float dy) {
    const float a = p ? alpha : 0.0f, g = p ? g2d : 0.0f;
    const float one_m_a = 1.0f - a;
    // 1 - alpha is in [0.01, 1] (alpha <= alpha_max) and T is normal: one rcp.approx.ftz (~1 ulp)
    // instead of __fdividef's denormal-range handling; T_before is not bit-exact anyway
    float rcp;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rcp) : "f"(one_m_a));
    const float t_before = p ? T * rcp : T;
    const float w = t_before * a;
    auto put = [&](int k, float x) { vv[k] = ACC ? vv[k] + x : x; };
    put(6, w * dL0);
    put(7, w * dL1);
    put(8, w * dL2);
    const float diff = (dL0 * r2.x + dL1 * r2.y + dL2 * r2.z) - B;
    const float sv = clamped ? 0.0f : t_before * diff * g;
    const float sx = sv * dx, sy = sv * dy;
    put(0, sv);
    put(1, sx);
    put(2, sy);
    put(3, sx * dx);
    put(4, sx * dy);
    put(5, sy * dy);
    B = B + a * diff;
    T = t_before;
}

// Warp-reduce the 18 values of staged entries ja (v[0..8]) and jb (v[9..17]) and add them to
// the per-Gaussian accumulator (common.cuh kG2Stride records): groups 0-2 (moments, colour) as
// they are, the warp's commit counts (from the callers: ballots or one add-reduction) in the 4th slot of
// group 2's record.
__device__ __forceinline__ void emit_entry_grads(const float v[18], int lane, int cnt_a, int cnt_b, uint32_t ja,
                                                 uint32_t jb, uint32_t a_gid, float4* __restrict__ grad2d) {
    float r[3];
    warp_reduce18(v, lane, r);
    const bool eb = lane & 16;
    const int grp = (lane & 8) ? 2 : (lane >> 2) & 1;
    const int cnt = eb ? cnt_b : cnt_a;
    const bool mine = (lane & 3) == 0 && (lane & 12) != 12 && cnt > 0;
    if (mine) {
        const uint32_t gid = lds_u32(a_gid + 4u * (eb ? jb : ja));
        red_add_v4(grad2d + kG2Stride * (size_t)gid + grp, r[0], r[1], r[2], grp == 2 ? (float)cnt : 0.0f);
    }
}

// Blend backward (gradients.cpp:73-123): per pixel, walk the tile list back to front from the
// pixel's last committed sample, re-evaluating the forward gates; b = colour behind the sample
// (normalised), exactly the reference recursion; T_before = T_after / (1 - alpha).
// Per staged Gaussian the 9 per-pixel contributions (d_mean2d 2, d_conic 3 (01 = 10),
// d_opacity, d_colour 3) plus a commit count are warp-reduced and added straight to the
// per-Gaussian accumulator with four red.global.add.v4.f32 per (warp, Gaussian): no shared
// accumulation, no flush barrier.
// With target != nullptr, dL/dC = sign(C - target)/n (l1_loss, loss.cpp:63-76) is fused in and
// the CTA's L1 partial sum is written to loss_partials[block].
template <bool THR, int BW, int BH>
__device__ __forceinline__ void blend_backward_block(int bid, CamParams cp, const uint32_t* __restrict__ ranges,
                                                            TileTails tt, const uint32_t* __restrict__ pair_gauss,
                                                            const ProjRec* __restrict__ rec,
                                                            const float* __restrict__ t_final,
                                                            const int32_t* __restrict__ last_index, float bg0,
                                                            float bg1, float bg2, const float* __restrict__ d_color,
                                                            const float* __restrict__ color,
                                                            const float* __restrict__ target, float inv_n,
                                                            float* __restrict__ loss_partials,
                                                            float4* __restrict__ grad2d) {
    __shared__ StageSmem<BW * BH> sm;
    __shared__ StageRaw<BW * BH> raw;
    __shared__ float s_red[BW * BH / 32];
    __shared__ int s_maxlast[BW * BH / 32];
    constexpr int nthreads = BW * BH;  // (every launch uses BW * BH threads)
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nwarps = nthreads >> 5;
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
    const size_t pix = inside ? (size_t)py * cp.width + px : 0;

    float dL0 = 0.f, dL1 = 0.f, dL2 = 0.f;
    float l = 0.0f;
    if (inside) {
        if (target) {
            float* dl[3] = {&dL0, &dL1, &dL2};
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const float dd = color[3 * pix + c] - target[3 * pix + c];
                l += fabsf(dd);
                *dl[c] = dd > 0.0f ? inv_n : (dd < 0.0f ? -inv_n : 0.0f);
            }
        } else {
            dL0 = d_color[3 * pix];
            dL1 = d_color[3 * pix + 1];
            dL2 = d_color[3 * pix + 2];
        }
    }
    if (target && loss_partials) {
        const float ws = warp_sum(l);
        if (lane == 0) s_red[warp] = ws;
    }
    const int my_last = inside ? last_index[pix] : -1;
    const int wl = (int)__reduce_max_sync(0xffffffffu, (unsigned)(my_last + 1)) - 1;
    if (lane == 0) s_maxlast[warp] = wl;
    __syncthreads();
    if (target && loss_partials && tid == 0) {
        float s = 0.0f;
        for (int w = 0; w < nwarps; ++w) s += s_red[w];
        loss_partials[bid] = s;
    }
    int block_last = -1;
    for (int w = 0; w < nwarps; ++w) block_last = max(block_last, s_maxlast[w]);
    const uint32_t start = ranges[2 * tile];
    if (block_last < (int)start) return;  // nothing committed in this block
    __shared__ ListTail s_tail;
    uint32_t vend;
    const int split = list_tail_setup(tt.tails, tt.st_list, tt.st_cover, tile, cp.tiles_x, ranges[2 * tile + 1], vend,
                                      &s_tail, tid == 0, []() { __syncthreads(); });

    const float amax_c = cp.alpha_max, cmin = cp.contribution_min;
    const float x = (float)px + 0.5f, y = (float)py + 0.5f;
    const uint32_t mybits = (1u << lx) | (1u << (16 + ly));
    const uint32_t wcols = 0xffu << (lx & ~7), wrows = 0xfu << (16 + (ly & ~3));
    const uint32_t a_r0 = smem_base(sm.r0), a_r1 = smem_base(sm.r1), a_r2 = smem_base(sm.r2);
    const uint32_t a_idx = smem_base(sm.idx), a_gid = smem_base(sm.gid);
    float T = inside ? t_final[pix] : 1.0f;
    float B = dL0 * bg0 + dL1 * bg1 + dL2 * bg2;

    auto pos = [&](int b, int t) -> int {
        const int i = block_last - b * nthreads - t;
        return i >= (int)start ? i : -1;
    };
    StagePipe<BW * BH, decltype(pos)> pipe(pos, pair_gauss, rec, &raw, split, &s_tail);
    pipe.start();
    const int nb = (block_last + 1 - (int)start + nthreads - 1) / nthreads;
    for (int b = 0; b < nb; ++b) {
        const int cnt = pipe.stage(b, true, bx0, bx1, by0, by1, sm);
        // Two staged entries per iteration: their gates are independent instruction streams (the
        // branch-free gate), the per-pixel recursion then commits them in list order (j first: the
        // batch is staged back to front), and one 18-value transpose reduction serves both.
        for (int j = 0; j < cnt; j += 2) {
            const bool has_b = j + 1 < cnt;
            const uint32_t jb = has_b ? (uint32_t)(j + 1) : (uint32_t)j;
            const int idx_a = (int)lds_u32(a_idx + 4u * j);
            const int idx_b = has_b ? (int)lds_u32(a_idx + 4u * jb) : INT_MAX;
            const float4 r1a = lds_f4(a_r1 + 16u * j);
            const float4 r1b = lds_f4(a_r1 + 16u * jb);
            const uint32_t ma = __float_as_uint(r1a.z), mb = __float_as_uint(r1b.z);
            // warp-uniform: above every commit of this warp, or the effective rect misses its patch
            const bool wa = idx_a <= wl && (ma & wrows) && (ma & wcols);
            const bool wb = idx_b <= wl && (mb & wrows) && (mb & wcols);
            if (!wa && !wb) continue;
            const float4 r0a = lds_f4(a_r0 + 16u * j), r0b = lds_f4(a_r0 + 16u * jb);
            float alpha_a, g_a, dxa, dya, alpha_b, g_b, dxb, dyb;
            bool cl_a, cl_b;
            bool ga = gate_sample_nb<THR>(r0a, r1a, mybits, x, y, amax_c, cmin, alpha_a, g_a, cl_a, dxa, dya);
            bool gb = gate_sample_nb<THR>(r0b, r1b, mybits, x, y, amax_c, cmin, alpha_b, g_b, cl_b, dxb, dyb);
            ga = ga && wa && idx_a <= my_last;
            gb = gb && wb && idx_b <= my_last;
            // v: (dmean.x, dmean.y, dconic00 | dconic01, dconic11, dopacity | dcolour rgb | commits)
            // for entry a in v[0..11], entry b in v[12..23]
            float v[18];  // assigned by the two commits (entry a: v[0..8], b: v[9..17])
            commit_sample<false>(ga, v, T, B, dL0, dL1, dL2, lds_f4(a_r2 + 16u * j), alpha_a, g_a, cl_a, dxa, dya);
            commit_sample<false>(gb, v + 9, T, B, dL0, dL1, dL2, lds_f4(a_r2 + 16u * jb), alpha_b, g_b, cl_b, dxb,
                                 dyb);
            const int cnt_a = __popc(__ballot_sync(0xffffffffu, ga)), cnt_b = __popc(__ballot_sync(0xffffffffu, gb));
            const bool any_a = cnt_a > 0, any_b = cnt_b > 0;
#ifdef SPLAT_STATS
            {
                const unsigned el_a = __ballot_sync(0xffffffffu, wa && idx_a <= my_last);
                const unsigned el_b = __ballot_sync(0xffffffffu, wb && idx_b <= my_last);
                const unsigned ca = __ballot_sync(0xffffffffu, ga), cb = __ballot_sync(0xffffffffu, gb);
                if (lane == 0) {
                    atomicAdd(&g_bstats[0], (unsigned long long)(wa + wb));
                    atomicAdd(&g_bstats[1], (unsigned long long)(any_a + any_b));
                    atomicAdd(&g_bstats[2], (unsigned long long)(__popc(el_a) + __popc(el_b)));
                    atomicAdd(&g_bstats[3], (unsigned long long)(__popc(ca) + __popc(cb)));
                    atomicAdd(&g_bstats[4], 1ull);
                }
            }
#endif
            if (any_a || any_b) emit_entry_grads(v, lane, cnt_a, cnt_b, (uint32_t)j, jb, a_gid, grad2d);
        }
        // the next stage() starts with a barrier before it overwrites the staging area
    }
    pipe.finish();
}

// Two pixels per thread: one warp per 8 x 8 block, lane (lx, ly) owns pixels (lx, ly) ["A", top
// half] and (lx, ly + 4) ["B", bottom half].  The per-pixel recursion and gates are those of
// blend_backward_block; per staged pair of entries the two pixels' contributions are added in
// registers before ONE 18-value warp reduction, which now covers 64 pixels (half the reduction
// work per pixel), and the two pixel chains are independent instruction streams.  Entries whose
// effective rect misses a half skip that half's gates (warp-uniform).
struct PixBwd {
    float T, B, dL0, dL1, dL2, x, y;
    int last;
    uint32_t bits;
};

template <bool THR, bool COMPACT>
__device__ __forceinline__ void blend_backward_block_px2(int bid, CamParams cp, const uint32_t* __restrict__ ranges,
                                                         TileTails tt, const uint32_t* __restrict__ pair_gauss,
                                                         const ProjRec* __restrict__ rec,
                                                         const float* __restrict__ t_final,
                                                         const int32_t* __restrict__ last_index, float bg0, float bg1,
                                                         float bg2, const float* __restrict__ d_color,
                                                         const float* __restrict__ color,
                                                         const float* __restrict__ target, float inv_n,
                                                         float* __restrict__ loss_partials,
                                                         float4* __restrict__ grad2d,
                                                         const uint32_t* __restrict__ bidx, int bcnt) {
    constexpr int BW = 8, BH = 8;
    __shared__ StageSmem<32> sm;
    __shared__ StageRaw<32> raw;
    const int lane = threadIdx.x;
    const int ts = cp.tile_size;
    const int subs_x = ts / BW, nsub = subs_x * (ts / BH);
    const int tile = bid / nsub, sub = bid - tile * nsub;
    const int tx = tile % cp.tiles_x, ty = tile / cp.tiles_x;
    const int sx = sub % subs_x, sy = sub / subs_x;
    const int bx0 = tx * ts + sx * BW, by0 = ty * ts + sy * BH;
    const int bx1 = min(bx0 + BW, cp.width), by1 = min(by0 + BH, cp.height);
    const int lx = lane & 7, ly = lane >> 3;
    PixBwd P[2];
    float l = 0.0f;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int px = bx0 + lx, py = by0 + ly + 4 * h;
        const bool inside = px < cp.width && py < cp.height;
        const size_t pix = inside ? (size_t)py * cp.width + px : 0;
        PixBwd& q = P[h];
        q.dL0 = q.dL1 = q.dL2 = 0.0f;
        if (inside) {
            if (target) {
                const float d0 = color[3 * pix] - target[3 * pix];
                const float d1 = color[3 * pix + 1] - target[3 * pix + 1];
                const float d2 = color[3 * pix + 2] - target[3 * pix + 2];
                l += fabsf(d0) + fabsf(d1) + fabsf(d2);
                q.dL0 = d0 > 0.0f ? inv_n : (d0 < 0.0f ? -inv_n : 0.0f);
                q.dL1 = d1 > 0.0f ? inv_n : (d1 < 0.0f ? -inv_n : 0.0f);
                q.dL2 = d2 > 0.0f ? inv_n : (d2 < 0.0f ? -inv_n : 0.0f);
            } else {
                q.dL0 = d_color[3 * pix];
                q.dL1 = d_color[3 * pix + 1];
                q.dL2 = d_color[3 * pix + 2];
            }
        }
        q.last = inside ? last_index[pix] : -1;
        q.T = inside ? t_final[pix] : 1.0f;
        q.B = q.dL0 * bg0 + q.dL1 * bg1 + q.dL2 * bg2;
        q.x = (float)px + 0.5f;
        q.y = (float)py + 0.5f;
        q.bits = (1u << lx) | (1u << (16 + ly + 4 * h));
    }
    if (target && loss_partials) {
        const float ws = warp_sum(l);
        if (lane == 0) loss_partials[bid] = ws;
    }
    if (COMPACT) {  // tile-list positions -> positions in the block's staged list (bidx increases)
        // (the few blocks with more than kBlockListSmem staged entries search bidx in global memory)
        __shared__ uint32_t s_bidx[kBlockListSmem];
        const bool in_smem = bcnt <= kBlockListSmem;
        if (in_smem) {
            for (int i = lane; i < bcnt; i += 32) s_bidx[i] = bidx[i];
            __syncwarp();
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            if (P[h].last < 0) continue;
            int lo = 0, hi = bcnt - 1;
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if ((int)(in_smem ? s_bidx[mid] : __ldg(bidx + mid)) <= P[h].last) lo = mid;
                else hi = mid - 1;
            }
            P[h].last = lo;
        }
        __syncwarp();
    }
    const int wlA = (int)__reduce_max_sync(0xffffffffu, (unsigned)(P[0].last + 1)) - 1;
    const int wlB = (int)__reduce_max_sync(0xffffffffu, (unsigned)(P[1].last + 1)) - 1;
    const int block_last = max(wlA, wlB);
    // COMPACT: the forward's staged (block-culled) list of this block, positions 0.. (last_index
    // holds positions in it); else the tile list from ranges, culled again while staging
    const uint32_t start = COMPACT ? 0u : ranges[2 * tile];
    if (block_last < (int)start) return;  // nothing committed in this block
    const uint32_t* list = COMPACT ? pair_gauss + (size_t)bid * kBlockList : pair_gauss;
    __shared__ ListTail s_tail;
    uint32_t vend;
    const int split = COMPACT ? INT_MAX
                              : list_tail_setup(tt.tails, tt.st_list, tt.st_cover, tile, cp.tiles_x,
                                                ranges[2 * tile + 1], vend, &s_tail, lane == 0, []() { __syncwarp(); });

    const float amax_c = cp.alpha_max, cmin = cp.contribution_min;
    constexpr uint32_t kRowsA = 0xfu << 16, kRowsB = 0xf0u << 16;
    const uint32_t a_r0 = smem_base(sm.r0), a_r1 = smem_base(sm.r1), a_r2 = smem_base(sm.r2);
    const uint32_t a_idx = smem_base(sm.idx), a_gid = smem_base(sm.gid);

    auto pos = [&](int b, int t) -> int {
        const int i = block_last - b * 32 - t;
        return i >= (int)start ? i : -1;
    };
    StagePipe<32, decltype(pos), !COMPACT> pipe(pos, list, rec, &raw, split, &s_tail);
    pipe.start();
    const int nb = (block_last + 1 - (int)start + 31) / 32;
    for (int b = 0; b < nb; ++b) {
        const int cnt = pipe.stage(b, true, bx0, bx1, by0, by1, sm);
        for (int j = 0; j < cnt; j += 2) {
            const bool has_b = j + 1 < cnt;
            const uint32_t jb = has_b ? (uint32_t)(j + 1) : (uint32_t)j;
            const int idx_a = (int)lds_u32(a_idx + 4u * j);
            const int idx_b = has_b ? (int)lds_u32(a_idx + 4u * jb) : INT_MAX;
            const float4 r1a = lds_f4(a_r1 + 16u * j);
            const float4 r1b = lds_f4(a_r1 + 16u * jb);
            const uint32_t ma = __float_as_uint(r1a.z), mb = __float_as_uint(r1b.z);
            // warp-uniform per half: above every commit of the half, or the rect misses the half
            const bool waA = idx_a <= wlA && (ma & kRowsA), waB = idx_a <= wlB && (ma & kRowsB);
            const bool wbA = idx_b <= wlA && (mb & kRowsA), wbB = idx_b <= wlB && (mb & kRowsB);
            if (!(waA || waB || wbA || wbB)) continue;
            const float4 r0a = lds_f4(a_r0 + 16u * j), r0b = lds_f4(a_r0 + 16u * jb);
            float v[18];
            uint32_t ncommit;  // this lane's commits: entry a in the low half-word, b in the high
            // the lane's two pixels share their column: dx and the dx-only products once per entry
            const float dxa = __fsub_rn(r0a.x, P[0].x), dxb = __fsub_rn(r0b.x, P[0].x);
            const float adxa = __fmul_rn(__fmul_rn(r0a.z, dxa), dxa), adxb = __fmul_rn(__fmul_rn(r0b.z, dxb), dxb);
            const float wdxa = __fmul_rn(r0a.w, dxa), wdxb = __fmul_rn(r0b.w, dxb);
            // one half's gates and commits; the first half evaluated assigns v (ACC false)
            auto run_half = [&](auto acc, const int h) {
                constexpr bool ACC = decltype(acc)::value;
                const bool wa = h == 0 ? waA : waB, wb = h == 0 ? wbA : wbB;
                PixBwd& q = P[h];
                float alpha_a, g_a, dya, alpha_b, g_b, dyb;
                bool cl_a, cl_b;
                bool ga = gate_sample_col<THR>(r0a, r1a, q.bits, dxa, adxa, wdxa, q.y, amax_c, cmin, alpha_a, g_a, cl_a,
                                               dya);
                bool gb = gate_sample_col<THR>(r0b, r1b, q.bits, dxb, adxb, wdxb, q.y, amax_c, cmin, alpha_b, g_b, cl_b,
                                               dyb);
                ga = ga && wa && idx_a <= q.last;
                gb = gb && wb && idx_b <= q.last;
                commit_sample<ACC>(ga, v, q.T, q.B, q.dL0, q.dL1, q.dL2, lds_f4(a_r2 + 16u * j), alpha_a, g_a,
                                   cl_a, dxa, dya);
                commit_sample<ACC>(gb, v + 9, q.T, q.B, q.dL0, q.dL1, q.dL2, lds_f4(a_r2 + 16u * jb), alpha_b,
                                   g_b, cl_b, dxb, dyb);
                const uint32_t nh = (ga ? 1u : 0u) + (gb ? 0x10000u : 0u);
                ncommit = ACC ? ncommit + nh : nh;
#ifdef SPLAT_STATS
                {  // [0] half-entries evaluated, [1] of which with a commit, [2] eligible lanes, [3] commits
                    const unsigned ca = __ballot_sync(0xffffffffu, ga), cb = __ballot_sync(0xffffffffu, gb);
                    const unsigned ea = __ballot_sync(0xffffffffu, wa && idx_a <= q.last);
                    const unsigned eb = __ballot_sync(0xffffffffu, wb && idx_b <= q.last);
                    if (lane == 0) {
                        atomicAdd(&g_bstats[0], (unsigned long long)(wa + wb));
                        atomicAdd(&g_bstats[1], (unsigned long long)((ca != 0) + (cb != 0)));
                        atomicAdd(&g_bstats[2], (unsigned long long)(__popc(ea) + __popc(eb)));
                        atomicAdd(&g_bstats[3], (unsigned long long)(__popc(ca) + __popc(cb)));
                        atomicAdd(&g_bstats[7], (unsigned long long)(wa != wb));  // half with one eligible entry
                    }
                }
#endif
            };
            // (the skip test above guarantees at least one half)
            if (waA || wbA) {
                run_half(std::false_type{}, 0);
                if (waB || wbB) run_half(std::true_type{}, 1);
            } else {
                run_half(std::false_type{}, 1);
            }
            // the warp's commit counts of both entries in one reduction (<= 64 each)
            const uint32_t nc = __reduce_add_sync(0xffffffffu, ncommit);
            const int cnt_a = (int)(nc & 0xffffu), cnt_b = (int)(nc >> 16);
            const bool any_a = cnt_a > 0, any_b = cnt_b > 0;
#ifdef SPLAT_STATS
            if (lane == 0) {
                atomicAdd(&g_bstats[4], 1ull);
                atomicAdd(&g_bstats[5], (unsigned long long)(any_a + any_b));
                atomicAdd(&g_bstats[6], (unsigned long long)(any_a != any_b));  // single-entry reductions
            }
#endif
            if (any_a || any_b) emit_entry_grads(v, lane, cnt_a, cnt_b, (uint32_t)j, jb, a_gid, grad2d);
        }
    }
    pipe.finish();
}

template <bool THR>
__global__ void __launch_bounds__(32) blend_backward_px2_persistent(
    CamParams cp, const uint32_t* __restrict__ ranges, const uint32_t* __restrict__ pair_gauss,
    const ProjRec* __restrict__ rec, const float* __restrict__ t_final, const int32_t* __restrict__ last_index,
    float bg0, float bg1, float bg2, const float* __restrict__ d_color, const float* __restrict__ color,
    const float* __restrict__ target, float inv_n, float* __restrict__ loss_partials, float4* __restrict__ grad2d,
    int nblocks, int* __restrict__ counter, const uint32_t* __restrict__ blist, const uint32_t* __restrict__ bidx,
    const int32_t* __restrict__ bcount, const uint32_t* __restrict__ cls_cnt, const uint32_t* __restrict__ cls_list,
    TileTails tt) {
    // Work order: the forward filed every block under a cost class (heaviest first); lane l holds
    // the exclusive starts of classes 2l and 2l + 1, so the k-th pull maps to (class, rank) with
    // two ballots.  Without classes the blocks go in raster order.
    const int lane = threadIdx.x;
    uint32_t e0 = 0, e1 = 0;
    if (cls_cnt) {
        const uint32_t c0 = cls_cnt[2 * lane], c1 = cls_cnt[2 * lane + 1];
        uint32_t incl = c0 + c1;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += u;
        }
        e0 = incl - c0 - c1;
        e1 = e0 + c0;
    }
    for (;;) {
        int b = 0;
        if (threadIdx.x == 0) b = pull_work(counter, nblocks);
        b = __shfl_sync(0xffffffffu, b, 0);
        if (b >= nblocks) break;
        if (cls_cnt) {
            const unsigned m0 = __ballot_sync(0xffffffffu, e0 <= (uint32_t)b);
            const unsigned m1 = __ballot_sync(0xffffffffu, e1 <= (uint32_t)b);
            const int c = __popc(m0) + __popc(m1) - 1;
            const uint32_t ex = __shfl_sync(0xffffffffu, (c & 1) ? e1 : e0, c >> 1);
            b = (int)cls_list[(size_t)c * nblocks + ((uint32_t)b - ex)];
        }
        const int bc = blist ? bcount[b] : kBlockList + 1;
        if (bc <= kBlockList)
            blend_backward_block_px2<THR, true>(b, cp, ranges, tt, blist, rec, t_final, last_index, bg0, bg1, bg2,
                                                d_color, color, target, inv_n, loss_partials, grad2d,
                                                bidx + (size_t)b * kBlockList, bc);
        else
            blend_backward_block_px2<THR, false>(b, cp, ranges, tt, pair_gauss, rec, t_final, last_index, bg0, bg1, bg2,
                                                 d_color, color, target, inv_n, loss_partials, grad2d, nullptr, 0);
        __syncwarp();
    }
}

template <bool THR, int BW, int BH>
__global__ void __launch_bounds__(BW * BH) blend_backward_kernel(CamParams cp, const uint32_t* __restrict__ ranges,
                                                            TileTails tt, const uint32_t* __restrict__ pair_gauss,
                                                            const ProjRec* __restrict__ rec,
                                                            const float* __restrict__ t_final,
                                                            const int32_t* __restrict__ last_index, float bg0,
                                                            float bg1, float bg2, const float* __restrict__ d_color,
                                                            const float* __restrict__ color,
                                                            const float* __restrict__ target, float inv_n,
                                                            float* __restrict__ loss_partials,
                                                            float4* __restrict__ grad2d) {
    blend_backward_block<THR, BW, BH>((int)blockIdx.x, cp, ranges, tt, pair_gauss, rec, t_final, last_index, bg0, bg1, bg2, d_color, color, target, inv_n, loss_partials, grad2d);
}

template <bool THR, int BW, int BH>
__global__ void __launch_bounds__(BW * BH) blend_backward_persistent(CamParams cp, const uint32_t* __restrict__ ranges,
                                                            TileTails tt, const uint32_t* __restrict__ pair_gauss,
                                                            const ProjRec* __restrict__ rec,
                                                            const float* __restrict__ t_final,
                                                            const int32_t* __restrict__ last_index, float bg0,
                                                            float bg1, float bg2, const float* __restrict__ d_color,
                                                            const float* __restrict__ color,
                                                            const float* __restrict__ target, float inv_n,
                                                            float* __restrict__ loss_partials,
                                                            float4* __restrict__ grad2d,
                                                            int nblocks, int* __restrict__ counter) {
    __shared__ int s_bid;
    for (;;) {
        __syncthreads();
        if (threadIdx.x == 0) s_bid = pull_work(counter, nblocks);
        __syncthreads();
        const int b = s_bid;
        if (b >= nblocks) break;
        blend_backward_block<THR, BW, BH>(b, cp, ranges, tt, pair_gauss, rec, t_final, last_index, bg0, bg1, bg2, d_color, color, target, inv_n, loss_partials, grad2d);
    }
}

constexpr int kL1Threads = 256;
constexpr int kL1Items = 8;

__global__ void __launch_bounds__(kL1Threads) l1_kernel(const float* __restrict__ a, const float* __restrict__ b,
                                                      int64_t n, float* __restrict__ grad,
                                                      float* __restrict__ partials) {
    __shared__ float s_red[kL1Threads / 32];
    const float inv_n = 1.0f / (float)n;
    float l = 0.0f;
    const int64_t base = (int64_t)blockIdx.x * kL1Threads * kL1Items;
#pragma unroll
    for (int k = 0; k < kL1Items; ++k) {
        const int64_t i = base + (int64_t)k * kL1Threads + threadIdx.x;
        if (i < n) {
            const float d = a[i] - b[i];
            l += fabsf(d);
            if (grad) grad[i] = d > 0.0f ? inv_n : (d < 0.0f ? -inv_n : 0.0f);
        }
    }
    l = warp_sum(l);
    if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = l;
    __syncthreads();
    if (threadIdx.x == 0) {
        float s = 0.0f;
        for (int w = 0; w < kL1Threads / 32; ++w) s += s_red[w];
        partials[blockIdx.x] = s;
    }
}

// Deterministic final sum (fixed order, fp64 accumulation).  1024 threads, 4 independent
// accumulators per thread so the partial loads are in flight together.
constexpr int kLossThreads = 1024;
__global__ void __launch_bounds__(kLossThreads) loss_reduce_kernel(const float* __restrict__ partials, int n,
                                                                   float inv_n, float* __restrict__ loss) {
    // one CTA; 16 independent loads in flight per thread, fp64 accumulation (order fixed by n)
    __shared__ double s[kLossThreads / 32];
    constexpr int kU = 16;
    double acc = 0.0;
    for (int base = 0; base < n; base += kLossThreads * kU) {
        float v[kU];
#pragma unroll
        for (int k = 0; k < kU; ++k) {
            const int i = base + k * kLossThreads + threadIdx.x;
            v[k] = i < n ? partials[i] : 0.0f;
        }
#pragma unroll
        for (int k = 0; k < kU; ++k) acc += (double)v[k];
    }
    double w = acc;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = w;
    __syncthreads();
    if (threadIdx.x < 32) {
        w = threadIdx.x < kLossThreads / 32 ? s[threadIdx.x] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
        if (threadIdx.x == 0) *loss = (float)w * inv_n;
    }
}

// adam_delta (optimizer.cpp:29-36) with every fp64 operation explicitly rounded (no DFMA), so
// the update is bit-identical to the reference's.  One element: returns the new parameter and
// writes the new moments.  mf == 0 (eps > 0) gives delta = +-0 exactly (0 / positive), so the three fp64
// divisions and the square root (whose zero operands take the slow library paths) are skipped.
__device__ __forceinline__ float adam_one(float p, float gr, float& m, float& v, double l, double b1, double omb1,
                                          double b2, double omb2, double eps, double bias1, double bias2) {
    const double g = (double)gr;
    const float mf = (float)__dadd_rn(__dmul_rn(b1, (double)m), __dmul_rn(omb1, g));
    const float vf = (float)__dadd_rn(__dmul_rn(b2, (double)v), __dmul_rn(__dmul_rn(omb2, g), g));
    m = mf;
    v = vf;
    float delta;
    if (mf == 0.0f && vf >= 0.0f && vf < INFINITY && eps > 0.0) {
        delta = copysignf(0.0f, mf);  // l * (+-0 / bias1) / (sqrt(v_hat) + eps), all factors positive
    } else {
        const double m_hat = __ddiv_rn((double)mf, bias1);
        const double v_hat = __ddiv_rn((double)vf, bias2);
        delta = (float)__ddiv_rn(__dmul_rn(l, m_hat), __dadd_rn(__dsqrt_rn(v_hat), eps));
    }
    return __fsub_rn(p, delta);
}

// Four consecutive elements per thread (float4 traffic when the group is 16-byte aligned), so four
// independent fp64 chains are in flight per thread.  SH: per-48 rows, coefficients k >= 3 use
// lr_alt (rows start at multiples of 48, so a 4-element group never straddles a row).
template <bool SH, bool VEC>
__global__ void __launch_bounds__(256) adam_kernel(float* __restrict__ param, const float* __restrict__ grad,
                                                   float* __restrict__ m, float* __restrict__ v, int64_t count,
                                                   double lr, double lr_alt, double b1, double omb1, double b2,
                                                   double omb2, double eps, double bias1, double bias2,
                                                   int sh_phase) {
    pdl_wait();
    const int64_t i0 = 4 * ((int64_t)blockIdx.x * blockDim.x + threadIdx.x);
    if (i0 >= count) return;
    // position of element i0 inside its 48-value SH row (sh_phase: the row position of element 0,
    // nonzero when a shard of the packed buffer starts mid-row); a 4-group may straddle rows then
    const int r0 = SH ? (int)((i0 + sh_phase) % 48) : 0;
    if (VEC && i0 + 4 <= count) {
        float4 p4 = *reinterpret_cast<const float4*>(param + i0);
        const float4 g4 = __ldg(reinterpret_cast<const float4*>(grad + i0));
        float4 m4 = *reinterpret_cast<const float4*>(m + i0);
        float4 v4 = *reinterpret_cast<const float4*>(v + i0);
        p4.x = adam_one(p4.x, g4.x, m4.x, v4.x, SH && r0 % 48 >= 3 ? lr_alt : lr, b1, omb1, b2, omb2, eps, bias1, bias2);
        p4.y = adam_one(p4.y, g4.y, m4.y, v4.y, SH && (r0 + 1) % 48 >= 3 ? lr_alt : lr, b1, omb1, b2, omb2, eps, bias1, bias2);
        p4.z = adam_one(p4.z, g4.z, m4.z, v4.z, SH && (r0 + 2) % 48 >= 3 ? lr_alt : lr, b1, omb1, b2, omb2, eps, bias1, bias2);
        p4.w = adam_one(p4.w, g4.w, m4.w, v4.w, SH && (r0 + 3) % 48 >= 3 ? lr_alt : lr, b1, omb1, b2, omb2, eps, bias1, bias2);
        *reinterpret_cast<float4*>(param + i0) = p4;
        *reinterpret_cast<float4*>(m + i0) = m4;
        *reinterpret_cast<float4*>(v + i0) = v4;
        return;
    }
    for (int k = 0; k < 4 && i0 + k < count; ++k) {
        const int64_t i = i0 + k;
        float mm = m[i], vv = v[i];
        param[i] = adam_one(param[i], grad[i], mm, vv, SH && (r0 + k) % 48 >= 3 ? lr_alt : lr, b1, omb1, b2, omb2, eps,
                            bias1, bias2);
        m[i] = mm;
        v[i] = vv;
    }
}

// normalized_quat (gaussian_set.hpp:15-20) in place, optimizer.cpp:69
__global__ void quat_normalize_kernel(float* __restrict__ q, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float* p = q + 4 * (size_t)i;
    const float w = p[0], x = p[1], y = p[2], z = p[3];
    const float s = __fadd_rn(__fadd_rn(__fmul_rn(w, w), __fmul_rn(x, x)), __fadd_rn(__fmul_rn(y, y), __fmul_rn(z, z)));
    const float nn = __fsqrt_rn(s);
    if (!(nn > 0.0f)) {
        p[0] = 1.0f; p[1] = p[2] = p[3] = 0.0f;
        return;
    }
    p[0] = __fdiv_rn(w, nn); p[1] = __fdiv_rn(x, nn); p[2] = __fdiv_rn(y, nn); p[3] = __fdiv_rn(z, nn);
}

inline unsigned blocks_for(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

}  // namespace

cudaError_t launch_blend_backward(LaunchCtx& lc, const CamParams& cp, const uint32_t* ranges, TileTails tt,
                                  const uint32_t* pair_gauss, const ProjRec* rec, const float* t_final,
                                  const int32_t* last_index, const float bg[3], const float* d_color,
                                  const float* color, const float* target, float* loss_partials, float* grad2d,
                                  const uint32_t* blist, const uint32_t* bidx, const int32_t* bcount,
                                  const uint32_t* cls_cnt, const uint32_t* cls_list) {
    const int ts = cp.tile_size;
    const unsigned grid = (unsigned)(cp.tiles_x * cp.tiles_y * (ts / cp.block_w) * (ts / cp.block_h));
    const float inv_n = 1.0f / (float)(3 * (int64_t)cp.width * cp.height);
    {
        LaunchScope ls_(lc, "blend_backward");
#define BLEND_BWD_SHAPE(T, W, H)                                                                                  \
    do {                                                                                                          \
        if (lc.persistent_blend && lc.work_counters) {                                                            \
            static int per_sm = 0;                                                                                \
            if (!per_sm) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, blend_backward_persistent<T, W, H>, \
                                                                      W * H, 0);                                  \
            const unsigned pg = (unsigned)(lc.num_sms * (per_sm > 0 ? per_sm : 1));                              \
            blend_backward_persistent<T, W, H><<<pg < grid ? pg : grid, W * H, 0, lc.stream>>>(                  \
                cp, ranges, tt, pair_gauss, rec, t_final, last_index, bg[0], bg[1], bg[2], d_color, color, target,  \
                inv_n, loss_partials, reinterpret_cast<float4*>(grad2d), (int)grid, lc.work_counters + 1);       \
        } else {                                                                                                  \
            blend_backward_kernel<T, W, H><<<grid, W * H, 0, lc.stream>>>(                                       \
                cp, ranges, tt, pair_gauss, rec, t_final, last_index, bg[0], bg[1], bg[2], d_color, color, target,  \
                inv_n, loss_partials, reinterpret_cast<float4*>(grad2d));                                         \
        }                                                                                                         \
    } while (0)
#define BLEND_BWD(T)                                             \
    do {                                                         \
        if (cp.block_w == 16) BLEND_BWD_SHAPE(T, 16, 16);        \
        else if (cp.block_h == 8) BLEND_BWD_SHAPE(T, 8, 8);      \
        else BLEND_BWD_SHAPE(T, 8, 4);                           \
    } while (0)
        if (lc.bwd_px2 && cp.block_w == 8 && cp.block_h == 8 && lc.work_counters) {
            static int per_sm[2] = {0, 0};
            const int k = cp.apply_thresholds ? 1 : 0;
            if (!per_sm[k]) {
                if (k) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[k], blend_backward_px2_persistent<true>, 32, 0);
                else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[k], blend_backward_px2_persistent<false>, 32, 0);
            }
            unsigned pg = (unsigned)(lc.num_sms * (per_sm[k] > 0 ? per_sm[k] : 1));
            if (pg > grid) pg = grid;
            if (k)
                blend_backward_px2_persistent<true><<<pg, 32, 0, lc.stream>>>(
                    cp, ranges, pair_gauss, rec, t_final, last_index, bg[0], bg[1], bg[2], d_color, color, target,
                    inv_n, loss_partials, reinterpret_cast<float4*>(grad2d), (int)grid, lc.work_counters + 1, blist,
                    bidx, bcount, cls_cnt, cls_list, tt);
            else
                blend_backward_px2_persistent<false><<<pg, 32, 0, lc.stream>>>(
                    cp, ranges, pair_gauss, rec, t_final, last_index, bg[0], bg[1], bg[2], d_color, color, target,
                    inv_n, loss_partials, reinterpret_cast<float4*>(grad2d), (int)grid, lc.work_counters + 1, blist,
                    bidx, bcount, cls_cnt, cls_list, tt);
        } else if (cp.apply_thresholds) BLEND_BWD(true);
        else BLEND_BWD(false);
#undef BLEND_BWD
#undef BLEND_BWD_SHAPE
    }
    lc.count++;
    return cudaGetLastError();
}

// Device floats straight into mapped pinned host memory (the per-view losses of a training step):
// a kernel instead of a copy-engine transfer, which would queue behind bulk host copies.
// The per-view losses to mapped host memory, then (seq != 0) a sequence number in the slot after
// them once the values are visible system-wide: the host polls that word instead of waiting for
// the stream (a synchronisation's wake-up costs more than the polling).
__global__ void copy_to_host_kernel(const float* __restrict__ src, float* dst_mapped, int n, uint32_t seq) {
    pdl_wait();
    for (int i = threadIdx.x; i < n; i += blockDim.x) reinterpret_cast<volatile float*>(dst_mapped)[i] = src[i];
    if (seq) {
        __threadfence_system();
        __syncthreads();
        if (threadIdx.x == 0) reinterpret_cast<volatile uint32_t*>(dst_mapped)[n] = seq;
    }
}

cudaError_t launch_copy_to_host(LaunchCtx& lc, const float* src, float* dst_mapped, int n, uint32_t seq) {
    if (n <= 0) return cudaSuccess;
    const cudaError_t e = launch_pdl(lc.stream, copy_to_host_kernel, dim3(1), dim3(128), 0, src, dst_mapped, n, seq);
    lc.count++;
    return e;
}

cudaError_t launch_loss_reduce(LaunchCtx& lc, const float* partials, int n, float inv_n, float* loss) {
    {
        LaunchScope ls_(lc, "loss_reduce");
        loss_reduce_kernel<<<1, kLossThreads, 0, lc.stream>>>(partials, n, inv_n, loss);
    }
    lc.count++;
    return cudaGetLastError();
}

int l1_partials_count(int64_t n) { return (int)((n + kL1Threads * kL1Items - 1) / (kL1Threads * kL1Items)); }

cudaError_t launch_l1(LaunchCtx& lc, const float* a, const float* b, int64_t n, float* grad, float* partials,
                      int n_partials) {
    if (n == 0) return cudaSuccess;
    l1_kernel<<<n_partials, kL1Threads, 0, lc.stream>>>(a, b, n, grad, partials);
    lc.count++;
    return cudaGetLastError();
}

cudaError_t launch_adam(LaunchCtx& lc, const AdamGroupArgs& a, double beta1, double beta2, double eps, double bias1,
                        double bias2) {
    if (a.count == 0) return cudaSuccess;
    {
        LaunchScope ls_(lc, "adam");
        const bool vec = ((reinterpret_cast<uintptr_t>(a.param) | reinterpret_cast<uintptr_t>(a.grad) |
                           reinterpret_cast<uintptr_t>(a.m) | reinterpret_cast<uintptr_t>(a.v)) & 15u) == 0;
        const unsigned grid = blocks_for((a.count + 3) / 4, 256);
#define ADAM_LAUNCH(SH, VEC)                                                                                      \
    launch_pdl(lc.stream, adam_kernel<SH, VEC>, dim3(grid), dim3(256), 0, a.param, a.grad, a.m, a.v, a.count, a.lr,  \
               a.lr_alt, beta1, 1.0 - beta1, beta2, 1.0 - beta2, eps, bias1, bias2, a.sh_phase)
        if (a.sh_layout) {
            if (vec) ADAM_LAUNCH(true, true);
            else ADAM_LAUNCH(true, false);
        } else {
            if (vec) ADAM_LAUNCH(false, true);
            else ADAM_LAUNCH(false, false);
        }
#undef ADAM_LAUNCH
    }
    lc.count++;
    return cudaGetLastError();
}

cudaError_t launch_quat_normalize(LaunchCtx& lc, float* rotations, int n) {
    if (n == 0) return cudaSuccess;
    {
        LaunchScope ls_(lc, "quat_normalize");
        quat_normalize_kernel<<<blocks_for(n, 256), 256, 0, lc.stream>>>(rotations, n);
    }
    lc.count++;
    return cudaGetLastError();
}

}  // namespace splat_b200

extern "C" int splat_debug_bstats(unsigned long long* out, int reset) {
#ifdef SPLAT_STATS
    cudaDeviceSynchronize();
    if (cudaMemcpyFromSymbol(out, splat_b200::g_bstats, sizeof(unsigned long long) * 8) != cudaSuccess) return 3;
    if (reset) {
        unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        cudaMemcpyToSymbol(splat_b200::g_bstats, z, sizeof(z));
    }
    return 0;
#else
    (void)out;
    (void)reset;
    return -1;
#endif
}
