// common.cuh — shared device-side definitions for the sm_100a rasterizer kernels.
//
// Bit-exactness contract: everything that decides an integer output
// (pixel rects, tile keys, per-tile lists, gates, argmax) or a forward image value is computed
// with correctly rounded, non-contracted IEEE operations in the reference's operation order
// (as fixed by oracle/compat/Eigen/Dense), and with the shared splat_expf.  forward.cu is
// compiled with --fmad=false; the per-sample gate below uses explicit _rn intrinsics so the
// backward (compiled with FMA contraction on) replays the forward's alphas bit for bit.
#pragma once

#include <climits>
#include <cstdint>
#include <cuda_runtime.h>

#include "splat_expf.h"

namespace splat_b200 {

constexpr int kBlock = 256;  // threads per tile CTA (16 x 16 pixels)

// 2D gradient accumulator of blend_backward: 3 float4 per Gaussian in moment form (backward.cu
// commit_sample), (S0, Sx, Sy, 0), (Sxx, Sxy, Syy, 0), (dcolour rgb, committed (warp, pixel) samples).
constexpr int kG2Stride = 3;
constexpr size_t grad2d_bytes(size_t n) { return n * 16 * kG2Stride; }

// Projected Gaussian record, 48 B (3 x float4), indexed by Gaussian id:
//   r0 = (mean2d.x, mean2d.y, conic0, conic1)
//   r1 = (conic2, opacity, eff x0 | x1 << 16, eff y0 | y1 << 16)
//   r2 = (color.r, color.g, color.b, cut)
// The effective rect is the reference pixel rect (rasterizer.cpp:63-68) intersected with the
// bounding box of the ellipse where alpha can reach the contribution floor; cut = ln(cmin /
// opacity) - 1e-3 (-inf in exact mode).  The reference rect itself (which defines the tile lists)
// is kept in a separate uint2 array for binning.
struct __align__(16) ProjRec {
    float4 r0, r1, r2;
};

// Auxiliary record for depth rendering (rasterizer.cpp:278-281): world center, symmetric
// inverse 3D covariance (or identity-flagged degenerate), 48 B.
//   a0 = (cx, cy, cz, degenerate ? 1 : 0), a1 = (i00, i01, i02, i11), a2 = (i12, i22, 0, 0)
struct __align__(16) AuxRec {
    float4 a0, a1, a2;
};

// normalized_quat / rotation_from_quat (gaussian_set.hpp:15-37) in the reference's operation
// order; bit-exact only in translation units compiled with --fmad=false (chain.cu, densify.cu).
__device__ __forceinline__ void normalized_quat(float w, float x, float y, float z, float q[4]) {
    const float n = sqrtf((w * w + x * x) + (y * y + z * z));
    if (!(n > 0.0f)) {
        q[0] = 1.0f; q[1] = q[2] = q[3] = 0.0f;
        return;
    }
    q[0] = w / n; q[1] = x / n; q[2] = y / n; q[3] = z / n;
}

__device__ __forceinline__ void rotation_from_quat(const float qr[4], float r[9]) {
    float q[4];
    normalized_quat(qr[0], qr[1], qr[2], qr[3], q);
    const float w = q[0], x = q[1], y = q[2], z = q[3];
    r[0] = 1.0f - 2.0f * (y * y + z * z);
    r[1] = 2.0f * (x * y - w * z);
    r[2] = 2.0f * (x * z + w * y);
    r[3] = 2.0f * (x * y + w * z);
    r[4] = 1.0f - 2.0f * (x * x + z * z);
    r[5] = 2.0f * (y * z - w * x);
    r[6] = 2.0f * (x * z - w * y);
    r[7] = 2.0f * (y * z + w * x);
    r[8] = 1.0f - 2.0f * (x * x + y * y);
}

// Camera + raster constants passed by value to kernels.
struct CamParams {
    int width, height;
    float fx, fy, cx, cy;
    float R[9];
    float t[3];
    float center[3];  // -(R^T t), computed on the host in the reference's order
    float znear;
    int tile_size, tiles_x, tiles_y;
    int block_w, block_h;  // pixel block of one blend CTA (16x16, 8x8 or 8x4; divides the tile)
    int apply_thresholds;
    float lowpass, radius_sigmas, alpha_max, contribution_min, transmittance_min;
    float log_cond_limit;  // float(log(1e12))
};

// Programmatic dependent launch (PDL): kernels launched with launch_pdl (internal.h) may start
// while their predecessor in the stream finishes; pdl_wait() blocks until the predecessor grid has
// completed and its memory is visible (a no-op for a normal launch), and pdl_trigger() lets the
// successor's CTAs be scheduled once every CTA of this grid has issued it.  Every PDL-launched
// kernel waits before touching global memory.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Work queue of the persistent blend kernels (one thread per CTA calls it): returns the next pixel
// block.  The last CTA to run dry re-zeroes the queue and its exit count (counter[8]), so the
// counter is zero at rest and no memset precedes a launch.
__device__ __forceinline__ int pull_work(int* counter, int nblocks) {
    const int b = atomicAdd(counter, 1);
    if (b >= nblocks && atomicAdd(counter + 8, 1) == (int)gridDim.x - 1) {
        atomicExch(counter, 0);
        atomicExch(counter + 8, 0);
    }
    return b;
}

__device__ __forceinline__ uint32_t pack_range(int lo, int hi) {
    return (uint32_t)lo | ((uint32_t)hi << 16);
}
__device__ __forceinline__ int range_lo(float f) { return (int)(__float_as_uint(f) & 0xffffu); }
__device__ __forceinline__ int range_hi(float f) { return (int)(__float_as_uint(f) >> 16); }

// Per-sample gate of traverse_pixel (rasterizer.hpp:125-143), shared by the forward and the
// backward so both see identical alphas.  r1 is the STAGED record (stage_batch): r1.z holds the
// block-relative pixel masks of the effective rect (columns in bits 0-15, rows in 16-31) and r1.w
// the cut.  Returns false when the sample is skipped: outside the rect, power > 0, power below the
// cut (alpha would be below the floor), or alpha below the contribution floor.  The extra skips
// only ever drop samples the reference skips too (see may_contribute / preprocess), and all
// arithmetic deciding the committed set is explicitly rounded: no FMA contraction.
template <bool THR>
__device__ __forceinline__ bool gate_sample(const float4& r0, const float4& r1, uint32_t mybits, float x, float y,
                                            float alpha_max, float contribution_min, float& alpha, float& g2d,
                                            bool& clamped, float& dx, float& dy) {
    if ((__float_as_uint(r1.z) & mybits) != mybits) return false;
    dx = __fsub_rn(r0.x, x);
    dy = __fsub_rn(r0.y, y);
    // power = -0.5 * (c0 dx dx + c2 dy dy) - c1 dx dy
    const float a = __fmul_rn(__fmul_rn(r0.z, dx), dx);
    const float b = __fmul_rn(__fmul_rn(r1.x, dy), dy);
    const float m = __fmul_rn(-0.5f, __fadd_rn(a, b));
    const float power = __fsub_rn(m, __fmul_rn(__fmul_rn(r0.w, dx), dy));
    if (power > 0.0f) return false;
    clamped = false;
    if (THR) {
        if (power < r1.w) return false;
        g2d = splat_expf_core(power);  // argument in [cut, 0]: bit-identical to splat_expf
        alpha = __fmul_rn(r1.y, g2d);
        if (alpha > alpha_max) {
            alpha = alpha_max;
            clamped = true;
        }
        if (alpha < contribution_min) return false;
    } else {
        g2d = splat_expf(power);
        alpha = __fmul_rn(r1.y, g2d);
    }
    return true;
}

// Branch-free form of gate_sample: the same explicitly rounded operations (identical alpha for
// every sample that passes), but every step is computed and the skips are folded into the
// returned predicate, so two samples' gates can be evaluated as independent instruction streams.
template <bool THR>
__device__ __forceinline__ bool gate_sample_nb(const float4& r0, const float4& r1, uint32_t mybits, float x, float y,
                                               float alpha_max, float contribution_min, float& alpha, float& g2d,
                                               bool& clamped, float& dx, float& dy) {
    const bool inrect = (__float_as_uint(r1.z) & mybits) == mybits;
    dx = __fsub_rn(r0.x, x);
    dy = __fsub_rn(r0.y, y);
    const float a = __fmul_rn(__fmul_rn(r0.z, dx), dx);
    const float b = __fmul_rn(__fmul_rn(r1.x, dy), dy);
    const float m = __fmul_rn(-0.5f, __fadd_rn(a, b));
    const float power = __fsub_rn(m, __fmul_rn(__fmul_rn(r0.w, dx), dy));
    bool ok = inrect && !(power > 0.0f);
    if (THR) {
        ok = ok && !(power < r1.w);
        // unconditional: measured faster than a branch around it for the lanes that need it
        // (forward 301 -> 311 us, backward 491 -> 538 us)
        g2d = splat_expf_gate(power);  // meaningless (never used) outside [cut, 0]
        alpha = __fmul_rn(r1.y, g2d);
        clamped = alpha > alpha_max;
        alpha = clamped ? alpha_max : alpha;
        ok = ok && !(alpha < contribution_min);
    } else {
        g2d = splat_expf(power);
        alpha = __fmul_rn(r1.y, g2d);
        clamped = false;
    }
    return ok;
}

// gate_sample_nb with the column terms precomputed (the two pixels of a backward lane share x):
// dx = mean.x - x, adx = (conic0 dx) dx, wdx = conic1 dx — the same rounded operations, so the
// same alpha bits.
template <bool THR>
__device__ __forceinline__ bool gate_sample_col(const float4& r0, const float4& r1, uint32_t mybits, float dx,
                                                float adx, float wdx, float y, float alpha_max, float contribution_min,
                                                float& alpha, float& g2d, bool& clamped, float& dy) {
    const bool inrect = (__float_as_uint(r1.z) & mybits) == mybits;
    dy = __fsub_rn(r0.y, y);
    const float b = __fmul_rn(__fmul_rn(r1.x, dy), dy);
    const float m = __fmul_rn(-0.5f, __fadd_rn(adx, b));
    const float power = __fsub_rn(m, __fmul_rn(wdx, dy));
    bool ok = inrect && !(power > 0.0f);
    if (THR) {
        ok = ok && !(power < r1.w);
        g2d = splat_expf_gate(power);  // meaningless (never used) outside [cut, 0]
        alpha = __fmul_rn(r1.y, g2d);
        clamped = alpha > alpha_max;
        alpha = clamped ? alpha_max : alpha;
        ok = ok && !(alpha < contribution_min);
    } else {
        g2d = splat_expf(power);
        alpha = __fmul_rn(r1.y, g2d);
        clamped = false;
    }
    return ok;
}

// Exactness-preserving block cull.  The Gaussian can pass the alpha gate somewhere in the pixel
// block [bx0, bx1) x [by0, by1) only if (a) its pixel rect meets the block and (b) the maximum of
// power = -q(dx, dy) / 2 over the block's pixel centres reaches cut = ln(cmin / opacity) - 1e-3
// (r2.w, written by preprocess; -inf in exact mode).  (b) bounds the discrete maximum by the
// continuous one over the box of pixel centres: q is a positive-definite quadratic, so its
// minimum over a box is 0 when the box holds the origin and otherwise lies on an edge, where it
// is a clamped 1-D vertex.  The 1e-3 margin in the exponent dwarfs every rounding involved (q is
// evaluated to ~1e-6 relative, splat_expf to 1 ulp), so a culled sample would have been skipped
// by the per-pixel gate anyway: the committed set, and every output bit, are unchanged.
// (b) alone, over the pixel box [X0, X1) x [Y0, Y1) (non-empty): r0 = (mean, conic0, conic1), c =
// conic2.
__device__ __forceinline__ bool quad_box_reaches(const float4& r0, float c, float cut, int X0, int X1, int Y0,
                                                 int Y1) {
    if (!(cut > -INFINITY)) return true;
    // dx = mean.x - (px + 0.5) over px in [X0, X1 - 1]
    const float dxl = r0.x - ((float)X1 - 0.5f), dxh = r0.x - ((float)X0 + 0.5f);
    const float dyl = r0.y - ((float)Y1 - 0.5f), dyh = r0.y - ((float)Y0 + 0.5f);
    float qmin = 0.0f;
    const bool inside = dxl <= 0.0f && dxh >= 0.0f && dyl <= 0.0f && dyh >= 0.0f;
    if (!inside) {
        const float a = r0.z, b = r0.w;
        // q minus a rounding bound proportional to the magnitudes of its terms: the per-pixel
        // gate evaluates the same quadratic in another order, and for elongated Gaussians the
        // terms cancel (|terms| >> q), so the cull must not trust q beyond ~1e-5 of sum |terms|.
        // Explicit FMAs and approximate reciprocals (forward.cu is compiled --fmad=false for the
        // gates): the cull only needs q to ~1e-6 relative, far inside its 1e-5 bound and the
        // 1e-3 margin in cut, and an approximate vertex moves q by O(error^2) at the minimum.
        auto q_lo = [&](float dx, float dy) {
            const float t0 = __fmul_rn(__fmul_rn(a, dx), dx), t1 = __fmul_rn(__fmul_rn(2.0f * b, dx), dy);
            const float t2 = __fmul_rn(__fmul_rn(c, dy), dy);
            return __fmaf_rn(-1e-5f, t0 + fabsf(t1) + t2, t0 + t1 + t2);
        };
        // Only edges facing the centre (the origin of (dx, dy)) can hold the minimum: at a
        // boundary minimiser p, -grad q(p) lies in the box's outward normal cone, and convexity
        // (q(0) <= q(p)) puts the centre on the outer side of that edge's line.  At most one
        // x-edge and one y-edge face it; the edge picked when none faces only adds a box point.
        const float ia = __fdividef(1.0f, a), ic = __fdividef(1.0f, c);
        const float ex = dxl > 0.0f ? dxl : dxh, ey = dyl > 0.0f ? dyl : dyh;
        const float y_at_x = fminf(fmaxf(-b * ex * ic, dyl), dyh);
        const float x_at_y = fminf(fmaxf(-b * ey * ia, dxl), dxh);
        qmin = fminf(q_lo(ex, y_at_x), q_lo(x_at_y, ey));
    }
    return -0.5f * qmin >= cut;
}

__device__ __forceinline__ bool may_contribute(const float4& r0, const float4& r1, float cut, int bx0, int bx1,
                                               int by0, int by1) {
    const int X0 = max(range_lo(r1.z), bx0), X1 = min(range_hi(r1.z), bx1);
    const int Y0 = max(range_lo(r1.w), by0), Y1 = min(range_hi(r1.w), by1);
    if (X0 >= X1 || Y0 >= Y1) return false;
    return quad_box_reaches(r0, r1.x, cut, X0, X1, Y0, Y1);
}

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm volatile("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Stage one batch of list entries [idx_of(0), ...) in shared memory, keeping only Gaussians that
// pass the exact block cull (common.cuh may_contribute); order is preserved by a ballot/prefix
// compaction.  Returns the number of staged entries.  s_idx keeps each entry's absolute position
// in the sorted pair array (the "list position" of the reference).
// 32-bit shared-window loads.  nvcc re-derives the shared window base (S2R SR_CgaCtaId + LEA)
// inside hot loops when it addresses __shared__ arrays by name; taking the base once as a 32-bit
// shared address, laundered through an empty asm so it stays in a register, and loading with
// ld.shared keeps the inner loops free of that overhead.
__device__ __forceinline__ uint32_t smem_base(const void* p) {
    uint32_t a = (uint32_t)__cvta_generic_to_shared(p);
    asm volatile("" : "+r"(a));
    return a;
}
__device__ __forceinline__ float4 lds_f4(uint32_t a) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}

// Shared-memory staging area of one batch (one per CTA).
template <int CAP>
struct StageSmem {
    float4 r0[CAP];
    float4 r1[CAP];
    float4 r2[CAP];
    uint32_t gid[CAP];
    int idx[CAP];
    int wcnt[(CAP + 31) / 32];
};

// Stage one batch of list entries in shared memory, keeping only Gaussians that pass the exact
// block cull (may_contribute); order is preserved by a ballot/prefix compaction.  Returns the
// number of staged entries.  sm.idx keeps each entry's absolute position in the sorted pair
// array (the reference's list position); sm.r1 is rewritten to (conic2, opacity, pixel masks of
// the effective rect relative to the block, cut) for gate_sample.
template <int CAP, typename IdxFn>
__device__ __forceinline__ int stage_batch(IdxFn idx_of, int count, const uint32_t* __restrict__ pair_gauss,
                                           const ProjRec* __restrict__ rec, int bx0, int bx1, int by0, int by1,
                                           StageSmem<CAP>& sm) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    bool keep = false;
    ProjRec rr;
    uint32_t gid = 0;
    int idx = 0;
    if (tid < count) {
        idx = idx_of(tid);
        gid = pair_gauss[idx];
        rr = rec[gid];
        keep = may_contribute(rr.r0, rr.r1, rr.r2.w, bx0, bx1, by0, by1);
    }
    const unsigned m = __ballot_sync(0xffffffffu, keep);
    if (lane == 0) sm.wcnt[warp] = __popc(m);
    __syncthreads();
    int off = 0, total = 0;
    for (int w = 0; w < nwarps; ++w) {
        const int c = sm.wcnt[w];
        off += w < warp ? c : 0;
        total += c;
    }
    if (keep) {
        const int pos = off + __popc(m & lanemask_lt());
        const int X0 = max(range_lo(rr.r1.z), bx0) - bx0, X1 = min(range_hi(rr.r1.z), bx1) - bx0;
        const int Y0 = max(range_lo(rr.r1.w), by0) - by0, Y1 = min(range_hi(rr.r1.w), by1) - by0;
        const uint32_t cols = ((1u << X1) - 1u) & ~((1u << X0) - 1u);
        const uint32_t rows = ((1u << Y1) - 1u) & ~((1u << Y0) - 1u);
        sm.r0[pos] = rr.r0;
        sm.r1[pos] = make_float4(rr.r1.x, rr.r1.y, __uint_as_float(cols | (rows << 16)), rr.r2.w);
        sm.r2[pos] = rr.r2;
        sm.gid[pos] = gid;
        sm.idx[pos] = idx;
    }
    __syncthreads();
    return total;
}


// ---- pipelined staging ------------------------------------------------------------------------
// stage_batch gathers each batch with two dependent round trips (list entry -> Gaussian id ->
// 48-byte record) right before the batch is needed, so every batch starts with the whole CTA
// stalled on L2.  StagePipe overlaps that latency with the previous batch's blending: while batch
// b is blended, batch b+1's records are already copied into a raw shared buffer by cp.async
// (their ids were loaded one batch earlier) and batch b+2's ids are in flight into registers.
// stage() then only culls + compacts from shared memory.  Same staged content, same order.
__device__ __forceinline__ void cp_async16(uint32_t smem_addr, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

template <int CAP>
struct StageRaw {
    float4 r[CAP][3];  // one raw ProjRec per thread slot
};

// A tile list whose materialised part stops at a prefix (binning.cu, kListPrefix): positions from
// `split` on are read from the tile's supertile list instead, from entry `first` on, skipping the
// entries whose cover misses the tile (bit `bit`) — the same entries in the same (depth) order as
// the full tile list.  Kept in shared memory (the staging loops read it only past the prefix).
struct ListTail {
    const uint32_t* gauss;  // supertile list (Gaussian ids)
    const uint16_t* cover;  // their 16-bit tile covers
    uint32_t first;         // supertile-list index of virtual position `split`
    uint32_t bit;           // the tile's bit in the covers
};

// Tile t's list: positions [start, mend) in pair_gauss, then (tails[2 t] < tails[2 t + 1]) the
// supertile-list entries [tails[2 t], tails[2 t + 1]) as virtual positions [mend, end).  Sets up
// *tail (call with the CTA / warp converged; `sync` orders the write against earlier readers and
// the pipe's first loads) and returns the split position (INT_MAX when the list is complete).
template <typename Sync>
__device__ __forceinline__ int list_tail_setup(const uint32_t* __restrict__ tails, const uint32_t* __restrict__ st_gauss,
                                               const uint16_t* __restrict__ st_cover, int tile, int tiles_x,
                                               uint32_t mend, uint32_t& end, ListTail* tail, bool leader, Sync sync) {
    end = mend;
    if (!tails) return INT_MAX;
    const uint32_t t0 = tails[2 * tile], t1 = tails[2 * tile + 1];
    if (t0 >= t1) return INT_MAX;
    end = mend + (t1 - t0);
    sync();  // every reader of the previous block's tail is past it
    if (leader) {
        const int tx = tile % tiles_x, ty = tile / tiles_x;
        tail->gauss = st_gauss;
        tail->cover = st_cover;
        tail->first = t0;
        tail->bit = (uint32_t)((ty & 3) * 4 + (tx & 3));  // binning.cu's cover bit (4 x 4 tiles per supertile)
    }
    sync();
    return (int)mend;
}

// PosFn pos(b, t): list position of thread t's entry in batch b, or -1 when batch b has no entry t.
// CULL = false: the list is already block-culled (the forward's per-block list): keep every entry.
template <int CAP, typename PosFn, bool CULL = true, int ITEMS = 1>
struct StagePipe {
    // every user launches CAP / ITEMS threads: compile-time counts let the per-batch warp-count
    // loops unroll (they ran as runtime loops over blockDim)
    static constexpr int kThreads = CAP / ITEMS, kWarps = kThreads / 32;
    // ITEMS entries per thread and batch: slot s = q * blockDim.x + tid holds list position
    // pos(b, s); batches are CAP = ITEMS * blockDim.x entries, compacted in slot order.
    PosFn pos;
    const uint32_t* __restrict__ pair_gauss;
    const ProjRec* __restrict__ rec;
    StageRaw<CAP>* raw;
    int split;              // positions >= split come from *tail (list_tail_setup)
    const ListTail* tail;
    int idx_f[ITEMS];       // entries whose records are in flight to raw (batch b)
    uint32_t gid_f[ITEMS];
    int idx_n[ITEMS];       // entries of batch b + 1, ids loaded into gid_n
    uint32_t gid_n[ITEMS];

    __device__ __forceinline__ StagePipe(PosFn p, const uint32_t* pg, const ProjRec* rc, StageRaw<CAP>* rw,
                                         int split_ = INT_MAX, const ListTail* tail_ = nullptr)
        : pos(p), pair_gauss(pg), rec(rc), raw(rw), split(split_), tail(tail_) {}

    // Gaussian id at list position idx (idx < 0: none); a tail entry whose cover misses the tile
    // becomes an empty slot (idx = -1).
    __device__ __forceinline__ uint32_t fetch(int& idx) const {
        if (idx < 0) return 0u;
        if (idx < split) return __ldg(pair_gauss + idx);
        const uint32_t e = tail->first + (uint32_t)(idx - split);
        const uint32_t cv = __ldg(tail->cover + e), gid = __ldg(tail->gauss + e);
        if (!((cv >> tail->bit) & 1u)) {
            idx = -1;
            return 0u;
        }
        return gid;
    }

    __device__ __forceinline__ void launch_copy() {
#pragma unroll
        for (int q = 0; q < ITEMS; ++q)
            if (idx_f[q] >= 0) {
                const float4* src = reinterpret_cast<const float4*>(rec + gid_f[q]);
                const uint32_t dst =
                    (uint32_t)__cvta_generic_to_shared(&raw->r[q * kThreads + threadIdx.x][0]);
                cp_async16(dst, src);
                cp_async16(dst + 16u, src + 1);
                cp_async16(dst + 32u, src + 2);
            }
        cp_async_commit();
    }

    // Batch 0 in flight, batch 1's ids loading.
    __device__ __forceinline__ void start() {
#pragma unroll
        for (int q = 0; q < ITEMS; ++q) {
            const int sl = q * kThreads + threadIdx.x;
            idx_f[q] = pos(0, sl);
            gid_f[q] = fetch(idx_f[q]);
        }
        launch_copy();
#pragma unroll
        for (int q = 0; q < ITEMS; ++q) {
            const int sl = q * kThreads + threadIdx.x;
            idx_n[q] = pos(1, sl);
            gid_n[q] = fetch(idx_n[q]);
        }
    }

    // Stage batch b (whose records are in flight): cull + compact into sm, then launch batch
    // b+1's copies and batch b+2's id loads.  Returns the staged count, or -1 when no thread of
    // the CTA is `active` (every thread gets the same answer; nothing is staged then).
    __device__ __forceinline__ int stage(int b, bool active, int bx0, int bx1, int by0, int by1, StageSmem<CAP>& sm) {
        const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
        constexpr int nwarps = kWarps;
        cp_async_wait_all();
        // raw is complete and visible; every thread is done reading the previous staging area
        if (__syncthreads_count(active) == 0) return -1;
        bool keep[ITEMS];
        unsigned m[ITEMS];
#pragma unroll
        for (int q = 0; q < ITEMS; ++q) {
            keep[q] = false;
            if (idx_f[q] >= 0) {
                const int sl = q * kThreads + tid;
                keep[q] = CULL ? may_contribute(raw->r[sl][0], raw->r[sl][1], raw->r[sl][2].w, bx0, bx1, by0, by1)
                               : true;
            }
            m[q] = __ballot_sync(0xffffffffu, keep[q]);
            if (lane == 0) sm.wcnt[q * nwarps + warp] = __popc(m[q]);
        }
        __syncthreads();
        int total = 0;
        for (int w = 0; w < ITEMS * nwarps; ++w) total += sm.wcnt[w];
        const unsigned lt = lanemask_lt();
#pragma unroll
        for (int q = 0; q < ITEMS; ++q) {
            if (!keep[q]) continue;
            int off = 0;
            for (int w = 0; w < q * nwarps + warp; ++w) off += sm.wcnt[w];
            const int p = off + __popc(m[q] & lt);
            const int sl = q * kThreads + tid;  // re-read from shared memory: no records held across the barrier
            ProjRec r;
            r.r0 = raw->r[sl][0];
            r.r1 = raw->r[sl][1];
            r.r2 = raw->r[sl][2];
            const int X0 = max(range_lo(r.r1.z), bx0) - bx0, X1 = min(range_hi(r.r1.z), bx1) - bx0;
            const int Y0 = max(range_lo(r.r1.w), by0) - by0, Y1 = min(range_hi(r.r1.w), by1) - by0;
            const uint32_t cols = ((1u << X1) - 1u) & ~((1u << X0) - 1u);
            const uint32_t rows = ((1u << Y1) - 1u) & ~((1u << Y0) - 1u);
            sm.r0[p] = r.r0;
            sm.r1[p] = make_float4(r.r1.x, r.r1.y, __uint_as_float(cols | (rows << 16)), r.r2.w);
            sm.r2[p] = r.r2;
            sm.gid[p] = gid_f[q];
            sm.idx[p] = idx_f[q];
        }
        __syncthreads();  // staged batch visible; raw reads done
#pragma unroll
        for (int q = 0; q < ITEMS; ++q) {
            idx_f[q] = idx_n[q];
            gid_f[q] = gid_n[q];
        }
        launch_copy();
#pragma unroll
        for (int q = 0; q < ITEMS; ++q) {
            const int sl = q * kThreads + tid;
            idx_n[q] = pos(b + 2, sl);
            gid_n[q] = fetch(idx_n[q]);
        }
        return total;
    }

    // No copy may still be writing raw when the CTA moves on (persistent kernels reuse it).
    __device__ __forceinline__ void finish() { cp_async_wait_all(); }
};

}  // namespace splat_b200
