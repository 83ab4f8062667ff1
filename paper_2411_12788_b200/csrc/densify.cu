// densify.cu — on-device consumers of the importance pass:
// quantile thresholds (quantile.hpp:16-46), per-view visibility masks (build_masks,
// visibility.cpp:9-37), critical identification (identify_critical, densify.cpp:32-103),
// aggressive cloning + plan application (densify.cpp:105-130, 159-195), importance pruning
// (simplify.cpp:94-107) and row gathers for GaussianSet::select / OptimState::remap
// (gaussian_set.hpp:96-110, optimizer.cpp:73-108).
//
// These run every few hundred iterations (trainer.cpp:211-342), so the host reads back the few
// scalars the reference's control flow branches on (candidate counts, order statistics); the
// per-Gaussian work is elementwise kernels + the hand-written radix sort (sort.cu) for the
// order statistics and the score ordering.  Arithmetic that decides integer outcomes follows
// the reference's operation order with explicitly rounded float ops and the shared
// splat_expf / splat_logf (include/splat_expf.h), so selections and cloned parameters are
// bit-identical to the mode-B reference build.
#include <cstdint>

#include "common.cuh"
#include "internal.h"

namespace splat_b200 {

namespace {

inline unsigned blocks_for(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

// Orderable unsigned keys: a < b as floats  <=>  key(a) < key(b) as unsigned (no NaNs).
__device__ __forceinline__ uint32_t f32_key(float f) {
    const uint32_t u = __float_as_uint(f);
    return (u >> 31) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ uint64_t f64_key(double d) {
    const uint64_t u = (uint64_t)__double_as_longlong(d);
    return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

// Compaction of the selected entries' keys (sel == nullptr: all), in index order; vals = index.
template <typename T>
__global__ void select_keys_kernel(const T* __restrict__ v, const uint8_t* __restrict__ sel, int n,
                                   const uint32_t* __restrict__ offsets, uint32_t* __restrict__ key_lo,
                                   uint32_t* __restrict__ key_hi, uint32_t* __restrict__ vals) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || (sel && !sel[i])) return;
    const uint32_t o = sel ? offsets[i] : (uint32_t)i;
    if constexpr (sizeof(T) == 4) {
        key_lo[o] = f32_key((float)v[i]);
    } else {
        const uint64_t k = f64_key((double)v[i]);
        key_lo[o] = (uint32_t)k;
        key_hi[o] = (uint32_t)(k >> 32);
    }
    vals[o] = (uint32_t)i;
}

__global__ void flags_from_bytes_kernel(const uint8_t* __restrict__ sel, int n, uint32_t* __restrict__ flags) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) flags[i] = sel[i] ? 1u : 0u;
}

__global__ void gather_u32_kernel(const uint32_t* __restrict__ src, const uint32_t* __restrict__ idx, int n,
                                  uint32_t* __restrict__ dst) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = src[idx[i]];
}

// count of entries with v > tau (and sel), device-wide
template <typename T>
__global__ void count_above_kernel(const T* __restrict__ v, const uint8_t* __restrict__ sel, int n, T tau,
                                   uint32_t* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const bool hit = i < n && (!sel || sel[i]) && v[i] > tau;
    const unsigned m = __ballot_sync(0xffffffffu, hit);
    if ((threadIdx.x & 31) == 0 && m) atomicAdd(out, (uint32_t)__popc(m));
}

// visibility.cpp:21-33: importance > tau, or (keep-all edge rule) importance > 0
__global__ void visibility_mask_kernel(const float* __restrict__ imp, int n, float tau, int keep_all,
                                       uint8_t* __restrict__ mask) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    mask[i] = keep_all ? (imp[i] > 0.0f) : (imp[i] > tau);
}

// densify.cpp:62-73 (MaxWeight): critical = ever_max && (keep_all || best > tau); also the
// candidate flags (ever_max) for the other criteria.
__global__ void maxweight_critical_kernel(const float* __restrict__ best, const int64_t* __restrict__ max_count,
                                          int n, float tau, int keep_all, uint8_t* __restrict__ critical) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const bool ever = max_count[i] > 0;
    critical[i] = ever && (keep_all || best[i] > tau);
}

__global__ void ever_max_kernel(const int64_t* __restrict__ max_count, int n, uint8_t* __restrict__ ever) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) ever[i] = max_count[i] > 0;
}

// densify.cpp:75-102: score per criterion, as an orderable 64-bit key for a DESCENDING stable
// sort (ties keep index order): key = ~f64_key(score).
__global__ void score_keys_kernel(int criterion, const float* __restrict__ opacity_logits,
                                  const double* __restrict__ summed, const double* __restrict__ random, int n,
                                  uint32_t* __restrict__ key_lo, uint32_t* __restrict__ key_hi,
                                  uint32_t* __restrict__ vals) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double s;
    if (criterion == SPLAT_CRITERION_OPACITY) {
        // set.opacity(i) = sigmoid(logit) in float (types.hpp:58-60), then widened to double
        const float e = splat_expf(-opacity_logits[i]);
        s = (double)__fdiv_rn(1.0f, __fadd_rn(1.0f, e));
    } else if (criterion == SPLAT_CRITERION_ACCUM_WEIGHT) {
        s = summed[i];
    } else {
        s = random[i];
    }
    const uint64_t k = ~f64_key(s);
    key_lo[i] = (uint32_t)k;
    key_hi[i] = (uint32_t)(k >> 32);
    vals[i] = (uint32_t)i;
}

__global__ void mark_first_kernel(const uint32_t* __restrict__ order, int count, uint8_t* __restrict__ critical) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r < count) critical[order[r]] = 1;
}

// aggressive_clone flags (densify.cpp:113-114): critical and opacity > 1e-7 (float sigmoid)
__global__ void clone_flags_kernel(const float* __restrict__ logits, const uint8_t* __restrict__ critical, int n,
                                   uint32_t* __restrict__ flags) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    bool f = false;
    if (critical[i]) {
        const float alpha = __fdiv_rn(1.0f, __fadd_rn(1.0f, splat_expf(-logits[i])));
        f = alpha > 1e-7f;
    }
    flags[i] = f ? 1u : 0u;
}

// aggressive_clone + apply_densify_plan (AggressiveClone mode): the clone's new opacity logit
// and log-scale shift (densify.cpp:115-121, operation order kept, explicitly rounded), written
// over row i and into appended row n + rank; moment_source per densify.cpp:164-170, 191-193.
__global__ void clone_apply_kernel(splat_params_mut p, const uint32_t* __restrict__ flags,
                                   const uint32_t* __restrict__ rank, int n, int32_t* __restrict__ moment_source) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const bool f = flags[i] != 0;
    if (moment_source) moment_source[i] = f ? -1 : i;
    if (!f) return;
    const int j = n + (int)rank[i];
    if (moment_source) moment_source[j] = -1;
    float alpha = __fdiv_rn(1.0f, __fadd_rn(1.0f, splat_expf(-p.opacity_logits[i])));
    alpha = fminf(alpha, __fsub_rn(1.0f, 1e-7f));
    const float sqrt2 = __fsqrt_rn(2.0f);
    const float alpha_new = __fsub_rn(1.0f, __fsqrt_rn(__fsub_rn(1.0f, alpha)));
    const float denom = __fsub_rn(__fmul_rn(2.0f, alpha_new), __fdiv_rn(__fmul_rn(alpha_new, alpha_new), sqrt2));
    const float k = __fdiv_rn(__fmul_rn(alpha, alpha), __fmul_rn(denom, denom));
    const float shift = __fmul_rn(0.5f, splat_logf(k));
    const float logit_new = splat_logf(__fdiv_rn(alpha_new, __fsub_rn(1.0f, alpha_new)));
    p.opacity_logits[i] = logit_new;
    p.opacity_logits[j] = logit_new;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const float ls = __fadd_rn(p.log_scales[3 * i + c], shift);
        p.log_scales[3 * i + c] = ls;
        p.log_scales[3 * j + c] = ls;
        p.centers[3 * j + c] = p.centers[3 * i + c];
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) p.rotations[4 * j + c] = p.rotations[4 * i + c];
    for (int c = 0; c < 48; ++c) p.sh[48 * (size_t)j + c] = p.sh[48 * (size_t)i + c];
}

__global__ void keep_flags_kernel(const double* __restrict__ v, int n, double tau, int keep_all,
                                  uint32_t* __restrict__ flags) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) flags[i] = (keep_all || v[i] > tau) ? 1u : 0u;
}

__global__ void compact_index_kernel(const uint32_t* __restrict__ flags, const uint32_t* __restrict__ offsets,
                                     int n, int32_t* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n && flags[i]) out[offsets[i]] = i;
}

// dst[r][c] = src[source[r]][c], zero row for source[r] < 0
__global__ void gather_rows_kernel(const float* __restrict__ src, int width, const int32_t* __restrict__ source,
                                   int64_t total, float* __restrict__ dst) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= total) return;
    const int64_t r = t / width, c = t - r * width;
    const int32_t s = source[r];
    dst[t] = s >= 0 ? src[(int64_t)s * width + c] : 0.0f;
}

// importance_sample keys (simplify.cpp:51-58): key = log(u) / w for w > 0 (log(u) drawn on the
// host), as a DESCENDING orderable 64-bit key; rows with w <= 0 (or NaN) get the all-ones key
// (sorted after every keyed row) and a filler flag.
__global__ void sample_keys_kernel(const double* __restrict__ imp, const double* __restrict__ logu, int n,
                                   uint32_t* __restrict__ key_lo, uint32_t* __restrict__ key_hi,
                                   uint32_t* __restrict__ vals, uint32_t* __restrict__ zero_flags) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double w = imp[i];
    const bool keyed = w > 0.0;
    const uint64_t k = keyed ? ~f64_key(__ddiv_rn(logu[i], w)) : ~0ull;
    key_lo[i] = (uint32_t)k;
    key_hi[i] = (uint32_t)(k >> 32);
    vals[i] = (uint32_t)i;
    zero_flags[i] = keyed ? 0u : 1u;
}

__global__ void mark_list_kernel(const int32_t* __restrict__ idx, int count, uint8_t* __restrict__ sel) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r < count) sel[idx[r]] = 1;
}

// vanilla_clone_split classification (densify.cpp:142-149): 0 untouched, 1 clone, 2 split.
// keep = not split; new rows = 1 (clone) / 2 (split); split rank flag.
__global__ void vcs_classify_kernel(const float* __restrict__ log_scales, const float* __restrict__ accum,
                                    const int32_t* __restrict__ count, int n, float grad_threshold,
                                    float scale_limit, uint32_t* __restrict__ keep, uint32_t* __restrict__ fresh,
                                    uint32_t* __restrict__ split) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int kind = 0;
    const int c = count[i];
    if (c > 0) {
        const float avg = __fdiv_rn(accum[i], (float)c);
        if (avg > grad_threshold) {
            // Vec3f scale = exp(log_scales) (gaussian_set.hpp:84); maxCoeff as std::max in order
            float m = splat_expf(log_scales[3 * i]);
            const float s1 = splat_expf(log_scales[3 * i + 1]);
            const float s2 = splat_expf(log_scales[3 * i + 2]);
            m = m < s1 ? s1 : m;
            m = m < s2 ? s2 : m;
            kind = m <= scale_limit ? 1 : 2;
        }
    }
    keep[i] = kind == 2 ? 0u : 1u;
    fresh[i] = (uint32_t)kind;
    split[i] = kind == 2 ? 1u : 0u;
}

// output row sources: kept rows in index order, then each clone's copy / split's two children
__global__ void vcs_sources_kernel(const uint32_t* __restrict__ keep, const uint32_t* __restrict__ keep_off,
                                   const uint32_t* __restrict__ fresh, const uint32_t* __restrict__ fresh_off,
                                   int n, int n_keep, int32_t* __restrict__ src, int32_t* __restrict__ moment_source) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (keep[i]) {
        src[keep_off[i]] = i;
        if (moment_source) moment_source[keep_off[i]] = i;
    }
    const uint32_t f = fresh[i];
    for (uint32_t c = 0; c < f; ++c) {
        const size_t r = (size_t)n_keep + fresh_off[i] + c;
        src[r] = i;
        if (moment_source) moment_source[r] = -1;
    }
}

// split children (densify.cpp:150-160): centre + R(q) (s .* n), log-scales - log(1.6); the
// normals of split j arrive in draw order, three per child, and Vec3f n(g(), g(), g()) takes
// them right to left (GCC's argument evaluation order, pinned against the reference build).
__global__ void vcs_split_kernel(splat_gaussians in, const uint32_t* __restrict__ fresh,
                                 const uint32_t* __restrict__ fresh_off, const uint32_t* __restrict__ split_rank,
                                 const float* __restrict__ normals, int n_keep, float split_shift,
                                 float* __restrict__ centers, float* __restrict__ log_scales) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= in.n || fresh[i] != 2) return;
    float q[4], rot[9], sc[3], c0[3], ls[3];
#pragma unroll
    for (int k = 0; k < 4; ++k) q[k] = in.rotations[4 * (size_t)i + k];
    rotation_from_quat(q, rot);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        ls[k] = in.log_scales[3 * (size_t)i + k];
        sc[k] = splat_expf(ls[k]);
        c0[k] = in.centers[3 * (size_t)i + k];
    }
    const float* nrm = normals + 6 * (size_t)split_rank[i];
#pragma unroll
    for (int child = 0; child < 2; ++child) {
        const size_t r = (size_t)n_keep + fresh_off[i] + child;
        float v[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) v[k] = __fmul_rn(sc[k], nrm[3 * child + 2 - k]);
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const float d = __fadd_rn(__fmul_rn(rot[3 * k], v[0]),
                                      __fadd_rn(__fmul_rn(rot[3 * k + 1], v[1]), __fmul_rn(rot[3 * k + 2], v[2])));
            centers[3 * r + k] = __fadd_rn(c0[k], d);
            log_scales[3 * r + k] = __fsub_rn(ls[k], split_shift);
        }
    }
}

}  // namespace

cudaError_t launch_select_keys_f32(LaunchCtx& lc, const float* v, const uint8_t* sel, int n, const uint32_t* offsets,
                                   uint32_t* key, uint32_t* vals) {
    if (n == 0) return cudaSuccess;
    LaunchScope s(lc, "select_keys");
    select_keys_kernel<float><<<blocks_for(n, 256), 256, 0, lc.stream>>>(v, sel, n, offsets, key, nullptr, vals);
    lc.count++;
    return cudaGetLastError();
}

cudaError_t launch_select_keys_f64(LaunchCtx& lc, const double* v, const uint8_t* sel, int n,
                                   const uint32_t* offsets, uint32_t* key_lo, uint32_t* key_hi, uint32_t* vals) {
    if (n == 0) return cudaSuccess;
    LaunchScope s(lc, "select_keys");
    select_keys_kernel<double><<<blocks_for(n, 256), 256, 0, lc.stream>>>(v, sel, n, offsets, key_lo, key_hi, vals);
    lc.count++;
    return cudaGetLastError();
}

cudaError_t launch_flags_from_bytes(LaunchCtx& lc, const uint8_t* sel, int n, uint32_t* flags) {
    if (n == 0) return cudaSuccess;
    flags_from_bytes_kernel<<<blocks_for(n, 256), 256, 0, lc.stream>>>(sel, n, flags);
    lc.count++;
    return cudaGetLastError();
}

cudaError_t launch_gather_u32(LaunchCtx& lc, const uint32_t* src, const uint32_t* idx, int n, uint32_t* dst) {
    if (n == 0) return cudaSuccess;
    gather_u32_kernel<<<blocks_for(n, 256), 256, 0, lc.stream>>>(src, idx, n, dst);
    lc.count++;
    return cudaGetLastError();
}

cudaError_t launch_count_above_f32(LaunchCtx& lc, const float* v, const uint8_t* sel, int n, float tau, uint32_t* out) {
    cudaError_t e = cudaMemsetAsync(out, 0, 4, lc.stream);
    if (e != cudaSuccess || n == 0) return e;
    count_above_kernel<float><<<blocks_for(n, 256), 256, 0, lc.stream>>>(v, sel, n, tau, out);
    lc.count++;
    return cudaGetLastError();
}

cudaError_t launch_count_above_f64(LaunchCtx& lc, const double* v, const uint8_t* sel, int n, double tau,
                                   uint32_t* out) {
    cudaError_t e = cudaMemsetAsync(out, 0, 4, lc.stream);
    if (e != cudaSuccess || n == 0) return e;
    count_above_kernel<double><<<blocks_for(n, 256), 256, 0, lc.stream>>>(v, sel, n, tau, out);
    lc.count++;
    return cudaGetLastError();
}

cudaError_t launch_visibility_mask(LaunchCtx& lc, const float* imp, int n, float tau, int keep_all, uint8_t* mask) {
    if (n == 0) return cudaSuccess;
    LaunchScope s(lc, "visibility_mask");
    visibility_mask_kernel<<<blocks_for(n, 256), 256, 0, lc.stream>>>(imp, n, tau, keep_all, mask);
    lc.count++;
    return cudaGetLastError();
}

cudaError_t launch_maxweight_critical(LaunchCtx& lc, const float* best, const int64_t* max_count, int n, float tau,
                                      int keep_all, uint8_t* critical) {
    if (n == 0) return cudaSuccess;
    maxweight_critical_kernel<<<blocks_for(n, 256), 256, 0, lc.stream>>>(best, max_count, n, tau, keep_all, critical);
    lc.count++;
    return cudaGetLastError();
}

cudaError_t launch_ever_max(LaunchCtx& lc, const int64_t* max_count, int n, uint8_t* ever) {
    if (n == 0) return cudaSuccess;
    ever_max_kernel<<<blocks_for(n, 256), 256, 0, lc.stream>>>(max_count, n, ever);
    lc.count++;
    return cudaGetLastError();
}

cudaError_t launch_score_keys(LaunchCtx& lc, int criterion, const float* logits, const double* summed,
                              const double* random, int n, uint32_t* key_lo, uint32_t* key_hi, uint32_t* vals) {
    if (n == 0) return cudaSuccess;
    score_keys_kernel<<<blocks_for(n, 256), 256, 0, lc.stream>>>(criterion, logits, summed, random, n, key_lo, key_hi,
                                                                 vals);
    lc.count++;
    return cudaGetLastError();
}

cudaError_t launch_mark_first(LaunchCtx& lc, const uint32_t* order, int count, uint8_t* critical) {
    if (count == 0) return cudaSuccess;
    mark_first_kernel<<<blocks_for(count, 256), 256, 0, lc.stream>>>(order, count, critical);
    lc.count++;
    return cudaGetLastError();
}

cudaError_t launch_clone_flags(LaunchCtx& lc, const float* logits, const uint8_t* critical, int n, uint32_t* flags) {
    if (n == 0) return cudaSuccess;
    clone_flags_kernel<<<blocks_for(n, 256), 256, 0, lc.stream>>>(logits, critical, n, flags);
    lc.count++;
    return cudaGetLastError();
}

cudaError_t launch_clone_apply(LaunchCtx& lc, const splat_params_mut& p, const uint32_t* flags, const uint32_t* rank,
                               int n, int32_t* moment_source) {
    if (n == 0) return cudaSuccess;
    LaunchScope s(lc, "clone_apply");
    clone_apply_kernel<<<blocks_for(n, 256), 256, 0, lc.stream>>>(p, flags, rank, n, moment_source);
    lc.count++;
    return cudaGetLastError();
}

cudaError_t launch_keep_flags(LaunchCtx& lc, const double* v, int n, double tau, int keep_all, uint32_t* flags) {
    if (n == 0) return cudaSuccess;
    keep_flags_kernel<<<blocks_for(n, 256), 256, 0, lc.stream>>>(v, n, tau, keep_all, flags);
    lc.count++;
    return cudaGetLastError();
}

cudaError_t launch_compact_index(LaunchCtx& lc, const uint32_t* flags, const uint32_t* offsets, int n, int32_t* out) {
    if (n == 0) return cudaSuccess;
    compact_index_kernel<<<blocks_for(n, 256), 256, 0, lc.stream>>>(flags, offsets, n, out);
    lc.count++;
    return cudaGetLastError();
}

cudaError_t launch_gather_rows(LaunchCtx& lc, const float* src, int width, const int32_t* source, int n_rows,
                               float* dst) {
    const int64_t total = (int64_t)width * n_rows;
    if (total == 0) return cudaSuccess;
    LaunchScope s(lc, "gather_rows");
    gather_rows_kernel<<<blocks_for(total, 256), 256, 0, lc.stream>>>(src, width, source, total, dst);
    lc.count++;
    return cudaGetLastError();
}

cudaError_t launch_sample_keys(LaunchCtx& lc, const double* imp, const double* logu, int n, uint32_t* key_lo,
                               uint32_t* key_hi, uint32_t* vals, uint32_t* zero_flags) {
    if (n == 0) return cudaSuccess;
    sample_keys_kernel<<<blocks_for(n, 256), 256, 0, lc.stream>>>(imp, logu, n, key_lo, key_hi, vals, zero_flags);
    lc.count++;
    return cudaGetLastError();
}

cudaError_t launch_mark_list(LaunchCtx& lc, const int32_t* idx, int count, uint8_t* sel) {
    if (count == 0) return cudaSuccess;
    mark_list_kernel<<<blocks_for(count, 256), 256, 0, lc.stream>>>(idx, count, sel);
    lc.count++;
    return cudaGetLastError();
}

cudaError_t launch_vcs_classify(LaunchCtx& lc, const float* log_scales, const float* accum, const int32_t* count,
                                int n, float grad_threshold, float scale_limit, uint32_t* keep, uint32_t* fresh,
                                uint32_t* split) {
    if (n == 0) return cudaSuccess;
    vcs_classify_kernel<<<blocks_for(n, 256), 256, 0, lc.stream>>>(log_scales, accum, count, n, grad_threshold,
                                                                   scale_limit, keep, fresh, split);
    lc.count++;
    return cudaGetLastError();
}

cudaError_t launch_vcs_sources(LaunchCtx& lc, const uint32_t* keep, const uint32_t* keep_off, const uint32_t* fresh,
                               const uint32_t* fresh_off, int n, int n_keep, int32_t* src, int32_t* moment_source) {
    if (n == 0) return cudaSuccess;
    vcs_sources_kernel<<<blocks_for(n, 256), 256, 0, lc.stream>>>(keep, keep_off, fresh, fresh_off, n, n_keep, src,
                                                                  moment_source);
    lc.count++;
    return cudaGetLastError();
}

cudaError_t launch_vcs_split(LaunchCtx& lc, const splat_gaussians& in, const uint32_t* fresh, const uint32_t* fresh_off,
                             const uint32_t* split_rank, const float* normals, int n_keep, float split_shift,
                             float* centers, float* log_scales) {
    if (in.n == 0) return cudaSuccess;
    vcs_split_kernel<<<blocks_for(in.n, 256), 256, 0, lc.stream>>>(in, fresh, fresh_off, split_rank, normals, n_keep,
                                                                    split_shift, centers, log_scales);
    lc.count++;
    return cudaGetLastError();
}

}  // namespace splat_b200
