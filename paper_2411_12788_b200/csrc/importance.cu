// importance.cu — K12: per-view visibility bitmask and the global importance reduction.
//
// Consumers of accumulate_importance over many views (BASELINE config 3):
//   * per view k, visible[k][i] = max_weight_k[i] > threshold (config 3 rule; the reference's
//     build_masks uses a per-view quantile of importance instead, visibility.cpp:15-33 — out of
//     scope this round), packed 32 Gaussians per word;
//   * global_importance (simplify.cpp:13-34): accum_weight[i] += importance_k[i] in fp64 and
//     intersections[i] += max_pixel_count_k[i], views added in order, exactly the reference's
//     accumulation (one add per view per Gaussian).
// HBM-bound: 12 B read + 12.125 B written per Gaussian per view.
#include <cstdint>

#include "common.cuh"
#include "internal.h"

namespace splat_b200 {

namespace {

__global__ void __launch_bounds__(256) visibility_update_kernel(const float* __restrict__ importance,
                                                               const float* __restrict__ max_weight,
                                                               const int32_t* __restrict__ max_count, int n,
                                                               float threshold, uint32_t* __restrict__ bitmask,
                                                               double* __restrict__ accum,
                                                               int64_t* __restrict__ counts,
                                                               float* __restrict__ max_all) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const bool in = i < n;
    const bool vis = in && max_weight[i] > threshold;
    const unsigned word = __ballot_sync(0xffffffffu, vis);
    if (bitmask && (threadIdx.x & 31) == 0 && (i >> 5) < (n + 31) / 32) bitmask[i >> 5] = word;
    if (!in) return;
    if (accum) accum[i] += (double)importance[i];
    if (counts) counts[i] += max_count[i];
    if (max_all) max_all[i] = fmaxf(max_all[i], max_weight[i]);
}

}  // namespace

cudaError_t launch_visibility_update(LaunchCtx& lc, const float* importance, const float* max_weight,
                                     const int32_t* max_count, int n, float threshold, uint32_t* bitmask,
                                     double* accum, int64_t* counts, float* max_all) {
    if (n == 0) return cudaSuccess;
    LaunchScope s(lc, "visibility_update");
    visibility_update_kernel<<<(unsigned)((n + 255) / 256), 256, 0, lc.stream>>>(importance, max_weight, max_count, n,
                                                                               threshold, bitmask, accum, counts,
                                                                               max_all);
    lc.count++;
    return cudaGetLastError();
}

}  // namespace splat_b200
