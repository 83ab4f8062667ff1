// spatial.cu — depth-reinitialisation tail on device: third-nearest-
// neighbour distances (third_neighbor_distances, spatial.cpp:101-121) and the fresh Gaussian set
// built from sampled points (depth_reinitialize, densify.cpp:237-251).
//
// The k-th neighbour distance is the k-th smallest of all |p_j - p_i| (j != i), whatever index
// finds it, so the GPU uses its own uniform grid (dense cell array sized from the point bounds,
// counting sort of points by cell) and searches Chebyshev rings around each query until ring
// r's lower distance bound r*h exceeds the current k-th distance.  Distances use the reference's
// float order (difference, x^2 + (y^2 + z^2), correctly rounded sqrt), so every distance — and
// the selected k-th one — is bit-identical to the reference's.
#include <algorithm>
#include <cfloat>
#include <cstdint>
#include <cstring>

#include "common.cuh"
#include "internal.h"

namespace splat_b200 {

namespace {

inline unsigned blocks_for(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

__device__ __forceinline__ uint32_t ord_key(float f) {
    const uint32_t u = __float_as_uint(f);
    return (u >> 31) ? ~u : (u | 0x80000000u);
}

// bounds[0..2] = ordered keys of the minima, [3..5] = of the maxima (atomics on ordered keys)
__global__ void bounds_kernel(const float* __restrict__ p, int m, uint32_t* __restrict__ bounds) {
    uint32_t lo[3] = {0xffffffffu, 0xffffffffu, 0xffffffffu}, hi[3] = {0u, 0u, 0u};
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const uint32_t k = ord_key(p[3 * i + c]);
            lo[c] = min(lo[c], k);
            hi[c] = max(hi[c], k);
        }
#pragma unroll
    for (int c = 0; c < 3; ++c) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            lo[c] = min(lo[c], __shfl_xor_sync(0xffffffffu, lo[c], o));
            hi[c] = max(hi[c], __shfl_xor_sync(0xffffffffu, hi[c], o));
        }
        if ((threadIdx.x & 31) == 0) {
            atomicMin(&bounds[c], lo[c]);
            atomicMax(&bounds[3 + c], hi[c]);
        }
    }
}

__device__ __forceinline__ int grid_cell(const KnnGrid& g, float x, float y, float z, int* ix, int* iy, int* iz) {
    *ix = min(max((int)((x - g.ox) * g.inv_h), 0), g.nx - 1);
    *iy = min(max((int)((y - g.oy) * g.inv_h), 0), g.ny - 1);
    *iz = min(max((int)((z - g.oz) * g.inv_h), 0), g.nz - 1);
    return (*iz * g.ny + *iy) * g.nx + *ix;
}

__global__ void cell_count_kernel(const float* __restrict__ p, int m, KnnGrid g, uint32_t* __restrict__ cell_of,
                                  uint32_t* __restrict__ count) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    int ix, iy, iz;
    const int c = grid_cell(g, p[3 * i], p[3 * i + 1], p[3 * i + 2], &ix, &iy, &iz);
    cell_of[i] = (uint32_t)c;
    atomicAdd(&count[c], 1u);
}

// start[c] = exclusive scan of counts; cursor copy gets consumed by the scatter
__global__ void cell_scatter_kernel(const uint32_t* __restrict__ cell_of, int m, uint32_t* __restrict__ cursor,
                                    uint32_t* __restrict__ sorted) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    sorted[atomicAdd(&cursor[cell_of[i]], 1u)] = (uint32_t)i;
}

// k-th (k <= 3) smallest distance from point i to the other points; out = max(kth, min_dist).
__global__ void __launch_bounds__(128) knn_kernel(const float* __restrict__ p, int m, KnnGrid g,
                                                  const uint32_t* __restrict__ start, const uint32_t* __restrict__ sorted,
                                                  int k, float min_dist, float* __restrict__ out) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= m) return;
    const int i = (int)sorted[t];  // cell-sorted query order: neighbouring threads share cells
    const float qx = p[3 * i], qy = p[3 * i + 1], qz = p[3 * i + 2];
    int cx, cy, cz;
    grid_cell(g, qx, qy, qz, &cx, &cy, &cz);
    float d[3] = {INFINITY, INFINITY, INFINITY};
    int found = 0;
    const int max_ring = max(max(g.nx, g.ny), g.nz);
    for (int r = 0; r <= max_ring; ++r) {
        for (int dz = -r; dz <= r; ++dz) {
            const int iz = cz + dz;
            if (iz < 0 || iz >= g.nz) continue;
            for (int dy = -r; dy <= r; ++dy) {
                const int iy = cy + dy;
                if (iy < 0 || iy >= g.ny) continue;
                const bool face = abs(dz) == r || abs(dy) == r;
                for (int dx = -r; dx <= r; dx += (face || r == 0) ? 1 : 2 * r) {
                    const int ix = cx + dx;
                    if (ix < 0 || ix >= g.nx) continue;
                    const int c = (iz * g.ny + iy) * g.nx + ix;
                    for (uint32_t q = start[c]; q < start[c + 1]; ++q) {
                        const int j = (int)sorted[q];
                        if (j == i) continue;
                        // (points_[j] - q).norm(): difference, x^2 + (y^2 + z^2), sqrt
                        const float ex = __fsub_rn(p[3 * j], qx), ey = __fsub_rn(p[3 * j + 1], qy),
                                    ez = __fsub_rn(p[3 * j + 2], qz);
                        const float dist = __fsqrt_rn(
                            __fadd_rn(__fmul_rn(ex, ex), __fadd_rn(__fmul_rn(ey, ey), __fmul_rn(ez, ez))));
                        ++found;
                        if (dist < d[2]) {
                            if (dist < d[1]) {
                                d[2] = d[1];
                                if (dist < d[0]) {
                                    d[1] = d[0];
                                    d[0] = dist;
                                } else {
                                    d[1] = dist;
                                }
                            } else {
                                d[2] = dist;
                            }
                        }
                    }
                }
            }
        }
        // every point of ring r + 1 is at least r * h away (minus rounding): done once that
        // bound clears the current k-th distance
        if (found >= k && (float)r * g.h * 0.99999f > d[k - 1]) break;
    }
    const float kth = found >= k ? d[k - 1] : INFINITY;
    out[i] = fmaxf(kth, min_dist);
}

// densify.cpp:243-251: centers = points, isotropic log-scales log(nn3), identity rotation,
// opacity logit(0.1), SH DC = (rgb - 0.5) / C0 and the higher bands zero.
__global__ void reinit_set_kernel(const float* __restrict__ points, const float* __restrict__ colors,
                                  const float* __restrict__ nn3, int m, splat_params_mut out) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= m) return;
    const float ls = splat_logf(nn3[r]);
    const float logit01 = splat_logf(__fdiv_rn(0.1f, __fsub_rn(1.0f, 0.1f)));
    const float c0 = (float)0.28209479177387814;  // T(kSH_C0)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        out.centers[3 * r + c] = points[3 * r + c];
        out.log_scales[3 * r + c] = ls;
    }
    out.rotations[4 * r] = 1.0f;
    out.rotations[4 * r + 1] = 0.0f;
    out.rotations[4 * r + 2] = 0.0f;
    out.rotations[4 * r + 3] = 0.0f;
    out.opacity_logits[r] = logit01;
    float* sh = out.sh + 48 * (size_t)r;
#pragma unroll
    for (int c = 0; c < 3; ++c) sh[c] = colors ? __fdiv_rn(__fsub_rn(colors[3 * r + c], 0.5f), c0) : 0.0f;
    for (int c = 3; c < 48; ++c) sh[c] = 0.0f;
}

// n <= 256: the reference's brute force (same value; kept for symmetry with spatial.cpp:107-117)
__global__ void knn_brute_kernel(const float* __restrict__ p, int m, int k, float min_dist, float* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    float d[3] = {INFINITY, INFINITY, INFINITY};
    for (int j = 0; j < m; ++j) {
        if (j == i) continue;
        const float ex = __fsub_rn(p[3 * j], p[3 * i]), ey = __fsub_rn(p[3 * j + 1], p[3 * i + 1]),
                    ez = __fsub_rn(p[3 * j + 2], p[3 * i + 2]);
        const float dist =
            __fsqrt_rn(__fadd_rn(__fmul_rn(ex, ex), __fadd_rn(__fmul_rn(ey, ey), __fmul_rn(ez, ez))));
        if (dist < d[2]) {
            if (dist < d[1]) {
                d[2] = d[1];
                if (dist < d[0]) {
                    d[1] = d[0];
                    d[0] = dist;
                } else {
                    d[1] = dist;
                }
            } else {
                d[2] = dist;
            }
        }
    }
    out[i] = fmaxf(d[k - 1], min_dist);
}

__global__ void fill_kernel(float* __restrict__ out, int m, float v) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m) out[i] = v;
}

float ord_to_float(uint32_t k) {
    const uint32_t u = (k >> 31) ? (k & 0x7fffffffu) : ~k;
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}

}  // namespace

cudaError_t launch_point_bounds(LaunchCtx& lc, const float* p, int m, uint32_t* bounds6) {
    static const uint32_t init[6] = {0xffffffffu, 0xffffffffu, 0xffffffffu, 0u, 0u, 0u};
    cudaError_t e = cudaMemcpyAsync(bounds6, init, sizeof(init), cudaMemcpyHostToDevice, lc.stream);
    if (e != cudaSuccess || m == 0) return e;
    bounds_kernel<<<(unsigned)std::min<int64_t>(blocks_for(m, 256), lc.num_sms * 4), 256, 0, lc.stream>>>(p, m, bounds6);
    lc.count++;
    return cudaGetLastError();
}

void decode_bounds(const uint32_t* keys6, float lo[3], float hi[3]) {
    for (int c = 0; c < 3; ++c) {
        lo[c] = ord_to_float(keys6[c]);
        hi[c] = ord_to_float(keys6[3 + c]);
    }
}

cudaError_t launch_grid_build(LaunchCtx& lc, const float* p, int m, const KnnGrid& g, uint32_t* cell_of,
                              uint32_t* start, uint32_t* cursor, uint32_t* sorted, uint32_t* scan_tmp) {
    const size_t ncells = (size_t)g.nx * g.ny * g.nz;
    cudaError_t e = cudaMemsetAsync(cursor, 0, ncells * 4, lc.stream);
    if (e != cudaSuccess) return e;
    {
        LaunchScope s(lc, "knn_grid");
        cell_count_kernel<<<blocks_for(m, 256), 256, 0, lc.stream>>>(p, m, g, cell_of, cursor);
        lc.count++;
    }
    e = exclusive_scan_u32(lc, cursor, start, ncells, scan_tmp, start + ncells);
    if (e != cudaSuccess) return e;
    e = cudaMemcpyAsync(cursor, start, ncells * 4, cudaMemcpyDeviceToDevice, lc.stream);
    if (e != cudaSuccess) return e;
    cell_scatter_kernel<<<blocks_for(m, 256), 256, 0, lc.stream>>>(cell_of, m, cursor, sorted);
    lc.count++;
    return cudaGetLastError();
}

cudaError_t launch_knn(LaunchCtx& lc, const float* p, int m, const KnnGrid& g, const uint32_t* start,
                       const uint32_t* sorted, int k, float min_dist, float* out) {
    LaunchScope s(lc, "knn");
    knn_kernel<<<blocks_for(m, 128), 128, 0, lc.stream>>>(p, m, g, start, sorted, k, min_dist, out);
    lc.count++;
    return cudaGetLastError();
}

cudaError_t launch_knn_brute(LaunchCtx& lc, const float* p, int m, int k, float min_dist, float* out) {
    if (m == 0) return cudaSuccess;
    knn_brute_kernel<<<blocks_for(m, 128), 128, 0, lc.stream>>>(p, m, k, min_dist, out);
    lc.count++;
    return cudaGetLastError();
}

cudaError_t launch_fill(LaunchCtx& lc, float* out, int m, float v) {
    if (m == 0) return cudaSuccess;
    fill_kernel<<<blocks_for(m, 256), 256, 0, lc.stream>>>(out, m, v);
    lc.count++;
    return cudaGetLastError();
}

cudaError_t launch_reinit_set(LaunchCtx& lc, const float* points, const float* colors, const float* nn3, int m,
                              const splat_params_mut& out) {
    if (m == 0) return cudaSuccess;
    LaunchScope s(lc, "reinit_set");
    reinit_set_kernel<<<blocks_for(m, 256), 256, 0, lc.stream>>>(points, colors, nn3, m, out);
    lc.count++;
    return cudaGetLastError();
}

}  // namespace splat_b200
