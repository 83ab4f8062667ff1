// internal.h — host-side declarations shared by the CUDA translation units and the C-ABI layer.
#pragma once

#include <cstddef>
#include <cstdint>
#include <string>
#include <utility>

#include <cuda_runtime.h>

#include "splat_b200.h"

namespace splat_b200 {

struct CamParams;
struct ProjRec;
struct AuxRec;

struct ProfileState;

struct LaunchCtx {
    cudaStream_t stream = nullptr;
    int64_t count = 0;  // kernels launched (bench accounting)
    int num_sms = 148;
    int* work_counters = nullptr;  // device ints, zero at rest: [0] fwd / [1] bwd work queues (+8: exit
                                   // counts), [4 + p] chain touched-list lengths
    int chain_parity = 0;
    bool persistent_blend = true;  // blend kernels as persistent CTAs pulling pixel blocks
    bool bwd_px2 = true;           // 8 x 8 backward: one warp, two pixels per thread
    ProfileState* prof = nullptr;  // non-null while per-kernel CUDA-event timing is on
    // Bracket one kernel launch with CUDA events on `stream` (no-ops when profiling is off).
    void prof_begin(const char* name);
    void prof_end();
};

// Launch with programmatic stream serialisation (the kernel must call pdl_wait() first).
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(cudaStream_t s, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// RAII bracket: LaunchScope s(lc, "name"); kernel<<<...>>>;
struct LaunchScope {
    LaunchCtx& lc;
    LaunchScope(LaunchCtx& l, const char* name) : lc(l) { lc.prof_begin(name); }
    ~LaunchScope() { lc.prof_end(); }
};

// ---- sort.cu ------------------------------------------------------------------------------
size_t scan_temp_words(uint64_t n);
size_t radix_hist_words(uint64_t n, int bits);
cudaError_t exclusive_scan_u32(LaunchCtx& lc, const uint32_t* in, uint32_t* out, uint64_t n,
                               uint32_t* tmp, uint32_t* total_dev);
// Same, with a dedicated tmp that is zero at rest (allocated zeroed; the kernel re-zeroes it):
// no memset launch before the scan.
cudaError_t exclusive_scan_u32_zeroed(LaunchCtx& lc, const uint32_t* in, uint32_t* out, uint64_t n, uint32_t* tmp);
// out[i] = sum_{r < i} in[idx[r]] (gather fused into the single-pass scan)
cudaError_t exclusive_scan_gather_u32(LaunchCtx& lc, const uint32_t* in, const uint32_t* idx, uint32_t* out,
                                      uint64_t n, uint32_t* tmp, uint32_t* total_dev);
// Stable LSD sort of (keys, vals) on key bits [begin_bit, end_bit). Result lands in keys/vals
// or, when *result_in_alt, in keys_alt/vals_alt.
// key_range (nullable; 2 words, zero at rest, re-zeroed by the sort): the sort first reduces
// [max(~key), max(key)] over the keys other than 0xFFFFFFFF (the survivors), derives its passes from
// that range and sums each pass's histogram in its rank phase; the 0xFFFFFFFF keys come out last in
// no particular order.  Without it a phase 0 histograms all 4 byte digits (stable for every key).
// Whole sort as one cooperative kernel (result in keys_alt / vals_alt); returns
// cudaErrorCooperativeLaunchTooLarge when N does not fit one resident wave of 4096-key tiles.
size_t radix_coop_count_words(uint64_t n);
cudaError_t radix_sort_coop(LaunchCtx& lc, uint32_t* keys, uint32_t* vals, uint32_t* keys_alt, uint32_t* vals_alt,
                            uint32_t* keys_tmp, uint32_t* vals_tmp, uint64_t n, uint32_t* work,
                            uint32_t* key_range = nullptr);
cudaError_t radix_sort_pairs(LaunchCtx& lc, uint32_t* keys, uint32_t* vals, uint32_t* keys_alt,
                             uint32_t* vals_alt, uint64_t n, int begin_bit, int end_bit,
                             uint32_t* hist, uint32_t* scan_tmp, bool* result_in_alt);

// ---- forward.cu ---------------------------------------------------------------------------
struct GaussianPtrs {
    const float* centers;
    const float* log_scales;
    const float* rotations;
    const float* opacity_logits;
    const float* sh;
    int n;
    int sh_degree;
};

// K1: per-Gaussian projection. Writes rec/aux (aux may be null), depth keys (0xFFFFFFFF when
// culled), identity values and per-Gaussian SUPERTILE counts (0 = culled);
// counters[0] += survivors, counters[1] += supertile pairs Ps, counters[2] += tile pairs P.
cudaError_t launch_preprocess(LaunchCtx& lc, const GaussianPtrs& g, const CamParams& cp,
                              const uint8_t* mask, ProjRec* rec, AuxRec* aux, uint32_t* keys,
                              uint32_t* vals, uint32_t* tile_counts, uint32_t* n_survivors_dev,
                              float* depth_out, uint2* rect_ref, uint32_t* host_counts = nullptr,
                              float4* proj_dbg = nullptr, uint32_t* cls_cnt = nullptr, uint32_t* tcls_cnt = nullptr);

// [survivors, Ps, P] to the host's mapped memory + the counters re-zeroed (one warp), on a side
// stream so the depth sort does not queue behind it.
cudaError_t launch_publish_counts(cudaStream_t s, uint32_t* n_survivors_dev, uint32_t* host_counts, uint32_t* cls_cnt,
                                  uint32_t* tcls_cnt);

// ---- binning.cu ---------------------------------------------------------------------------
constexpr int kTailNoteWord = 9;  // host_counters[9]: a forward walked past a tile-list prefix
constexpr int kKeyRangeWord = 8;  // counters[8..9]: the depth sort's key-range scratch (zero at rest)
constexpr int kCostClasses = 64;  // work-order cost classes of the persistent blend kernels

struct BinningArgs {
    const uint32_t* order;       // survivors in (depth, index) order
    const uint32_t* st_offsets;  // exclusive scan of supertile counts in depth order
    const uint2* rect_ref;  // reference pixel rects (x0 | x1 << 16, y0 | y1 << 16)
    int n_surv;
    uint64_t st_pairs;
    int tile_size, tiles_x, tiles_y, st_x, st_y, st_bits;
    uint32_t* st_key[2];    // fallback path only
    uint32_t* st_gauss[2];  // [0]: supertile lists (chunked path); both: sort ping-pong (fallback)
    uint32_t* st_cnt;       // [st_chunk_words] chunked path: (supertile, chunk) counts / offsets
    uint32_t* st_scan_tmp;  // [scan_temp_words] zero at rest, for the st_cnt scan only
    uint32_t* st_ranges;   // [2 * n_st]
    uint16_t* st_cover;     // [st_pairs] tile cover (16 bits) of each supertile list entry
    uint32_t* l2_tmp;      // [bin_l2_words] level-2 piece map and per-piece tile counts
    uint32_t* ranges;      // [2 * n_tiles] out: [start, end) of each tile's list in pair_gauss
    uint32_t* pair_gauss;  // [16 * st_pairs] out: per-tile lists of Gaussian ids (capacity layout)
    uint32_t* hist;
    uint32_t* scan_tmp;
    // the forward's work order (chunked path only; nullable): [64 counters | 64 x n_tiles lists],
    // every tile filed under its list-length class as its range is written
    uint32_t* tcls;
    // List prefixes: each tile's list is materialised up to list_prefix entries (0xffffffff: all);
    // tails[2 t .. 2 t + 1] = [first, end) of the rest in the supertile list (empty: complete), read
    // through StagePipe / ListTail.  *st_list receives the supertile list the tails index.
    uint32_t list_prefix;
    uint32_t* tails;
    const uint32_t** st_list;
};
// Materialise the rest of every tile list of the last launch_binning(a) (the bit-exact getters);
// tails become empty.
cudaError_t complete_tile_lists(LaunchCtx& lc, const BinningArgs& a, const uint32_t* st_list);
int supertile_side();
// Capacity (entries) of the per-tile list buffer: every tile of supertile s gets L_s slots.
size_t bin_l2_pieces(uint64_t st_pairs, int n_st);
size_t bin_l2_words(uint64_t st_pairs, int n_st);
inline size_t tile_list_capacity(uint64_t st_pairs) { return (size_t)st_pairs * 16; }
// Chunked supertile pass (no pair sort) when the supertile count fits shared memory; otherwise
// the fallback needs st_offsets (exclusive scan of supertile counts in depth order) and st_key.
bool st_chunked(int n_st);
int st_chunks(int n_surv);
size_t st_chunk_words(int n_surv, int n_st);
cudaError_t launch_binning(LaunchCtx& lc, const BinningArgs& a);

struct FwdOutputs {
    float* color;            // [H][W][3] or null
    float* alpha;            // [H][W] or null
    float* depth;            // [H][W] or null (needs aux)
    float* transmittance;    // [H][W] or null
    int32_t* max_contributor;// [H][W] or null
    float* importance;       // [n] or null (report)
    float* max_weight;       // [n] or null
    int32_t* max_pixel_count;// [n] or null
    float* t_final;          // [H][W] backward state or null
    int32_t* last_index;     // [H][W] backward state or null
    // Per 8 x 8 block, the staged (block-culled) list entries the forward walked, for the
    // backward to replay without re-culling: blist[block][kBlockList] Gaussian ids, bidx the same
    // entries' tile-list positions (increasing), bcount[block] = entries walked (> kBlockList:
    // not stored, the backward re-culls the tile list).
    uint32_t* blist;         // or null
    uint32_t* bidx;
    int32_t* bcount;
    // Work order for the backward: block b appends itself to cost class c = 63 - min(63, entries
    // walked / 16) (heaviest first): cls_list[c * n_blocks + rank], rank from cls_cnt[c] (64
    // counters, zeroed by publish_counts before the forward).  Null: not recorded.
    uint32_t* cls_cnt;
    uint32_t* cls_list;
    int n_blocks;
    // tile-list tails (BinningArgs::tails; null: lists complete); *tail_note (mapped host memory)
    // is set when a block walks into a tail
    const uint32_t* tails;
    const uint32_t* st_list;
    const uint16_t* st_cover;
    uint32_t* tail_note;
};

constexpr int kBlockList = 2048;      // replay-list capacity per 8 x 8 block
constexpr int kBlockListSmem = 512;   // entries the backward maps through shared memory

// traverse_pixel statistics (V visits, C commits) of the last forward's lists: out[0..1] += (V, C).
cudaError_t launch_traversal_counts(LaunchCtx& lc, const CamParams& cp, const uint32_t* ranges,
                                    const uint32_t* pair_gauss, const ProjRec* rec, const uint2* rect_ref,
                                    unsigned long long* out);

// K6 (+K7 depth epilogue): per-tile front-to-back blend.
cudaError_t launch_blend_forward(LaunchCtx& lc, const CamParams& cp, const uint32_t* ranges,
                                 const uint32_t* pair_gauss, const ProjRec* rec, const AuxRec* aux,
                                 const float bg[3], const FwdOutputs& out, const uint32_t* tcls = nullptr);

// Depth unprojection + stride-rule compaction over one rendered view.
cudaError_t launch_unproject(LaunchCtx& lc, const CamParams& cp, const int32_t* max_contributor,
                             const float* alpha, const float* depth, int rule, float alpha_threshold,
                             int64_t view_index, int32_t stride, int64_t seed, float* points,
                             int32_t* pixel, int64_t capacity, int32_t* count_dev, uint32_t* flags,
                             uint32_t* offsets, uint32_t* scan_tmp, bool append = false,
                             int32_t* view_out = nullptr);

// ---- importance.cu ------------------------------------------------------------------------
cudaError_t launch_visibility_update(LaunchCtx& lc, const float* importance, const float* max_weight,
                                     const int32_t* max_count, int n, float threshold, uint32_t* bitmask,
                                     double* accum, int64_t* counts, float* max_all = nullptr);

// ---- backward.cu --------------------------------------------------------------------------
// Per-Gaussian 2D gradient accumulator, 64 B (4 x float4, w unused):
//   g0 = (d_mean.x, d_mean.y, d_conic00), g1 = (d_conic01, d_conic11, d_opacity),
//   g2 = d_colour, g3.x = committed samples (touched flag)
struct Grad2D;

// The tile lists' tails (BinningArgs::tails, StagePipe) for the kernels that walk tile lists.
struct TileTails {
    const uint32_t* tails;  // null: lists complete
    const uint32_t* st_list;
    const uint16_t* st_cover;
};
cudaError_t launch_blend_backward(LaunchCtx& lc, const CamParams& cp, const uint32_t* ranges, TileTails tt,
                                  const uint32_t* pair_gauss, const ProjRec* rec,
                                  const float* t_final, const int32_t* last_index, const float bg[3],
                                  const float* d_color, const float* color, const float* target,
                                  float* loss_partials, float* grad2d,
                                  const uint32_t* blist = nullptr, const uint32_t* bidx = nullptr,
                                  const int32_t* bcount = nullptr, const uint32_t* cls_cnt = nullptr,
                                  const uint32_t* cls_list = nullptr);
cudaError_t launch_loss_reduce(LaunchCtx& lc, const float* partials, int n, float inv_n, float* loss);
cudaError_t launch_copy_to_host(LaunchCtx& lc, const float* src, float* dst_mapped, int n, uint32_t seq = 0);
// K10 chain.  list: scratch of n_surv + 1 words (touched-Gaussian list; touched <= survivors).
// prezeroed: a fresh (accumulate = 0) gradient whose rows were already zero-filled (side stream);
// only touched rows are written.
cudaError_t launch_chain(LaunchCtx& lc, const GaussianPtrs& g, const CamParams& cp, float* grad2d,
                         const ProjRec* rec, const splat_param_grads& out, int accumulate, int n_surv,
                         uint32_t* list, bool prezeroed = false);
cudaError_t launch_l1(LaunchCtx& lc, const float* a, const float* b, int64_t n, float* grad,
                      float* partials, int n_partials);
int l1_partials_count(int64_t n);

struct AdamGroupArgs {
    float* param;
    const float* grad;
    float* m;
    float* v;
    int64_t count;
    double lr;
    double lr_alt;   // for SH: lr of coefficients k >= 3 (rest)
    int sh_layout;   // 1: per-48 row, first 3 use lr, rest lr_alt
    int sh_phase = 0;  // SH: row position (0..47) of element 0 (a shard starting mid-row)
};
cudaError_t launch_adam(LaunchCtx& lc, const AdamGroupArgs& a, double beta1, double beta2, double eps,
                        double bias1, double bias2);
cudaError_t launch_quat_normalize(LaunchCtx& lc, float* rotations, int n);

// densify.cu: selection keys, counts, masks, critical flags, clone, gathers.
cudaError_t launch_select_keys_f32(LaunchCtx& lc, const float* v, const uint8_t* sel, int n, const uint32_t* offsets,
                                   uint32_t* key, uint32_t* vals);
cudaError_t launch_select_keys_f64(LaunchCtx& lc, const double* v, const uint8_t* sel, int n,
                                   const uint32_t* offsets, uint32_t* key_lo, uint32_t* key_hi, uint32_t* vals);
cudaError_t launch_flags_from_bytes(LaunchCtx& lc, const uint8_t* sel, int n, uint32_t* flags);
cudaError_t launch_gather_u32(LaunchCtx& lc, const uint32_t* src, const uint32_t* idx, int n, uint32_t* dst);
cudaError_t launch_count_above_f32(LaunchCtx& lc, const float* v, const uint8_t* sel, int n, float tau, uint32_t* out);
cudaError_t launch_count_above_f64(LaunchCtx& lc, const double* v, const uint8_t* sel, int n, double tau,
                                   uint32_t* out);
cudaError_t launch_visibility_mask(LaunchCtx& lc, const float* imp, int n, float tau, int keep_all, uint8_t* mask);
cudaError_t launch_maxweight_critical(LaunchCtx& lc, const float* best, const int64_t* max_count, int n, float tau,
                                      int keep_all, uint8_t* critical);
cudaError_t launch_ever_max(LaunchCtx& lc, const int64_t* max_count, int n, uint8_t* ever);
cudaError_t launch_score_keys(LaunchCtx& lc, int criterion, const float* logits, const double* summed,
                              const double* random, int n, uint32_t* key_lo, uint32_t* key_hi, uint32_t* vals);
cudaError_t launch_mark_first(LaunchCtx& lc, const uint32_t* order, int count, uint8_t* critical);
cudaError_t launch_clone_flags(LaunchCtx& lc, const float* logits, const uint8_t* critical, int n, uint32_t* flags);
cudaError_t launch_clone_apply(LaunchCtx& lc, const splat_params_mut& p, const uint32_t* flags, const uint32_t* rank,
                               int n, int32_t* moment_source);
cudaError_t launch_keep_flags(LaunchCtx& lc, const double* v, int n, double tau, int keep_all, uint32_t* flags);
cudaError_t launch_compact_index(LaunchCtx& lc, const uint32_t* flags, const uint32_t* offsets, int n, int32_t* out);
cudaError_t launch_gather_rows(LaunchCtx& lc, const float* src, int width, const int32_t* source, int n_rows,
                               float* dst);
// importance_sample (simplify.cpp:36-92) and vanilla_clone_split (densify.cpp:132-163)
cudaError_t launch_sample_keys(LaunchCtx& lc, const double* imp, const double* logu, int n, uint32_t* key_lo,
                               uint32_t* key_hi, uint32_t* vals, uint32_t* zero_flags);
cudaError_t launch_mark_list(LaunchCtx& lc, const int32_t* idx, int count, uint8_t* sel);
cudaError_t launch_vcs_classify(LaunchCtx& lc, const float* log_scales, const float* accum, const int32_t* count,
                                int n, float grad_threshold, float scale_limit, uint32_t* keep, uint32_t* fresh,
                                uint32_t* split);
cudaError_t launch_vcs_sources(LaunchCtx& lc, const uint32_t* keep, const uint32_t* keep_off, const uint32_t* fresh,
                               const uint32_t* fresh_off, int n, int n_keep, int32_t* src, int32_t* moment_source);
cudaError_t launch_vcs_split(LaunchCtx& lc, const splat_gaussians& in, const uint32_t* fresh, const uint32_t* fresh_off,
                             const uint32_t* split_rank, const float* normals, int n_keep, float split_shift,
                             float* centers, float* log_scales);

// ssim.cu: mean SSIM (lambda < 0) or the photometric loss into value_dev,
// optional gradient; tmp = 3 w h ch floats when grad != null, partials = 2 ssim_partials_count.
size_t ssim_partials_count(int w, int h, int ch);
cudaError_t launch_ssim(LaunchCtx& lc, const float* a, const float* b, int w, int h, int ch, float lambda,
                        float* grad, float* value_dev, float* tmp, double* partials);

// spatial.cu: uniform-grid k-NN and the depth-reinit fresh set.
struct KnnGrid {
    float ox, oy, oz, h, inv_h;
    int nx, ny, nz;
};
cudaError_t launch_point_bounds(LaunchCtx& lc, const float* p, int m, uint32_t* bounds6);
void decode_bounds(const uint32_t* keys6, float lo[3], float hi[3]);
cudaError_t launch_grid_build(LaunchCtx& lc, const float* p, int m, const KnnGrid& g, uint32_t* cell_of,
                              uint32_t* start, uint32_t* cursor, uint32_t* sorted, uint32_t* scan_tmp);
cudaError_t launch_knn(LaunchCtx& lc, const float* p, int m, const KnnGrid& g, const uint32_t* start,
                       const uint32_t* sorted, int k, float min_dist, float* out);
cudaError_t launch_knn_brute(LaunchCtx& lc, const float* p, int m, int k, float min_dist, float* out);
cudaError_t launch_fill(LaunchCtx& lc, float* out, int m, float v);
cudaError_t launch_reinit_set(LaunchCtx& lc, const float* points, const float* colors, const float* nn3, int m,
                              const splat_params_mut& out);


// ---- comm.cu: the library's NCCL communicator (libnccl bound at run time) -------------------
struct Comm;
int comm_unique_id(void* id_out, std::string* err);
Comm* comm_create(int nranks, int rank, const void* id, std::string* err);
void comm_destroy(Comm* c);
int comm_ranks(const Comm* c);
int comm_rank(const Comm* c);
int comm_reduce_scatter(Comm* c, const float* send, float* recv, size_t recv_count, cudaStream_t s, std::string* err);
int comm_all_gather(Comm* c, const float* send, float* recv, size_t send_count, cudaStream_t s, std::string* err);
int comm_all_reduce(Comm* c, const void* send, void* recv, size_t count, int dtype, int op, cudaStream_t s,
                    std::string* err);

}  // namespace splat_b200
