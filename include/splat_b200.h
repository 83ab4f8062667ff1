/*
 * splat_b200.h — C-ABI drop-in boundary for the Mini-Splatting2 optimisation hot path
 * (tile-based differentiable Gaussian rasterizer, blending-weight importance, depth
 * rendering + unprojection) implemented as hand-written sm_100a CUDA kernels.
 *
 * Every entry point replaces one reference C++ function (paths relative to
 * /root/reference/proj):
 *
 *   splat_render                 <- render<float>              include/splat/rasterizer.hpp:72-76
 *                                                               src/rasterizer.cpp:175-182
 *   splat_accumulate_importance  <- accumulate_importance<float> rasterizer.hpp:79-82,
 *                                                               rasterizer.cpp:184-193
 *   splat_render_backward        <- render_backward<float>     include/splat/gradients.hpp:52-56,
 *                                                               src/gradients.cpp:45-222
 *   splat_l1_loss                <- l1_loss<float>             include/splat/loss.hpp:9-10,
 *                                                               src/loss.cpp:63-76
 *   splat_render_backward_l1     <- l1_loss + render_backward fused (trainer.cpp:228-239 with
 *                                   lambda_dssim = 0)
 *   splat_adam_step              <- OptimState::step           include/splat/optimizer.hpp:41,
 *                                                               src/optimizer.cpp:40-71
 *   splat_depth_unproject        <- depth_reinitialize unprojection loop src/densify.cpp:207-222
 *   splat_project_debug / splat_tiles_debug <- project<float> (rasterizer.cpp:10-90) and
 *                                   detail::bin_tiles (rasterizer.hpp:156-174), exposed for
 *                                   bit-exact checks of rects, sort keys, lists and ranges.
 *
 * Conventions (mirroring the reference):
 *   - Gaussian storage is the reference's GaussianSetT<float> layout: centers [N][3],
 *     log_scales [N][3], rotations [N][4] (w,x,y,z), opacity_logits [N], sh [N][48]
 *     coefficient-major (sh[k*3+c]).
 *   - Images are H x W x C row-major, channel-interleaved (types.hpp:24-52).
 *   - Pointers named *_dev are device memory; everything else is host memory.
 *   - All calls are asynchronous on the context stream unless documented otherwise.
 *   - Exceptions of the reference map to status codes: std::invalid_argument ->
 *     SPLAT_ERR_INVALID_ARGUMENT, std::logic_error -> SPLAT_ERR_LOGIC,
 *     std::runtime_error -> SPLAT_ERR_RUNTIME.  splat_last_error() returns the message.
 */
#ifndef SPLAT_B200_H
#define SPLAT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPLAT_SH_COEFFS 16
#define SPLAT_SH_VALUES 48
#define SPLAT_GRAD_FLOATS 59 /* 3 + 3 + 4 + 1 + 48 floats per Gaussian */

typedef enum splat_status {
    SPLAT_OK = 0,
    SPLAT_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument in the reference */
    SPLAT_ERR_LOGIC = 2,            /* std::logic_error (arrays / rows out of sync) */
    SPLAT_ERR_RUNTIME = 3,          /* std::runtime_error (e.g. no valid depth pixel) */
    SPLAT_ERR_CUDA = 4,
    SPLAT_ERR_OUT_OF_MEMORY = 5,
    SPLAT_ERR_NO_FORWARD_STATE = 6, /* fused/reuse call without a matching forward */
    SPLAT_ERR_NCCL = 7              /* NCCL missing or a collective failed (view-parallel exchange) */
} splat_status;

/* Mirrors CameraT<float> (camera.hpp:12-22). rotation is row-major world->camera. */
typedef struct splat_camera {
    int32_t width, height;
    float fx, fy, cx, cy;
    float rotation[9];
    float translation[3];
    float znear, zfar;
} splat_camera;

/* Mirrors RasterConfig (rasterizer.hpp:17-25) field for field. */
typedef struct splat_raster_config {
    int32_t tile_size;          /* 16 */
    int32_t apply_thresholds;   /* 1; 0 = exact mode (no gates, full-image rects) */
    double transmittance_min;   /* 1e-4 */
    double contribution_min;    /* 1/255 */
    double alpha_max;           /* 0.99 */
    double lowpass;             /* 0.3 */
    double radius_sigmas;       /* 3.0 */
} splat_raster_config;

/* GaussianSetT<float> (gaussian_set.hpp:60-81) as plain arrays. */
typedef struct splat_gaussians {
    const float* centers;        /* [n][3] */
    const float* log_scales;     /* [n][3] */
    const float* rotations;      /* [n][4] (w,x,y,z) */
    const float* opacity_logits; /* [n] */
    const float* sh;             /* [n][48] coefficient-major */
    int32_t n;
    int32_t active_sh_degree;
} splat_gaussians;

/* RenderOutput<float> (rasterizer.hpp:43-51); every field may be NULL. */
typedef struct splat_render_outputs {
    float* color;            /* [H][W][3] */
    float* alpha;            /* [H][W] */
    float* depth;            /* [H][W] */
    float* transmittance;    /* [H][W] */
    int32_t* max_contributor;/* [H][W], -1 = background */
} splat_render_outputs;

/* ImportanceReport<float> (rasterizer.hpp:54-61). */
typedef struct splat_importance_outputs {
    float* importance;        /* [n] sum of blend weights */
    float* max_weight;        /* [n] */
    int32_t* max_pixel_count; /* [n] */
} splat_importance_outputs;

/* ParamGrads<float> (gradients.hpp:14-46). */
typedef struct splat_param_grads {
    float* d_centers;        /* [n][3] */
    float* d_log_scales;     /* [n][3] */
    float* d_rotations;      /* [n][4] */
    float* d_opacity_logits; /* [n] */
    float* d_sh;             /* [n][48] */
    float* grad2d_accum;     /* [n] (may be NULL) */
    int32_t* grad2d_count;   /* [n] (may be NULL) */
} splat_param_grads;

/* AdamConfig + LrSchedule (optimizer.hpp:12-32). */
typedef struct splat_adam_config {
    double beta1, beta2, eps;
    double lr_init, lr_final;
    int32_t max_steps;
    int32_t _pad;
    double scene_extent;
    double lr_sh_dc, lr_sh_rest, lr_opacity, lr_scale, lr_rotation;
} splat_adam_config;

/* Parameter groups for splat_adam_step's group_mask. */
#define SPLAT_GROUP_CENTERS   1u
#define SPLAT_GROUP_SCALES    2u
#define SPLAT_GROUP_ROTATIONS 4u
#define SPLAT_GROUP_OPACITY   8u
#define SPLAT_GROUP_SH        16u
#define SPLAT_GROUP_ALL       31u

/* Mutable parameter pointers (device) for the optimizer. */
typedef struct splat_params_mut {
    float* centers;
    float* log_scales;
    float* rotations;
    float* opacity_logits;
    float* sh;
    int32_t n;
    int32_t active_sh_degree;
} splat_params_mut;

/* Adam moments, same layout as the parameters (optimizer.hpp:69-76). */
typedef struct splat_adam_moments {
    float *m_centers, *v_centers;
    float *m_log_scales, *v_log_scales;
    float *m_rotations, *v_rotations;
    float *m_opacity, *v_opacity;
    float *m_sh, *v_sh;
} splat_adam_moments;

/* Pixel validity rule for splat_depth_unproject. */
#define SPLAT_DEPTH_RULE_ARGMAX 0 /* max_contributor >= 0 (densify.cpp:216) */
#define SPLAT_DEPTH_RULE_ALPHA  1 /* accumulated alpha > alpha_threshold (BASELINE cfg 2) */

typedef struct splat_ctx splat_ctx;

/* ---- context ------------------------------------------------------------------------ */
int splat_ctx_create(int device, splat_ctx** out);
int splat_ctx_destroy(splat_ctx* ctx);
/* Use an external cudaStream_t (e.g. torch's current stream); NULL = legacy default. */
int splat_ctx_set_stream(splat_ctx* ctx, void* cuda_stream);
int splat_sync(splat_ctx* ctx);
const char* splat_last_error(const splat_ctx* ctx);
/* Number of kernels this context launched since creation (for bench accounting). */
int64_t splat_kernel_launches(const splat_ctx* ctx);

/* Per-kernel CUDA-event timing on the context stream (bench accounting). While enabled,
 * every launch is bracketed by events; splat_profile_read synchronises, writes up to
 * max_kernels entries (names '\n'-separated into `names`, total milliseconds, launch counts)
 * and resets the accumulators. */
int splat_profile_enable(splat_ctx* ctx, int on);
int splat_profile_read(splat_ctx* ctx, char* names, int names_bytes, double* total_ms,
                       int64_t* counts, int max_kernels, int* n_kernels);

/* ---- forward ------------------------------------------------------------------------ */
/* render<float>: g/mask/out are device pointers; background is host float[3]. The context
 * keeps the forward state (sorted tile lists, projected records, per-pixel T_final and last
 * contributor) for a following splat_render_backward(reuse_forward=1) / _l1 / unproject.
 * report may be NULL (render without ImportanceReport). */
int splat_render(splat_ctx* ctx, const splat_gaussians* g_dev, const splat_camera* cam,
                 const splat_raster_config* cfg, const uint8_t* mask_dev,
                 const float background[3], const splat_render_outputs* out_dev,
                 const splat_importance_outputs* report_dev);

int splat_accumulate_importance(splat_ctx* ctx, const splat_gaussians* g_dev,
                                const splat_camera* cam, const splat_raster_config* cfg,
                                const uint8_t* mask_dev,
                                const splat_importance_outputs* report_dev);

/* ---- backward ----------------------------------------------------------------------- */
/* render_backward<float>. accumulate=0 zeroes grads first (reference returns fresh
 * ParamGrads); accumulate=1 adds (ParamGrads::add, gradients.hpp:35-45). reuse_forward=1
 * reuses the state of the immediately preceding splat_render on the same inputs. */
int splat_render_backward(splat_ctx* ctx, const splat_gaussians* g_dev,
                          const splat_camera* cam, const splat_raster_config* cfg,
                          const float* d_color_dev, const uint8_t* mask_dev,
                          const float background[3], const splat_param_grads* grads_dev,
                          int accumulate, int reuse_forward);

/* l1_loss<float>: loss_dev (device float scalar) may be NULL, grad_dev may be NULL. */
int splat_l1_loss(splat_ctx* ctx, const float* a_dev, const float* b_dev, int64_t count,
                  float* grad_dev, float* loss_dev);

/* Fused L1 + backward against target_dev, using the colour of the preceding splat_render
 * (which must have run on the same inputs). loss_dev may be NULL. */
int splat_render_backward_l1(splat_ctx* ctx, const splat_gaussians* g_dev,
                             const splat_camera* cam, const splat_raster_config* cfg,
                             const float* target_dev, const uint8_t* mask_dev,
                             const float background[3], const splat_param_grads* grads_dev,
                             int accumulate, float* loss_dev);

/* ---- optimizer ---------------------------------------------------------------------- */
/* OptimState::step. *step_count is the host-side step counter t (read, then incremented),
 * exactly as OptimState::t_ (optimizer.cpp:45-47). Groups not in group_mask are left
 * untouched; quaternion renormalisation (optimizer.cpp:69) runs iff
 * SPLAT_GROUP_ROTATIONS is in the mask. */
int splat_adam_step(splat_ctx* ctx, const splat_params_mut* params_dev,
                    const splat_param_grads* grads_dev, const splat_adam_moments* moments_dev,
                    const splat_adam_config* cfg, int32_t* step_count, uint32_t group_mask);

/* OptimState::step on a shard of the packed parameter layout (the view-parallel step, SURVEY
 * §8e: reduce-scatter -> sharded Adam -> all-gather).  params_flat / m_flat / v_flat are the
 * packed [centers 3n | log_scales 3n | rotations 4n | opacity n | sh 48n] buffers (+ padding);
 * elements [begin, begin + count) are updated from grad_shard[count] (the reduce-scattered
 * gradient), each with its group's learning rate (position lr at step `step`, the count BEFORE
 * this step, as OptimState::step uses it; bias corrections of step + 1).  Padding elements (>= 59n)
 * and groups outside group_mask are skipped.  The quaternion renormalisation (optimizer.cpp:69)
 * is NOT applied: call splat_quat_normalize on the gathered rotations. */
int splat_adam_step_range(splat_ctx* ctx, float* params_flat, const float* grad_shard_dev, float* m_flat,
                          float* v_flat, int32_t n, int64_t begin, int64_t count, const splat_adam_config* cfg,
                          int32_t step, uint32_t group_mask);
/* normalized_quat (gaussian_set.hpp:15-20) over n (w,x,y,z) rows in place (optimizer.cpp:69). */
int splat_quat_normalize(splat_ctx* ctx, float* rotations_dev, int32_t n);

/* ---- depth unprojection ------------------------------------------------------------- */
/* For the preceding splat_render: every valid pixel (rule) whose raster index satisfies
 * (view_index*H*W + pixel + seed) % stride == 0 is unprojected to
 * cam.center() + depth * cam.ray_direction(px, py) (densify.cpp:213-220). Points are
 * written compacted in raster order: points_dev [capacity][3], pixel_dev [capacity].
 * *count_dev receives the number of selected pixels (may exceed capacity: nothing is
 * written past capacity). stride = 1 selects every valid pixel. */
int splat_depth_unproject(splat_ctx* ctx, const splat_camera* cam, int rule,
                          float alpha_threshold, int64_t view_index, int32_t stride,
                          int64_t seed, float* points_dev, int32_t* pixel_dev,
                          int64_t capacity, int32_t* count_dev);

/* ---- importance over views (BASELINE config 3) ------------------------------------- */
/* After splat_accumulate_importance for view k: bitmask_dev[(n+31)/32] (may be NULL) gets bit i
 * set iff max_weight[i] > threshold (the config-3 visibility rule), and the running
 * global_importance (simplify.cpp:13-34) is updated: accum_dev[i] += (double)importance[i],
 * counts_dev[i] += max_pixel_count[i] (either may be NULL).  Views added in call order give the
 * reference's fp64 sums for the same per-view importance. */
int splat_visibility_update(splat_ctx* ctx, const splat_importance_outputs* report_dev, int32_t n,
                            float threshold, uint32_t* bitmask_dev, double* accum_dev,
                            int64_t* counts_dev);
/* The same, plus max_all_dev[i] = max(max_all_dev[i], max_weight[i]) (may be NULL): the
 * per-Gaussian maximum blending weight over all views so far (the quantity the view-parallel
 * pass max-reduces across ranks). */
int splat_visibility_update_max(splat_ctx* ctx, const splat_importance_outputs* report_dev, int32_t n,
                                float threshold, uint32_t* bitmask_dev, double* accum_dev,
                                int64_t* counts_dev, float* max_all_dev);

/* ---- whole multi-view passes (BASELINE configs 3 and 2) ------------------------------ */
/* build_masks / global_importance over n_views views (visibility.cpp:9-37, simplify.cpp:13-34):
 * for each view k, splat_accumulate_importance then splat_visibility_update_max into
 * masks_dev[k * mask_words ..] (mask_words >= (n+31)/32), accum_dev, counts_dev and max_all_dev
 * (nullable) — the same results as that loop (updates applied in view order), with consecutive
 * views' rasterisation overlapped on an internal twin context. */
int splat_visibility_pass(splat_ctx* ctx, const splat_gaussians* g, const splat_camera* cams, int32_t n_views,
                          const splat_raster_config* cfg, float threshold, uint32_t* masks_dev, int64_t mask_words,
                          double* accum_dev, int64_t* counts_dev, float* max_all_dev);
/* depth_reinitialize's unprojection over n_views views (densify.cpp:207-222): for view k, a
 * depth render and splat_depth_unproject with view_index first_view + k; the points of all views
 * are appended in view order (raster order within a view) to points_dev [capacity][3],
 * pixel_dev [capacity] and view_dev [capacity] (nullable: the view index of each point);
 * *count_dev = the total (may exceed capacity: nothing is written past it).  Views overlap on an
 * internal twin context as in splat_visibility_pass. */
int splat_depth_points(splat_ctx* ctx, const splat_gaussians* g, const splat_camera* cams, int32_t n_views,
                       const splat_raster_config* cfg, int rule, float alpha_threshold, int64_t first_view,
                       int32_t stride, int64_t seed, float* points_dev, int32_t* view_dev, int32_t* pixel_dev,
                       int64_t capacity, int32_t* count_dev);

/* ---- depth re-initialisation tail (densify.cpp:227-251, spatial.cpp:9-121; §8f rank 2) ---- */
/* third_neighbor_distances: out_dev[i] = max(distance from point i to its k-th nearest other
 * point, min_dist), k = min(3, m - 1) (all min_dist when m < 2); points_dev [m][3].  Exact (the
 * k-th smallest of all pairwise float distances, computed in the reference's order). */
int splat_third_neighbor_distances(splat_ctx* ctx, const float* points_dev, int32_t m, float min_dist,
                                   float* out_dev);
/* The fresh set depth_reinitialize builds from sampled points (densify.cpp:237-251): centers =
 * points, log-scales = log(third-neighbour distance) (isotropic), rotation (1,0,0,0), opacity
 * logit(0.1), SH DC = (rgb - 0.5) / C0 from colors_dev [m][3] (NULL: 0), higher bands 0.  out
 * holds m rows (out->n is ignored). */
int splat_reinit_gaussians(splat_ctx* ctx, const float* points_dev, const float* colors_dev, int32_t m,
                           float min_dist, const splat_params_mut* out);

/* ---- native training step (trainer.cpp:208-240, one process) ------------------------------ */
/* One optimisation step over n_views views, the body of the reference's training iteration run
 * natively: for each view, render (splat_render), the loss (L1, or photometric_loss with
 * lambda_dssim > 0) and render_backward with gradients summed over the views
 * (ParamGrads::add), then OptimState::step on group_mask.  targets[k] is view k's H x W x 3
 * target: device memory, or, with targets_on_host != 0, host memory (pinned for an asynchronous
 * copy) that is copied on a side stream while the view's forward runs.  loss_host (nullable,
 * n_views floats) receives each view's loss: the call returns once the losses are on the host
 * (with the L1 loss that is before the chain and the optimiser step have finished: they complete
 * on the context's stream, ahead of anything queued there later, so the next call needs no
 * synchronisation; read parameters on another stream only after synchronising with it).
 * Without loss_host nothing is synchronised (loss_dev, nullable, gets the losses on the device). */
int splat_train_step(splat_ctx* ctx, const splat_params_mut* params, const splat_param_grads* grads,
                     const splat_adam_moments* moments, const splat_adam_config* adam, int32_t* step_count,
                     uint32_t group_mask, const splat_camera* cams, int32_t n_views, const float* const* targets,
                     int targets_on_host, const splat_raster_config* cfg, const float background[3],
                     float lambda_dssim, float* loss_dev, float* loss_host);
/* With a communicator on ctx (splat_comm_init), splat_train_step is the view-parallel step of
 * one rank: its views' gradients are summed locally, then splat_exchange_step replaces the plain
 * OptimState::step.  This needs the packed layout for params, grads and moments (each group
 * right after the previous one: centers, centers + 3n, + 6n, + 10n, + 11n) with at least
 * splat_exchange_len(n, nranks, buckets) floats per buffer (zero padding after 59n). */

/* ---- view-parallel exchange over the library's own NCCL communicator ---------
 * One process per GPU, each holding a replica of the Gaussians and training its own views.
 * splat_comm_unique_id on one rank, its 128 bytes broadcast by the caller (MPI, torch, a file),
 * then splat_comm_init on every rank (libnccl is loaded at run time).  The exchange:
 * reduce-scatter(sum) of the packed gradient in `buckets` pieces on a communication stream ->
 * OptimState::step on this rank's shard of each bucket (splat_adam_step_range, overlapping the
 * later buckets' reduce-scatter) -> in-place all-gather of the updated parameters ->
 * rotation renormalisation.  Only this rank's shards of m and v are kept current. */
#define SPLAT_UNIQUE_ID_BYTES 128
int splat_comm_unique_id(void* id_out);
int splat_comm_init(splat_ctx* ctx, int32_t nranks, int32_t rank, const void* unique_id, int32_t buckets);
int splat_comm_destroy(splat_ctx* ctx);
/* Padded packed length: 59 n rounded up to a multiple of nranks * buckets * 4 floats. */
int64_t splat_exchange_len(int32_t n, int32_t nranks, int32_t buckets);
/* The exchange + optimiser step on packed flats of flat_len floats (>= splat_exchange_len);
 * *step_count is OptimState's count (incremented).  Without a communicator: the plain step. */
int splat_exchange_step(splat_ctx* ctx, float* params_flat, const float* grads_flat, float* m_flat, float* v_flat,
                        int32_t n, int64_t flat_len, const splat_adam_config* cfg, int32_t* step_count,
                        uint32_t group_mask);
/* In-place all-reduce over the communicator on ctx's stream (the config-3 importance sums / max
 * weights / argmax counts across ranks).  dtype: SPLAT_DTYPE_*; op: SPLAT_OP_*. */
#define SPLAT_DTYPE_INT32 2
#define SPLAT_DTYPE_INT64 4
#define SPLAT_DTYPE_FLOAT32 7
#define SPLAT_DTYPE_FLOAT64 8
#define SPLAT_OP_SUM 0
#define SPLAT_OP_MAX 2
int splat_allreduce(splat_ctx* ctx, void* buf_dev, int64_t count, int32_t dtype, int32_t op);

/* ---- SSIM and the photometric loss (loss.cpp:78-153) -------------- */
/* ssim<float>: value_dev (device float) = mean SSIM of H x W x ch images a, b with the 11-tap
 * sigma-1.5 window; grad_dev (nullable) = d mean SSIM / d a.  Per-pixel values are the
 * reference's bit for bit; the image mean is summed in fp64 (the reference: one float sum). */
int splat_ssim(splat_ctx* ctx, const float* a_dev, const float* b_dev, int32_t width, int32_t height,
               int32_t channels, float* grad_dev, float* value_dev);
/* photometric_loss<float> (loss.cpp:136-147): (1 - lambda) l1 + lambda (1 - ssim) and its
 * gradient (nullable) with respect to `rendered`. */
int splat_photometric_loss(splat_ctx* ctx, const float* rendered_dev, const float* target_dev, int32_t width,
                           int32_t height, int32_t channels, float lambda, float* grad_dev, float* value_dev);
/* The training step's loss + backward with lambda_dssim (trainer.cpp:226-239): after splat_render
 * on the same inputs, photometric_loss(colour, target, lambda) -> dL/dC -> render_backward.
 * loss_dev (nullable) receives the loss. */
int splat_render_backward_photometric(splat_ctx* ctx, const splat_gaussians* g, const splat_camera* cam,
                                      const splat_raster_config* cfg, const float* target_dev,
                                      const uint8_t* mask_dev, const float background[3],
                                      const splat_param_grads* grads, int accumulate, float lambda,
                                      float* loss_dev);

/* ---- densification and simplification on device ---------- */
/* These run every few hundred iterations; each synchronises the context stream once or twice
 * to read back the scalars the reference's control flow branches on. */

/* quantile_threshold (quantile.hpp:16-28) over the entries of values_dev[n] selected by
 * sel_dev[i] != 0 (NULL: all entries): the (1 - keep_q) linear-interpolation order statistic,
 * computed in double from the two neighbouring sorted values.  *count_out = selected entries.
 * SPLAT_ERR_INVALID_ARGUMENT for an empty selection or keep_q outside (0, 1), as the reference
 * throws std::invalid_argument. */
int splat_quantile_threshold(splat_ctx* ctx, const float* values_dev, const uint8_t* sel_dev, int32_t n,
                             double keep_q, float* tau_out, int32_t* count_out);
int splat_quantile_threshold_f64(splat_ctx* ctx, const double* values_dev, const uint8_t* sel_dev, int32_t n,
                                 double keep_q, double* tau_out, int32_t* count_out);

/* build_masks (visibility.cpp:9-37), one view: from that view's accumulate_importance
 * importance_dev[n], mask_dev[n] = importance > tau with tau the keep_q quantile over the
 * strictly positive importances; when nothing exceeds tau every positive entry is kept; all
 * zero when nothing is positive.  The byte mask is what splat_render / accumulate_importance
 * take as `mask` (VisibilityTable::mask_for). */
int splat_visibility_mask(splat_ctx* ctx, const float* importance_dev, int32_t n, double keep_q, uint8_t* mask_dev);

/* identify_critical (densify.cpp:32-103) from the per-view statistics accumulated by
 * splat_visibility_update_max over the views: best_weight_dev (max over views of max_weight),
 * max_count_sum_dev (sum over views of max_pixel_count: > 0 iff "ever the max contributor")
 * and summed_importance_dev (fp64).  MaxWeight: critical = ever_max && best > tau (tau the keep_q
 * quantile over the ever_max candidates, keep-all edge rule); the other criteria take the same
 * count of Gaussians by score, descending, ties by index: opacity (float sigmoid), summed
 * importance, or caller-drawn random_scores_dev (the reference draws uniform doubles from its
 * std::mt19937).  critical_dev[n] bytes (0/1); *count_out = CriticalSelection::count. */
#define SPLAT_CRITERION_RANDOM 0
#define SPLAT_CRITERION_OPACITY 1
#define SPLAT_CRITERION_ACCUM_WEIGHT 2
#define SPLAT_CRITERION_MAX_WEIGHT 3
int splat_identify_critical(splat_ctx* ctx, const splat_gaussians* g, const float* best_weight_dev,
                            const int64_t* max_count_sum_dev, const double* summed_importance_dev, int criterion,
                            double keep_q, const double* random_scores_dev, uint8_t* critical_dev,
                            int32_t* count_out);

/* aggressive_clone + apply_densify_plan (densify.cpp:105-130, 159-195), in place: p holds p->n
 * rows in arrays with room for `capacity` rows.  Every critical row with opacity > 1e-7 gets
 * alpha_new = 1 - sqrt(1 - alpha) (alpha clamped to 1 - 1e-7), opacity logit(alpha_new) and
 * log-scales + ln(k)/2, and an identical copy is appended, in index order.
 * moment_source_dev[new n]: old row for Adam moments, -1 = zeroed (both copies of a clone and
 * every appended row).  *n_out = new row count.  SPLAT_ERR_INVALID_ARGUMENT when capacity is too
 * small (*n_out then = the rows needed; nothing is modified). */
int splat_aggressive_clone(splat_ctx* ctx, const splat_params_mut* p, int64_t capacity, const uint8_t* critical_dev,
                           int32_t* moment_source_dev, int32_t* n_out);

/* importance_prune (simplify.cpp:94-107): kept_dev = ascending indices with
 * importance > tau (select_above_quantile over all n entries, keep-all edge rule);
 * *n_kept = their count.  Follow with splat_gather_rows (GaussianSet::select) and, for Adam,
 * the same gather of the moments (OptimState::keep). */
int splat_importance_prune(splat_ctx* ctx, const double* importance_dev, int32_t n, double keep_q, int32_t* kept_dev,
                           int32_t* n_kept);

/* ---- the reference's random draws (include/splat_rng.h; host side, no device work) ---------
 * splat_rng is a std::mt19937 (densify.cpp:35, 134, 198: the trainer's engine passed by
 * reference): create it from a seed, or move a caller's engine in and out with the state words
 * libstdc++ streams (operator<< / >>: x[0..623] then the index _M_p), so a C++ caller's
 * std::mt19937& advances exactly as the reference's call would advance it. */
typedef struct splat_rng splat_rng;
int splat_rng_create(uint32_t seed, splat_rng** out);
void splat_rng_destroy(splat_rng* rng);
int splat_rng_get_state(const splat_rng* rng, uint32_t words_out[625]);
int splat_rng_set_state(splat_rng* rng, const uint32_t words[625]);
/* identify_critical's Random scores (densify.cpp:78-80): n uniform doubles in [0, 1) from rng,
 * written to out (host or device pointer: out_on_device selects). */
int splat_random_scores(splat_ctx* ctx, splat_rng* rng, int32_t n, double* out, int out_on_device);
/* depth_reinitialize's sample draw (densify.cpp:227-235): the first `take` entries of a partial
 * Fisher-Yates over [0, pool) with uniform_int_distribution<int> on rng -> idx_dev[take]. */
int splat_pool_sample(splat_ctx* ctx, splat_rng* rng, int32_t pool, int32_t take, int32_t* idx_dev);

/* importance_sample (simplify.cpp:36-92): target_count rows drawn without replacement with
 * probability proportional to importance_dev (fp64) by Efraimidis-Spirakis keys log(u)/w from
 * std::mt19937_64(seed) (u drawn on the host, keys + the 64-bit stable sort on the device, ties by
 * index); non-positive weights only fill a deficit (uniform partial Fisher-Yates over them, in
 * index order); no positive weight: a uniform draw.  kept_dev = ascending indices, *n_kept =
 * target_count.  SPLAT_ERR_INVALID_ARGUMENT when target_count is outside [1, n]. */
int splat_importance_sample(splat_ctx* ctx, const double* importance_dev, int32_t n, int32_t target_count,
                            uint64_t seed, int32_t* kept_dev, int32_t* n_kept);

/* vanilla_clone_split + apply_densify_plan, Progressive mode (densify.cpp:132-163, 182-191).
 * Rows of `in` with grad2d_count > 0 and grad2d_accum / count > grad_threshold are cloned when
 * max(exp(log_scale)) <= scale_threshold * scene_extent, else split: two children at centre +
 * R(q) (exp(log_scale) .* n), n ~ N(0, I3) from rng (normal_distribution<float>, drawn on the host
 * in the reference's order), log-scales - log(1.6).  `out` (capacity rows, must not alias `in`)
 * receives the kept rows (split rows removed) in index order, then the new rows in index order;
 * moment_source_dev[*n_out]: old row for kept rows, -1 for new rows.  *n_clone / *n_split may be
 * NULL.  SPLAT_ERR_INVALID_ARGUMENT when capacity is too small (*n_out = rows needed, rng and
 * out untouched). */
int splat_vanilla_clone_split(splat_ctx* ctx, const splat_gaussians* in, const float* grad2d_accum_dev,
                              const int32_t* grad2d_count_dev, float grad_threshold, float scale_threshold,
                              float scene_extent, splat_rng* rng, const splat_params_mut* out, int64_t capacity,
                              int32_t* moment_source_dev, int32_t* n_out, int32_t* n_clone, int32_t* n_split);

/* Row gather: dst[r][c] = src[source[r]][c] for r < n_rows, c < width; source[r] < 0 gives a zero
 * row (OptimState::remap, optimizer.cpp:73-108; GaussianSet::select, gaussian_set.hpp:96-110).
 * src and dst must not overlap. */
int splat_gather_rows(splat_ctx* ctx, const float* src_dev, int32_t width, const int32_t* source_dev, int32_t n_rows,
                      float* dst_dev);

/* ---- primitives (exposed for tests and microbenchmarks) ------------------------------ */
/* Stable LSD radix sort of (keys, vals) on key bits [begin_bit, end_bit), n pairs, device
 * pointers; the result lands in keys/vals or, when *result_in_alt, in keys_alt/vals_alt. */
int splat_sort_pairs(splat_ctx* ctx, uint32_t* keys_dev, uint32_t* vals_dev, uint32_t* keys_alt_dev,
                     uint32_t* vals_alt_dev, int64_t n, int begin_bit, int end_bit, int* result_in_alt);
/* Exclusive prefix sum of n uint32 (in place allowed); total_dev may be NULL. */
int splat_exclusive_scan(splat_ctx* ctx, const uint32_t* in_dev, uint32_t* out_dev, int64_t n,
                         uint32_t* total_dev);

/* ---- bit-exact debug views of the preceding forward (host outputs, synchronous) ------ */
/* n_survivors / n_pairs of the last forward. */
int splat_forward_counts(splat_ctx* ctx, int64_t* n_survivors, int64_t* n_pairs,
                         int32_t* tiles_x, int32_t* tiles_y);
/* ProjectedGaussian<float> (rasterizer.hpp:27-41). */
typedef struct splat_projected {
    float mean2d[2];
    float cov2d[3];          /* xx, xy, yy after the low-pass */
    float conic[3];
    float depth_mean;
    int32_t radius;
    int32_t index;
    float opacity;
    float color[3];
    int32_t x0, x1, y0, y1;  /* pixel rect, half-open */
    float center_world[3];
    float cov_world_inv[9];  /* row-major (symmetric: the cofactor inverse is exactly symmetric) */
    int32_t cov_degenerate;
} splat_projected;
/* project<float> (rasterizer.cpp:10-90): the survivors' records sorted by (depth, index), written
 * to out_host[0 .. *count) (host memory, capacity records; SPLAT_ERR_INVALID_ARGUMENT with *count
 * set when it is too small).  Runs the forward (also leaves its state for the debug getters). */
int splat_project(splat_ctx* ctx, const splat_gaussians* g, const splat_camera* cam, const splat_raster_config* cfg,
                  const uint8_t* mask, splat_projected* out_host, int64_t capacity, int32_t* count);

/* traverse_pixel statistics of the last forward (rasterizer.hpp:116-147; SURVEY §8d's V and C):
 * list entries visited (the breaking sample included) and samples committed, summed over the
 * pixels.  A measurement pass (one plain thread per pixel over the per-tile lists), synchronous. */
int splat_traversal_counts(splat_ctx* ctx, int64_t* visits, int64_t* commits);
/* Per Gaussian (index order): rect[4] = x0,x1,y0,y1 (0,0,0,0 when culled), radius,
 * depth bits, survivor flag. Any pointer may be NULL. */
int splat_project_debug(splat_ctx* ctx, int32_t* rect, int32_t* radius, float* depth,
                        uint8_t* survivor, float* mean2d, float* conic, float* color,
                        float* opacity);
/* Sorted pairs: key_tile[p], gaussian[p] for p < n_pairs (per-tile lists, depth-ordered),
 * ranges[2*t] = start, ranges[2*t+1] = end, depth_order[r] = r-th survivor (by
 * (depth, index)). Any pointer may be NULL. */
int splat_tiles_debug(splat_ctx* ctx, int32_t* key_tile, int32_t* gaussian, int32_t* ranges,
                      int32_t* depth_order);

#ifdef __cplusplus
}
#endif

#endif /* SPLAT_B200_H */
