/*
 * splat_oracle.h — CPU parity oracle for the Mini-Splatting2 rasterizer hot path.
 *
 * TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load the oracle libraries (liboracle, oracle/_ref).  The
 * product path (paper_2411_12788_b200/) never calls into this directory.
 *
 * Two implementations export this same C interface:
 *   - oracle/splat_oracle.c   : a plain-C restatement of the reference algorithm, function by
 *                               function (symbols prefixed oracle_);
 *   - oracle/ref_capi.cpp     : the reference's OWN sources (/root/reference/proj/src), compiled
 *                               in place against oracle/compat/Eigen (symbols prefixed ref_),
 *                               built into oracle/_ref/ by oracle/Makefile.
 * The restatement is pinned against the reference build (bitwise, tests/test_oracle_pin.py)
 * and against the reference's own known-answer tests (tests/golden/).
 *
 * Exp modes: liboracle.so / libsplat_ref.so use splat_expf (include/splat_expf.h), the
 * exp the CUDA kernels use ("mode B", bit-exact parity); liboracle_libm.so /
 * libsplat_ref_libm.so use glibc expf ("mode A", the reference exactly as shipped).
 */
#ifndef SPLAT_ORACLE_H
#define SPLAT_ORACLE_H

#include "splat_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

#ifndef ORACLE_FN
#define ORACLE_FN(name) oracle_##name
#endif

const char* ORACLE_FN(last_error)(void);

/* project<float> (rasterizer.cpp:10-90), results scattered per Gaussian index.
 * order[r] = index of the r-th survivor in (depth, index) order; *n_survivors its length. */
int ORACLE_FN(project)(const splat_gaussians* g, const splat_camera* cam,
                       const splat_raster_config* cfg, const uint8_t* mask,
                       int32_t* n_survivors, int32_t* order, int32_t* rect, int32_t* radius,
                       float* depth, float* mean2d, float* conic, float* color, float* opacity);

/* detail::bin_tiles (rasterizer.hpp:156-174) as CSR over Gaussian indices:
 * ranges[2t], ranges[2t+1] = [start, end) into gaussian[]. *n_pairs always receives P;
 * gaussian is written only when capacity >= P (pass capacity 0 to query). */
int ORACLE_FN(tiles)(const splat_gaussians* g, const splat_camera* cam,
                     const splat_raster_config* cfg, const uint8_t* mask, int64_t* n_pairs,
                     int32_t* ranges, int32_t* gaussian, int64_t capacity);

/* render<float> with optional ImportanceReport (rasterizer.cpp:96-182). Any output may be
 * NULL. stats (nullable, int64[2]) receives list visits V and committed blends C. */
int ORACLE_FN(render)(const splat_gaussians* g, const splat_camera* cam,
                      const splat_raster_config* cfg, const uint8_t* mask, const float bg[3],
                      float* color, float* alpha, float* depth, float* transmittance,
                      int32_t* max_contributor, float* importance, float* max_weight,
                      int32_t* max_pixel_count, int64_t* stats);

/* render_backward<float> (gradients.cpp:45-222). Grad arrays are overwritten (fresh
 * ParamGrads). grad2d_accum / grad2d_count may be NULL. */
int ORACLE_FN(render_backward)(const splat_gaussians* g, const splat_camera* cam,
                               const splat_raster_config* cfg, const float* d_color,
                               const uint8_t* mask, const float bg[3], float* d_centers,
                               float* d_log_scales, float* d_rotations, float* d_opacity,
                               float* d_sh, float* grad2d_accum, int32_t* grad2d_count);

/* l1_loss<float> (loss.cpp:63-76). grad may be NULL. */
float ORACLE_FN(l1_loss)(const float* a, const float* b, int64_t count, float* grad);

/* OptimState::step (optimizer.cpp:40-71) on arrays; params/moments updated in place.
 * Groups outside group_mask are skipped; rotations are renormalised iff rotations are in
 * the mask (all groups = the reference exactly). */
int ORACLE_FN(adam_step)(float* centers, float* log_scales, float* rotations,
                         float* opacity_logits, float* sh, int32_t n, const float* d_centers,
                         const float* d_log_scales, const float* d_rotations,
                         const float* d_opacity, const float* d_sh, float* m, float* v,
                         const splat_adam_config* cfg, int32_t* step_count,
                         uint32_t group_mask);

/* LrSchedule::at (optimizer.cpp:8-12). */
double ORACLE_FN(lr_at)(const splat_adam_config* cfg, int32_t step);

/* depth_reinitialize unprojection (densify.cpp:207-222) over one rendered view, with the
 * selection rule of splat_depth_unproject (include/splat_b200.h). */
int ORACLE_FN(unproject)(const splat_camera* cam, const int32_t* max_contributor,
                         const float* alpha, const float* depth, int rule,
                         float alpha_threshold, int64_t view_index, int32_t stride,
                         int64_t seed, float* points, int32_t* pixel, int64_t capacity,
                         int64_t* count);

/* ---- densification / simplification (contracts as in splat_b200.h) ---- */
int ORACLE_FN(quantile_threshold)(const float* values, const uint8_t* sel, int32_t n, double keep_q, float* tau,
                                  int32_t* count);
int ORACLE_FN(quantile_threshold_f64)(const double* values, const uint8_t* sel, int32_t n, double keep_q,
                                      double* tau, int32_t* count);
int ORACLE_FN(visibility_mask)(const float* importance, int32_t n, double keep_q, uint8_t* mask);
int ORACLE_FN(identify_critical)(const splat_gaussians* g, const float* best, const int64_t* max_count_sum,
                                 const double* summed, int criterion, double keep_q, const double* random,
                                 uint8_t* critical, int32_t* count_out);
int ORACLE_FN(aggressive_clone)(float* centers, float* log_scales, float* rotations, float* opacity_logits, float* sh,
                                int32_t n, int64_t capacity, const uint8_t* critical, int32_t* moment_source,
                                int32_t* n_out);
int ORACLE_FN(importance_prune)(const double* importance, int32_t n, double keep_q, int32_t* kept, int32_t* n_kept);

/* ssim<float> (loss.cpp:78-134) on H x W x ch images: mean SSIM, grad_a nullable. */
float ORACLE_FN(ssim)(const float* a, const float* b, int w, int h, int ch, float* grad_a);
/* photometric_loss<float> (loss.cpp:136-147). */
float ORACLE_FN(photometric_loss)(const float* rendered, const float* target, int w, int h, int ch, float lambda,
                                  float* grad);
/* the normalised 11-tap window gaussian_kernel builds (loss.cpp:13-22) */
void ORACLE_FN(ssim_window)(float* out11);

/* third_neighbor_distances (spatial.cpp:101-121) and depth_reinitialize's fresh set
 * (densify.cpp:237-251); contracts as splat_third_neighbor_distances / splat_reinit_gaussians. */
int ORACLE_FN(third_neighbor_distances)(const float* points, int32_t m, float min_dist, float* out);
int ORACLE_FN(reinit_gaussians)(const float* points, const float* colors, int32_t m, float min_dist, float* centers,
                                float* log_scales, float* rotations, float* opacity_logits, float* sh);

/* The exp the library was built with (splat_expf or glibc expf). */
/* The reference's random draws (include/splat_rng.h) and the §8f functions that consume them
 * (oracle_ restatement; the ref_ build exports its own wrappers in ref_capi.cpp). */
int ORACLE_FN(rng_normal_f32)(uint32_t seed, int32_t n, float* out);
int ORACLE_FN(rng_mixed_64)(uint64_t seed, int32_t n, const int32_t* kinds, const int32_t* lo, const int32_t* hi,
                            double* out);
int ORACLE_FN(rng_uniform_f64_32)(uint32_t seed, int32_t n, double* out);
int ORACLE_FN(rng_fisher_yates)(uint32_t seed, int32_t pool, int32_t take, int32_t* idx_out);
int ORACLE_FN(importance_sample)(const double* importance, int32_t n, int32_t target, uint64_t seed, int32_t* kept,
                                 int32_t* n_kept);
int ORACLE_FN(vanilla_clone_split)(const splat_gaussians* g, const float* grad2d_accum, const int32_t* grad2d_count,
                                   float grad_threshold, float scale_threshold, float scene_extent, uint32_t seed,
                                   float* centers, float* log_scales, float* rotations, float* opacity_logits,
                                   float* sh, int64_t capacity, int32_t* moment_source, int32_t* n_out,
                                   int32_t* n_clone, int32_t* n_split);
int ORACLE_FN(adam_step_range)(float* params, const float* grad_shard, float* m, float* v, int32_t n, int64_t begin,
                               int64_t count, const splat_adam_config* cfg, int32_t step, uint32_t group_mask);
int ORACLE_FN(quat_normalize)(float* rotations, int32_t n);
float ORACLE_FN(exp)(float x);

#ifdef __cplusplus
}
#endif

#endif /* SPLAT_ORACLE_H */
