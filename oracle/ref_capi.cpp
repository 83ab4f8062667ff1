// oracle/ref_capi.cpp — C interface over the reference's OWN hot-path code.
//
// TEST INFRASTRUCTURE ONLY.  Built by oracle/Makefile into oracle/_ref/libsplat_ref*.so from
// /root/reference/proj/src/*.cpp compiled in place (never copied) against the Eigen-subset
// shim in oracle/compat.  Exposes the splat_oracle.h interface with the ref_ prefix so the
// tests can run the reference itself next to the C restatement (oracle/splat_oracle.c) and
// the CUDA kernels, plus a few reference-only entry points (Adam from fresh moments,
// depth_reinitialize) used to pin the restatement.
#define ORACLE_FN(name) ref_##name
#include "splat_oracle.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "splat/densify.hpp"
#include "splat/gradients.hpp"
#include "splat/loss.hpp"
#include "splat/optimizer.hpp"
#include "splat/ply_io.hpp"
#include "splat/rasterizer.hpp"
#include "splat/simplify.hpp"
#include "splat/spatial.hpp"
#include "splat/visibility.hpp"

using namespace splat;

namespace {

std::string g_err;

int map_exception(const std::exception& e, int code) {
    g_err = e.what();
    return code;
}

#define REF_TRY try {
#define REF_CATCH                                                        \
    }                                                                    \
    catch (const std::invalid_argument& e) {                             \
        return map_exception(e, SPLAT_ERR_INVALID_ARGUMENT);             \
    }                                                                    \
    catch (const std::logic_error& e) {                                  \
        return map_exception(e, SPLAT_ERR_LOGIC);                        \
    }                                                                    \
    catch (const std::runtime_error& e) {                                \
        return map_exception(e, SPLAT_ERR_RUNTIME);                      \
    }                                                                    \
    catch (const std::exception& e) {                                    \
        return map_exception(e, SPLAT_ERR_RUNTIME);                      \
    }

GaussianSet to_set(const splat_gaussians* g) {
    GaussianSet s;
    s.active_sh_degree = g->active_sh_degree;
    s.resize(g->n);
    for (int i = 0; i < g->n; ++i) {
        s.centers[i] = Vec3f(g->centers[3 * i], g->centers[3 * i + 1], g->centers[3 * i + 2]);
        s.log_scales[i] = Vec3f(g->log_scales[3 * i], g->log_scales[3 * i + 1], g->log_scales[3 * i + 2]);
        s.rotations[i] = Vec4f(g->rotations[4 * i], g->rotations[4 * i + 1], g->rotations[4 * i + 2],
                               g->rotations[4 * i + 3]);
        s.opacity_logits[i] = g->opacity_logits[i];
    }
    if (g->n > 0) std::memcpy(s.sh.data(), g->sh, sizeof(float) * 48 * static_cast<size_t>(g->n));
    return s;
}

Camera to_cam(const splat_camera* c) {
    Camera cam;
    cam.width = c->width;
    cam.height = c->height;
    cam.fx = c->fx;
    cam.fy = c->fy;
    cam.cx = c->cx;
    cam.cy = c->cy;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) cam.rotation(i, j) = c->rotation[i * 3 + j];
    cam.translation = Vec3f(c->translation[0], c->translation[1], c->translation[2]);
    cam.znear = c->znear;
    cam.zfar = c->zfar;
    return cam;
}

RasterConfig to_cfg(const splat_raster_config* c) {
    RasterConfig r;
    r.tile_size = c->tile_size;
    r.transmittance_min = c->transmittance_min;
    r.contribution_min = c->contribution_min;
    r.alpha_max = c->alpha_max;
    r.lowpass = c->lowpass;
    r.radius_sigmas = c->radius_sigmas;
    r.apply_thresholds = c->apply_thresholds != 0;
    return r;
}

std::vector<char> to_mask(const uint8_t* m, int n) {
    std::vector<char> v(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) v[i] = static_cast<char>(m[i]);
    return v;
}

AdamConfig to_adam(const splat_adam_config* c) {
    AdamConfig a;
    a.beta1 = c->beta1;
    a.beta2 = c->beta2;
    a.eps = c->eps;
    a.position.lr_init = c->lr_init;
    a.position.lr_final = c->lr_final;
    a.position.max_steps = c->max_steps;
    a.scene_extent = c->scene_extent;
    a.lr_sh_dc = c->lr_sh_dc;
    a.lr_sh_rest = c->lr_sh_rest;
    a.lr_opacity = c->lr_opacity;
    a.lr_scale = c->lr_scale;
    a.lr_rotation = c->lr_rotation;
    return a;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

float ref_exp(float x) { return std::exp(x); }

int ref_project(const splat_gaussians* g, const splat_camera* c, const splat_raster_config* cf,
                const uint8_t* mask, int32_t* n_survivors, int32_t* order, int32_t* rect,
                int32_t* radius, float* depth, float* mean2d, float* conic, float* color,
                float* opacity) {
    REF_TRY
    const GaussianSet set = to_set(g);
    const Camera cam = to_cam(c);
    std::vector<char> mv;
    if (mask) mv = to_mask(mask, g->n);
    const auto proj = project<float>(set, cam, to_cfg(cf), mask ? &mv : nullptr);
    *n_survivors = static_cast<int32_t>(proj.size());
    for (size_t r = 0; r < proj.size(); ++r) {
        const auto& pg = proj[r];
        const int i = pg.index;
        if (order) order[r] = i;
        if (rect) {
            rect[4 * i] = pg.x0;
            rect[4 * i + 1] = pg.x1;
            rect[4 * i + 2] = pg.y0;
            rect[4 * i + 3] = pg.y1;
        }
        if (radius) radius[i] = pg.radius;
        if (depth) depth[i] = pg.depth_mean;
        if (mean2d) {
            mean2d[2 * i] = pg.mean2d[0];
            mean2d[2 * i + 1] = pg.mean2d[1];
        }
        if (conic)
            for (int k = 0; k < 3; ++k) conic[3 * i + k] = pg.conic[k];
        if (color)
            for (int k = 0; k < 3; ++k) color[3 * i + k] = pg.color[k];
        if (opacity) opacity[i] = pg.opacity;
    }
    return 0;
    REF_CATCH
}

int ref_tiles(const splat_gaussians* g, const splat_camera* c, const splat_raster_config* cf,
              const uint8_t* mask, int64_t* n_pairs, int32_t* ranges, int32_t* gaussian,
              int64_t capacity) {
    REF_TRY
    const GaussianSet set = to_set(g);
    const Camera cam = to_cam(c);
    cam.validate();
    std::vector<char> mv;
    if (mask) mv = to_mask(mask, g->n);
    const RasterConfig cfg = to_cfg(cf);
    const auto proj = project<float>(set, cam, cfg, mask ? &mv : nullptr);
    const auto grid = detail::bin_tiles(proj, cam.width, cam.height, cfg.tile_size);
    int64_t total = 0;
    for (size_t t = 0; t < grid.lists.size(); ++t) {
        if (ranges) {
            ranges[2 * t] = static_cast<int32_t>(total);
            ranges[2 * t + 1] = static_cast<int32_t>(total + grid.lists[t].size());
        }
        total += static_cast<int64_t>(grid.lists[t].size());
    }
    *n_pairs = total;
    if (gaussian && capacity >= total) {
        int64_t k = 0;
        for (const auto& list : grid.lists)
            for (int pos : list) gaussian[k++] = proj[pos].index;
    }
    return 0;
    REF_CATCH
}

int ref_render(const splat_gaussians* g, const splat_camera* c, const splat_raster_config* cf,
               const uint8_t* mask, const float bg[3], float* color, float* alpha, float* depth,
               float* transmittance, int32_t* max_contributor, float* importance,
               float* max_weight, int32_t* max_pixel_count, int64_t* stats) {
    REF_TRY
    const GaussianSet set = to_set(g);
    const Camera cam = to_cam(c);
    std::vector<char> mv;
    if (mask) mv = to_mask(mask, g->n);
    ImportanceReport<float> report;
    const bool want_report = importance || max_weight || max_pixel_count;
    const auto out = render<float>(set, cam, to_cfg(cf), mask ? &mv : nullptr,
                                   Vec3f(bg[0], bg[1], bg[2]), want_report ? &report : nullptr);
    const size_t hw = static_cast<size_t>(cam.width) * cam.height;
    if (color) std::memcpy(color, out.color.data.data(), sizeof(float) * hw * 3);
    if (alpha) std::memcpy(alpha, out.alpha.data.data(), sizeof(float) * hw);
    if (depth) std::memcpy(depth, out.depth.data.data(), sizeof(float) * hw);
    if (transmittance) std::memcpy(transmittance, out.transmittance.data.data(), sizeof(float) * hw);
    if (max_contributor) std::memcpy(max_contributor, out.max_contributor.data(), sizeof(int32_t) * hw);
    if (importance) std::memcpy(importance, report.importance.data(), sizeof(float) * g->n);
    if (max_weight) std::memcpy(max_weight, report.max_weight.data(), sizeof(float) * g->n);
    if (max_pixel_count)
        std::memcpy(max_pixel_count, report.max_pixel_count.data(), sizeof(int32_t) * g->n);
    if (stats) stats[0] = stats[1] = -1;
    return 0;
    REF_CATCH
}

int ref_accumulate_importance(const splat_gaussians* g, const splat_camera* c,
                              const splat_raster_config* cf, const uint8_t* mask,
                              float* importance, float* max_weight, int32_t* max_pixel_count) {
    REF_TRY
    const GaussianSet set = to_set(g);
    std::vector<char> mv;
    if (mask) mv = to_mask(mask, g->n);
    const auto rep = accumulate_importance<float>(set, to_cam(c), to_cfg(cf), mask ? &mv : nullptr);
    std::memcpy(importance, rep.importance.data(), sizeof(float) * g->n);
    std::memcpy(max_weight, rep.max_weight.data(), sizeof(float) * g->n);
    std::memcpy(max_pixel_count, rep.max_pixel_count.data(), sizeof(int32_t) * g->n);
    return 0;
    REF_CATCH
}

int ref_render_backward(const splat_gaussians* g, const splat_camera* c,
                        const splat_raster_config* cf, const float* d_color, const uint8_t* mask,
                        const float bg[3], float* d_centers, float* d_log_scales,
                        float* d_rotations, float* d_opacity, float* d_sh, float* grad2d_accum,
                        int32_t* grad2d_count) {
    REF_TRY
    const GaussianSet set = to_set(g);
    const Camera cam = to_cam(c);
    std::vector<char> mv;
    if (mask) mv = to_mask(mask, g->n);
    Imagef dc(cam.width, cam.height, 3);
    std::memcpy(dc.data.data(), d_color, sizeof(float) * dc.data.size());
    const auto gr = render_backward<float>(set, cam, to_cfg(cf), dc, mask ? &mv : nullptr,
                                           Vec3f(bg[0], bg[1], bg[2]));
    for (int i = 0; i < g->n; ++i) {
        for (int k = 0; k < 3; ++k) {
            d_centers[3 * i + k] = gr.d_centers[i][k];
            d_log_scales[3 * i + k] = gr.d_log_scales[i][k];
        }
        for (int k = 0; k < 4; ++k) d_rotations[4 * i + k] = gr.d_rotations[i][k];
        d_opacity[i] = gr.d_opacity_logits[i];
        if (grad2d_accum) grad2d_accum[i] = gr.grad2d_accum[i];
        if (grad2d_count) grad2d_count[i] = gr.grad2d_count[i];
    }
    if (g->n > 0) std::memcpy(d_sh, gr.d_sh.data(), sizeof(float) * 48 * static_cast<size_t>(g->n));
    return 0;
    REF_CATCH
}

float ref_l1_loss(const float* a, const float* b, int64_t count, float* grad) {
    Imagef ia(static_cast<int>(count), 1, 1), ib(static_cast<int>(count), 1, 1), ig;
    std::memcpy(ia.data.data(), a, sizeof(float) * count);
    std::memcpy(ib.data.data(), b, sizeof(float) * count);
    const float l = l1_loss<float>(ia, ib, grad ? &ig : nullptr);
    if (grad) std::memcpy(grad, ig.data.data(), sizeof(float) * count);
    return l;
}

double ref_lr_at(const splat_adam_config* cfg, int32_t step) {
    return to_adam(cfg).position.at(step);
}

// `steps` reference OptimState::step calls from fresh (zero) moments with the same grads.
int ref_adam_steps(float* centers, float* log_scales, float* rotations, float* opacity_logits,
                   float* sh, int32_t n, const float* d_centers, const float* d_log_scales,
                   const float* d_rotations, const float* d_opacity, const float* d_sh,
                   const splat_adam_config* cfg, int32_t steps) {
    REF_TRY
    splat_gaussians gv{centers, log_scales, rotations, opacity_logits, sh, n, 3};
    GaussianSet set = to_set(&gv);
    ParamGrads<float> gr;
    gr.resize_zero(n);
    for (int i = 0; i < n; ++i) {
        gr.d_centers[i] = Vec3f(d_centers[3 * i], d_centers[3 * i + 1], d_centers[3 * i + 2]);
        gr.d_log_scales[i] = Vec3f(d_log_scales[3 * i], d_log_scales[3 * i + 1], d_log_scales[3 * i + 2]);
        gr.d_rotations[i] = Vec4f(d_rotations[4 * i], d_rotations[4 * i + 1], d_rotations[4 * i + 2],
                                  d_rotations[4 * i + 3]);
        gr.d_opacity_logits[i] = d_opacity[i];
    }
    if (n > 0) std::memcpy(gr.d_sh.data(), d_sh, sizeof(float) * 48 * static_cast<size_t>(n));
    OptimState opt(to_adam(cfg), n);
    for (int s = 0; s < steps; ++s) opt.step(set, gr);
    for (int i = 0; i < n; ++i) {
        for (int k = 0; k < 3; ++k) {
            centers[3 * i + k] = set.centers[i][k];
            log_scales[3 * i + k] = set.log_scales[i][k];
        }
        for (int k = 0; k < 4; ++k) rotations[4 * i + k] = set.rotations[i][k];
        opacity_logits[i] = set.opacity_logits[i];
    }
    if (n > 0) std::memcpy(sh, set.sh.data(), sizeof(float) * 48 * static_cast<size_t>(n));
    return 0;
    REF_CATCH
}

// depth_reinitialize (densify.cpp:197-253) over one view; writes the fresh set's centers
// (a seeded permutation of the unprojected pool when sample_count >= pool size).
int ref_depth_reinitialize(const splat_gaussians* g, const splat_camera* c,
                           const splat_raster_config* cf, const float* image,
                           int32_t sample_count, uint32_t seed, float* centers_out,
                           int32_t* count_out) {
    REF_TRY
    const GaussianSet set = to_set(g);
    const Camera cam = to_cam(c);
    Imagef img(cam.width, cam.height, 3);
    std::memcpy(img.data.data(), image, sizeof(float) * img.data.size());
    std::mt19937 rng(seed);
    const GaussianSet fresh = depth_reinitialize(set, {cam}, {img}, sample_count, to_cfg(cf), rng);
    *count_out = fresh.size();
    for (int i = 0; i < fresh.size(); ++i)
        for (int k = 0; k < 3; ++k) centers_out[3 * i + k] = fresh.centers[i][k];
    return 0;
    REF_CATCH
}

// global_importance (simplify.cpp:13-34) over several views: fp64 Σ importance and Σ counts.
int ref_global_importance(const splat_gaussians* g, const splat_camera* cams, int32_t n_cams,
                          const splat_raster_config* cf, double* accum_weight,
                          int32_t* intersections) {
    REF_TRY
    const GaussianSet set = to_set(g);
    std::vector<Camera> cv;
    for (int k = 0; k < n_cams; ++k) cv.push_back(to_cam(&cams[k]));
    const auto gi = global_importance(set, cv, to_cfg(cf));
    for (int i = 0; i < g->n; ++i) {
        accum_weight[i] = gi.accum_weight[i];
        intersections[i] = gi.intersections[i];
    }
    return 0;
    REF_CATCH
}


// render_backward<double> on the float inputs promoted to double: an fp64 "truth" used to show
// that the GPU's float gradients are as close to exact as the reference's own float path.
int ref_render_backward_f64(const splat_gaussians* g, const splat_camera* c, const splat_raster_config* cf,
                            const float* d_color, const uint8_t* mask, const float bg[3], double* d_centers,
                            double* d_log_scales, double* d_rotations, double* d_opacity, double* d_sh) {
    REF_TRY
    const GaussianSetT<double> set = to_set(g).cast<double>();
    const CameraT<double> cam = to_cam(c).cast<double>();
    std::vector<char> mv;
    if (mask) mv = to_mask(mask, g->n);
    Image<double> dc(cam.width, cam.height, 3);
    for (size_t k = 0; k < dc.data.size(); ++k) dc.data[k] = d_color[k];
    const auto gr = render_backward<double>(set, cam, to_cfg(cf), dc, mask ? &mv : nullptr,
                                            Vec3<double>(bg[0], bg[1], bg[2]));
    for (int i = 0; i < g->n; ++i) {
        for (int k = 0; k < 3; ++k) {
            d_centers[3 * i + k] = gr.d_centers[i][k];
            d_log_scales[3 * i + k] = gr.d_log_scales[i][k];
        }
        for (int k = 0; k < 4; ++k) d_rotations[4 * i + k] = gr.d_rotations[i][k];
        d_opacity[i] = gr.d_opacity_logits[i];
    }
    for (size_t k = 0; k < gr.d_sh.size(); ++k) d_sh[k] = gr.d_sh[k];
    return 0;
    REF_CATCH
}


// ---- CPU baseline: one config-1 training view through the reference's own API ---------------
// A scene handle owns a GaussianSet + OptimState so the timed call runs only reference code:
// render<float> -> l1_loss -> render_backward<float> -> OptimState::step with only d_centers
// populated (config 1: Adam on means; zero grads + zero moments leave the other groups unchanged,
// test_optimizer.cpp:147-159).
struct RefScene {
    GaussianSet set;
    OptimState opt;
    RefScene(GaussianSet s, const AdamConfig& c) : set(std::move(s)), opt(c, 0) { opt.reinit(set.size()); }
};

void* ref_scene_create(const splat_gaussians* g, const splat_adam_config* cfg) {
    try {
        return new RefScene(to_set(g), to_adam(cfg));
    } catch (...) {
        return nullptr;
    }
}

void ref_scene_destroy(void* h) { delete static_cast<RefScene*>(h); }

int ref_train_view(void* h, const splat_camera* c, const splat_raster_config* cf, const float* target,
                   float* loss_out) {
    REF_TRY
    RefScene& sc = *static_cast<RefScene*>(h);
    const Camera cam = to_cam(c);
    const RasterConfig cfg = to_cfg(cf);
    const auto out = render<float>(sc.set, cam, cfg);
    Imagef tgt(cam.width, cam.height, 3), d_color;
    std::memcpy(tgt.data.data(), target, sizeof(float) * tgt.data.size());
    const float loss = l1_loss<float>(out.color, tgt, &d_color);
    ParamGrads<float> g = render_backward<float>(sc.set, cam, cfg, d_color);
    ParamGrads<float> means;
    means.resize_zero(sc.set.size());
    means.d_centers = g.d_centers;
    sc.opt.step(sc.set, means);
    if (loss_out) *loss_out = loss;
    return 0;
    REF_CATCH
}

// ---- densification / simplification, the reference's own functions ---------

// The uniform draws identify_critical's Random criterion makes from a fresh std::mt19937(seed)
// (densify.cpp:78-81), exported so the restatement and the GPU can be fed the same scores.
int ref_random_scores(uint32_t seed, int32_t n, double* out) {
    std::mt19937 rng(seed);
    std::uniform_real_distribution<double> u(0.0, 1.0);
    for (int i = 0; i < n; ++i) out[i] = u(rng);
    return 0;
}

// identify_critical (densify.cpp:32-103); masks: optional [n_cams][n] bytes (VisibilityTable).
int ref_identify_critical_views(const splat_gaussians* g, const splat_camera* cams, int32_t n_cams,
                                const splat_raster_config* cf, int criterion, double keep_q, uint32_t seed,
                                const uint8_t* masks, uint8_t* critical, int32_t* count) {
    REF_TRY
    const GaussianSet set = to_set(g);
    std::vector<Camera> cv;
    for (int k = 0; k < n_cams; ++k) cv.push_back(to_cam(&cams[k]));
    VisibilityTable table;
    if (masks) {
        table.gaussian_count = g->n;
        for (int k = 0; k < n_cams; ++k)
            table.masks.emplace_back(masks + (size_t)k * g->n, masks + (size_t)(k + 1) * g->n);
    }
    std::mt19937 rng(seed);
    const IdentCriterion crit = criterion == SPLAT_CRITERION_RANDOM    ? IdentCriterion::Random
                                : criterion == SPLAT_CRITERION_OPACITY ? IdentCriterion::Opacity
                                : criterion == SPLAT_CRITERION_ACCUM_WEIGHT ? IdentCriterion::AccumWeight
                                                                            : IdentCriterion::MaxWeight;
    const CriticalSelection sel = identify_critical(set, cv, crit, keep_q, to_cfg(cf), rng, masks ? &table : nullptr);
    for (int i = 0; i < g->n; ++i) critical[i] = sel.critical[i] ? 1 : 0;
    *count = sel.count;
    return 0;
    REF_CATCH
}

// aggressive_clone + apply_densify_plan (densify.cpp:105-130, 159-195): the applied set written
// to the output arrays (capacity rows), moment_source, new row count.
int ref_aggressive_clone_apply(const splat_gaussians* g, const uint8_t* critical, float* centers, float* log_scales,
                         float* rotations, float* opacity_logits, float* sh, int64_t capacity,
                         int32_t* moment_source, int32_t* n_out) {
    REF_TRY
    const GaussianSet set = to_set(g);
    std::vector<char> crit(critical, critical + g->n);
    const DensifyPlan plan = aggressive_clone(set, crit);
    const DensifyApplied out = apply_densify_plan(set, plan);
    const int m = out.set.size();
    *n_out = m;
    if (m > capacity) throw std::invalid_argument("ref_aggressive_clone: capacity");
    for (int i = 0; i < m; ++i) {
        for (int c = 0; c < 3; ++c) {
            centers[3 * i + c] = out.set.centers[i][c];
            log_scales[3 * i + c] = out.set.log_scales[i][c];
        }
        for (int c = 0; c < 4; ++c) rotations[4 * i + c] = out.set.rotations[i][c];
        opacity_logits[i] = out.set.opacity_logits[i];
        moment_source[i] = out.moment_source[i];
    }
    if (m > 0) std::memcpy(sh, out.set.sh.data(), sizeof(float) * 48 * static_cast<size_t>(m));
    return 0;
    REF_CATCH
}

// build_masks (visibility.cpp:9-37): masks [n_cams][n] bytes.
int ref_build_masks(const splat_gaussians* g, const splat_camera* cams, int32_t n_cams, const splat_raster_config* cf,
                    double keep_q, uint8_t* masks) {
    REF_TRY
    const GaussianSet set = to_set(g);
    std::vector<Camera> cv;
    for (int k = 0; k < n_cams; ++k) cv.push_back(to_cam(&cams[k]));
    const VisibilityTable t = build_masks(set, cv, keep_q, to_cfg(cf));
    for (int k = 0; k < n_cams; ++k)
        for (int i = 0; i < g->n; ++i) masks[(size_t)k * g->n + i] = t.masks[k][i] ? 1 : 0;
    return 0;
    REF_CATCH
}

// importance_prune (simplify.cpp:94-107) on a set of n rows: the kept indices.
int ref_importance_prune_set(const splat_gaussians* g, const double* importance, double keep_q, int32_t* kept,
                         int32_t* n_kept) {
    REF_TRY
    const GaussianSet set = to_set(g);
    std::vector<double> imp(importance, importance + g->n);
    const SimplifyResult r = importance_prune(set, imp, keep_q);
    for (size_t k = 0; k < r.kept.size(); ++k) kept[k] = r.kept[k];
    *n_kept = static_cast<int32_t>(r.kept.size());
    return 0;
    REF_CATCH
}

// ssim / photometric_loss (loss.cpp:78-147) on H x W x ch images.
float ref_ssim(const float* a, const float* b, int w, int h, int ch, float* grad_a) {
    Imagef ia(w, h, ch), ib(w, h, ch), ig;
    std::memcpy(ia.data.data(), a, sizeof(float) * ia.size());
    std::memcpy(ib.data.data(), b, sizeof(float) * ib.size());
    const float s = ssim<float>(ia, ib, grad_a ? &ig : nullptr);
    if (grad_a) std::memcpy(grad_a, ig.data.data(), sizeof(float) * ig.size());
    return s;
}

float ref_photometric_loss(const float* rendered, const float* target, int w, int h, int ch, float lambda,
                           float* grad) {
    Imagef ia(w, h, ch), ib(w, h, ch), ig;
    std::memcpy(ia.data.data(), rendered, sizeof(float) * ia.size());
    std::memcpy(ib.data.data(), target, sizeof(float) * ib.size());
    const float l = photometric_loss<float>(ia, ib, lambda, grad ? &ig : nullptr);
    if (grad) std::memcpy(grad, ig.data.data(), sizeof(float) * ig.size());
    return l;
}

// ---- depth re-initialisation tail (densify.cpp:227-251, spatial.cpp:101-121) -------------
int ref_third_neighbor_distances(const float* points, int32_t m, float min_dist, float* out) {
    REF_TRY
    std::vector<Vec3f> p(m);
    for (int i = 0; i < m; ++i) p[i] = Vec3f(points[3 * i], points[3 * i + 1], points[3 * i + 2]);
    const std::vector<float> d = third_neighbor_distances(p, min_dist);
    for (int i = 0; i < m; ++i) out[i] = d[i];
    return 0;
    REF_CATCH
}

// The pool indices depth_reinitialize's partial Fisher-Yates draws (densify.cpp:227-235) from a
// fresh std::mt19937(seed) — the reference's sampling, exported so the device path can be fed it.
int ref_fisher_yates(uint32_t seed, int32_t pool, int32_t take, int32_t* idx_out) {
    std::mt19937 rng(seed);
    std::vector<int> idx(pool);
    for (int i = 0; i < pool; ++i) idx[i] = i;
    for (int r = 0; r < take; ++r) {
        std::uniform_int_distribution<int> pick(r, pool - 1);
        std::swap(idx[r], idx[pick(rng)]);
    }
    for (int r = 0; r < take; ++r) idx_out[r] = idx[r];
    return 0;
}

// depth_reinitialize over several views with their images: the fresh set, rows = min(sample_count, pool).
int ref_depth_reinitialize_views(const splat_gaussians* g, const splat_camera* cams, int32_t n_cams,
                                 const splat_raster_config* cf, const float* images, int32_t sample_count,
                                 uint32_t seed, float* centers, float* log_scales, float* rotations,
                                 float* opacity_logits, float* sh, int32_t* count_out) {
    REF_TRY
    const GaussianSet set = to_set(g);
    std::vector<Camera> cv;
    std::vector<Imagef> imgs;
    size_t off = 0;
    for (int k = 0; k < n_cams; ++k) {
        cv.push_back(to_cam(&cams[k]));
        Imagef img(cv.back().width, cv.back().height, 3);
        std::memcpy(img.data.data(), images + off, sizeof(float) * img.data.size());
        off += img.data.size();
        imgs.push_back(std::move(img));
    }
    std::mt19937 rng(seed);
    const GaussianSet fresh = depth_reinitialize(set, cv, imgs, sample_count, to_cfg(cf), rng);
    const int m = fresh.size();
    *count_out = m;
    for (int i = 0; i < m; ++i) {
        for (int c = 0; c < 3; ++c) {
            centers[3 * i + c] = fresh.centers[i][c];
            log_scales[3 * i + c] = fresh.log_scales[i][c];
        }
        for (int c = 0; c < 4; ++c) rotations[4 * i + c] = fresh.rotations[i][c];
        opacity_logits[i] = fresh.opacity_logits[i];
    }
    if (m > 0) std::memcpy(sh, fresh.sh.data(), sizeof(float) * 48 * static_cast<size_t>(m));
    return 0;
    REF_CATCH
}

// ---- the reference's random draws and the draw-consuming §8f functions ---------------------
// std::normal_distribution<float>(0, 1) on a fresh std::mt19937(seed), one distribution object
// (the draws vanilla_clone_split makes, densify.cpp:141, 154).
int ref_rng_normal_f32(uint32_t seed, int32_t n, float* out) {
    std::mt19937 rng(seed);
    std::normal_distribution<float> gauss(0.f, 1.f);
    for (int i = 0; i < n; ++i) out[i] = gauss(rng);
    return 0;
}

// uniform_real_distribution<double> / uniform_int_distribution<int>(lo[i], hi[i]) interleaved on a
// fresh std::mt19937_64(seed): kinds[i] = 0 real, 1 int (the engine importance_sample uses).
int ref_rng_mixed_64(uint64_t seed, int32_t n, const int32_t* kinds, const int32_t* lo, const int32_t* hi,
                     double* out) {
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> u(0.0, 1.0);
    for (int i = 0; i < n; ++i) {
        if (kinds[i] == 0) {
            out[i] = u(rng);
        } else {
            std::uniform_int_distribution<int> pick(lo[i], hi[i]);
            out[i] = pick(rng);
        }
    }
    return 0;
}

// importance_sample (simplify.cpp:36-92): kept indices (ascending), target_count of them.
int ref_importance_sample_set(const splat_gaussians* g, const double* importance, int32_t target, uint64_t seed,
                              int32_t* kept, int32_t* n_kept) {
    REF_TRY
    const GaussianSet set = to_set(g);
    std::vector<double> imp(importance, importance + g->n);
    const SimplifyResult r = importance_sample(set, imp, target, seed);
    for (size_t k = 0; k < r.kept.size(); ++k) kept[k] = r.kept[k];
    *n_kept = static_cast<int32_t>(r.kept.size());
    return 0;
    REF_CATCH
}

// vanilla_clone_split + apply_densify_plan (densify.cpp:132-195, Progressive mode) with a fresh
// std::mt19937(seed): the resulting set (capacity rows), moment sources, clone / split counts.
int ref_vanilla_clone_split_apply(const splat_gaussians* g, const float* grad2d_accum, const int32_t* grad2d_count,
                                  float grad_threshold, float scale_threshold, float scene_extent, uint32_t seed,
                                  float* centers, float* log_scales, float* rotations, float* opacity_logits, float* sh,
                                  int64_t capacity, int32_t* moment_source, int32_t* n_out, int32_t* n_clone,
                                  int32_t* n_split) {
    REF_TRY
    const GaussianSet set = to_set(g);
    ParamGrads<float> grads;
    grads.resize_zero(g->n);
    for (int i = 0; i < g->n; ++i) {
        grads.grad2d_accum[i] = grad2d_accum[i];
        grads.grad2d_count[i] = grad2d_count[i];
    }
    std::mt19937 rng(seed);
    const DensifyPlan plan = vanilla_clone_split(set, grads, grad_threshold, scale_threshold, scene_extent, rng);
    const DensifyApplied out = apply_densify_plan(set, plan);
    const int m = out.set.size();
    *n_out = m;
    *n_clone = static_cast<int32_t>(plan.clone_indices.size());
    *n_split = static_cast<int32_t>(plan.split_indices.size());
    if (m > capacity) throw std::invalid_argument("vanilla_clone_split: capacity too small");
    for (int i = 0; i < m; ++i) {
        for (int c = 0; c < 3; ++c) {
            centers[3 * i + c] = out.set.centers[i][c];
            log_scales[3 * i + c] = out.set.log_scales[i][c];
        }
        for (int c = 0; c < 4; ++c) rotations[4 * i + c] = out.set.rotations[i][c];
        opacity_logits[i] = out.set.opacity_logits[i];
        moment_source[i] = out.moment_source[i];
    }
    if (m > 0) std::memcpy(sh, out.set.sh.data(), sizeof(float) * 48 * static_cast<size_t>(m));
    return 0;
    REF_CATCH
}

// ---- PLY checkpoints (ply_io.cpp) ------------------------------------------------------
int ref_write_ply(const char* path, const splat_gaussians* g) {
    REF_TRY
    write_ply(path, to_set(g));
    return 0;
    REF_CATCH
}

// read_ply into caller arrays with room for `capacity` rows; *n_out = rows in the file.
int ref_read_ply(const char* path, float* centers, float* log_scales, float* rotations, float* opacity_logits,
                 float* sh, int32_t capacity, int32_t* n_out) {
    REF_TRY
    const GaussianSet s = read_ply(path);
    *n_out = s.size();
    if (s.size() > capacity) throw std::invalid_argument("ref_read_ply: capacity");
    for (int i = 0; i < s.size(); ++i) {
        for (int c = 0; c < 3; ++c) {
            centers[3 * i + c] = s.centers[i][c];
            log_scales[3 * i + c] = s.log_scales[i][c];
        }
        for (int c = 0; c < 4; ++c) rotations[4 * i + c] = s.rotations[i][c];
        opacity_logits[i] = s.opacity_logits[i];
    }
    if (s.size() > 0) std::memcpy(sh, s.sh.data(), sizeof(float) * 48 * static_cast<size_t>(s.size()));
    return 0;
    REF_CATCH
}

}  // extern "C"
