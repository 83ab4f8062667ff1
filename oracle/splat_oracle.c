/*
 * splat_oracle.c — plain-C restatement of the reference rasterizer hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see splat_oracle.h).  Follows /root/reference/proj function by
 * function, in the reference's operation order as fixed by oracle/compat/Eigen/Dense
 * (halving reductions: sum3 = a + (b + c), sum4 = (a + b) + (c + d); left-associative
 * products with materialised intermediates).  Compile with -ffp-contract=off.
 *
 * EXP selects the exponential: splat_expf (mode B, default) or glibc expf (mode A).
 */
#include "splat_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "splat_expf.h"

#ifdef ORACLE_USE_LIBM_EXP
#define EXP expf
#define LOG logf
#else
#define EXP splat_expf
#define LOG splat_logf
#endif

#define SPLAT_RNG_LOGF LOG
#include "splat_rng.h"

static char g_err[256];
static int fail(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}
const char* ORACLE_FN(last_error)(void) { return g_err; }
float ORACLE_FN(exp)(float x) { return EXP(x); }

/* ---- small fixed-size helpers (shim order) ---------------------------------------- */
static inline float dot3(const float* a, const float* b) { return a[0] * b[0] + (a[1] * b[1] + a[2] * b[2]); }
static inline float sq3(const float* a) { return a[0] * a[0] + (a[1] * a[1] + a[2] * a[2]); }
static inline float sq4(const float* a) { return (a[0] * a[0] + a[1] * a[1]) + (a[2] * a[2] + a[3] * a[3]); }
static inline float sigmoidf_(float x) { return 1.0f / (1.0f + EXP(-x)); } /* types.hpp:58-60 */
static inline float fmax_std(float a, float b) { return (a < b) ? b : a; } /* std::max */
static inline float fmin_std(float a, float b) { return (b < a) ? b : a; } /* std::min */

/* SH constants (sh.hpp:14-22), cast double -> float as T(kSH_*) does. */
static const double kC0 = 0.28209479177387814;
static const double kC1 = 0.4886025119029199;
static const double kC2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                              -1.0925484305920792, 0.5462742152960396};
static const double kC3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                              0.3731763325901154, -0.4570457994644658, 1.445305721320277,
                              -0.5900435899266435};

/* sh_basis (sh.hpp:27-51) */
static void sh_basis(const float* dir, int degree, float* b) {
    for (int i = 0; i < 16; ++i) b[i] = 0.0f;
    b[0] = (float)kC0;
    if (degree < 1) return;
    const float x = dir[0], y = dir[1], z = dir[2];
    b[1] = -(float)kC1 * y;
    b[2] = (float)kC1 * z;
    b[3] = -(float)kC1 * x;
    if (degree < 2) return;
    const float xx = x * x, yy = y * y, zz = z * z;
    b[4] = (float)kC2[0] * x * y;
    b[5] = (float)kC2[1] * y * z;
    b[6] = (float)kC2[2] * (2.0f * zz - xx - yy);
    b[7] = (float)kC2[3] * x * z;
    b[8] = (float)kC2[4] * (xx - yy);
    if (degree < 3) return;
    b[9] = (float)kC3[0] * y * (3.0f * xx - yy);
    b[10] = (float)kC3[1] * x * y * z;
    b[11] = (float)kC3[2] * y * (4.0f * zz - xx - yy);
    b[12] = (float)kC3[3] * z * (2.0f * zz - 3.0f * xx - 3.0f * yy);
    b[13] = (float)kC3[4] * x * (4.0f * zz - xx - yy);
    b[14] = (float)kC3[5] * z * (xx - yy);
    b[15] = (float)kC3[6] * x * (xx - 3.0f * yy);
}

/* sh_basis_grad (sh.hpp:55-79); g[k][0..2] */
static void sh_basis_grad(const float* dir, int degree, float g[16][3]) {
    memset(g, 0, sizeof(float) * 48);
    if (degree < 1) return;
    const float x = dir[0], y = dir[1], z = dir[2];
    const float c1 = (float)kC1;
    g[1][0] = 0.0f; g[1][1] = -c1; g[1][2] = 0.0f;
    g[2][0] = 0.0f; g[2][1] = 0.0f; g[2][2] = c1;
    g[3][0] = -c1; g[3][1] = 0.0f; g[3][2] = 0.0f;
    if (degree < 2) return;
    const float xx = x * x, yy = y * y, zz = z * z;
#define SET3(k, C, a, b, c) do { const float cc_ = (float)(C); g[k][0] = cc_ * (a); g[k][1] = cc_ * (b); g[k][2] = cc_ * (c); } while (0)
    SET3(4, kC2[0], y, x, 0.0f);
    SET3(5, kC2[1], 0.0f, z, y);
    SET3(6, kC2[2], -2.0f * x, -2.0f * y, 4.0f * z);
    SET3(7, kC2[3], z, 0.0f, x);
    SET3(8, kC2[4], 2.0f * x, -2.0f * y, 0.0f);
    if (degree < 3) return;
    SET3(9, kC3[0], 6.0f * x * y, 3.0f * xx - 3.0f * yy, 0.0f);
    SET3(10, kC3[1], y * z, x * z, x * y);
    SET3(11, kC3[2], -2.0f * x * y, 4.0f * zz - xx - 3.0f * yy, 8.0f * y * z);
    SET3(12, kC3[3], -6.0f * x * z, -6.0f * y * z, 6.0f * zz - 3.0f * xx - 3.0f * yy);
    SET3(13, kC3[4], 4.0f * zz - 3.0f * xx - yy, -2.0f * x * y, 8.0f * x * z);
    SET3(14, kC3[5], 2.0f * x * z, -2.0f * y * z, xx - yy);
    SET3(15, kC3[6], 3.0f * xx - 3.0f * yy, -6.0f * x * y, 0.0f);
#undef SET3
}

static inline int sh_coeffs(int degree) { return (degree + 1) * (degree + 1); }

/* sh_to_color (sh.hpp:84-100) */
static void sh_to_color(const float* sh, const float* dir, int degree, float* rgb, int* clamped) {
    float b[16];
    sh_basis(dir, degree, b);
    rgb[0] = rgb[1] = rgb[2] = 0.5f;
    const int n = sh_coeffs(degree);
    for (int k = 0; k < n; ++k)
        for (int c = 0; c < 3; ++c) rgb[c] += b[k] * sh[k * 3 + c];
    for (int c = 0; c < 3; ++c) {
        const int neg = rgb[c] < 0.0f;
        if (clamped) clamped[c] = neg;
        if (neg) rgb[c] = 0.0f;
    }
}

/* normalized_quat (gaussian_set.hpp:15-20) */
static void normalized_quat(const float* q, float* out) {
    const float n = sqrtf(sq4(q));
    if (!(n > 0.0f)) {
        out[0] = 1.0f; out[1] = out[2] = out[3] = 0.0f;
        return;
    }
    for (int k = 0; k < 4; ++k) out[k] = q[k] / n;
}

/* rotation_from_quat (gaussian_set.hpp:23-37), row-major r[i*3+j] */
static void rotation_from_quat(const float* q_raw, float* r) {
    float q[4];
    normalized_quat(q_raw, q);
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

/* covariance_from_params (gaussian_set.hpp:41-55); cov row-major */
static void covariance(const float* log_scale, const float* rot, float* cov) {
    float r[9], s[3], m[9];
    rotation_from_quat(rot, r);
    for (int k = 0; k < 3; ++k) s[k] = EXP(log_scale[k]);
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) m[i * 3 + j] = r[i * 3 + j] * s[j];
    for (int i = 0; i < 3; ++i)
        for (int j = i; j < 3; ++j) {
            const float v = dot3(&m[i * 3], &m[j * 3]);
            cov[i * 3 + j] = v;
            cov[j * 3 + i] = v;
        }
}

/* Mat3 inverse with Eigen's cofactor scheme (see compat/Eigen/Dense) */
static void inverse3(const float* m, float* r) {
#define M(i, j) m[(i) * 3 + (j)]
#define COF(i, j) (M(((i) + 1) % 3, ((j) + 1) % 3) * M(((i) + 2) % 3, ((j) + 2) % 3) - \
                   M(((i) + 1) % 3, ((j) + 2) % 3) * M(((i) + 2) % 3, ((j) + 1) % 3))
    const float c00 = COF(0, 0), c10 = COF(1, 0), c20 = COF(2, 0);
    const float det = c00 * M(0, 0) + (c10 * M(1, 0) + c20 * M(2, 0));
    const float invdet = 1.0f / det;
    r[1 * 3 + 0] = COF(0, 1) * invdet;
    r[1 * 3 + 1] = COF(1, 1) * invdet;
    r[2 * 3 + 0] = COF(0, 2) * invdet;
    r[1 * 3 + 2] = COF(2, 1) * invdet;
    r[2 * 3 + 1] = COF(1, 2) * invdet;
    r[2 * 3 + 2] = COF(2, 2) * invdet;
    r[0] = c00 * invdet;
    r[1] = c10 * invdet;
    r[2] = c20 * invdet;
#undef COF
#undef M
}

/* camera.hpp:23-36 */
static void cam_to_camera(const splat_camera* c, const float* p, float* out) {
    for (int i = 0; i < 3; ++i) out[i] = dot3(&c->rotation[i * 3], p) + c->translation[i];
}
static void cam_center(const splat_camera* c, float* out) {
    for (int i = 0; i < 3; ++i) {
        const float col[3] = {c->rotation[i], c->rotation[3 + i], c->rotation[6 + i]};
        out[i] = -dot3(col, c->translation);
    }
}
static void cam_ray_direction(const splat_camera* c, int px, int py, float* out) {
    float d[3] = {((float)px + 0.5f - c->cx) / c->fx, ((float)py + 0.5f - c->cy) / c->fy, 1.0f};
    const float z = sq3(d);
    if (z > 0.0f) {
        const float n = sqrtf(z);
        for (int k = 0; k < 3; ++k) d[k] /= n;
    }
    for (int i = 0; i < 3; ++i) {
        const float col[3] = {c->rotation[i], c->rotation[3 + i], c->rotation[6 + i]};
        out[i] = dot3(col, d);
    }
}
static int camera_validate(const splat_camera* c) {
    if (c->width < 1 || c->height < 1) return fail(SPLAT_ERR_INVALID_ARGUMENT, "camera: degenerate image size");
    if (!(c->znear > 0.0f) || !(c->zfar > c->znear))
        return fail(SPLAT_ERR_INVALID_ARGUMENT, "camera: need 0 < znear < zfar");
    /* rotation * rotation^T - I, max |.| <= 1e-6 (camera.hpp:38-41) */
    float worst = 0.0f;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            const float v = dot3(&c->rotation[i * 3], &c->rotation[j * 3]) - (i == j ? 1.0f : 0.0f);
            worst = fmax_std(worst, fabsf(v));
        }
    if (!(worst <= 1e-6f)) return fail(SPLAT_ERR_INVALID_ARGUMENT, "camera: rotation not orthonormal");
    return 0;
}

/* ProjectedGaussian (rasterizer.hpp:27-41) */
typedef struct {
    float mean2d[2], cov2d[3], conic[3], depth;
    int radius, index;
    float opacity, color[3];
    int x0, x1, y0, y1;
    float center[3], cov_inv[9];
    int degenerate;
} proj_t;

static int cmp_proj(const void* a, const void* b) {
    const proj_t* p = (const proj_t*)a;
    const proj_t* q = (const proj_t*)b;
    if (p->depth != q->depth) return p->depth < q->depth ? -1 : 1;
    return (p->index > q->index) - (p->index < q->index);
}

/* project<T> (rasterizer.cpp:10-90). Returns survivors sorted by (depth, index). */
static int project_impl(const splat_gaussians* g, const splat_camera* cam, const splat_raster_config* cfg,
                        const uint8_t* mask, proj_t** out, int* n_out) {
    const int n = g->n;
    proj_t* proj = (proj_t*)malloc(sizeof(proj_t) * (size_t)(n > 0 ? n : 1));
    if (!proj) return fail(SPLAT_ERR_OUT_OF_MEMORY, "oracle: out of memory");
    int np = 0;
    float cc[3];
    cam_center(cam, cc);
    const int exact = !cfg->apply_thresholds;
    const float log_cond_limit = (float)log(1e12);
    const float fx = cam->fx, fy = cam->fy;
    const float* R = cam->rotation;
    for (int i = 0; i < n; ++i) {
        if (mask && !mask[i]) continue;
        const float* p = &g->centers[3 * i];
        float pc[3];
        cam_to_camera(cam, p, pc);
        const float z = pc[2];
        if (z <= cam->znear) continue;
        proj_t pg;
        memset(&pg, 0, sizeof pg);
        pg.index = i;
        pg.depth = z;
        pg.mean2d[0] = fx * pc[0] / pc[2] + cam->cx;
        pg.mean2d[1] = fy * pc[1] / pc[2] + cam->cy;
        float cov3d[9];
        covariance(&g->log_scales[3 * i], &g->rotations[4 * i], cov3d);
        /* J (2x3) row-major */
        const float J[6] = {fx / z, 0.0f, -fx * pc[0] / (z * z), 0.0f, fy / z, -fy * pc[1] / (z * z)};
        float Mm[6], A[6], V[4];
        for (int r = 0; r < 2; ++r)
            for (int c = 0; c < 3; ++c)
                Mm[r * 3 + c] = J[r * 3 + 0] * R[0 * 3 + c] + (J[r * 3 + 1] * R[1 * 3 + c] + J[r * 3 + 2] * R[2 * 3 + c]);
        for (int r = 0; r < 2; ++r)
            for (int c = 0; c < 3; ++c)
                A[r * 3 + c] = Mm[r * 3 + 0] * cov3d[0 * 3 + c] + (Mm[r * 3 + 1] * cov3d[1 * 3 + c] + Mm[r * 3 + 2] * cov3d[2 * 3 + c]);
        for (int r = 0; r < 2; ++r)
            for (int c = 0; c < 2; ++c)
                V[r * 2 + c] = A[r * 3 + 0] * Mm[c * 3 + 0] + (A[r * 3 + 1] * Mm[c * 3 + 1] + A[r * 3 + 2] * Mm[c * 3 + 2]);
        pg.cov2d[0] = V[0] + (float)cfg->lowpass;
        pg.cov2d[1] = V[1];
        pg.cov2d[2] = V[3] + (float)cfg->lowpass;
        const float det = pg.cov2d[0] * pg.cov2d[2] - pg.cov2d[1] * pg.cov2d[1];
        if (!(det > 0.0f)) continue;
        const float inv_det = 1.0f / det;
        pg.conic[0] = pg.cov2d[2] * inv_det;
        pg.conic[1] = -pg.cov2d[1] * inv_det;
        pg.conic[2] = pg.cov2d[0] * inv_det;
        if (exact) {
            pg.radius = cam->width > cam->height ? cam->width : cam->height;
            pg.x0 = 0; pg.x1 = cam->width;
            pg.y0 = 0; pg.y1 = cam->height;
        } else {
            const float mid = 0.5f * (pg.cov2d[0] + pg.cov2d[2]);
            const float lambda_max = mid + sqrtf(fmax_std(mid * mid - det, 0.0f));
            pg.radius = (int)ceilf((float)cfg->radius_sigmas * sqrtf(lambda_max));
            int v;
            v = (int)ceilf(pg.mean2d[0] - (float)pg.radius - 0.5f); pg.x0 = v > 0 ? v : 0;
            v = (int)floorf(pg.mean2d[0] + (float)pg.radius - 0.5f) + 1; pg.x1 = v < cam->width ? v : cam->width;
            v = (int)ceilf(pg.mean2d[1] - (float)pg.radius - 0.5f); pg.y0 = v > 0 ? v : 0;
            v = (int)floorf(pg.mean2d[1] + (float)pg.radius - 0.5f) + 1; pg.y1 = v < cam->height ? v : cam->height;
            if (pg.x0 >= pg.x1 || pg.y0 >= pg.y1) continue;
        }
        pg.opacity = sigmoidf_(g->opacity_logits[i]);
        float u[3] = {p[0] - cc[0], p[1] - cc[1], p[2] - cc[2]};
        const float zz = sq3(u);
        if (zz > 0.0f) {
            const float nrm = sqrtf(zz);
            for (int k = 0; k < 3; ++k) u[k] = u[k] / nrm;
        }
        int clamped[3];
        sh_to_color(&g->sh[48 * (size_t)i], u, g->active_sh_degree, pg.color, clamped);
        for (int k = 0; k < 3; ++k) pg.center[k] = p[k];
        const float* s = &g->log_scales[3 * i];
        const float smax = fmax_std(fmax_std(s[0], s[1]), s[2]);
        const float smin = fmin_std(fmin_std(s[0], s[1]), s[2]);
        pg.degenerate = 2.0f * (smax - smin) > log_cond_limit;
        if (pg.degenerate) {
            for (int k = 0; k < 9; ++k) pg.cov_inv[k] = (k % 4 == 0) ? 1.0f : 0.0f;
        } else {
            inverse3(cov3d, pg.cov_inv);
        }
        proj[np++] = pg;
    }
    qsort(proj, (size_t)np, sizeof(proj_t), cmp_proj);
    *out = proj;
    *n_out = np;
    return 0;
}

static int check_inputs(const splat_gaussians* g, const splat_camera* cam) {
    if (g->n < 0) return fail(SPLAT_ERR_LOGIC, "GaussianSet parallel arrays out of sync");
    if (g->n > 0 && (!g->centers || !g->log_scales || !g->rotations || !g->opacity_logits || !g->sh))
        return fail(SPLAT_ERR_LOGIC, "GaussianSet parallel arrays out of sync");
    return camera_validate(cam);
}

int ORACLE_FN(project)(const splat_gaussians* g, const splat_camera* cam, const splat_raster_config* cfg,
                       const uint8_t* mask, int32_t* n_survivors, int32_t* order, int32_t* rect,
                       int32_t* radius, float* depth, float* mean2d, float* conic, float* color,
                       float* opacity) {
    int rc = check_inputs(g, cam);
    if (rc) return rc;
    proj_t* proj;
    int np;
    if ((rc = project_impl(g, cam, cfg, mask, &proj, &np))) return rc;
    *n_survivors = np;
    for (int r = 0; r < np; ++r) {
        const proj_t* pg = &proj[r];
        const int i = pg->index;
        if (order) order[r] = i;
        if (rect) { rect[4 * i] = pg->x0; rect[4 * i + 1] = pg->x1; rect[4 * i + 2] = pg->y0; rect[4 * i + 3] = pg->y1; }
        if (radius) radius[i] = pg->radius;
        if (depth) depth[i] = pg->depth;
        if (mean2d) { mean2d[2 * i] = pg->mean2d[0]; mean2d[2 * i + 1] = pg->mean2d[1]; }
        if (conic) { for (int k = 0; k < 3; ++k) conic[3 * i + k] = pg->conic[k]; }
        if (color) { for (int k = 0; k < 3; ++k) color[3 * i + k] = pg->color[k]; }
        if (opacity) opacity[i] = pg->opacity;
    }
    free(proj);
    return 0;
}

/* bin_tiles (rasterizer.hpp:156-174): CSR of positions into proj */
typedef struct {
    int tiles_x, tiles_y;
    int64_t* start; /* tiles + 1 */
    int32_t* pos;
} grid_t;

static int bin_tiles(const proj_t* proj, int np, int w, int h, int ts, grid_t* grid) {
    grid->tiles_x = (w + ts - 1) / ts;
    grid->tiles_y = (h + ts - 1) / ts;
    const int nt = grid->tiles_x * grid->tiles_y;
    grid->start = (int64_t*)calloc((size_t)nt + 1, sizeof(int64_t));
    if (!grid->start) return fail(SPLAT_ERR_OUT_OF_MEMORY, "oracle: out of memory");
    for (int p = 0; p < np; ++p) {
        const proj_t* pg = &proj[p];
        for (int ty = pg->y0 / ts; ty <= (pg->y1 - 1) / ts; ++ty)
            for (int tx = pg->x0 / ts; tx <= (pg->x1 - 1) / ts; ++tx) grid->start[ty * grid->tiles_x + tx + 1]++;
    }
    for (int t = 0; t < nt; ++t) grid->start[t + 1] += grid->start[t];
    grid->pos = (int32_t*)malloc(sizeof(int32_t) * (size_t)(grid->start[nt] > 0 ? grid->start[nt] : 1));
    int64_t* fillp = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nt > 0 ? nt : 1));
    if (!grid->pos || !fillp) return fail(SPLAT_ERR_OUT_OF_MEMORY, "oracle: out of memory");
    for (int t = 0; t < nt; ++t) fillp[t] = grid->start[t];
    for (int p = 0; p < np; ++p) {
        const proj_t* pg = &proj[p];
        for (int ty = pg->y0 / ts; ty <= (pg->y1 - 1) / ts; ++ty)
            for (int tx = pg->x0 / ts; tx <= (pg->x1 - 1) / ts; ++tx) grid->pos[fillp[ty * grid->tiles_x + tx]++] = p;
    }
    free(fillp);
    return 0;
}
static void free_grid(grid_t* g) { free(g->start); free(g->pos); }

int ORACLE_FN(tiles)(const splat_gaussians* g, const splat_camera* cam, const splat_raster_config* cfg,
                     const uint8_t* mask, int64_t* n_pairs, int32_t* ranges, int32_t* gaussian, int64_t capacity) {
    int rc = check_inputs(g, cam);
    if (rc) return rc;
    if (cfg->tile_size < 1) return fail(SPLAT_ERR_INVALID_ARGUMENT, "tile_size < 1");
    proj_t* proj;
    int np;
    if ((rc = project_impl(g, cam, cfg, mask, &proj, &np))) return rc;
    grid_t grid;
    if ((rc = bin_tiles(proj, np, cam->width, cam->height, cfg->tile_size, &grid))) { free(proj); return rc; }
    const int nt = grid.tiles_x * grid.tiles_y;
    *n_pairs = grid.start[nt];
    if (ranges)
        for (int t = 0; t < nt; ++t) { ranges[2 * t] = (int32_t)grid.start[t]; ranges[2 * t + 1] = (int32_t)grid.start[t + 1]; }
    if (gaussian && capacity >= grid.start[nt])
        for (int64_t k = 0; k < grid.start[nt]; ++k) gaussian[k] = proj[grid.pos[k]].index;
    free_grid(&grid);
    free(proj);
    return 0;
}

/* depth_along_ray (rasterizer.hpp:87-96) */
static float depth_along_ray(const float* center, const float* ci, const float* origin, const float* dir) {
    const float rel[3] = {center[0] - origin[0], center[1] - origin[1], center[2] - origin[2]};
    float cd[3];
    for (int i = 0; i < 3; ++i) cd[i] = dot3(&ci[i * 3], dir);
    const float denom = dot3(dir, cd);
    const float t = dot3(rel, cd) / denom;
    if (!(t > 0.0f) || !isfinite(t)) return dot3(rel, dir);
    return t;
}

int ORACLE_FN(render)(const splat_gaussians* g, const splat_camera* cam, const splat_raster_config* cfg,
                      const uint8_t* mask, const float bg[3], float* color, float* alpha, float* depth,
                      float* transmittance, int32_t* max_contributor, float* importance, float* max_weight,
                      int32_t* max_pixel_count, int64_t* stats) {
    int rc = check_inputs(g, cam);
    if (rc) return rc;
    if (cfg->tile_size < 1) return fail(SPLAT_ERR_INVALID_ARGUMENT, "tile_size < 1");
    const int w = cam->width, h = cam->height, ts = cfg->tile_size;
    proj_t* proj;
    int np;
    if ((rc = project_impl(g, cam, cfg, mask, &proj, &np))) return rc;
    grid_t grid;
    if ((rc = bin_tiles(proj, np, w, h, ts, &grid))) { free(proj); return rc; }
    if (color) memset(color, 0, sizeof(float) * (size_t)w * h * 3);
    if (alpha) memset(alpha, 0, sizeof(float) * (size_t)w * h);
    if (depth) memset(depth, 0, sizeof(float) * (size_t)w * h);
    if (transmittance) memset(transmittance, 0, sizeof(float) * (size_t)w * h);
    if (max_contributor) for (size_t k = 0; k < (size_t)w * h; ++k) max_contributor[k] = -1;
    if (importance) memset(importance, 0, sizeof(float) * (size_t)g->n);
    if (max_weight) memset(max_weight, 0, sizeof(float) * (size_t)g->n);
    if (max_pixel_count) memset(max_pixel_count, 0, sizeof(int32_t) * (size_t)g->n);
    const int thr = cfg->apply_thresholds;
    const float a_max = (float)cfg->alpha_max, c_min = (float)cfg->contribution_min, t_min = (float)cfg->transmittance_min;
    float origin[3];
    cam_center(cam, origin);
    int64_t visits = 0, commits = 0;
    for (int ty = 0; ty < grid.tiles_y; ++ty)
        for (int tx = 0; tx < grid.tiles_x; ++tx) {
            const int t = ty * grid.tiles_x + tx;
            const int px1 = (tx + 1) * ts < w ? (tx + 1) * ts : w;
            const int py1 = (ty + 1) * ts < h ? (ty + 1) * ts : h;
            for (int py = ty * ts; py < py1; ++py)
                for (int px = tx * ts; px < px1; ++px) {
                    float acc[3] = {0.0f, 0.0f, 0.0f};
                    float w_max = 0.0f;
                    int pos_max = -1;
                    /* traverse_pixel (rasterizer.hpp:116-147) */
                    const float x = (float)px + 0.5f, y = (float)py + 0.5f;
                    float trans = 1.0f;
                    for (int64_t k = grid.start[t]; k < grid.start[t + 1]; ++k) {
                        const int pos = grid.pos[k];
                        const proj_t* pg = &proj[pos];
                        ++visits;
                        if (px < pg->x0 || px >= pg->x1 || py < pg->y0 || py >= pg->y1) continue;
                        const float dx = pg->mean2d[0] - x;
                        const float dy = pg->mean2d[1] - y;
                        const float power = -0.5f * (pg->conic[0] * dx * dx + pg->conic[2] * dy * dy) - pg->conic[1] * dx * dy;
                        if (power > 0.0f) continue;
                        const float g2d = EXP(power);
                        float a = pg->opacity * g2d;
                        if (thr) {
                            if (a > a_max) a = a_max;
                            if (a < c_min) continue;
                        }
                        const float next = trans * (1.0f - a);
                        if (thr && next < t_min) break;
                        const float wgt = trans * a;
                        ++commits;
                        /* visitor (rasterizer.cpp:136-149) */
                        for (int c = 0; c < 3; ++c) acc[c] += wgt * pg->color[c];
                        if (wgt > w_max) { w_max = wgt; pos_max = pos; }
                        if (importance) importance[pg->index] += wgt;
                        if (max_weight && wgt > max_weight[pg->index]) max_weight[pg->index] = wgt;
                        trans = next;
                    }
                    if (max_pixel_count && pos_max >= 0) max_pixel_count[proj[pos_max].index]++;
                    const size_t pix = (size_t)py * w + px;
                    for (int c = 0; c < 3; ++c) acc[c] += trans * bg[c];
                    if (color) for (int c = 0; c < 3; ++c) color[pix * 3 + c] = acc[c];
                    if (alpha) alpha[pix] = 1.0f - trans;
                    if (transmittance) transmittance[pix] = trans;
                    if (pos_max >= 0) {
                        const proj_t* pg = &proj[pos_max];
                        if (max_contributor) max_contributor[pix] = pg->index;
                        if (depth) {
                            float dir[3];
                            cam_ray_direction(cam, px, py, dir);
                            float d;
                            if (pg->degenerate) {
                                const float rel[3] = {pg->center[0] - origin[0], pg->center[1] - origin[1], pg->center[2] - origin[2]};
                                d = dot3(rel, dir);
                            } else {
                                d = depth_along_ray(pg->center, pg->cov_inv, origin, dir);
                            }
                            depth[pix] = d;
                        }
                    }
                }
        }
    if (stats) { stats[0] = visits; stats[1] = commits; }
    free_grid(&grid);
    free(proj);
    return 0;
}

typedef struct {
    int pos;
    float alpha, g2d, weight, t_before;
    int clamped;
} sample_t;

int ORACLE_FN(render_backward)(const splat_gaussians* g, const splat_camera* cam, const splat_raster_config* cfg,
                               const float* d_color, const uint8_t* mask, const float bg[3], float* d_centers,
                               float* d_log_scales, float* d_rotations, float* d_opacity, float* d_sh,
                               float* grad2d_accum, int32_t* grad2d_count) {
    int rc = check_inputs(g, cam);
    if (rc) return rc;
    if (!d_color) return fail(SPLAT_ERR_INVALID_ARGUMENT, "render_backward: dLoss/dColor shape mismatch");
    const int n = g->n;
    memset(d_centers, 0, sizeof(float) * 3 * (size_t)n);
    memset(d_log_scales, 0, sizeof(float) * 3 * (size_t)n);
    memset(d_rotations, 0, sizeof(float) * 4 * (size_t)n);
    memset(d_opacity, 0, sizeof(float) * (size_t)n);
    memset(d_sh, 0, sizeof(float) * 48 * (size_t)n);
    if (grad2d_accum) memset(grad2d_accum, 0, sizeof(float) * (size_t)n);
    if (grad2d_count) memset(grad2d_count, 0, sizeof(int32_t) * (size_t)n);
    const int w = cam->width, h = cam->height, ts = cfg->tile_size;
    proj_t* proj;
    int np;
    if ((rc = project_impl(g, cam, cfg, mask, &proj, &np))) return rc;
    if (np == 0) { free(proj); return 0; }
    grid_t grid;
    if ((rc = bin_tiles(proj, np, w, h, ts, &grid))) { free(proj); return rc; }
    float* dcol = (float*)calloc((size_t)np * 3, sizeof(float));
    float* dmean = (float*)calloc((size_t)np * 2, sizeof(float));
    float* dconic = (float*)calloc((size_t)np * 4, sizeof(float));
    float* dopac = (float*)calloc((size_t)np, sizeof(float));
    char* touched = (char*)calloc((size_t)np, 1);
    size_t cap = 64;
    sample_t* samples = (sample_t*)malloc(sizeof(sample_t) * cap);
    const int thr = cfg->apply_thresholds;
    const float a_max = (float)cfg->alpha_max, c_min = (float)cfg->contribution_min, t_min = (float)cfg->transmittance_min;
    for (int ty = 0; ty < grid.tiles_y; ++ty)
        for (int tx = 0; tx < grid.tiles_x; ++tx) {
            const int t = ty * grid.tiles_x + tx;
            if (grid.start[t] == grid.start[t + 1]) continue;
            const int px1 = (tx + 1) * ts < w ? (tx + 1) * ts : w;
            const int py1 = (ty + 1) * ts < h ? (ty + 1) * ts : h;
            for (int py = ty * ts; py < py1; ++py)
                for (int px = tx * ts; px < px1; ++px) {
                    size_t ns = 0;
                    const float x = (float)px + 0.5f, y = (float)py + 0.5f;
                    float trans = 1.0f;
                    for (int64_t k = grid.start[t]; k < grid.start[t + 1]; ++k) {
                        const int pos = grid.pos[k];
                        const proj_t* pg = &proj[pos];
                        if (px < pg->x0 || px >= pg->x1 || py < pg->y0 || py >= pg->y1) continue;
                        const float dx = pg->mean2d[0] - x;
                        const float dy = pg->mean2d[1] - y;
                        const float power = -0.5f * (pg->conic[0] * dx * dx + pg->conic[2] * dy * dy) - pg->conic[1] * dx * dy;
                        if (power > 0.0f) continue;
                        const float g2d = EXP(power);
                        float a = pg->opacity * g2d;
                        int clamped = 0;
                        if (thr) {
                            if (a > a_max) { a = a_max; clamped = 1; }
                            if (a < c_min) continue;
                        }
                        const float next = trans * (1.0f - a);
                        if (thr && next < t_min) break;
                        if (ns == cap) { cap *= 2; samples = (sample_t*)realloc(samples, sizeof(sample_t) * cap); }
                        samples[ns].pos = pos; samples[ns].alpha = a; samples[ns].g2d = g2d;
                        samples[ns].weight = trans * a; samples[ns].t_before = trans; samples[ns].clamped = clamped;
                        ++ns;
                        trans = next;
                    }
                    if (ns == 0) continue;
                    const size_t pix = (size_t)py * w + px;
                    const float dL[3] = {d_color[pix * 3], d_color[pix * 3 + 1], d_color[pix * 3 + 2]};
                    float b[3] = {bg[0], bg[1], bg[2]};
                    for (size_t si = ns; si-- > 0;) {
                        const sample_t* s = &samples[si];
                        const proj_t* pg = &proj[s->pos];
                        touched[s->pos] = 1;
                        for (int c = 0; c < 3; ++c) dcol[s->pos * 3 + c] += s->weight * dL[c];
                        float tmp[3];
                        for (int c = 0; c < 3; ++c) tmp[c] = s->t_before * (pg->color[c] - b[c]);
                        const float da = dot3(dL, tmp);
                        if (!s->clamped) {
                            dopac[s->pos] += da * s->g2d;
                            const float dpower = da * pg->opacity * s->g2d;
                            const float dx = pg->mean2d[0] - x;
                            const float dy = pg->mean2d[1] - y;
                            dmean[s->pos * 2] += dpower * (-(pg->conic[0] * dx + pg->conic[1] * dy));
                            dmean[s->pos * 2 + 1] += dpower * (-(pg->conic[2] * dy + pg->conic[1] * dx));
                            float* dq = &dconic[s->pos * 4]; /* (0,0),(0,1),(1,0),(1,1) */
                            dq[0] += dpower * -0.5f * dx * dx;
                            dq[1] += dpower * -0.5f * dx * dy;
                            dq[2] += dpower * -0.5f * dx * dy;
                            dq[3] += dpower * -0.5f * dy * dy;
                        }
                        float t1[3], t2[3];
                        for (int c = 0; c < 3; ++c) t1[c] = s->alpha * pg->color[c];
                        const float oma = 1.0f - s->alpha;
                        for (int c = 0; c < 3; ++c) t2[c] = oma * b[c];
                        for (int c = 0; c < 3; ++c) b[c] = t1[c] + t2[c];
                    }
                }
        }
    free(samples);

    /* per-Gaussian chain (gradients.cpp:127-220) */
    float cc[3];
    cam_center(cam, cc);
    const float fx = cam->fx, fy = cam->fy;
    const float* Rc = cam->rotation;
    for (int pos = 0; pos < np; ++pos) {
        if (!touched[pos]) continue;
        const proj_t* pg = &proj[pos];
        const int i = pg->index;
        const float* dm = &dmean[pos * 2];
        if (grad2d_accum) grad2d_accum[i] += sqrtf(dm[0] * dm[0] + dm[1] * dm[1]);
        if (grad2d_count) grad2d_count[i] += 1;
        /* dV = (-Q) * dQ * Q, row-major 2x2 */
        const float Qn[4] = {-pg->conic[0], -pg->conic[1], -pg->conic[1], -pg->conic[2]};
        const float Q[4] = {pg->conic[0], pg->conic[1], pg->conic[1], pg->conic[2]};
        const float* dQ = &dconic[pos * 4];
        float N[4], dV[4];
        for (int r = 0; r < 2; ++r)
            for (int c = 0; c < 2; ++c) N[r * 2 + c] = Qn[r * 2] * dQ[c] + Qn[r * 2 + 1] * dQ[2 + c];
        for (int r = 0; r < 2; ++r)
            for (int c = 0; c < 2; ++c) dV[r * 2 + c] = N[r * 2] * Q[c] + N[r * 2 + 1] * Q[2 + c];
        const float* p = &g->centers[3 * i];
        float pc[3];
        cam_to_camera(cam, p, pc);
        const float z = pc[2];
        const float J[6] = {fx / z, 0.0f, -fx * pc[0] / (z * z), 0.0f, fy / z, -fy * pc[1] / (z * z)};
        float Mm[6];
        for (int r = 0; r < 2; ++r)
            for (int c = 0; c < 3; ++c)
                Mm[r * 3 + c] = J[r * 3 + 0] * Rc[0 * 3 + c] + (J[r * 3 + 1] * Rc[1 * 3 + c] + J[r * 3 + 2] * Rc[2 * 3 + c]);
        float cov3d[9];
        covariance(&g->log_scales[3 * i], &g->rotations[4 * i], cov3d);
        /* d_cov3d = M^T dV M */
        float P[6], D[9];
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 2; ++c) P[r * 2 + c] = Mm[0 * 3 + r] * dV[0 * 2 + c] + Mm[1 * 3 + r] * dV[1 * 2 + c];
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) D[r * 3 + c] = P[r * 2] * Mm[0 * 3 + c] + P[r * 2 + 1] * Mm[1 * 3 + c];
        /* dM = 2 dV M cov3d ; dJ = dM R^T */
        float dV2[4], E[6], F[6], dJ[6];
        for (int k = 0; k < 4; ++k) dV2[k] = 2.0f * dV[k];
        for (int r = 0; r < 2; ++r)
            for (int c = 0; c < 3; ++c) E[r * 3 + c] = dV2[r * 2] * Mm[0 * 3 + c] + dV2[r * 2 + 1] * Mm[1 * 3 + c];
        for (int r = 0; r < 2; ++r)
            for (int c = 0; c < 3; ++c)
                F[r * 3 + c] = E[r * 3 + 0] * cov3d[0 * 3 + c] + (E[r * 3 + 1] * cov3d[1 * 3 + c] + E[r * 3 + 2] * cov3d[2 * 3 + c]);
        for (int r = 0; r < 2; ++r)
            for (int c = 0; c < 3; ++c) dJ[r * 3 + c] = dot3(&F[r * 3], &Rc[c * 3]);
        float dp[3] = {0.0f, 0.0f, 0.0f};
        dp[0] += dJ[0 * 3 + 2] * (-fx / (z * z));
        dp[1] += dJ[1 * 3 + 2] * (-fy / (z * z));
        dp[2] += dJ[0 * 3 + 0] * (-fx / (z * z)) + dJ[0 * 3 + 2] * (2.0f * fx * pc[0] / (z * z * z)) +
                 dJ[1 * 3 + 1] * (-fy / (z * z)) + dJ[1 * 3 + 2] * (2.0f * fy * pc[1] / (z * z * z));
        dp[0] += dm[0] * fx / z;
        dp[1] += dm[1] * fy / z;
        dp[2] += dm[0] * (-fx * pc[0] / (z * z)) + dm[1] * (-fy * pc[1] / (z * z));
        for (int k = 0; k < 3; ++k) {
            const float col[3] = {Rc[k], Rc[3 + k], Rc[6 + k]};
            d_centers[3 * i + k] += dot3(col, dp);
        }
        /* cov3d = M3 M3^T, M3 = R(q) diag(exp(s)) */
        float qh[4], Rq[9], sc[3], M3[9], D2[9], G[9], H[9];
        normalized_quat(&g->rotations[4 * i], qh);
        rotation_from_quat(qh, Rq);
        for (int k = 0; k < 3; ++k) sc[k] = EXP(g->log_scales[3 * i + k]);
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) M3[r * 3 + c] = Rq[r * 3 + c] * sc[c];
        for (int k = 0; k < 9; ++k) D2[k] = 2.0f * D[k];
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c)
                G[r * 3 + c] = D2[r * 3 + 0] * M3[0 * 3 + c] + (D2[r * 3 + 1] * M3[1 * 3 + c] + D2[r * 3 + 2] * M3[2 * 3 + c]);
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) H[r * 3 + c] = G[r * 3 + c] * sc[c];
        for (int k = 0; k < 3; ++k) {
            const float dSkk = Rq[0 * 3 + k] * G[0 * 3 + k] + (Rq[1 * 3 + k] * G[1 * 3 + k] + Rq[2 * 3 + k] * G[2 * 3 + k]);
            d_log_scales[3 * i + k] += dSkk * sc[k];
        }
        /* quat_rotation_jacobians (gradients.cpp:25-41), row-major */
        const float w_ = qh[0], x_ = qh[1], y_ = qh[2], z_ = qh[3];
        float dRq[4][9] = {
            {0.0f, -z_, y_, z_, 0.0f, -x_, -y_, x_, 0.0f},
            {0.0f, y_, z_, y_, -2.0f * x_, -w_, z_, w_, -2.0f * x_},
            {-2.0f * y_, x_, w_, x_, 0.0f, z_, -w_, z_, -2.0f * y_},
            {-2.0f * z_, -w_, x_, w_, -2.0f * z_, y_, x_, y_, 0.0f}};
        float dqh[4];
        for (int k = 0; k < 4; ++k) {
            float e[9]; /* column-major element order of H .* dR_dq[k] */
            for (int c = 0; c < 3; ++c)
                for (int r = 0; r < 3; ++r) e[c * 3 + r] = H[r * 3 + c] * (dRq[k][r * 3 + c] * 2.0f);
            /* halving redux over 9: (e0+e1)+(e2+e3) + ((e4+e5) + (e6+(e7+e8))) */
            dqh[k] = ((e[0] + e[1]) + (e[2] + e[3])) + ((e[4] + e[5]) + (e[6] + (e[7] + e[8])));
        }
        const float qn = sqrtf(sq4(&g->rotations[4 * i]));
        if (qn > 1e-12f) {
            const float qd = (qh[0] * dqh[0] + qh[1] * dqh[1]) + (qh[2] * dqh[2] + qh[3] * dqh[3]);
            for (int k = 0; k < 4; ++k) d_rotations[4 * i + k] += (dqh[k] - qh[k] * qd) / qn;
        }
        d_opacity[i] += dopac[pos] * pg->opacity * (1.0f - pg->opacity);
        /* SH (gradients.cpp:192-219) */
        const float u[3] = {p[0] - cc[0], p[1] - cc[1], p[2] - cc[2]};
        const float len = sqrtf(sq3(u));
        const float dir[3] = {u[0] / len, u[1] / len, u[2] / len};
        float basis[16];
        const int deg = g->active_sh_degree;
        sh_basis(dir, deg, basis);
        float rgb[3];
        int clamped[3];
        const float* shp = &g->sh[48 * (size_t)i];
        sh_to_color(shp, dir, deg, rgb, clamped);
        float dc[3];
        for (int c = 0; c < 3; ++c) dc[c] = clamped[c] ? 0.0f : dcol[pos * 3 + c];
        const int nco = sh_coeffs(deg);
        float* dsh = &d_sh[48 * (size_t)i];
        for (int k = 0; k < nco; ++k)
            for (int c = 0; c < 3; ++c) dsh[k * 3 + c] += basis[k] * dc[c];
        if (deg > 0) {
            float gb[16][3];
            sh_basis_grad(dir, deg, gb);
            float ddir[3] = {0.0f, 0.0f, 0.0f};
            for (int k = 1; k < nco; ++k) {
                float coef = 0.0f;
                for (int c = 0; c < 3; ++c) coef += dc[c] * shp[k * 3 + c];
                for (int c = 0; c < 3; ++c) ddir[c] += gb[k][c] * coef;
            }
            const float dd = dot3(dir, ddir);
            for (int c = 0; c < 3; ++c) d_centers[3 * i + c] += (ddir[c] - dir[c] * dd) / len;
        }
    }
    free(dcol); free(dmean); free(dconic); free(dopac); free(touched);
    free_grid(&grid);
    free(proj);
    return 0;
}

float ORACLE_FN(l1_loss)(const float* a, const float* b, int64_t count, float* grad) {
    float sum = 0.0f;
    const float inv_n = 1.0f / (float)count;
    for (int64_t i = 0; i < count; ++i) {
        const float d = a[i] - b[i];
        sum += fabsf(d);
        if (grad) grad[i] = d > 0.0f ? inv_n : (d < 0.0f ? -inv_n : 0.0f);
    }
    return sum * inv_n;
}

double ORACLE_FN(lr_at)(const splat_adam_config* cfg, int32_t step) {
    if (step <= 0) return cfg->lr_init;
    double t = (double)step / (double)cfg->max_steps;
    if (t > 1.0) t = 1.0;
    return exp((1.0 - t) * log(cfg->lr_init) + t * log(cfg->lr_final));
}

/* adam_delta (optimizer.cpp:29-36) */
static inline float adam_delta(float* m, float* v, float g, double b1, double b2, double eps, double bias1,
                               double bias2, double lr) {
    *m = (float)(b1 * *m + (1.0 - b1) * g);
    *v = (float)(b2 * *v + (1.0 - b2) * (double)g * g);
    const double m_hat = *m / bias1;
    const double v_hat = *v / bias2;
    return (float)(lr * m_hat / (sqrt(v_hat) + eps));
}

int ORACLE_FN(adam_step)(float* centers, float* log_scales, float* rotations, float* opacity_logits, float* sh,
                         int32_t n, const float* d_centers, const float* d_log_scales, const float* d_rotations,
                         const float* d_opacity, const float* d_sh, float* m, float* v,
                         const splat_adam_config* cfg, int32_t* step_count, uint32_t group_mask) {
    const double lr_pos = ORACLE_FN(lr_at)(cfg, *step_count) * cfg->scene_extent;
    *step_count += 1;
    const double bias1 = 1.0 - pow(cfg->beta1, *step_count);
    const double bias2 = 1.0 - pow(cfg->beta2, *step_count);
    const double b1 = cfg->beta1, b2 = cfg->beta2, eps = cfg->eps;
    const size_t N = (size_t)n;
    float* mc = m; float* vc = v;
    float* ms = m + 3 * N; float* vs = v + 3 * N;
    float* mr = m + 6 * N; float* vr = v + 6 * N;
    float* mo = m + 10 * N; float* vo = v + 10 * N;
    float* mh = m + 11 * N; float* vh = v + 11 * N;
    for (size_t i = 0; i < N; ++i) {
        for (int k = 0; k < 3; ++k) {
            const size_t j = 3 * i + k;
            if (group_mask & SPLAT_GROUP_CENTERS)
                centers[j] -= adam_delta(&mc[j], &vc[j], d_centers[j], b1, b2, eps, bias1, bias2, lr_pos);
            if (group_mask & SPLAT_GROUP_SCALES)
                log_scales[j] -= adam_delta(&ms[j], &vs[j], d_log_scales[j], b1, b2, eps, bias1, bias2, cfg->lr_scale);
        }
        if (group_mask & SPLAT_GROUP_ROTATIONS)
            for (int k = 0; k < 4; ++k) {
                const size_t j = 4 * i + k;
                rotations[j] -= adam_delta(&mr[j], &vr[j], d_rotations[j], b1, b2, eps, bias1, bias2, cfg->lr_rotation);
            }
        if (group_mask & SPLAT_GROUP_OPACITY)
            opacity_logits[i] -= adam_delta(&mo[i], &vo[i], d_opacity[i], b1, b2, eps, bias1, bias2, cfg->lr_opacity);
        if (group_mask & SPLAT_GROUP_SH)
            for (int k = 0; k < 48; ++k) {
                const size_t j = 48 * i + k;
                sh[j] -= adam_delta(&mh[j], &vh[j], d_sh[j], b1, b2, eps, bias1, bias2, k < 3 ? cfg->lr_sh_dc : cfg->lr_sh_rest);
            }
        if (group_mask & SPLAT_GROUP_ROTATIONS) {
            float q[4];
            normalized_quat(&rotations[4 * i], q);
            for (int k = 0; k < 4; ++k) rotations[4 * i + k] = q[k];
        }
    }
    return 0;
}

int ORACLE_FN(unproject)(const splat_camera* cam, const int32_t* max_contributor, const float* alpha,
                         const float* depth, int rule, float alpha_threshold, int64_t view_index, int32_t stride,
                         int64_t seed, float* points, int32_t* pixel, int64_t capacity, int64_t* count) {
    if (stride < 1) return fail(SPLAT_ERR_INVALID_ARGUMENT, "unproject: stride < 1");
    const int w = cam->width, h = cam->height;
    const int64_t hw = (int64_t)w * h;
    float origin[3];
    cam_center(cam, origin);
    int64_t cnt = 0;
    for (int py = 0; py < h; ++py)
        for (int px = 0; px < w; ++px) {
            const int64_t pix = (int64_t)py * w + px;
            const int valid = rule == SPLAT_DEPTH_RULE_ALPHA ? (alpha[pix] > alpha_threshold) : (max_contributor[pix] >= 0);
            if (!valid) continue;
            const int64_t key = view_index * hw + pix + seed;
            if (((key % stride) + stride) % stride != 0) continue;
            if (cnt < capacity) {
                float dir[3];
                cam_ray_direction(cam, px, py, dir);
                const float d = depth[pix];
                for (int c = 0; c < 3; ++c) points[3 * cnt + c] = origin[c] + d * dir[c];
                pixel[cnt] = (int32_t)pix;
            }
            ++cnt;
        }
    *count = cnt;
    return 0;
}

/* ---- densification and simplification ----------------- */
static int cmp_f32(const void* a, const void* b) {
    const float x = *(const float*)a, y = *(const float*)b;
    return (x > y) - (x < y);
}
static int cmp_f64(const void* a, const void* b) {
    const double x = *(const double*)a, y = *(const double*)b;
    return (x > y) - (x < y);
}

/* quantile_threshold (quantile.hpp:16-28): sort, linear interpolation in double. */
int ORACLE_FN(quantile_threshold)(const float* values, const uint8_t* sel, int32_t n, double keep_q, float* tau,
                                  int32_t* count) {
    if (!(keep_q > 0.0 && keep_q < 1.0)) return fail(SPLAT_ERR_INVALID_ARGUMENT, "quantile_threshold: keep_q");
    float* v = (float*)malloc(sizeof(float) * (size_t)(n > 0 ? n : 1));
    int32_t m = 0;
    for (int32_t i = 0; i < n; ++i)
        if (!sel || sel[i]) v[m++] = values[i];
    if (count) *count = m;
    if (m == 0) {
        free(v);
        return fail(SPLAT_ERR_INVALID_ARGUMENT, "quantile_threshold: empty input");
    }
    qsort(v, (size_t)m, sizeof(float), cmp_f32);
    const double q = 1.0 - keep_q;
    const double h = q * (double)(m - 1);
    const size_t lo = (size_t)floor(h);
    const size_t hi = lo + 1 < (size_t)m - 1 ? lo + 1 : (size_t)m - 1;
    const double frac = h - (double)lo;
    *tau = (float)((double)v[lo] + frac * ((double)v[hi] - (double)v[lo]));
    free(v);
    return 0;
}

int ORACLE_FN(quantile_threshold_f64)(const double* values, const uint8_t* sel, int32_t n, double keep_q,
                                      double* tau, int32_t* count) {
    if (!(keep_q > 0.0 && keep_q < 1.0)) return fail(SPLAT_ERR_INVALID_ARGUMENT, "quantile_threshold: keep_q");
    double* v = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    int32_t m = 0;
    for (int32_t i = 0; i < n; ++i)
        if (!sel || sel[i]) v[m++] = values[i];
    if (count) *count = m;
    if (m == 0) {
        free(v);
        return fail(SPLAT_ERR_INVALID_ARGUMENT, "quantile_threshold: empty input");
    }
    qsort(v, (size_t)m, sizeof(double), cmp_f64);
    const double q = 1.0 - keep_q;
    const double h = q * (double)(m - 1);
    const size_t lo = (size_t)floor(h);
    const size_t hi = lo + 1 < (size_t)m - 1 ? lo + 1 : (size_t)m - 1;
    const double frac = h - (double)lo;
    *tau = v[lo] + frac * (v[hi] - v[lo]);
    free(v);
    return 0;
}

/* build_masks, one view (visibility.cpp:15-35). */
int ORACLE_FN(visibility_mask)(const float* importance, int32_t n, double keep_q, uint8_t* mask) {
    uint8_t* pos = (uint8_t*)malloc((size_t)(n > 0 ? n : 1));
    int any_pos = 0;
    for (int32_t i = 0; i < n; ++i) {
        pos[i] = importance[i] > 0.0f;
        any_pos |= pos[i];
        mask[i] = 0;
    }
    if (any_pos) {
        float tau;
        /* visibility.cpp:23: quantile_threshold(positive, float(keep_q)) */
        int rc = ORACLE_FN(quantile_threshold)(importance, pos, n, (double)(float)keep_q, &tau, NULL);
        if (rc) {
            free(pos);
            return rc;
        }
        int any = 0;
        for (int32_t i = 0; i < n; ++i) {
            mask[i] = importance[i] > tau;
            any |= mask[i];
        }
        if (!any)
            for (int32_t i = 0; i < n; ++i) mask[i] = importance[i] > 0.0f;
    }
    free(pos);
    return 0;
}

typedef struct {
    double score;
    int32_t idx;
} scored_t;
static int cmp_scored(const void* a, const void* b) { /* densify.cpp:96-99: score desc, index asc */
    const scored_t* x = (const scored_t*)a;
    const scored_t* y = (const scored_t*)b;
    if (x->score != y->score) return x->score > y->score ? -1 : 1;
    return (x->idx > y->idx) - (x->idx < y->idx);
}

/* identify_critical (densify.cpp:32-103) from the per-view statistics (best weight = max over
 * views of max_weight, max_count_sum > 0 = ever the max contributor, fp64 summed importance). */
int ORACLE_FN(identify_critical)(const splat_gaussians* g, const float* best, const int64_t* max_count_sum,
                                 const double* summed, int criterion, double keep_q, const double* random,
                                 uint8_t* critical, int32_t* count_out) {
    const int32_t n = g->n;
    *count_out = 0;
    uint8_t* ever = (uint8_t*)malloc((size_t)(n > 0 ? n : 1));
    int32_t m = 0;
    for (int32_t i = 0; i < n; ++i) {
        ever[i] = max_count_sum[i] > 0;
        m += ever[i];
        critical[i] = 0;
    }
    if (m == 0) {
        free(ever);
        return 0;
    }
    float tau;
    /* densify.cpp:63: quantile_threshold(candidate_weights, float(keep_q)) */
    int rc = ORACLE_FN(quantile_threshold)(best, ever, n, (double)(float)keep_q, &tau, NULL);
    if (rc) {
        free(ever);
        return rc;
    }
    int32_t count = 0;
    for (int32_t i = 0; i < n; ++i)
        if (ever[i] && best[i] > tau) ++count;
    const int keep_all = count == 0;
    if (keep_all) count = m;
    *count_out = count;
    if (criterion == SPLAT_CRITERION_MAX_WEIGHT) {
        for (int32_t i = 0; i < n; ++i) critical[i] = ever[i] && (keep_all || best[i] > tau);
        free(ever);
        return 0;
    }
    scored_t* sc = (scored_t*)malloc(sizeof(scored_t) * (size_t)n);
    for (int32_t i = 0; i < n; ++i) {
        double s;
        if (criterion == SPLAT_CRITERION_OPACITY)
            s = (double)sigmoidf_(g->opacity_logits[i]);
        else if (criterion == SPLAT_CRITERION_ACCUM_WEIGHT)
            s = summed[i];
        else
            s = random[i];
        sc[i].score = s;
        sc[i].idx = i;
    }
    qsort(sc, (size_t)n, sizeof(scored_t), cmp_scored);
    for (int32_t r = 0; r < count; ++r) critical[sc[r].idx] = 1;
    free(sc);
    free(ever);
    return 0;
}

/* aggressive_clone + apply_densify_plan (densify.cpp:105-130, 159-195) on arrays with room for
 * capacity rows; same contract as splat_aggressive_clone. */
int ORACLE_FN(aggressive_clone)(float* centers, float* log_scales, float* rotations, float* opacity_logits, float* sh,
                                int32_t n, int64_t capacity, const uint8_t* critical, int32_t* moment_source,
                                int32_t* n_out) {
    int32_t clones = 0;
    for (int32_t i = 0; i < n; ++i)
        if (critical[i] && sigmoidf_(opacity_logits[i]) > 1e-7f) ++clones;
    *n_out = n + clones;
    if ((int64_t)n + clones > capacity) return fail(SPLAT_ERR_INVALID_ARGUMENT, "aggressive_clone: capacity");
    const float sqrt2 = sqrtf(2.f);
    int32_t j = n;
    for (int32_t i = 0; i < n; ++i) {
        if (moment_source) moment_source[i] = i;
        if (!critical[i]) continue;
        float alpha = sigmoidf_(opacity_logits[i]);
        if (alpha <= 1e-7f) continue;
        alpha = fmin_std(alpha, 1.f - 1e-7f);
        const float alpha_new = 1.f - sqrtf(1.f - alpha);
        const float denom = 2.f * alpha_new - alpha_new * alpha_new / sqrt2;
        const float k = (alpha * alpha) / (denom * denom);
        const float shift = 0.5f * LOG(k);
        const float logit_new = LOG(alpha_new / (1.f - alpha_new)); /* logit, types.hpp:63-65 */
        opacity_logits[i] = logit_new;
        for (int c = 0; c < 3; ++c) log_scales[3 * i + c] = log_scales[3 * i + c] + shift;
        if (moment_source) {
            moment_source[i] = -1;
            moment_source[j] = -1;
        }
        memcpy(centers + 3 * (size_t)j, centers + 3 * (size_t)i, 12);
        memcpy(log_scales + 3 * (size_t)j, log_scales + 3 * (size_t)i, 12);
        memcpy(rotations + 4 * (size_t)j, rotations + 4 * (size_t)i, 16);
        opacity_logits[j] = logit_new;
        memcpy(sh + 48 * (size_t)j, sh + 48 * (size_t)i, 192);
        ++j;
    }
    return 0;
}

/* importance_prune (simplify.cpp:94-107): kept = ascending indices selected by
 * select_above_quantile (quantile.hpp:33-46). */
int ORACLE_FN(importance_prune)(const double* importance, int32_t n, double keep_q, int32_t* kept, int32_t* n_kept) {
    double tau;
    int rc = ORACLE_FN(quantile_threshold_f64)(importance, NULL, n, keep_q, &tau, NULL);
    if (rc) return rc;
    int32_t k = 0, any = 0;
    for (int32_t i = 0; i < n; ++i) any |= importance[i] > tau;
    for (int32_t i = 0; i < n; ++i)
        if (!any || importance[i] > tau) kept[k++] = i;
    *n_kept = k;
    return 0;
}

/* OptimState::step restricted to elements [begin, begin + count) of the packed layout (the
 * sharded step of the view-parallel exchange, splat_adam_step_range): the per-element update of
 * optimizer.cpp:53-68 with the element's group learning rate, no quaternion renormalisation. */
int ORACLE_FN(adam_step_range)(float* params, const float* grad_shard, float* m, float* v, int32_t n, int64_t begin,
                               int64_t count, const splat_adam_config* cfg, int32_t step, uint32_t group_mask) {
    const double lr_pos = ORACLE_FN(lr_at)(cfg, step) * cfg->scene_extent;
    const double bias1 = 1.0 - pow(cfg->beta1, step + 1);
    const double bias2 = 1.0 - pow(cfg->beta2, step + 1);
    const int64_t N = n;
    for (int64_t e = begin; e < begin + count && e < 59 * N; ++e) {
        uint32_t bit;
        double lr;
        if (e < 3 * N) { bit = SPLAT_GROUP_CENTERS; lr = lr_pos; }
        else if (e < 6 * N) { bit = SPLAT_GROUP_SCALES; lr = cfg->lr_scale; }
        else if (e < 10 * N) { bit = SPLAT_GROUP_ROTATIONS; lr = cfg->lr_rotation; }
        else if (e < 11 * N) { bit = SPLAT_GROUP_OPACITY; lr = cfg->lr_opacity; }
        else { bit = SPLAT_GROUP_SH; lr = (e - 11 * N) % 48 < 3 ? cfg->lr_sh_dc : cfg->lr_sh_rest; }
        if (!(group_mask & bit)) continue;
        params[e] -= adam_delta(&m[e], &v[e], grad_shard[e - begin], cfg->beta1, cfg->beta2, cfg->eps, bias1, bias2, lr);
    }
    return 0;
}

/* normalized_quat over n rows in place (optimizer.cpp:69). */
int ORACLE_FN(quat_normalize)(float* rotations, int32_t n) {
    for (int32_t i = 0; i < n; ++i) {
        float q[4];
        normalized_quat(&rotations[4 * (size_t)i], q);
        for (int k = 0; k < 4; ++k) rotations[4 * (size_t)i + k] = q[k];
    }
    return 0;
}

/* ---- the reference's random draws (include/splat_rng.h) and their consumers -------------- */
/* std::normal_distribution<float>(0, 1) on std::mt19937(seed), one distribution object. */
int ORACLE_FN(rng_normal_f32)(uint32_t seed, int32_t n, float* out) {
    splat_mt19937 g;
    splat_normal_f32 d = {0.0f, 0};
    splat_mt19937_seed(&g, seed);
    for (int32_t i = 0; i < n; ++i) out[i] = splat_normal_f32_next(&d, &g, 0.0f, 1.0f);
    return 0;
}

/* kinds[i] = 0: uniform_real_distribution<double>(0, 1), 1: uniform_int_distribution<int>(lo, hi),
 * interleaved on one std::mt19937_64(seed). */
int ORACLE_FN(rng_mixed_64)(uint64_t seed, int32_t n, const int32_t* kinds, const int32_t* lo, const int32_t* hi,
                            double* out) {
    splat_mt19937_64 g;
    splat_mt19937_64_seed(&g, seed);
    for (int32_t i = 0; i < n; ++i)
        out[i] = kinds[i] == 0 ? splat_canonical_f64_64(&g) : (double)splat_uniform_int_64(&g, lo[i], hi[i]);
    return 0;
}

/* std::uniform_real_distribution<double>(0, 1) on std::mt19937(seed) (densify.cpp:78-80). */
int ORACLE_FN(rng_uniform_f64_32)(uint32_t seed, int32_t n, double* out) {
    splat_mt19937 g;
    splat_mt19937_seed(&g, seed);
    for (int32_t i = 0; i < n; ++i) out[i] = splat_canonical_f64_32(&g);
    return 0;
}

/* depth_reinitialize's pool draw (densify.cpp:227-235) from std::mt19937(seed). */
int ORACLE_FN(rng_fisher_yates)(uint32_t seed, int32_t pool, int32_t take, int32_t* idx_out) {
    splat_mt19937 g;
    splat_mt19937_seed(&g, seed);
    int32_t* idx = (int32_t*)malloc(sizeof(int32_t) * (size_t)(pool > 0 ? pool : 1));
    splat_partial_fisher_yates(&g, idx, pool, take);
    memcpy(idx_out, idx, sizeof(int32_t) * (size_t)take);
    free(idx);
    return 0;
}

typedef struct {
    double key;
    int32_t idx;
} keyed_t;
static int cmp_keyed(const void* a, const void* b) { /* simplify.cpp:72-75: key desc, index asc */
    const keyed_t* x = (const keyed_t*)a;
    const keyed_t* y = (const keyed_t*)b;
    if (x->key != y->key) return x->key > y->key ? -1 : 1;
    return (x->idx > y->idx) - (x->idx < y->idx);
}
static int cmp_i32(const void* a, const void* b) {
    const int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
    return (x > y) - (x < y);
}

/* importance_sample (simplify.cpp:36-92): Efraimidis-Spirakis keys log(u)/w on std::mt19937_64(seed),
 * the target_count largest (ties by index), a uniform filler from the zero-weight rows, or a
 * uniform draw when no weight is positive; kept ascending. */
int ORACLE_FN(importance_sample)(const double* importance, int32_t n, int32_t target, uint64_t seed, int32_t* kept,
                                 int32_t* n_kept) {
    if (target < 1 || target > n) return fail(SPLAT_ERR_INVALID_ARGUMENT, "importance_sample: target_count out of range");
    splat_mt19937_64 g;
    splat_mt19937_64_seed(&g, seed);
    keyed_t* keyed = (keyed_t*)malloc(sizeof(keyed_t) * (size_t)n);
    int32_t* zero = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
    int32_t nk = 0, nz = 0;
    for (int32_t i = 0; i < n; ++i) {
        double u = splat_canonical_f64_64(&g);
        if (u < 1e-300) u = 1e-300; /* std::max(u, 1e-300) */
        if (importance[i] > 0.0) {
            keyed[nk].key = log(u) / importance[i];
            keyed[nk].idx = i;
            ++nk;
        } else {
            zero[nz++] = i;
        }
    }
    int32_t k = 0;
    if (nk == 0) {
        int32_t* idx = zero; /* every row has zero weight: idx = 0..n-1 */
        for (int32_t i = 0; i < n; ++i) idx[i] = i;
        for (int32_t r = 0; r < target; ++r) {
            const int32_t j = splat_uniform_int_64(&g, r, n - 1);
            const int32_t t = idx[r];
            idx[r] = idx[j];
            idx[j] = t;
        }
        for (int32_t r = 0; r < target; ++r) kept[k++] = idx[r];
    } else {
        const int32_t from_weighted = target < nk ? target : nk;
        qsort(keyed, (size_t)nk, sizeof(keyed_t), cmp_keyed);
        for (int32_t r = 0; r < from_weighted; ++r) kept[k++] = keyed[r].idx;
        int32_t deficit = target - from_weighted;
        for (int32_t r = 0; deficit > 0; --deficit, ++r) {
            const int32_t j = splat_uniform_int_64(&g, r, nz - 1);
            const int32_t t = zero[r];
            zero[r] = zero[j];
            zero[j] = t;
            kept[k++] = zero[r];
        }
    }
    qsort(kept, (size_t)k, sizeof(int32_t), cmp_i32);
    *n_kept = k;
    free(keyed);
    free(zero);
    return 0;
}

/* vanilla_clone_split + apply_densify_plan, Progressive mode (densify.cpp:132-163, 182-195): rows
 * whose mean 2D gradient exceeds grad_threshold are cloned (max scale <= scale_threshold * extent)
 * or split into two children at centre + R(q) (s .* n), n ~ N(0, I) from std::mt19937(seed),
 * log-scales - log(1.6).  Output: the kept rows in index order, then the new rows in index order;
 * moment_source = old row for kept rows, -1 for new rows. */
int ORACLE_FN(vanilla_clone_split)(const splat_gaussians* g, const float* grad2d_accum, const int32_t* grad2d_count,
                                   float grad_threshold, float scale_threshold, float scene_extent, uint32_t seed,
                                   float* centers, float* log_scales, float* rotations, float* opacity_logits,
                                   float* sh, int64_t capacity, int32_t* moment_source, int32_t* n_out,
                                   int32_t* n_clone, int32_t* n_split) {
    const int32_t n = g->n;
    uint8_t* kind = (uint8_t*)malloc((size_t)(n > 0 ? n : 1));
    int32_t nc = 0, ns = 0;
    for (int32_t i = 0; i < n; ++i) {
        kind[i] = 0;
        if (grad2d_count[i] <= 0) continue;
        const float avg = grad2d_accum[i] / (float)grad2d_count[i];
        if (avg <= grad_threshold) continue;
        float sc[3];
        for (int c = 0; c < 3; ++c) sc[c] = EXP(g->log_scales[3 * i + c]);
        float mx = sc[0];
        for (int c = 1; c < 3; ++c) mx = fmax_std(mx, sc[c]);
        if (mx <= scale_threshold * scene_extent) {
            kind[i] = 1;
            ++nc;
        } else {
            kind[i] = 2;
            ++ns;
        }
    }
    const int64_t m = (int64_t)n - ns + nc + 2 * (int64_t)ns;
    *n_out = (int32_t)m;
    *n_clone = nc;
    *n_split = ns;
    if (m > capacity) {
        free(kind);
        return fail(SPLAT_ERR_INVALID_ARGUMENT, "vanilla_clone_split: capacity too small");
    }
    int64_t r = 0;
    for (int32_t i = 0; i < n; ++i) { /* kept rows (apply_densify_plan: select(keep)) */
        if (kind[i] == 2) continue;
        memcpy(centers + 3 * r, g->centers + 3 * (size_t)i, 12);
        memcpy(log_scales + 3 * r, g->log_scales + 3 * (size_t)i, 12);
        memcpy(rotations + 4 * r, g->rotations + 4 * (size_t)i, 16);
        opacity_logits[r] = g->opacity_logits[i];
        memcpy(sh + 48 * r, g->sh + 48 * (size_t)i, 192);
        moment_source[r] = i;
        ++r;
    }
    splat_mt19937 rng;
    splat_normal_f32 gauss = {0.0f, 0};
    splat_mt19937_seed(&rng, seed);
    const float split_shift = LOG(1.6f);
    for (int32_t i = 0; i < n; ++i) { /* plan.new_rows, appended in index order */
        if (kind[i] == 0) continue;
        const int children = kind[i] == 1 ? 1 : 2;
        float rot[9], sc[3];
        if (kind[i] == 2) {
            rotation_from_quat(g->rotations + 4 * (size_t)i, rot);
            for (int c = 0; c < 3; ++c) sc[c] = EXP(g->log_scales[3 * i + c]);
        }
        for (int child = 0; child < children; ++child) {
            memcpy(centers + 3 * r, g->centers + 3 * (size_t)i, 12);
            memcpy(log_scales + 3 * r, g->log_scales + 3 * (size_t)i, 12);
            memcpy(rotations + 4 * r, g->rotations + 4 * (size_t)i, 16);
            opacity_logits[r] = g->opacity_logits[i];
            memcpy(sh + 48 * r, g->sh + 48 * (size_t)i, 192);
            moment_source[r] = -1;
            if (kind[i] == 2) {
                float nv[3], v[3];
                /* Vec3f n(gauss(rng), gauss(rng), gauss(rng)): GCC evaluates the three arguments
                 * right to left (pinned against the reference build) */
                nv[2] = splat_normal_f32_next(&gauss, &rng, 0.0f, 1.0f);
                nv[1] = splat_normal_f32_next(&gauss, &rng, 0.0f, 1.0f);
                nv[0] = splat_normal_f32_next(&gauss, &rng, 0.0f, 1.0f);
                for (int c = 0; c < 3; ++c) v[c] = sc[c] * nv[c];
                for (int c = 0; c < 3; ++c)
                    centers[3 * r + c] = g->centers[3 * (size_t)i + c] + dot3(&rot[3 * c], v);
                for (int c = 0; c < 3; ++c) log_scales[3 * r + c] = g->log_scales[3 * (size_t)i + c] - split_shift;
            }
            ++r;
        }
    }
    free(kind);
    return 0;
}

/* ---- SSIM and the photometric loss (loss.cpp:10-153) ------------- */
#define SSIM_W 11
/* gaussian_kernel (loss.cpp:13-22) */
static void ssim_kernel(float k[SSIM_W]) {
    float sum = 0.0f;
    for (int i = 0; i < SSIM_W; ++i) {
        const float d = (float)(i - SSIM_W / 2);
        k[i] = EXP(-d * d / (float)(2 * 1.5 * 1.5));
        sum += k[i];
    }
    for (int i = 0; i < SSIM_W; ++i) k[i] /= sum;
}

void ORACLE_FN(ssim_window)(float* out11) { ssim_kernel(out11); }

/* blur (loss.cpp:26-53): separable "same" convolution, zero padding by skipping. */
static void ssim_blur(const float* img, int w, int h, int ch, const float k[SSIM_W], float* out, float* tmp) {
    const int half = SSIM_W / 2;
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x)
            for (int c = 0; c < ch; ++c) {
                float acc = 0.0f;
                for (int q = -half; q <= half; ++q) {
                    const int xx = x + q;
                    if (xx < 0 || xx >= w) continue;
                    acc += k[q + half] * img[((size_t)y * w + xx) * ch + c];
                }
                tmp[((size_t)y * w + x) * ch + c] = acc;
            }
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x)
            for (int c = 0; c < ch; ++c) {
                float acc = 0.0f;
                for (int q = -half; q <= half; ++q) {
                    const int yy = y + q;
                    if (yy < 0 || yy >= h) continue;
                    acc += k[q + half] * tmp[((size_t)yy * w + x) * ch + c];
                }
                out[((size_t)y * w + x) * ch + c] = acc;
            }
}

/* ssim<float> (loss.cpp:78-134): mean SSIM; grad_a (nullable) = d mean SSIM / d a. */
float ORACLE_FN(ssim)(const float* a, const float* b, int w, int h, int ch, float* grad_a) {
    const float c1 = (float)(0.01 * 0.01), c2 = (float)(0.03 * 0.03);
    float k[SSIM_W];
    ssim_kernel(k);
    const size_t n = (size_t)w * h * ch;
    float* buf = (float*)malloc(sizeof(float) * n * 12);
    float *aa = buf, *bb = buf + n, *ab = buf + 2 * n, *mu_a = buf + 3 * n, *mu_b = buf + 4 * n,
          *m_aa = buf + 5 * n, *m_bb = buf + 6 * n, *m_ab = buf + 7 * n, *tmp = buf + 8 * n, *t1 = buf + 9 * n,
          *t2 = buf + 10 * n, *t3 = buf + 11 * n;
    for (size_t i = 0; i < n; ++i) {
        aa[i] = a[i] * a[i];
        bb[i] = b[i] * b[i];
        ab[i] = a[i] * b[i];
    }
    ssim_blur(a, w, h, ch, k, mu_a, tmp);
    ssim_blur(b, w, h, ch, k, mu_b, tmp);
    ssim_blur(aa, w, h, ch, k, m_aa, tmp);
    ssim_blur(bb, w, h, ch, k, m_bb, tmp);
    ssim_blur(ab, w, h, ch, k, m_ab, tmp);
    const float inv_n = 1.0f / (float)n;
    float total = 0.0f;
    for (size_t i = 0; i < n; ++i) {
        const float ma = mu_a[i], mb = mu_b[i];
        const float va = m_aa[i] - ma * ma;
        const float vb = m_bb[i] - mb * mb;
        const float cov = m_ab[i] - ma * mb;
        const float a1 = 2.0f * ma * mb + c1;
        const float a2 = 2.0f * cov + c2;
        const float b1 = ma * ma + mb * mb + c1;
        const float b2 = va + vb + c2;
        const float sv = (a1 * a2) / (b1 * b2);
        total += sv;
        if (grad_a) {
            const float ds_dmu = 2.0f * (mb * a2 * b1 - ma * a1 * a2) / (b1 * b1 * b2);
            const float ds_dva = -a1 * a2 / (b1 * b2 * b2);
            const float ds_dcov = 2.0f * a1 / (b1 * b2);
            t1[i] = inv_n * (ds_dmu - 2.0f * ma * ds_dva - mb * ds_dcov);
            t2[i] = inv_n * ds_dva;
            t3[i] = inv_n * ds_dcov;
        }
    }
    if (grad_a) {
        float* g1 = aa; /* reuse */
        float* g2 = bb;
        float* g3 = ab;
        ssim_blur(t1, w, h, ch, k, g1, tmp);
        ssim_blur(t2, w, h, ch, k, g2, tmp);
        ssim_blur(t3, w, h, ch, k, g3, tmp);
        for (size_t i = 0; i < n; ++i) grad_a[i] = g1[i] + 2.0f * a[i] * g2[i] + b[i] * g3[i];
    }
    free(buf);
    return total * inv_n;
}

/* photometric_loss<float> (loss.cpp:136-147). grad nullable. */
float ORACLE_FN(photometric_loss)(const float* rendered, const float* target, int w, int h, int ch, float lambda,
                                  float* grad) {
    const size_t n = (size_t)w * h * ch;
    float* g_l1 = grad ? (float*)malloc(sizeof(float) * n) : NULL;
    float* g_s = grad ? (float*)malloc(sizeof(float) * n) : NULL;
    const float l1 = ORACLE_FN(l1_loss)(rendered, target, (int64_t)n, g_l1);
    const float sv = ORACLE_FN(ssim)(rendered, target, w, h, ch, g_s);
    if (grad)
        for (size_t i = 0; i < n; ++i) grad[i] = (1.0f - lambda) * g_l1[i] - lambda * g_s[i];
    free(g_l1);
    free(g_s);
    return (1.0f - lambda) * l1 + lambda * (1.0f - sv);
}

/* ---- depth re-initialisation tail (spatial.cpp:101-121, densify.cpp:237-251) ------------ */
/* third_neighbor_distances: the k-th smallest distance to the other points, by brute force
 * (spatial.cpp:107-117 restated for every n; the reference's grid gives the same values). */
int ORACLE_FN(third_neighbor_distances)(const float* p, int32_t m, float min_dist, float* out) {
    if (m < 2) {
        for (int32_t i = 0; i < m; ++i) out[i] = min_dist;
        return 0;
    }
    const int k = m - 1 < 3 ? m - 1 : 3;
    for (int32_t i = 0; i < m; ++i) {
        float d[3] = {INFINITY, INFINITY, INFINITY};
        for (int32_t j = 0; j < m; ++j) {
            if (j == i) continue;
            const float e[3] = {p[3 * j] - p[3 * i], p[3 * j + 1] - p[3 * i + 1], p[3 * j + 2] - p[3 * i + 2]};
            const float dist = sqrtf(sq3(e));
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
        out[i] = fmax_std(d[k - 1], min_dist);
    }
    return 0;
}

/* The fresh set of depth_reinitialize (densify.cpp:237-251) from sampled points / colours. */
int ORACLE_FN(reinit_gaussians)(const float* points, const float* colors, int32_t m, float min_dist, float* centers,
                                float* log_scales, float* rotations, float* opacity_logits, float* sh) {
    float* nn3 = (float*)malloc(sizeof(float) * (size_t)(m > 0 ? m : 1));
    ORACLE_FN(third_neighbor_distances)(points, m, min_dist, nn3);
    const float logit01 = LOG(0.1f / (1.f - 0.1f));
    const float c0 = (float)0.28209479177387814;
    for (int32_t r = 0; r < m; ++r) {
        const float ls = LOG(nn3[r]);
        for (int c = 0; c < 3; ++c) {
            centers[3 * r + c] = points[3 * r + c];
            log_scales[3 * r + c] = ls;
        }
        rotations[4 * r] = 1.f;
        rotations[4 * r + 1] = rotations[4 * r + 2] = rotations[4 * r + 3] = 0.f;
        opacity_logits[r] = logit01;
        for (int c = 0; c < 48; ++c) sh[48 * (size_t)r + c] = 0.f;
        for (int c = 0; c < 3; ++c) sh[48 * (size_t)r + c] = colors ? (colors[3 * r + c] - 0.5f) / c0 : 0.f;
    }
    free(nn3);
    return 0;
}

