// splat_b200_adapter.hpp — drop-in for the reference's C++ API on top of the C-ABI.
//
// A maintainer of the reference adds this header (and links libsplat_b200.so + libcudart) and
// switches call sites from splat::render<float> / accumulate_importance<float> /
// render_backward<float> / OptimState::step to splat::gpu::*, with identical signatures,
// argument meaning and exceptions.  It includes the reference's own headers
// (splat/rasterizer.hpp, splat/gradients.hpp, splat/optimizer.hpp) and therefore compiles only
// inside the reference's build.
//
//   reference (rasterizer.hpp:72-82, gradients.hpp:52-56, optimizer.hpp:41)   this header
//   render<float>(set, cam, cfg, mask, bg, report)                         -> gpu::render(...)
//   accumulate_importance<float>(set, cam, cfg, mask)                      -> gpu::accumulate_importance(...)
//   render_backward<float>(set, cam, cfg, d_color, mask, bg)               -> gpu::render_backward(...)
//   OptimState(cfg, n).step(set, grads)                                    -> gpu::OptimState(cfg, n).step(...)
//
// Host std::vector storage is copied to/from HBM around each call (the reference's by-value
// semantics); a training loop that wants to stay resident uses the C-ABI directly on device
// pointers (paper_2411_12788_b200/trainer.py does).
#pragma once

#include <cuda_runtime.h>

#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "splat/gradients.hpp"
#include "splat/optimizer.hpp"
#include "splat/rasterizer.hpp"
#include "splat_b200.h"

namespace splat {
namespace gpu {

namespace detail {

inline void check_cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// Map a C-ABI status to the reference's exception types.
inline void check(splat_ctx* ctx, int rc) {
    if (rc == SPLAT_OK) return;
    const std::string msg = splat_last_error(ctx);
    if (rc == SPLAT_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
    if (rc == SPLAT_ERR_LOGIC) throw std::logic_error(msg);
    throw std::runtime_error(msg);
}

struct Buffer {
    void* p = nullptr;
    size_t bytes = 0;
    ~Buffer() {
        if (p) cudaFree(p);
    }
    void* ensure(size_t n) {
        if (n > bytes) {
            if (p) cudaFree(p);
            p = nullptr;
            check_cuda(cudaMalloc(&p, n), "cudaMalloc");
            bytes = n;
        }
        return p;
    }
};

inline void upload(Buffer& b, const void* src, size_t n) {
    if (n == 0) return;
    b.ensure(n);
    check_cuda(cudaMemcpy(b.p, src, n, cudaMemcpyHostToDevice), "upload");
}

inline void download(void* dst, const Buffer& b, size_t n) {
    if (n == 0) return;
    check_cuda(cudaMemcpy(dst, b.p, n, cudaMemcpyDeviceToHost), "download");
}

}  // namespace detail

// One CUDA context + scratch per thread (the reference's functions are reentrant per thread).
class Context {
public:
    explicit Context(int device = 0) {
        if (splat_ctx_create(device, &ctx_) != SPLAT_OK) throw std::runtime_error("splat_ctx_create failed");
    }
    ~Context() { splat_ctx_destroy(ctx_); }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    static Context& thread_default() {
        thread_local Context c;
        return c;
    }
    splat_ctx* get() const { return ctx_; }

    // Upload a GaussianSet (Vec3f / Vec4f are contiguous floats) and return the C-ABI view.
    splat_gaussians upload(const GaussianSet& set) {
        set.check_consistent();
        const size_t n = static_cast<size_t>(set.size());
        detail::upload(c_, set.centers.data(), n * 12);
        detail::upload(s_, set.log_scales.data(), n * 12);
        pack_rot_.resize(n * 4);
        for (size_t i = 0; i < n; ++i)
            for (int k = 0; k < 4; ++k) pack_rot_[4 * i + k] = set.rotations[i][k];
        detail::upload(r_, pack_rot_.data(), n * 16);
        detail::upload(o_, set.opacity_logits.data(), n * 4);
        detail::upload(h_, set.sh.data(), n * 192);
        return splat_gaussians{static_cast<const float*>(c_.p), static_cast<const float*>(s_.p),
                               static_cast<const float*>(r_.p), static_cast<const float*>(o_.p),
                               static_cast<const float*>(h_.p), set.size(), set.active_sh_degree};
    }
    const uint8_t* upload_mask(const std::vector<char>* mask, int n) {
        if (!mask) return nullptr;
        if (static_cast<int>(mask->size()) != n)
            throw std::invalid_argument("visibility mask size does not match Gaussian count");
        detail::upload(m_, mask->data(), mask->size());
        return static_cast<const uint8_t*>(m_.p);
    }
    detail::Buffer& scratch(int k) { return tmp_[k]; }

private:
    splat_ctx* ctx_ = nullptr;
    detail::Buffer c_, s_, r_, o_, h_, m_;
    detail::Buffer tmp_[12];
    std::vector<float> pack_rot_;
};

inline splat_camera to_c(const Camera& cam) {
    splat_camera c{};
    c.width = cam.width;
    c.height = cam.height;
    c.fx = cam.fx;
    c.fy = cam.fy;
    c.cx = cam.cx;
    c.cy = cam.cy;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) c.rotation[i * 3 + j] = cam.rotation(i, j);
    for (int i = 0; i < 3; ++i) c.translation[i] = cam.translation[i];
    c.znear = cam.znear;
    c.zfar = cam.zfar;
    return c;
}

inline splat_raster_config to_c(const RasterConfig& r) {
    return splat_raster_config{r.tile_size, r.apply_thresholds ? 1 : 0, r.transmittance_min, r.contribution_min,
                               r.alpha_max, r.lowpass, r.radius_sigmas};
}

// render<float> (rasterizer.hpp:72-76)
inline RenderOutput<float> render(const GaussianSet& set, const Camera& cam, const RasterConfig& cfg,
                                  const std::vector<char>* visibility_mask = nullptr,
                                  const Vec3f& background = Vec3f::Zero(),
                                  ImportanceReport<float>* report = nullptr,
                                  Context& ctx = Context::thread_default()) {
    cam.validate();
    const splat_gaussians g = ctx.upload(set);
    const uint8_t* mask = ctx.upload_mask(visibility_mask, set.size());
    const splat_camera c = to_c(cam);
    const splat_raster_config rc = to_c(cfg);
    const size_t hw = static_cast<size_t>(cam.width) * cam.height;
    const size_t n = static_cast<size_t>(set.size());
    auto f = [&](int k, size_t bytes) { return ctx.scratch(k).ensure(bytes > 0 ? bytes : 4); };
    splat_render_outputs out{static_cast<float*>(f(0, hw * 12)), static_cast<float*>(f(1, hw * 4)),
                             static_cast<float*>(f(2, hw * 4)), static_cast<float*>(f(3, hw * 4)),
                             static_cast<int32_t*>(f(4, hw * 4))};
    splat_importance_outputs rep{static_cast<float*>(f(5, n * 4)), static_cast<float*>(f(6, n * 4)),
                                 static_cast<int32_t*>(f(7, n * 4))};
    const float bg[3] = {background[0], background[1], background[2]};
    detail::check(ctx.get(), splat_render(ctx.get(), &g, &c, &rc, mask, bg, &out, report ? &rep : nullptr));
    RenderOutput<float> o;
    o.width = cam.width;
    o.height = cam.height;
    o.color = Imagef(cam.width, cam.height, 3);
    o.alpha = Imagef(cam.width, cam.height, 1);
    o.depth = Imagef(cam.width, cam.height, 1);
    o.transmittance = Imagef(cam.width, cam.height, 1);
    o.max_contributor.assign(hw, -1);
    detail::download(o.color.data.data(), ctx.scratch(0), hw * 12);
    detail::download(o.alpha.data.data(), ctx.scratch(1), hw * 4);
    detail::download(o.depth.data.data(), ctx.scratch(2), hw * 4);
    detail::download(o.transmittance.data.data(), ctx.scratch(3), hw * 4);
    detail::download(o.max_contributor.data(), ctx.scratch(4), hw * 4);
    if (report) {
        report->importance.assign(n, 0.f);
        report->max_weight.assign(n, 0.f);
        report->max_pixel_count.assign(n, 0);
        detail::download(report->importance.data(), ctx.scratch(5), n * 4);
        detail::download(report->max_weight.data(), ctx.scratch(6), n * 4);
        detail::download(report->max_pixel_count.data(), ctx.scratch(7), n * 4);
    }
    return o;
}

// accumulate_importance<float> (rasterizer.hpp:79-82)
inline ImportanceReport<float> accumulate_importance(const GaussianSet& set, const Camera& cam,
                                                     const RasterConfig& cfg,
                                                     const std::vector<char>* visibility_mask = nullptr,
                                                     Context& ctx = Context::thread_default()) {
    cam.validate();
    const splat_gaussians g = ctx.upload(set);
    const uint8_t* mask = ctx.upload_mask(visibility_mask, set.size());
    const splat_camera c = to_c(cam);
    const splat_raster_config rc = to_c(cfg);
    const size_t n = static_cast<size_t>(set.size());
    splat_importance_outputs rep{static_cast<float*>(ctx.scratch(5).ensure(n * 4 + 4)),
                                 static_cast<float*>(ctx.scratch(6).ensure(n * 4 + 4)),
                                 static_cast<int32_t*>(ctx.scratch(7).ensure(n * 4 + 4))};
    detail::check(ctx.get(), splat_accumulate_importance(ctx.get(), &g, &c, &rc, mask, &rep));
    ImportanceReport<float> r;
    r.importance.assign(n, 0.f);
    r.max_weight.assign(n, 0.f);
    r.max_pixel_count.assign(n, 0);
    detail::download(r.importance.data(), ctx.scratch(5), n * 4);
    detail::download(r.max_weight.data(), ctx.scratch(6), n * 4);
    detail::download(r.max_pixel_count.data(), ctx.scratch(7), n * 4);
    return r;
}

// render_backward<float> (gradients.hpp:52-56)
inline ParamGrads<float> render_backward(const GaussianSet& set, const Camera& cam, const RasterConfig& cfg,
                                         const Imagef& d_color, const std::vector<char>* visibility_mask = nullptr,
                                         const Vec3f& background = Vec3f::Zero(),
                                         Context& ctx = Context::thread_default()) {
    cam.validate();
    if (d_color.width != cam.width || d_color.height != cam.height || d_color.channels != 3)
        throw std::invalid_argument("render_backward: dLoss/dColor shape mismatch");
    const splat_gaussians g = ctx.upload(set);
    const uint8_t* mask = ctx.upload_mask(visibility_mask, set.size());
    const splat_camera c = to_c(cam);
    const splat_raster_config rc = to_c(cfg);
    const size_t n = static_cast<size_t>(set.size());
    detail::upload(ctx.scratch(8), d_color.data.data(), d_color.data.size() * 4);
    float* gb = static_cast<float*>(ctx.scratch(9).ensure(n * 59 * 4 + 4));
    float* acc = static_cast<float*>(ctx.scratch(10).ensure(n * 4 + 4));
    int32_t* cnt = static_cast<int32_t*>(ctx.scratch(11).ensure(n * 4 + 4));
    splat_param_grads pg{gb, gb + 3 * n, gb + 6 * n, gb + 10 * n, gb + 11 * n, acc, cnt};
    const float bg[3] = {background[0], background[1], background[2]};
    detail::check(ctx.get(), splat_render_backward(ctx.get(), &g, &c, &rc, static_cast<const float*>(ctx.scratch(8).p),
                                                   mask, bg, &pg, 0, 0));
    std::vector<float> h(n * 59);
    detail::download(h.data(), ctx.scratch(9), n * 59 * 4);
    ParamGrads<float> out;
    out.resize_zero(set.size());
    for (size_t i = 0; i < n; ++i) {
        out.d_centers[i] = Vec3f(h[3 * i], h[3 * i + 1], h[3 * i + 2]);
        out.d_log_scales[i] = Vec3f(h[3 * n + 3 * i], h[3 * n + 3 * i + 1], h[3 * n + 3 * i + 2]);
        out.d_rotations[i] = Vec4f(h[6 * n + 4 * i], h[6 * n + 4 * i + 1], h[6 * n + 4 * i + 2], h[6 * n + 4 * i + 3]);
        out.d_opacity_logits[i] = h[10 * n + i];
    }
    if (n) std::memcpy(out.d_sh.data(), h.data() + 11 * n, n * 48 * 4);
    detail::download(out.grad2d_accum.data(), ctx.scratch(10), n * 4);
    detail::download(out.grad2d_count.data(), ctx.scratch(11), n * 4);
    return out;
}

// OptimState (optimizer.hpp:37-76): moments live in HBM; step() updates `set` in place.
class OptimState {
public:
    explicit OptimState(const AdamConfig& config, int n = 0) : cfg_(config), n_(n) {
        m_.ensure(static_cast<size_t>(n) * 59 * 4 + 4);
        v_.ensure(static_cast<size_t>(n) * 59 * 4 + 4);
        detail::check_cuda(cudaMemset(m_.p, 0, m_.bytes), "memset");
        detail::check_cuda(cudaMemset(v_.p, 0, v_.bytes), "memset");
    }
    int size() const { return n_; }
    int step_count() const { return t_; }

    void step(GaussianSet& set, const ParamGrads<float>& grads, Context& ctx = Context::thread_default()) {
        if (set.size() != n_ || grads.size() != n_)
            throw std::logic_error("OptimState::step: moment/gradient rows out of sync with set");
        const size_t n = static_cast<size_t>(n_);
        std::vector<float> p(n * 59), g(n * 59);
        for (size_t i = 0; i < n; ++i) {
            for (int k = 0; k < 3; ++k) {
                p[3 * i + k] = set.centers[i][k];
                p[3 * n + 3 * i + k] = set.log_scales[i][k];
                g[3 * i + k] = grads.d_centers[i][k];
                g[3 * n + 3 * i + k] = grads.d_log_scales[i][k];
            }
            for (int k = 0; k < 4; ++k) {
                p[6 * n + 4 * i + k] = set.rotations[i][k];
                g[6 * n + 4 * i + k] = grads.d_rotations[i][k];
            }
            p[10 * n + i] = set.opacity_logits[i];
            g[10 * n + i] = grads.d_opacity_logits[i];
        }
        if (n) {
            std::memcpy(p.data() + 11 * n, set.sh.data(), n * 192);
            std::memcpy(g.data() + 11 * n, grads.d_sh.data(), n * 192);
        }
        detail::upload(pd_, p.data(), n * 59 * 4);
        detail::upload(gd_, g.data(), n * 59 * 4);
        float* P = static_cast<float*>(pd_.p);
        float* G = static_cast<float*>(gd_.p);
        float* M = static_cast<float*>(m_.p);
        float* V = static_cast<float*>(v_.p);
        splat_params_mut pm{P, P + 3 * n, P + 6 * n, P + 10 * n, P + 11 * n, n_, set.active_sh_degree};
        splat_param_grads gr{G, G + 3 * n, G + 6 * n, G + 10 * n, G + 11 * n, nullptr, nullptr};
        splat_adam_moments mo{M, V, M + 3 * n, V + 3 * n, M + 6 * n, V + 6 * n, M + 10 * n, V + 10 * n, M + 11 * n,
                              V + 11 * n};
        splat_adam_config ac{cfg_.beta1, cfg_.beta2, cfg_.eps, cfg_.position.lr_init, cfg_.position.lr_final,
                             cfg_.position.max_steps, 0, cfg_.scene_extent, cfg_.lr_sh_dc, cfg_.lr_sh_rest,
                             cfg_.lr_opacity, cfg_.lr_scale, cfg_.lr_rotation};
        detail::check(ctx.get(), splat_adam_step(ctx.get(), &pm, &gr, &mo, &ac, &t_, SPLAT_GROUP_ALL));
        detail::download(p.data(), pd_, n * 59 * 4);
        for (size_t i = 0; i < n; ++i) {
            set.centers[i] = Vec3f(p[3 * i], p[3 * i + 1], p[3 * i + 2]);
            set.log_scales[i] = Vec3f(p[3 * n + 3 * i], p[3 * n + 3 * i + 1], p[3 * n + 3 * i + 2]);
            set.rotations[i] = Vec4f(p[6 * n + 4 * i], p[6 * n + 4 * i + 1], p[6 * n + 4 * i + 2], p[6 * n + 4 * i + 3]);
            set.opacity_logits[i] = p[10 * n + i];
        }
        if (n) std::memcpy(set.sh.data(), p.data() + 11 * n, n * 192);
    }

private:
    AdamConfig cfg_;
    int n_ = 0;
    int t_ = 0;
    detail::Buffer m_, v_, pd_, gd_;
};

}  // namespace gpu
}  // namespace splat
