// splat_b200_adapter.hpp — drop-in for the reference's C++ API on top of the C-ABI.
//
// A maintainer of the reference adds this header (and links libsplat_b200.so + libcudart) and
// switches call sites from the reference's functions to splat::gpu::*, with identical signatures,
// argument meaning and exceptions.  It includes the reference's own headers
// and therefore compiles only inside the reference's build.
//
//   reference                                                               this header
//   project<float>(set, cam, cfg, mask)              rasterizer.hpp:67-70  -> gpu::project(...)
//   render<float>(set, cam, cfg, mask, bg, report)   rasterizer.hpp:72-76  -> gpu::render(...)
//   accumulate_importance<float>(set, cam, cfg, mask) rasterizer.hpp:79-82 -> gpu::accumulate_importance(...)
//   render_backward<float>(set, cam, cfg, d_color, mask, bg) gradients.hpp:52-56 -> gpu::render_backward(...)
//   l1_loss<float>(a, b, grad)                       loss.hpp:9-10         -> gpu::l1_loss(...)
//   OptimState(cfg, n).step(set, grads)              optimizer.hpp:41      -> gpu::OptimState(cfg, n).step(...)
//   depth_reinitialize(set, cams, images, k, cfg, rng) densify.hpp:77      -> gpu::depth_reinitialize(...)
//
// Data movement.  The reference passes host std::vectors by value, so by default every call
// copies the set to HBM (through pinned, double-buffered staging) and the results back.  A
// training loop can keep the set resident instead: Context::keep_resident(true) makes the
// context reuse its device copy while the set's storage (data pointers and size) and the
// caller's generation counter (Context::touch(), to be called after modifying the set on the
// host) are unchanged; gpu::OptimState::step updates the device copy in place and writes the new
// parameters back into the host set, so the copy stays valid across render -> backward -> step.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "splat/densify.hpp"
#include "splat/gradients.hpp"
#include "splat/loss.hpp"
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
    Buffer() = default;
    Buffer(const Buffer&) = delete;
    Buffer& operator=(const Buffer&) = delete;
    ~Buffer() {
        if (p) cudaFree(p);
    }
    void* ensure(size_t n) {
        if (n > bytes || !p) {
            if (p) cudaFree(p);
            p = nullptr;
            check_cuda(cudaMalloc(&p, n > 0 ? n : 4), "cudaMalloc");
            bytes = n > 0 ? n : 4;
        }
        return p;
    }
    template <typename T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

// Host <-> device copies of pageable memory through two pinned chunks: the CPU copy of chunk k + 1
// overlaps the DMA of chunk k.
class Staging {
public:
    static constexpr size_t kChunk = 8u << 20;
    ~Staging() {
        for (int k = 0; k < 2; ++k) {
            if (buf_[k]) cudaFreeHost(buf_[k]);
            if (ev_[k]) cudaEventDestroy(ev_[k]);
        }
    }
    void h2d(void* dst, const void* src, size_t n, cudaStream_t s) {
        init();
        const char* in = static_cast<const char*>(src);
        char* out = static_cast<char*>(dst);
        for (size_t off = 0, k = 0; off < n; off += kChunk, k ^= 1) {
            const size_t c = std::min(kChunk, n - off);
            check_cuda(cudaEventSynchronize(ev_[k]), "staging wait");  // chunk k's previous DMA done
            std::memcpy(buf_[k], in + off, c);
            check_cuda(cudaMemcpyAsync(out + off, buf_[k], c, cudaMemcpyHostToDevice, s), "upload");
            check_cuda(cudaEventRecord(ev_[k], s), "staging record");
        }
        check_cuda(cudaStreamSynchronize(s), "upload sync");
    }
    void d2h(void* dst, const void* src, size_t n, cudaStream_t s) {
        init();
        char* out = static_cast<char*>(dst);
        const char* in = static_cast<const char*>(src);
        size_t pending = 0, pending_off = 0;
        int pk = 0;
        for (size_t off = 0, k = 0; off < n; off += kChunk, k ^= 1) {
            const size_t c = std::min(kChunk, n - off);
            check_cuda(cudaMemcpyAsync(buf_[k], in + off, c, cudaMemcpyDeviceToHost, s), "download");
            check_cuda(cudaEventRecord(ev_[k], s), "staging record");
            if (pending) {  // the previous chunk's bytes leave the pinned buffer while this one lands
                check_cuda(cudaEventSynchronize(ev_[pk]), "staging wait");
                std::memcpy(out + pending_off, buf_[pk], pending);
            }
            pending = c;
            pending_off = off;
            pk = (int)k;
        }
        if (pending) {
            check_cuda(cudaEventSynchronize(ev_[pk]), "staging wait");
            std::memcpy(out + pending_off, buf_[pk], pending);
        }
    }

private:
    void init() {
        if (buf_[0]) return;
        for (int k = 0; k < 2; ++k) {
            check_cuda(cudaHostAlloc(&buf_[k], kChunk, cudaHostAllocDefault), "cudaHostAlloc");
            check_cuda(cudaEventCreateWithFlags(&ev_[k], cudaEventDisableTiming), "event");
            check_cuda(cudaEventRecord(ev_[k], 0), "event");
        }
    }
    void* buf_[2] = {nullptr, nullptr};
    cudaEvent_t ev_[2] = {nullptr, nullptr};
};

}  // namespace detail

// One C-ABI context + device buffers per host thread (the reference's functions are reentrant
// per thread).  The C-ABI calls run on the context's stream (the legacy default stream).
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
    cudaStream_t stream() const { return nullptr; }

    // Device-resident set (see the header comment).  touch(): the host set was modified.
    void keep_resident(bool on) {
        resident_ = on;
        valid_ = false;
    }
    void touch() { ++generation_; }

    void h2d(void* dst, const void* src, size_t n) {
        if (n) staging_.h2d(dst, src, n, stream());
    }
    void d2h(void* dst, const void* src, size_t n) {
        if (n) staging_.d2h(dst, src, n, stream());
    }

    // The set in HBM as one packed block [centers 3N | log_scales 3N | rotations 4N | opacity N |
    // sh 48N] (the layout the optimiser and the gradients share).
    splat_gaussians upload(const GaussianSet& set) {
        set.check_consistent();
        const size_t n = static_cast<size_t>(set.size());
        static_assert(sizeof(Vec3f) == 12 && sizeof(Vec4f) == 16, "packed Vec3f / Vec4f expected");
        if (!(resident_ && valid_ && matches(set))) {
            float* d = static_cast<float*>(set_.ensure(n * 59 * 4));
            h2d(d, set.centers.data(), n * 12);
            h2d(d + 3 * n, set.log_scales.data(), n * 12);
            h2d(d + 6 * n, set.rotations.data(), n * 16);
            h2d(d + 10 * n, set.opacity_logits.data(), n * 4);
            h2d(d + 11 * n, set.sh.data(), n * 192);
            remember(set);
        }
        return view(set);
    }
    // After the device copy was updated to equal `set` (gpu::OptimState::step).
    void remember(const GaussianSet& set) {
        key_ = {set.centers.data(), set.log_scales.data(), set.rotations.data(), set.opacity_logits.data(),
                set.sh.data(), set.size(), generation_};
        valid_ = true;
    }
    bool holds(const GaussianSet& set) const { return valid_ && matches(set); }
    float* set_dev() const { return set_.as<float>(); }
    splat_gaussians view(const GaussianSet& set) const {
        const size_t n = static_cast<size_t>(set.size());
        const float* d = set_.as<float>();
        return splat_gaussians{d, d + 3 * n, d + 6 * n, d + 10 * n, d + 11 * n, set.size(), set.active_sh_degree};
    }

    const uint8_t* upload_mask(const std::vector<char>* mask, int n) {
        if (!mask) return nullptr;
        if (static_cast<int>(mask->size()) != n)
            throw std::invalid_argument("visibility mask size does not match Gaussian count");
        m_.ensure(mask->size());
        h2d(m_.p, mask->data(), mask->size());
        return static_cast<const uint8_t*>(m_.p);
    }
    detail::Buffer& scratch(int k) { return tmp_[k]; }

private:
    struct Key {
        const void *c = nullptr, *s = nullptr, *r = nullptr, *o = nullptr, *h = nullptr;
        int n = -1;
        unsigned long long gen = 0;
    };
    bool matches(const GaussianSet& set) const {
        return key_.c == set.centers.data() && key_.s == set.log_scales.data() && key_.r == set.rotations.data() &&
               key_.o == set.opacity_logits.data() && key_.h == set.sh.data() && key_.n == set.size() &&
               key_.gen == generation_;
    }
    splat_ctx* ctx_ = nullptr;
    detail::Buffer set_, m_;
    detail::Buffer tmp_[16];
    detail::Staging staging_;
    bool resident_ = false, valid_ = false;
    unsigned long long generation_ = 0;
    Key key_;
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

// project<float> (rasterizer.hpp:67-70)
inline std::vector<ProjectedGaussian<float>> project(const GaussianSet& set, const Camera& cam, const RasterConfig& cfg,
                                                     const std::vector<char>* visibility_mask = nullptr,
                                                     Context& ctx = Context::thread_default()) {
    cam.validate();
    const splat_gaussians g = ctx.upload(set);
    const uint8_t* mask = ctx.upload_mask(visibility_mask, set.size());
    const splat_camera c = to_c(cam);
    const splat_raster_config rc = to_c(cfg);
    std::vector<splat_projected> raw(static_cast<size_t>(std::max(set.size(), 1)));
    int32_t count = 0;
    detail::check(ctx.get(), splat_project(ctx.get(), &g, &c, &rc, mask, raw.data(), (int64_t)raw.size(), &count));
    std::vector<ProjectedGaussian<float>> out(static_cast<size_t>(count));
    for (int r = 0; r < count; ++r) {
        const splat_projected& q = raw[r];
        ProjectedGaussian<float>& p = out[r];
        p.mean2d = Vec2f(q.mean2d[0], q.mean2d[1]);
        for (int k = 0; k < 3; ++k) {
            p.cov2d[k] = q.cov2d[k];
            p.conic[k] = q.conic[k];
        }
        p.depth_mean = q.depth_mean;
        p.radius = q.radius;
        p.index = q.index;
        p.opacity = q.opacity;
        p.color = Vec3f(q.color[0], q.color[1], q.color[2]);
        p.x0 = q.x0;
        p.x1 = q.x1;
        p.y0 = q.y0;
        p.y1 = q.y1;
        p.center_world = Vec3f(q.center_world[0], q.center_world[1], q.center_world[2]);
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) p.cov_world_inv(i, j) = q.cov_world_inv[3 * i + j];
        p.cov_degenerate = q.cov_degenerate != 0;
    }
    return out;
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
    auto f = [&](int k, size_t bytes) { return ctx.scratch(k).ensure(bytes); };
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
    ctx.d2h(o.color.data.data(), ctx.scratch(0).p, hw * 12);
    ctx.d2h(o.alpha.data.data(), ctx.scratch(1).p, hw * 4);
    ctx.d2h(o.depth.data.data(), ctx.scratch(2).p, hw * 4);
    ctx.d2h(o.transmittance.data.data(), ctx.scratch(3).p, hw * 4);
    ctx.d2h(o.max_contributor.data(), ctx.scratch(4).p, hw * 4);
    if (report) {
        report->importance.assign(n, 0.f);
        report->max_weight.assign(n, 0.f);
        report->max_pixel_count.assign(n, 0);
        ctx.d2h(report->importance.data(), ctx.scratch(5).p, n * 4);
        ctx.d2h(report->max_weight.data(), ctx.scratch(6).p, n * 4);
        ctx.d2h(report->max_pixel_count.data(), ctx.scratch(7).p, n * 4);
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
    splat_importance_outputs rep{static_cast<float*>(ctx.scratch(5).ensure(n * 4)),
                                 static_cast<float*>(ctx.scratch(6).ensure(n * 4)),
                                 static_cast<int32_t*>(ctx.scratch(7).ensure(n * 4))};
    detail::check(ctx.get(), splat_accumulate_importance(ctx.get(), &g, &c, &rc, mask, &rep));
    ImportanceReport<float> r;
    r.importance.assign(n, 0.f);
    r.max_weight.assign(n, 0.f);
    r.max_pixel_count.assign(n, 0);
    ctx.d2h(r.importance.data(), ctx.scratch(5).p, n * 4);
    ctx.d2h(r.max_weight.data(), ctx.scratch(6).p, n * 4);
    ctx.d2h(r.max_pixel_count.data(), ctx.scratch(7).p, n * 4);
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
    ctx.scratch(8).ensure(d_color.data.size() * 4);
    ctx.h2d(ctx.scratch(8).p, d_color.data.data(), d_color.data.size() * 4);
    float* gb = static_cast<float*>(ctx.scratch(9).ensure(n * 59 * 4));
    float* acc = static_cast<float*>(ctx.scratch(10).ensure(n * 4));
    int32_t* cnt = static_cast<int32_t*>(ctx.scratch(11).ensure(n * 4));
    splat_param_grads pg{gb, gb + 3 * n, gb + 6 * n, gb + 10 * n, gb + 11 * n, acc, cnt};
    const float bg[3] = {background[0], background[1], background[2]};
    detail::check(ctx.get(), splat_render_backward(ctx.get(), &g, &c, &rc, static_cast<const float*>(ctx.scratch(8).p),
                                                   mask, bg, &pg, 0, 0));
    ParamGrads<float> out;
    out.resize_zero(set.size());
    static_assert(sizeof(Vec3f) == 12 && sizeof(Vec4f) == 16, "packed Vec3f / Vec4f expected");
    ctx.d2h(out.d_centers.data(), gb, n * 12);
    ctx.d2h(out.d_log_scales.data(), gb + 3 * n, n * 12);
    ctx.d2h(out.d_rotations.data(), gb + 6 * n, n * 16);
    ctx.d2h(out.d_opacity_logits.data(), gb + 10 * n, n * 4);
    ctx.d2h(out.d_sh.data(), gb + 11 * n, n * 192);
    ctx.d2h(out.grad2d_accum.data(), acc, n * 4);
    ctx.d2h(out.grad2d_count.data(), cnt, n * 4);
    return out;
}

// l1_loss<float> (loss.hpp:9-10)
inline float l1_loss(const Imagef& a, const Imagef& b, Imagef* grad = nullptr,
                     Context& ctx = Context::thread_default()) {
    if (!a.same_shape(b)) throw std::invalid_argument("l1_loss: shape mismatch");
    const size_t n = a.size();
    if (grad) *grad = Imagef(a.width, a.height, a.channels);
    float* da = static_cast<float*>(ctx.scratch(12).ensure(n * 4));
    float* db = static_cast<float*>(ctx.scratch(13).ensure(n * 4));
    float* dg = static_cast<float*>(ctx.scratch(14).ensure(n * 4));
    float* dl = static_cast<float*>(ctx.scratch(15).ensure(4));
    ctx.h2d(da, a.data.data(), n * 4);
    ctx.h2d(db, b.data.data(), n * 4);
    detail::check(ctx.get(), splat_l1_loss(ctx.get(), da, db, (int64_t)n, grad ? dg : nullptr, dl));
    float loss = 0.f;
    ctx.d2h(&loss, dl, 4);
    if (grad) ctx.d2h(grad->data.data(), dg, n * 4);
    return loss;
}

// OptimState (optimizer.hpp:37-76): moments live in HBM; step() updates the set in place.
class OptimState {
public:
    explicit OptimState(const AdamConfig& config, int n = 0) : cfg_(config), n_(n) {
        m_.ensure(static_cast<size_t>(n) * 59 * 4);
        v_.ensure(static_cast<size_t>(n) * 59 * 4);
        detail::check_cuda(cudaMemset(m_.p, 0, m_.bytes), "memset");
        detail::check_cuda(cudaMemset(v_.p, 0, v_.bytes), "memset");
    }
    int size() const { return n_; }
    int step_count() const { return t_; }

    void step(GaussianSet& set, const ParamGrads<float>& grads, Context& ctx = Context::thread_default()) {
        if (set.size() != n_ || grads.size() != n_)
            throw std::logic_error("OptimState::step: moment/gradient rows out of sync with set");
        const size_t n = static_cast<size_t>(n_);
        ctx.upload(set);  // no copy when the context already holds this set
        float* P = ctx.set_dev();
        float* G = static_cast<float*>(gd_.ensure(n * 59 * 4));
        ctx.h2d(G, grads.d_centers.data(), n * 12);
        ctx.h2d(G + 3 * n, grads.d_log_scales.data(), n * 12);
        ctx.h2d(G + 6 * n, grads.d_rotations.data(), n * 16);
        ctx.h2d(G + 10 * n, grads.d_opacity_logits.data(), n * 4);
        ctx.h2d(G + 11 * n, grads.d_sh.data(), n * 192);
        float* M = m_.as<float>();
        float* V = v_.as<float>();
        splat_params_mut pm{P, P + 3 * n, P + 6 * n, P + 10 * n, P + 11 * n, n_, set.active_sh_degree};
        splat_param_grads gr{G, G + 3 * n, G + 6 * n, G + 10 * n, G + 11 * n, nullptr, nullptr};
        splat_adam_moments mo{M, V, M + 3 * n, V + 3 * n, M + 6 * n, V + 6 * n, M + 10 * n, V + 10 * n, M + 11 * n,
                              V + 11 * n};
        splat_adam_config ac{cfg_.beta1, cfg_.beta2, cfg_.eps, cfg_.position.lr_init, cfg_.position.lr_final,
                             cfg_.position.max_steps, 0, cfg_.scene_extent, cfg_.lr_sh_dc, cfg_.lr_sh_rest,
                             cfg_.lr_opacity, cfg_.lr_scale, cfg_.lr_rotation};
        detail::check(ctx.get(), splat_adam_step(ctx.get(), &pm, &gr, &mo, &ac, &t_, SPLAT_GROUP_ALL));
        ctx.d2h(set.centers.data(), P, n * 12);
        ctx.d2h(set.log_scales.data(), P + 3 * n, n * 12);
        ctx.d2h(set.rotations.data(), P + 6 * n, n * 16);
        ctx.d2h(set.opacity_logits.data(), P + 10 * n, n * 4);
        ctx.d2h(set.sh.data(), P + 11 * n, n * 192);
        ctx.remember(set);  // host and device copies agree again
    }

private:
    AdamConfig cfg_;
    int n_ = 0;
    int t_ = 0;
    detail::Buffer m_, v_, gd_;
};

namespace detail {
// std::mt19937 <-> splat_rng through the state libstdc++ streams (x[0..623] then the index).
inline void rng_in(splat_rng* r, const std::mt19937& g) {
    std::stringstream ss;
    ss << g;
    uint32_t w[625];
    for (int i = 0; i < 625; ++i) {
        unsigned long long v = 0;
        ss >> v;
        w[i] = (uint32_t)v;
    }
    if (splat_rng_set_state(r, w) != SPLAT_OK) throw std::runtime_error("rng state transfer");
}
inline void rng_out(const splat_rng* r, std::mt19937& g) {
    uint32_t w[625];
    if (splat_rng_get_state(r, w) != SPLAT_OK) throw std::runtime_error("rng state transfer");
    std::stringstream ss;
    for (int i = 0; i < 625; ++i) ss << w[i] << (i < 624 ? " " : "");
    ss >> g;
}
}  // namespace detail

// depth_reinitialize (densify.cpp:196-252): the renders, unprojection, the pool draw (advancing
// the caller's rng exactly as the reference does), 3rd-NN scales and the fresh set, on the GPU.
inline GaussianSet depth_reinitialize(const GaussianSet& set, const std::vector<Camera>& cameras,
                                      const std::vector<Imagef>& images, int sample_count, const RasterConfig& cfg,
                                      std::mt19937& rng, Context& ctx = Context::thread_default()) {
    if (cameras.empty()) throw std::invalid_argument("depth_reinitialize: no cameras");
    if (cameras.size() != images.size()) throw std::invalid_argument("depth_reinitialize: camera/image count mismatch");
    if (sample_count < 1) throw std::invalid_argument("depth_reinitialize: sample_count < 1");
    const splat_gaussians g = ctx.upload(set);
    const splat_raster_config rc = to_c(cfg);
    // pool: every pixel with a max contributor, view-major in raster order; its colour row
    std::vector<float> pts, cols;
    for (size_t k = 0; k < cameras.size(); ++k) {
        const Camera& cam = cameras[k];
        const Imagef& img = images[k];
        if (img.width != cam.width || img.height != cam.height || img.channels != 3)
            throw std::invalid_argument("depth_reinitialize: image does not match camera");
        cam.validate();
        const splat_camera c = to_c(cam);
        const size_t hw = static_cast<size_t>(cam.width) * cam.height;
        splat_render_outputs out{nullptr, static_cast<float*>(ctx.scratch(1).ensure(hw * 4)),
                                 static_cast<float*>(ctx.scratch(2).ensure(hw * 4)), nullptr,
                                 static_cast<int32_t*>(ctx.scratch(4).ensure(hw * 4))};
        const float bg[3] = {0.f, 0.f, 0.f};
        detail::check(ctx.get(), splat_render(ctx.get(), &g, &c, &rc, nullptr, bg, &out, nullptr));
        float* p = static_cast<float*>(ctx.scratch(12).ensure(hw * 12));
        int32_t* px = static_cast<int32_t*>(ctx.scratch(13).ensure(hw * 4));
        int32_t* cnt = static_cast<int32_t*>(ctx.scratch(15).ensure(4));
        detail::check(ctx.get(), splat_depth_unproject(ctx.get(), &c, SPLAT_DEPTH_RULE_ARGMAX, 0.5f, 0, 1, 0, p, px,
                                                       (int64_t)hw, cnt));
        int32_t m = 0;
        ctx.d2h(&m, cnt, 4);
        const size_t base = pts.size();
        pts.resize(base + 3 * (size_t)m);
        ctx.d2h(pts.data() + base, p, (size_t)m * 12);
        std::vector<int32_t> pix((size_t)m);
        ctx.d2h(pix.data(), px, (size_t)m * 4);
        for (int32_t j = 0; j < m; ++j)
            for (int ch = 0; ch < 3; ++ch) cols.push_back(img.data[3 * (size_t)pix[j] + ch]);
    }
    if (pts.empty()) throw std::runtime_error("depth_reinitialize: no valid depth pixels (model renders nothing)");
    const int pool = static_cast<int>(pts.size() / 3);
    const int take = std::min(sample_count, pool);
    splat_rng* r = nullptr;
    detail::check(ctx.get(), splat_rng_create(5489u, &r));
    struct RngGuard {
        splat_rng* r;
        ~RngGuard() { splat_rng_destroy(r); }
    } guard{r};
    detail::rng_in(r, rng);
    int32_t* idx = static_cast<int32_t*>(ctx.scratch(14).ensure((size_t)take * 4));
    detail::check(ctx.get(), splat_pool_sample(ctx.get(), r, pool, take, idx));
    detail::rng_out(r, rng);
    float* dp = static_cast<float*>(ctx.scratch(12).ensure(pts.size() * 4));
    float* dc = static_cast<float*>(ctx.scratch(13).ensure(cols.size() * 4));
    ctx.h2d(dp, pts.data(), pts.size() * 4);
    ctx.h2d(dc, cols.data(), cols.size() * 4);
    float* sp = static_cast<float*>(ctx.scratch(10).ensure((size_t)take * 12));
    float* sc = static_cast<float*>(ctx.scratch(11).ensure((size_t)take * 12));
    detail::check(ctx.get(), splat_gather_rows(ctx.get(), dp, 3, idx, take, sp));
    detail::check(ctx.get(), splat_gather_rows(ctx.get(), dc, 3, idx, take, sc));
    float* fresh = static_cast<float*>(ctx.scratch(9).ensure((size_t)take * 59 * 4));
    const size_t t = static_cast<size_t>(take);
    splat_params_mut out{fresh, fresh + 3 * t, fresh + 6 * t, fresh + 10 * t, fresh + 11 * t, take,
                         set.active_sh_degree};
    detail::check(ctx.get(), splat_reinit_gaussians(ctx.get(), sp, sc, take, 1e-7f, &out));
    GaussianSet res;
    res.active_sh_degree = set.active_sh_degree;
    res.resize(take);
    ctx.d2h(res.centers.data(), fresh, t * 12);
    ctx.d2h(res.log_scales.data(), fresh + 3 * t, t * 12);
    ctx.d2h(res.rotations.data(), fresh + 6 * t, t * 16);
    ctx.d2h(res.opacity_logits.data(), fresh + 10 * t, t * 4);
    ctx.d2h(res.sh.data(), fresh + 11 * t, t * 192);
    return res;
}

}  // namespace gpu
}  // namespace splat
