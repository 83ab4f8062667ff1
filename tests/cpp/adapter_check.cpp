// adapter_check.cpp — the drop-in, exercised in the reference's own C++ types (TEST).
//
// Builds the reference's test fixtures (tests/test_utils.hpp random_set / random_camera, included
// in place), runs the reference's CPU splat::render / render_backward / OptimState::step (mode-B
// build, oracle/_ref/libsplat_ref.so) and the GPU drop-ins of include/splat_b200_adapter.hpp on
// the same inputs, and checks forward images and Adam bit for bit, gradients within tolerance,
// and the reference's exceptions.  Built by oracle/Makefile (needs /root/reference); run on the
// GPU box by tests/test_adapter.py.
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <random>

#include "splat_b200_adapter.hpp"
#include "test_utils.hpp"

using namespace splat;

static int fails = 0;
#define EXPECT(c, ...)                 \
    do {                               \
        if (!(c)) {                    \
            std::printf("FAIL: " __VA_ARGS__); \
            std::printf("\n");         \
            ++fails;                   \
        }                              \
    } while (0)

static bool same(const std::vector<float>& a, const std::vector<float>& b) {
    return a.size() == b.size() && std::memcmp(a.data(), b.data(), a.size() * 4) == 0;
}

static double block_err(const std::vector<float>& g, const std::vector<float>& r) {
    double m = 0, e = 0;
    for (size_t i = 0; i < r.size(); ++i) {
        m = std::max(m, (double)std::fabs(r[i]));
        e = std::max(e, (double)std::fabs(g[i] - r[i]));
    }
    return m > 0 ? e / m : e;
}

template <class V>
static std::vector<float> flat(const std::vector<V>& v, int k) {
    std::vector<float> o;
    for (const auto& x : v)
        for (int i = 0; i < k; ++i) o.push_back(x[i]);
    return o;
}

// --time N: the drop-in at BASELINE config 1 scale (N Gaussians, 1237 x 822): one view's
// render -> l1_loss -> render_backward -> OptimState::step through the adapter, by value and with a
// resident set, views/s.
static int time_adapter(int n) {
    std::mt19937 rng(0);
    const auto set0 = testutil::random_set<float>(rng, n, 3);
    Camera cam = testutil::random_camera<float>(rng, 1237, 822);
    RasterConfig cfg;
    Imagef target(cam.width, cam.height, 3, 0.5f);
    for (int resident = 0; resident < 2; ++resident) {
        GaussianSet s = set0;
        gpu::Context ctx;
        ctx.keep_resident(resident != 0);
        gpu::OptimState opt(AdamConfig(), s.size());
        auto one = [&]() {
            const auto out = gpu::render(s, cam, cfg, nullptr, Vec3f::Zero(), nullptr, ctx);
            Imagef d_color;
            gpu::l1_loss(out.color, target, &d_color, ctx);
            const auto g = gpu::render_backward(s, cam, cfg, d_color, nullptr, Vec3f::Zero(), ctx);
            opt.step(s, g, ctx);
        };
        one();
        const auto t0 = std::chrono::steady_clock::now();
        const int iters = 5;
        for (int i = 0; i < iters; ++i) one();
        const double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        std::printf("ADAPTER_TIME resident=%d n=%d views_per_s=%.2f ms_per_view=%.1f\n", resident, n, iters / sec,
                    1000.0 * sec / iters);
    }
    return 0;
}

int main(int argc, char** argv) {
    if (argc > 2 && std::strcmp(argv[1], "--time") == 0) return time_adapter(std::atoi(argv[2]));
    for (int scene = 0; scene < 6; ++scene) {
        std::mt19937 rng(900u + scene);
        const auto set = testutil::random_set<float>(rng, 40 + 60 * scene, scene % 4);
        const auto cam = testutil::random_camera<float>(rng, 64 + 8 * scene, 48 + 4 * scene);
        RasterConfig cfg;
        if (scene == 5) cfg.apply_thresholds = false;
        if (scene == 4) cfg.tile_size = 32;
        const Vec3f bg(0.1f * scene, 0.2f, 0.3f);
        ImportanceReport<float> rr, gr;
        const auto ref = render<float>(set, cam, cfg, nullptr, bg, &rr);
        const auto got = gpu::render(set, cam, cfg, nullptr, bg, &gr);
        EXPECT(same(ref.color.data, got.color.data), "scene %d colour", scene);
        EXPECT(same(ref.alpha.data, got.alpha.data), "scene %d alpha", scene);
        EXPECT(same(ref.depth.data, got.depth.data), "scene %d depth", scene);
        EXPECT(ref.max_contributor == got.max_contributor, "scene %d argmax", scene);
        EXPECT(same(rr.max_weight, gr.max_weight), "scene %d max_weight", scene);
        EXPECT(rr.max_pixel_count == gr.max_pixel_count, "scene %d counts", scene);
        EXPECT(block_err(gr.importance, rr.importance) < 1e-5, "scene %d importance", scene);
        const auto imp = gpu::accumulate_importance(set, cam, cfg);
        EXPECT(same(imp.max_weight, rr.max_weight), "scene %d accumulate_importance", scene);

        Imagef d_color(cam.width, cam.height, 3);
        std::uniform_real_distribution<float> u(-1.f, 1.f);
        for (auto& v : d_color.data) v = u(rng);
        const auto gref = render_backward<float>(set, cam, cfg, d_color, nullptr, bg);
        const auto ggot = gpu::render_backward(set, cam, cfg, d_color, nullptr, bg);
        EXPECT(block_err(flat(ggot.d_centers, 3), flat(gref.d_centers, 3)) < 1e-4, "scene %d d_centers", scene);
        EXPECT(block_err(flat(ggot.d_log_scales, 3), flat(gref.d_log_scales, 3)) < 1e-4, "scene %d d_scales", scene);
        EXPECT(block_err(flat(ggot.d_rotations, 4), flat(gref.d_rotations, 4)) < 1e-4, "scene %d d_rot", scene);
        EXPECT(block_err(ggot.d_opacity_logits, gref.d_opacity_logits) < 1e-4, "scene %d d_opacity", scene);
        EXPECT(block_err(ggot.d_sh, gref.d_sh) < 1e-4, "scene %d d_sh", scene);
        EXPECT(ggot.grad2d_count == gref.grad2d_count, "scene %d grad2d_count", scene);

        AdamConfig ac;
        ac.scene_extent = 2.5;
        GaussianSet a = set, b = set;
        OptimState oa(ac, set.size());
        gpu::OptimState ob(ac, set.size());
        for (int s = 0; s < 3; ++s) {
            oa.step(a, gref);
            ob.step(b, gref);
        }
        EXPECT(flat(a.centers, 3) == flat(b.centers, 3) && flat(a.rotations, 4) == flat(b.rotations, 4) &&
                   a.sh == b.sh && a.opacity_logits == b.opacity_logits,
               "scene %d adam", scene);
    }
    // project<float>: the records, bit for bit (cov_world_inv: the cofactor inverse is symmetric)
    for (int scene = 0; scene < 3; ++scene) {
        std::mt19937 rng(700u + scene);
        const auto set = testutil::random_set<float>(rng, 80 + 40 * scene, 3);
        const auto cam = testutil::random_camera<float>(rng, 96, 64);
        RasterConfig cfg;
        if (scene == 2) cfg.apply_thresholds = false;
        const auto want = project<float>(set, cam, cfg);
        const auto got = gpu::project(set, cam, cfg);
        bool ok = want.size() == got.size();
        for (size_t r = 0; ok && r < want.size(); ++r) {
            const auto &a = want[r], &b = got[r];
            ok = a.index == b.index && a.radius == b.radius && a.x0 == b.x0 && a.x1 == b.x1 && a.y0 == b.y0 &&
                 a.y1 == b.y1 && a.depth_mean == b.depth_mean && a.mean2d == b.mean2d && a.opacity == b.opacity &&
                 a.color == b.color && a.center_world == b.center_world && a.cov_degenerate == b.cov_degenerate &&
                 a.cov_world_inv == b.cov_world_inv;
            for (int k = 0; k < 3; ++k) ok = ok && a.cov2d[k] == b.cov2d[k] && a.conic[k] == b.conic[k];
        }
        EXPECT(ok, "scene %d project", scene);
    }
    // l1_loss<float>: gradient bit for bit, the value within the reference's float-sum drift
    {
        std::mt19937 rng(5);
        std::uniform_real_distribution<float> u(0.f, 1.f);
        Imagef a(40, 30, 3), b(40, 30, 3), ga, gb;
        for (auto& v : a.data) v = u(rng);
        for (auto& v : b.data) v = u(rng);
        b.data[7] = a.data[7];  // a tie: zero gradient
        const float want = l1_loss<float>(a, b, &ga);
        const float got = gpu::l1_loss(a, b, &gb);
        EXPECT(same(ga.data, gb.data), "l1 gradient");
        EXPECT(std::fabs(want - got) <= 1e-5f * std::fabs(want), "l1 value %g vs %g", want, got);
        bool threw = false;
        try {
            gpu::l1_loss(a, Imagef(3, 3, 3));
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        EXPECT(threw, "l1 shape mismatch must throw std::invalid_argument");
    }
    // resident set across render -> backward -> step, three iterations, against the reference
    {
        std::mt19937 rng(77);
        const auto set0 = testutil::random_set<float>(rng, 300, 3);
        const auto cam = testutil::random_camera<float>(rng, 80, 64);
        RasterConfig cfg;
        AdamConfig ac;
        GaussianSet a = set0, b = set0;
        OptimState oa(ac, a.size());
        gpu::OptimState ob(ac, b.size());
        gpu::Context ctx;
        ctx.keep_resident(true);
        bool ok = true;
        for (int it = 0; it < 3; ++it) {
            const auto ra = render<float>(a, cam, cfg);
            const auto rb = gpu::render(b, cam, cfg, nullptr, Vec3f::Zero(), nullptr, ctx);
            ok = ok && same(ra.color.data, rb.color.data);
            Imagef d_color(cam.width, cam.height, 3, 0.001f * (it + 1));
            const auto gga = render_backward<float>(a, cam, cfg, d_color);
            oa.step(a, gga);
            ob.step(b, gga, ctx);  // identical gradients: Adam and renormalisation bit for bit
            ok = ok && flat(a.centers, 3) == flat(b.centers, 3) && a.sh == b.sh;
        }
        b.opacity_logits[0] += 1.0f;  // a host-side edit: touch() makes the next call re-upload
        a.opacity_logits[0] += 1.0f;
        ctx.touch();
        const auto ra = render<float>(a, cam, cfg);
        const auto rb = gpu::render(b, cam, cfg, nullptr, Vec3f::Zero(), nullptr, ctx);
        ok = ok && same(ra.color.data, rb.color.data);
        EXPECT(ok, "resident training loop");
    }
    // depth_reinitialize: the fresh set and the caller's rng advance exactly as the reference's
    {
        std::mt19937 rng(11);
        const auto set = testutil::random_set<float>(rng, 400, 3);
        std::vector<Camera> cams;
        std::vector<Imagef> imgs;
        std::uniform_real_distribution<float> u(0.f, 1.f);
        for (int k = 0; k < 3; ++k) {
            cams.push_back(testutil::random_camera<float>(rng, 64, 48));
            Imagef im(64, 48, 3);
            for (auto& v : im.data) v = u(rng);
            imgs.push_back(im);
        }
        std::mt19937 ra(123), rb(123);
        const GaussianSet want = depth_reinitialize(set, cams, imgs, 500, RasterConfig(), ra);
        const GaussianSet got = gpu::depth_reinitialize(set, cams, imgs, 500, RasterConfig(), rb);
        EXPECT(want.size() == got.size() && flat(want.centers, 3) == flat(got.centers, 3) &&
                   flat(want.log_scales, 3) == flat(got.log_scales, 3) && want.sh == got.sh &&
                   want.opacity_logits == got.opacity_logits,
               "depth_reinitialize fresh set");
        EXPECT(ra() == rb(), "depth_reinitialize rng advance");
    }
    // exceptions mirror the reference
    std::mt19937 rng(1);
    const auto set = testutil::random_set<float>(rng, 6, 1);
    auto cam = testutil::random_camera<float>(rng, 24, 24);
    const std::vector<char> short_mask{1, 0};
    bool threw = false;
    try {
        gpu::render(set, cam, RasterConfig(), &short_mask);
    } catch (const std::invalid_argument&) {
        threw = true;
    }
    EXPECT(threw, "short mask must throw std::invalid_argument");
    threw = false;
    try {
        gpu::render_backward(set, cam, RasterConfig(), Imagef(3, 3, 3));
    } catch (const std::invalid_argument&) {
        threw = true;
    }
    EXPECT(threw, "d_color shape must throw std::invalid_argument");
    std::printf("%s (%d failures)\n", fails ? "FAILED" : "PASSED", fails);
    return fails ? 1 : 0;
}
