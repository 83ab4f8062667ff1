// adapter_check.cpp — the drop-in, exercised in the reference's own C++ types (TEST).
//
// Builds the reference's test fixtures (tests/test_utils.hpp random_set / random_camera, included
// in place), runs the reference's CPU splat::render / render_backward / OptimState::step (mode-B
// build, oracle/_ref/libsplat_ref.so) and the GPU drop-ins of include/splat_b200_adapter.hpp on
// the same inputs, and checks forward images and Adam bit for bit, gradients within tolerance,
// and the reference's exceptions.  Built by oracle/Makefile (needs /root/reference); run on the
// GPU box by tests/test_adapter.py.
#include <cmath>
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

int main() {
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
