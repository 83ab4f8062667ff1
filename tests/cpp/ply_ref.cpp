// tests/cpp/ply_ref.cpp — TEST INFRASTRUCTURE: the reference's own write_ply / read_ply
// (ply_io.cpp, in oracle/_ref/libsplat_ref.so) as a command-line helper.  The Python
// interpreter of this image exports libstdc++ symbols that break std::fstream inside a dlopen'ed
// library, so tests/test_ply.py drives the reference's PLY code through this process instead.
//   ply_ref write <arrays.bin> <n> <out.ply>   arrays.bin = centers | log_scales | rotations |
//                                              opacity_logits | sh (float32, GaussianSet order)
//   ply_ref read <in.ply> <arrays.bin>         the same layout back
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "splat_b200.h"

extern "C" int ref_write_ply(const char* path, const splat_gaussians* g);
extern "C" int ref_read_ply(const char* path, float* centers, float* log_scales, float* rotations,
                            float* opacity_logits, float* sh, int32_t capacity, int32_t* n_out);
extern "C" const char* ref_last_error(void);

int main(int argc, char** argv) {
    if (argc < 4) return 2;
    const std::string mode = argv[1];
    if (mode == "write" && argc == 5) {
        const int n = std::atoi(argv[3]);
        std::vector<float> a((size_t)n * 59);
        FILE* f = std::fopen(argv[2], "rb");
        if (!f || std::fread(a.data(), 4, a.size(), f) != a.size()) return 3;
        std::fclose(f);
        float* p = a.data();
        splat_gaussians g{p, p + 3 * n, p + 6 * n, p + 10 * n, p + 11 * n, n, 3};
        const int rc = ref_write_ply(argv[4], &g);
        if (rc) std::fprintf(stderr, "%s\n", ref_last_error());
        return rc;
    }
    if (mode == "read") {
        int32_t n = 0;
        ref_read_ply(argv[2], nullptr, nullptr, nullptr, nullptr, nullptr, 0, &n);  // row count
        std::vector<float> a((size_t)(n > 0 ? n : 1) * 59);
        float* p = a.data();
        const int rc = ref_read_ply(argv[2], p, p + 3 * n, p + 6 * n, p + 10 * n, p + 11 * n, n, &n);
        if (rc) {
            std::fprintf(stderr, "%s\n", ref_last_error());
            return rc;
        }
        FILE* f = std::fopen(argv[3], "wb");
        if (!f) return 3;
        std::fwrite(a.data(), 4, (size_t)n * 59, f);
        std::fclose(f);
        return 0;
    }
    return 2;
}
