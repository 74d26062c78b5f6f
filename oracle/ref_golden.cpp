// ORACLE — TEST INFRASTRUCTURE. Links the unmodified reference library
// (oracle/_ref/libvgpu_ref.a) and writes golden vectors produced by the
// reference's OWN payload code path (PayloadRegistry::builtins().execute,
// proj/src/payload.cpp:21-46,:59-65) for seeded inputs:
//   mt19937(41) U(-1000, 1000), the generator of proj/tests/test_payload.cpp:63-79.
// Output (argv[1] directory): ref_vector_ops.bin = for each n in SIZES:
//   u64 n | f32 a[n] | f32 b[n] | f32 add[n] | f32 scale2[n]
// The generating command is oracle/make_golden.sh.
#include <cstdio>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "vgpu/payload.hpp"

int main(int argc, char** argv) {
    const std::string dir = argc > 1 ? argv[1] : ".";
    std::FILE* f = std::fopen((dir + "/ref_vector_ops.bin").c_str(), "wb");
    if (!f) return 1;
    std::mt19937 rng(41);
    std::uniform_real_distribution<float> d(-1000.f, 1000.f);
    const auto& reg = vgpu::PayloadRegistry::builtins();
    for (std::uint64_t n : {1ull, 7ull, 1024ull, 4099ull}) {
        std::vector<float> a(n), b(n);
        for (std::uint64_t i = 0; i < n; ++i) {
            a[i] = d(rng);
            b[i] = d(rng);
        }
        vgpu::Bytes in(8 * n);
        std::memcpy(in.data(), a.data(), 4 * n);
        std::memcpy(in.data() + 4 * n, b.data(), 4 * n);
        const vgpu::Bytes add = reg.execute("vector-add", in);
        const vgpu::Bytes sc = reg.execute("vector-scale", vgpu::Bytes(in.begin(), in.begin() + 4 * n));
        std::fwrite(&n, 8, 1, f);
        std::fwrite(a.data(), 4, n, f);
        std::fwrite(b.data(), 4, n, f);
        std::fwrite(add.data(), 1, add.size(), f);
        std::fwrite(sc.data(), 1, sc.size(), f);
    }
    std::fclose(f);
    return 0;
}
