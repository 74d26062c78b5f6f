// NPB MG right-hand side (zran3, NPB 3.x mg.f) for the nas-mg payload.
#include "vgpu/npb_mg.hpp"

#include <algorithm>
#include <array>
#include <cstring>
#include <stdexcept>

#include "vgpu_cuda.h"

namespace vgpu::npb {

namespace {

constexpr std::uint64_t kMask46 = (std::uint64_t{1} << 46) - 1;
constexpr std::uint64_t kA = 1220703125ull;  // 5^13

std::uint64_t powmod46(std::uint64_t a, std::uint64_t e) {
    std::uint64_t r = 1;
    for (; e; e >>= 1, a = (a * a) & kMask46)
        if (e & 1) r = (r * a) & kMask46;
    return r;
}

}  // namespace

MgClass mg_class(char cls) {
    switch (cls) {
        case 'S': return {32, 4, 0, 0.5307707005734e-04};
        case 'W': return {128, 4, 0, 0.6467329375339e-05};
        case 'A': return {256, 4, 0, 0.2433365309069e-05};
        case 'B': return {256, 20, 1, 0.1800564401355e-05};
        case 'C': return {512, 20, 1, 0.5706732285740e-06};
        default: throw std::invalid_argument(std::string("unknown NPB MG class ") + cls);
    }
}

std::vector<std::uint8_t> make_mg_input(std::uint32_t nx, std::uint32_t nit, std::uint32_t coeffs) {
    if (nx < 4 || nx > 512 || (nx & (nx - 1))) throw std::invalid_argument("nas-mg: nx must be a power of two in 4..512");
    const std::uint64_t pts = std::uint64_t{nx} * nx * nx;
    std::vector<std::uint8_t> out(vgpu_mg_input_bytes(nx));
    const vgpu_mg_header h{nx, nit, coeffs, 0};
    std::memcpy(out.data(), &h, sizeof h);
    // zran3's draws: point (i1, i2, i3) takes x0 a^(1 + i1 + nx (i2 + nx i3));
    // keep the 10 largest and 10 smallest as (value, index), index order
    // breaking ties like mg.f's strict comparisons (the first one met stays)
    std::array<std::pair<double, std::uint64_t>, 10> hi{}, lo{};
    hi.fill({0.0, 0});
    lo.fill({1.0, 0});
    const std::uint64_t row = powmod46(kA, nx), plane = powmod46(kA, std::uint64_t{nx} * nx);
    std::uint64_t x_plane = 314159265ull, idx = 0;
    for (std::uint32_t i3 = 0; i3 < nx; ++i3, x_plane = (x_plane * plane) & kMask46) {
        std::uint64_t x_row = x_plane;
        for (std::uint32_t i2 = 0; i2 < nx; ++i2, x_row = (x_row * row) & kMask46) {
            std::uint64_t x = x_row;
            for (std::uint32_t i1 = 0; i1 < nx; ++i1, ++idx) {
                x = (x * kA) & kMask46;
                const double z = static_cast<double>(x) * 0x1p-46;
                if (z > hi[0].first) {  // hi ascending: hi[0] = smallest kept
                    hi[0] = {z, idx};
                    for (int k = 0; k < 9 && hi[k].first > hi[k + 1].first; ++k) std::swap(hi[k], hi[k + 1]);
                }
                if (z < lo[0].first) {  // lo descending: lo[0] = largest kept
                    lo[0] = {z, idx};
                    for (int k = 0; k < 9 && lo[k].first < lo[k + 1].first; ++k) std::swap(lo[k], lo[k + 1]);
                }
            }
        }
    }
    double* v = reinterpret_cast<double*>(out.data() + sizeof h);
    std::fill(v, v + pts, 0.0);
    for (const auto& [z, i] : lo) v[i] = -1.0;
    for (const auto& [z, i] : hi) v[i] = 1.0;
    return out;
}

}  // namespace vgpu::npb
