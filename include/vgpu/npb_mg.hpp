// NPB MG problem builder: the SPMD program's side of the nas-mg payload.
//
// NPB MG times only its V-cycles; the right-hand side v is built before the
// timer by zran3 (NPB 3.x mg.f): nx^3 draws of the 46-bit LCG (seed
// 314159265, multiplier 5^13, i1 fastest), v = +1 at the 10 largest draws,
// -1 at the 10 smallest, 0 elsewhere. An MG client does the same here and
// sends v as the nas-mg input (include/vgpu_cuda.h: vgpu_mg_header | v).
#ifndef VGPU_NPB_MG_HPP
#define VGPU_NPB_MG_HPP

#include <cstdint>
#include <vector>

namespace vgpu::npb {

struct MgClass {
    std::uint32_t nx;      // grid points per dimension
    std::uint32_t nit;     // V-cycles
    std::uint32_t coeffs;  // smoother set (0: S/W/A, 1: B/C)
    double rnm2_verify;    // NPB's published ||r||_2 / sqrt(nx^3) after nit cycles
};

// NPB classes S, W, A, B, C; throws std::invalid_argument otherwise.
MgClass mg_class(char cls);

// The nas-mg input bytes: header + zran3's v (nx a power of two, 4..512).
std::vector<std::uint8_t> make_mg_input(std::uint32_t nx, std::uint32_t nit, std::uint32_t coeffs);

}  // namespace vgpu::npb

#endif
