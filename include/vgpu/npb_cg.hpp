// NPB CG problem builder: the SPMD program's side of the nas-cg payload.
//
// NPB CG times only its conj_grad iterations; the sparse matrix is built
// before the timer by makea (NPB 3.x cg.f makea/sprnvc/vecset/sparse). A CG
// client does the same here and sends the result as the nas-cg input
// (include/vgpu_cuda.h: vgpu_cg_header | rowstr | colidx | a). The matrix
// bits equal NPB's: the same 46-bit LCG stream (seed 314159265, multiplier
// 5^13, one draw discarded), the same rejection sampling of positions, and
// duplicate entries summed in NPB's order (increasing outer index).
#ifndef VGPU_NPB_CG_HPP
#define VGPU_NPB_CG_HPP

#include <cstdint>
#include <vector>

namespace vgpu::npb {

struct CgClass {
    std::uint32_t n;
    std::uint32_t nonzer;
    std::uint32_t niter;
    double shift;
    double zeta_verify;  // NPB's published zeta after niter iterations
};

// NPB classes S, W, A, B, C; throws std::invalid_argument otherwise.
CgClass cg_class(char cls);

// The nas-cg input bytes for an NPB-shaped problem (rcond = 0.1, 25 CG
// steps per outer iteration).
std::vector<std::uint8_t> make_cg_input(std::uint32_t n, std::uint32_t nonzer, std::uint32_t niter,
                                        double shift);

}  // namespace vgpu::npb

#endif
