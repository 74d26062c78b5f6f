// Electrostatics payload ("electrostatics"): direct Coulomb summation of
// point charges on a lattice, the VMD algorithm the paper benchmarks as ES
// (PAPER.md:431, :510 — 100K atoms, 25 iterations; no reference kernel:
// proj/src/bench/profiles.cpp:43 is a timing profile only).
//
//   V(p) = sum_i q_i / |p - a_i|,   p = (x h, y h, z h) on an nx x ny x nz
//   lattice (one z slice = one of the paper's iterations)
//
// B200 design: the sum is bound by the reciprocal square root (MUFU, 16
// per clock per SM, a quarter of the FMA rate), so everything else per
// atom-point is kept to two FMA-pipe ops: each thread owns kEsPts lattice
// points spaced kEsTx apart along x (dx of point u = dx_0 + u kEsTx h), the
// y/z part of r^2 is computed once per atom per thread, atoms stream
// through shared memory in tiles of kEsTile (float4 x, y, z, q) shared by
// the CTA's 128 threads. Partial sums are FP32 per tile and FP64 across
// tiles (one DADD per 512 atoms per point), which keeps the result within
// ~1e-6 of the binary64 oracle at 100K atoms.
#pragma once

#include <cstdint>

#include "vgpu_cuda.h"

namespace vgk {

constexpr int kEsTx = 16;       // threads along x
constexpr int kEsTy = 8;        // threads along y
constexpr int kEsThreads = kEsTx * kEsTy;
constexpr int kEsPts = 4;       // lattice points per thread along x
constexpr int kEsTile = 512;    // atoms per shared-memory tile
constexpr int kMaxEsJobs = 32;

struct EsJob {
    const float4* atoms;
    float* out;
    std::uint32_t natoms, nx, ny, nz;
    float h;
    std::uint32_t bx, by;       // CTAs along x and y (z: one per slice)
    std::uint32_t cta_begin;
};

struct EsTable {
    EsJob job[kMaxEsJobs];
    std::uint32_t njobs;
};

// MUFU.RSQ without rsqrtf's denormal rescaling (r^2 is never subnormal:
// atoms are off the lattice): one instruction per atom-point
__device__ __forceinline__ float es_rsqrt(float x) {
    float y;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__global__ void __launch_bounds__(kEsThreads) es_table_kernel(const __grid_constant__ EsTable table) {
    __shared__ float4 tile[kEsTile];
    int j = 0;
#pragma unroll 1
    for (int k = 1; k < static_cast<int>(table.njobs); ++k)
        if (table.job[k].cta_begin <= blockIdx.x) j = k;
    const EsJob& job = table.job[j];
    const std::uint32_t local = blockIdx.x - job.cta_begin;
    const std::uint32_t cz = local / (job.bx * job.by);
    const std::uint32_t cy = (local / job.bx) % job.by;
    const std::uint32_t cx = local % job.bx;
    const unsigned tx = threadIdx.x % kEsTx, ty = threadIdx.x / kEsTx;
    const std::uint32_t x0 = cx * (kEsTx * kEsPts) + tx;
    const std::uint32_t y = cy * kEsTy + ty;
    const float h = job.h;
    const float px = static_cast<float>(x0) * h, py = static_cast<float>(y) * h,
                pz = static_cast<float>(cz) * h;
    const float step = kEsTx * h;
    double total[kEsPts];
#pragma unroll
    for (int u = 0; u < kEsPts; ++u) total[u] = 0.0;
    for (std::uint32_t a0 = 0; a0 < job.natoms; a0 += kEsTile) {
        const std::uint32_t na = min(static_cast<std::uint32_t>(kEsTile), job.natoms - a0);
        __syncthreads();
        for (std::uint32_t i = threadIdx.x; i < na; i += kEsThreads) tile[i] = __ldg(job.atoms + a0 + i);
        __syncthreads();
        float acc[kEsPts];
#pragma unroll
        for (int u = 0; u < kEsPts; ++u) acc[u] = 0.0f;
#pragma unroll 4
        for (std::uint32_t i = 0; i < na; ++i) {
            const float4 at = tile[i];
            const float dy = py - at.y, dz = pz - at.z;
            const float dyz2 = fmaf(dy, dy, dz * dz);
            const float dx0 = px - at.x;
#pragma unroll
            for (int u = 0; u < kEsPts; ++u) {
                const float dx = fmaf(static_cast<float>(u), step, dx0);
                acc[u] = fmaf(at.w, es_rsqrt(fmaf(dx, dx, dyz2)), acc[u]);
            }
        }
#pragma unroll
        for (int u = 0; u < kEsPts; ++u) total[u] += static_cast<double>(acc[u]);
    }
    if (y >= job.ny) return;
    float* row = job.out + (static_cast<std::uint64_t>(cz) * job.ny + y) * job.nx;
#pragma unroll
    for (int u = 0; u < kEsPts; ++u) {
        const std::uint32_t x = x0 + u * kEsTx;
        if (x < job.nx) row[x] = static_cast<float>(total[u]);
    }
}

}  // namespace vgk
