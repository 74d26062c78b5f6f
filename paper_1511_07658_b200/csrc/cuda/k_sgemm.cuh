// FP32 matrix multiply C = A * B (row-major n x n), the paper's MM payload.
//
// No reference arithmetic (proj/src/bench/profiles.cpp:35 is a timing
// triple). Precision contract: true FP32 (SIMT FFMA) — relative Frobenius
// error vs the binary64 oracle <= 1e-5. No TF32 tensor-core rounding.
//
// Fast path (n % 128 == 0): 128x128x8 CTA tile, 256 threads, 8x8 outputs per
// thread in two 4x4 quadrants (rows ty*4 and 64+ty*4, cols tx*4 and
// 64+tx*4) so shared-memory reads are 128-bit and conflict-free; A is
// stored k-major (transposed, +4 padding) in shared memory; the next k-tile
// is prefetched into registers while the current one is multiplied
// (register double buffering, one barrier per k-tile). All SGEMM tasks of a
// batch share ONE launch (blockIdx.y = task) so 16 clients x 256 tiles fill
// the 148 SMs for many waves instead of leaving a ragged single wave.
// Generic path: 16x16 shared tiles with bounds checks, any n.
#pragma once

#include <cstdint>

namespace vgk {

constexpr int kGemmThreads = 256;
constexpr int kGemmBM = 128, kGemmBN = 128, kGemmBK = 8;
constexpr int kGemmPadA = 4;
constexpr int kMaxGemmJobs = 64;

struct GemmJob {
    const float* A;
    const float* B;
    float* C;
    std::uint32_t n;
    std::uint32_t tiles;  // fast path: (n/128)^2 ; generic: (ceil(n/16))^2
};

struct GemmTable {
    GemmJob job[kMaxGemmJobs];
    std::uint32_t njobs;
};

__global__ void __launch_bounds__(kGemmThreads, 2)
sgemm128_kernel(const __grid_constant__ GemmTable table) {
    const GemmJob& job = table.job[blockIdx.y];
    if (blockIdx.x >= job.tiles) return;
    const int n = static_cast<int>(job.n);
    const int tiles_n = n / kGemmBN;
    const int m0 = (blockIdx.x / tiles_n) * kGemmBM;
    const int n0 = (blockIdx.x % tiles_n) * kGemmBN;

    __shared__ __align__(16) float As[2][kGemmBK][kGemmBM + kGemmPadA];
    __shared__ __align__(16) float Bs[2][kGemmBK][kGemmBN];

    const int tid = threadIdx.x;
    const int ty = tid / 16, tx = tid % 16;
    // loader coordinates
    const int a_row = tid / 2, a_col = (tid % 2) * 4;
    const int b_row = tid / 32, b_col = (tid % 32) * 4;
    const float* Ag = job.A + static_cast<std::size_t>(m0 + a_row) * n + a_col;
    const float* Bg = job.B + static_cast<std::size_t>(b_row) * n + n0 + b_col;

    float acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.0f;

    float4 ra = *reinterpret_cast<const float4*>(Ag);
    float4 rb = *reinterpret_cast<const float4*>(Bg);
    As[0][a_col + 0][a_row] = ra.x;
    As[0][a_col + 1][a_row] = ra.y;
    As[0][a_col + 2][a_row] = ra.z;
    As[0][a_col + 3][a_row] = ra.w;
    *reinterpret_cast<float4*>(&Bs[0][b_row][b_col]) = rb;
    __syncthreads();

    const int ktiles = n / kGemmBK;
    for (int kt = 0; kt < ktiles; ++kt) {
        const int cur = kt & 1;
        if (kt + 1 < ktiles) {
            ra = *reinterpret_cast<const float4*>(Ag + (kt + 1) * kGemmBK);
            rb = *reinterpret_cast<const float4*>(Bg + static_cast<std::size_t>(kt + 1) * kGemmBK * n);
        }
#pragma unroll
        for (int k = 0; k < kGemmBK; ++k) {
            const float4 a0 = *reinterpret_cast<const float4*>(&As[cur][k][ty * 4]);
            const float4 a1 = *reinterpret_cast<const float4*>(&As[cur][k][64 + ty * 4]);
            const float4 b0 = *reinterpret_cast<const float4*>(&Bs[cur][k][tx * 4]);
            const float4 b1 = *reinterpret_cast<const float4*>(&Bs[cur][k][64 + tx * 4]);
            const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
            const float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
        if (kt + 1 < ktiles) {
            const int nxt = cur ^ 1;
            As[nxt][a_col + 0][a_row] = ra.x;
            As[nxt][a_col + 1][a_row] = ra.y;
            As[nxt][a_col + 2][a_row] = ra.z;
            As[nxt][a_col + 3][a_row] = ra.w;
            *reinterpret_cast<float4*>(&Bs[nxt][b_row][b_col]) = rb;
        }
        __syncthreads();
    }

#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int row = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
        float* crow = job.C + static_cast<std::size_t>(row) * n + n0;
        *reinterpret_cast<float4*>(crow + tx * 4) =
            make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
        *reinterpret_cast<float4*>(crow + 64 + tx * 4) =
            make_float4(acc[i][4], acc[i][5], acc[i][6], acc[i][7]);
    }
}

constexpr int kGemmSmallTile = 16;

__global__ void __launch_bounds__(kGemmSmallTile * kGemmSmallTile)
sgemm_generic_kernel(const __grid_constant__ GemmTable table) {
    const GemmJob& job = table.job[blockIdx.y];
    if (blockIdx.x >= job.tiles) return;
    const int n = static_cast<int>(job.n);
    const int tiles_n = (n + kGemmSmallTile - 1) / kGemmSmallTile;
    const int row = (blockIdx.x / tiles_n) * kGemmSmallTile + threadIdx.y;
    const int col = (blockIdx.x % tiles_n) * kGemmSmallTile + threadIdx.x;
    __shared__ float sa[kGemmSmallTile][kGemmSmallTile + 1];
    __shared__ float sb[kGemmSmallTile][kGemmSmallTile + 1];
    float acc = 0.0f;
    for (int k0 = 0; k0 < n; k0 += kGemmSmallTile) {
        const int ka = k0 + threadIdx.x, kb = k0 + threadIdx.y;
        sa[threadIdx.y][threadIdx.x] =
            (row < n && ka < n) ? job.A[static_cast<std::size_t>(row) * n + ka] : 0.0f;
        sb[threadIdx.y][threadIdx.x] =
            (kb < n && col < n) ? job.B[static_cast<std::size_t>(kb) * n + col] : 0.0f;
        __syncthreads();
#pragma unroll
        for (int k = 0; k < kGemmSmallTile; ++k)
            acc = fmaf(sa[threadIdx.y][k], sb[k][threadIdx.x], acc);
        __syncthreads();
    }
    if (row < n && col < n) job.C[static_cast<std::size_t>(row) * n + col] = acc;
}

}  // namespace vgk
