// NAS CG payload ("nas-cg"): the timed part of NPB CG (cg.f conj_grad and
// the outer zeta loop) on the CSR matrix the SPMD program sent.
//
// No reference arithmetic exists (proj/src/bench/profiles.cpp:41 is a timing
// profile only); the algorithm is NPB 3.x CG, restated in
// oracle/vgpu_oracle.c (vo_cg_run) and pinned there to NPB's published zeta
// values for classes S, W and A.
//
// B200 design: one thread-block CLUSTER per job (1..16 CTAs by matrix size,
// one CTA per SM: class S takes 1, W 4, A 16). Each CTA owns a contiguous
// slice of rows; its vector slices (x, z, r, q, p) live in the job's HBM
// workspace, the whole direction vector p is
// re-staged into shared memory after every update when it fits (n <= 24K,
// classes S..A), so the SpMV gathers p from shared memory and only the
// matrix streams from L2/HBM (12 B per nonzero: a f64 + colidx u32).
// Dot products reduce warp -> CTA (fixed order) -> cluster: every CTA reads
// the cluster's partials over DSMEM in rank order, so all CTAs hold the same
// bits and the result is deterministic run to run. Three cluster barriers
// per CG step (p . q, r . r, the p update), as NPB's data dependences need.
// SpMV: one warp per row, lanes stride the row, shuffle-tree sum.
#pragma once

#include <cooperative_groups.h>
#include <cstdint>

#include "vgpu_cuda.h"

namespace vgk {

namespace cgx = cooperative_groups;

constexpr int kCgThreads = 1024;
constexpr int kCgMaxCluster = 16;     // CTAs per job at most (non-portable size)
constexpr int kMaxCgJobs = 16;
constexpr std::uint32_t kCgStageMax = 24576;  // rows whose p fits in shared memory (192 KiB)

struct CgJob {
    const std::uint32_t* rowstr;
    const std::uint32_t* colidx;
    const double* a;
    double* x;
    double* z;
    double* p;
    double* q;
    double* r;
    vgpu_cg_result* out;
    std::uint32_t n, nnz, niter, cgitmax;
    double shift;
};

struct CgTable {
    CgJob job[kMaxCgJobs];
    std::uint32_t njobs;
};

__device__ __forceinline__ double cg_warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    return v;  // lane 0
}

struct CgReduce {
    double warp[kCgThreads / 32][3];
    double slot[2][3];  // this CTA's partials, read by every CTA over DSMEM
    double total[3];
};

// Sum W per-thread values over the whole cluster: warp tree, warps in
// order, CTAs in rank order (warp 0 of every CTA computes the same bits).
// The cluster barrier inside also orders every global write before it.
template <int W>
__device__ __forceinline__ void cg_cluster_sum(double (&v)[W], CgReduce& red, unsigned& parity,
                                               cgx::cluster_group& cluster, unsigned csize) {
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int w = 0; w < W; ++w) {
        const double s = cg_warp_sum(v[w]);
        if (lane == 0) red.warp[warp][w] = s;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
#pragma unroll
        for (int w = 0; w < W; ++w) {
            double s = 0.0;
#pragma unroll
            for (int k = 0; k < kCgThreads / 32; ++k) s += red.warp[k][w];
            red.slot[parity][w] = s;
        }
    }
    cluster.sync();
    if (warp == 0) {
        // lane c fetches CTA c's partials (one DSMEM round trip), lane 0
        // adds them in rank order
        double part[W];
        const double* src = lane < csize ? cluster.map_shared_rank(&red.slot[parity][0], lane) : nullptr;
#pragma unroll
        for (int w = 0; w < W; ++w) part[w] = src ? src[w] : 0.0;
#pragma unroll
        for (int w = 0; w < W; ++w) {
            double s = 0.0;
            for (unsigned c = 0; c < csize; ++c) s += __shfl_sync(0xffffffffu, part[w], c);
            if (lane == 0) red.total[w] = s;
        }
    }
    __syncthreads();
#pragma unroll
    for (int w = 0; w < W; ++w) v[w] = red.total[w];
    parity ^= 1u;
}

// y[row] = sum_k a[k] * v[colidx[k]] for this CTA's rows, one warp per row;
// lane 0 of the owning warp gets the row sum. Calls f(row, sum) on lane 0.
template <typename Gather, typename F>
__device__ __forceinline__ void cg_spmv(const CgJob& job, std::uint32_t r0, std::uint32_t r1,
                                        Gather gather, F f) {
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (std::uint32_t row = r0 + warp; row < r1; row += kCgThreads / 32) {
        const std::uint32_t k0 = __ldg(job.rowstr + row), k1 = __ldg(job.rowstr + row + 1);
        double s = 0.0;
        for (std::uint32_t k = k0 + lane; k < k1; k += 32) {
            const std::uint32_t c = min(__ldg(job.colidx + k), job.n - 1);  // malformed input stays in bounds
            s = fma(__ldg(job.a + k), gather(c), s);
        }
        s = cg_warp_sum(s);
        if (lane == 0) f(row, s);
    }
}

template <bool kStage>
__global__ void __launch_bounds__(kCgThreads, 1) cg_kernel(const __grid_constant__ CgTable table) {
    extern __shared__ double ps[];  // staged p (kStage)
    __shared__ CgReduce red;
    cgx::cluster_group cluster = cgx::this_cluster();
    const unsigned csize = cluster.num_blocks();
    const CgJob& job = table.job[blockIdx.x / csize];
    const unsigned rank = cluster.block_rank();
    const std::uint32_t n = job.n;
    const std::uint32_t r0 = static_cast<std::uint32_t>((static_cast<std::uint64_t>(n) * rank) / csize);
    const std::uint32_t r1 = static_cast<std::uint32_t>((static_cast<std::uint64_t>(n) * (rank + 1)) / csize);
    unsigned parity = 0;
    double* const x = job.x;
    double* const z = job.z;
    double* const p = job.p;
    double* const q = job.q;
    double* const r = job.r;

    auto stage_p = [&]() {
        if constexpr (kStage) {
            for (std::uint32_t i = threadIdx.x; i < n; i += kCgThreads) ps[i] = __ldcg(p + i);
            __syncthreads();
        }
    };
    auto gather_p = [&](std::uint32_t c) -> double {
        if constexpr (kStage) return ps[c];
        else return __ldcg(p + c);
    };

    for (std::uint32_t i = r0 + threadIdx.x; i < r1; i += kCgThreads) x[i] = 1.0;
    double zeta = 0.0, rnorm = 0.0;
    for (std::uint32_t it = 0; it < job.niter; ++it) {
        // conj_grad: q = z = 0, r = p = x, rho = r . r
        double v1[1] = {0.0};
        for (std::uint32_t i = r0 + threadIdx.x; i < r1; i += kCgThreads) {
            const double xi = x[i];
            z[i] = 0.0;
            r[i] = xi;
            p[i] = xi;
            v1[0] = fma(xi, xi, v1[0]);
        }
        cg_cluster_sum(v1, red, parity, cluster, csize);  // also publishes p
        double rho = v1[0];
        stage_p();
        for (std::uint32_t cgit = 0; cgit < job.cgitmax; ++cgit) {
            // q = A p, d = p . q
            double d[1] = {0.0};
            cg_spmv(job, r0, r1, gather_p, [&](std::uint32_t row, double s) {
                q[row] = s;
                d[0] = fma(p[row], s, d[0]);
            });
            cg_cluster_sum(d, red, parity, cluster, csize);
            const double alpha = rho / d[0];
            const double rho0 = rho;
            // z += alpha p, r -= alpha q, rho = r . r
            double rr[1] = {0.0};
            for (std::uint32_t i = r0 + threadIdx.x; i < r1; i += kCgThreads) {
                const double pi = p[i];
                z[i] = fma(alpha, pi, z[i]);
                const double ri = fma(-alpha, q[i], r[i]);
                r[i] = ri;
                rr[0] = fma(ri, ri, rr[0]);
            }
            cg_cluster_sum(rr, red, parity, cluster, csize);
            rho = rr[0];
            const double beta = rho / rho0;
            for (std::uint32_t i = r0 + threadIdx.x; i < r1; i += kCgThreads) p[i] = fma(beta, p[i], r[i]);
            cluster.sync();  // p complete before anyone gathers it
            stage_p();
        }
        // ||x - A z||, x . z, z . z (z complete: written before the last barriers)
        double s3[3] = {0.0, 0.0, 0.0};
        cg_spmv(job, r0, r1, [&](std::uint32_t c) { return __ldcg(z + c); },
                [&](std::uint32_t row, double s) {
                    const double xi = x[row], zi = z[row];
                    const double e = xi - s;
                    s3[0] = fma(e, e, s3[0]);
                    s3[1] = fma(xi, zi, s3[1]);
                    s3[2] = fma(zi, zi, s3[2]);
                });
        cg_cluster_sum(s3, red, parity, cluster, csize);
        rnorm = sqrt(s3[0]);
        zeta = job.shift + 1.0 / s3[1];
        const double scale = 1.0 / sqrt(s3[2]);
        for (std::uint32_t i = r0 + threadIdx.x; i < r1; i += kCgThreads) x[i] = scale * z[i];
    }
    if (rank == 0 && threadIdx.x == 0) {
        vgpu_cg_result res;
        res.zeta = zeta;
        res.rnorm = rnorm;
        res.niter = job.niter;
        res.n = n;
        res.nnz = job.nnz;
        *job.out = res;
    }
    // no CTA may exit while a peer can still read its shared memory
    cluster.sync();
}

}  // namespace vgk
