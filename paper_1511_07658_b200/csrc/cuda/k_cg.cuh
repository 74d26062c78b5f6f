// NAS CG payload ("nas-cg"): the timed part of NPB CG (cg.f conj_grad and
// the outer zeta loop) on the CSR matrix the SPMD program sent.
//
// No reference arithmetic exists (proj/src/bench/profiles.cpp:41 is a timing
// profile only); the algorithm is NPB 3.x CG, restated in
// oracle/vgpu_oracle.c (vo_cg_run) and pinned there to NPB's published zeta
// values for classes S, W and A.
//
// B200 design: one thread-block CLUSTER per job, one 1024-thread CTA per SM;
// the host picks the widest cluster (up to 16) at which the whole batch is
// co-resident (backend.cu cg_cluster_for). Each CTA owns a contiguous slice
// of rows. Vectors live in shared memory when they fit (classes S..A: the
// CTA's x, z, r, q slices and the whole p, new p slices PUSHED into every
// peer's copy over DSMEM), else p alone is staged there, else all stay in
// the job's HBM workspace (CgMode below); only the matrix streams from
// L2/HBM (12 B per nonzero: a f64 + colidx u32). Dot products reduce warp
// -> CTA -> cluster by one fixed shuffle tree over DSMEM partials in rank
// order, so all CTAs hold the same bits and the result repeats run to run.
// Three cluster barriers per CG step (p . q, r . r, the p update), as NPB's
// data dependences need. SpMV: row segments of 8/16/32 lanes, predicated
// load chains per lane, shuffle-tree sum (cg_spmv).
#pragma once

#include <cooperative_groups.h>
#include <cstdint>
#include <type_traits>

#include "vgpu_cuda.h"

namespace vgk {

namespace cgx = cooperative_groups;

constexpr int kCgThreads = 1024;
constexpr int kCgMaxCluster = 16;     // CTAs per job at most (non-portable size)
constexpr int kMaxCgJobs = 16;
constexpr int kCgMaxGridCtas = 32;  // CTAs per job in the grid variant (warp-0 reduction)
constexpr std::uint32_t kCgStageMax = 24576;  // rows whose p fits in shared memory (192 KiB)
constexpr std::uint32_t kCgSmemBytes = 224 * 1024;  // dynamic shared memory cap per CTA

// Group mode (kCgResident only): a job spans G clusters of the launch's
// width instead of one, so a job that would get one GPC's worth of SMs gets
// more of them (the host uses it for a launch with one large job). The
// clusters of a job exchange what crosses them through the job's HBM/L2
// workspace: each cluster's dot-product partial (one slot per group, summed
// by every CTA in group order, so all CTAs keep identical bits), each CTA's
// r slice (written before the r . r barrier, after which every CTA computes
// the whole p = r + beta p itself: no p pushes, two group barriers per CG
// step) and, once per outer iteration, z. The barrier between groups is a
// release counter per group. A job's clusters are only co-resident when nothing else holds
// the SMs, so the groups first JOIN: when all G arrive within the wait
// budget the job runs grouped; otherwise the first arrival claims the job
// and runs it alone (rows over its own cluster, the plain schedule) and the
// late clusters exit. Nothing ever waits without a bound on a cluster that
// may not be scheduled.
constexpr int kCgMaxGroups = 4;
enum CgGroupMode : unsigned { kCgGrouped = 1, kCgSolo = 2, kCgExit = 3 };

struct CgGroupSync {          // per job, zeroed before every launch
    unsigned state;           // arrivals (bits 0..15) | decision << 16 (1 grouped, 2 solo)
    unsigned pad0[31];
    unsigned seq[kCgMaxGroups];  // publish counter per group
    unsigned pad1[32 - kCgMaxGroups];
    double part[2][kCgMaxGroups][4];  // [slot][group][value]
};

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
    CgGroupSync* gsync;  // group mode only
    std::uint32_t n, nnz, niter, cgitmax;
    double shift;
};

struct CgTable {
    CgJob job[kMaxCgJobs];
    std::uint32_t njobs;
    std::uint32_t stage_n;     // doubles of staged p at the start of dynamic smem
    std::uint32_t own_rows;    // kCgResident: doubles per own vector slice after it
    std::uint32_t srow_words;  // room for a rowstr slice after them (u32 words)
    std::uint32_t groups;      // clusters per job (1: plain)
    std::uint32_t join_ns;     // group mode: how long the first arrival waits for the others
};

__device__ __forceinline__ unsigned cg_ld_acquire_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ std::uint64_t cg_globaltimer() {
    std::uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// A CTA's group-mode state, in shared memory (CTA-uniform; read only on
// the group paths, so the SpMV loop keeps its registers).
struct CgGroupCtx {
    unsigned groups, gidx, gseq;
    CgGroupSync* gs;
    double* gp;  // the workspace copies of r (every CG step) and z (every
    double* gz;  // outer iteration) that all CTAs of the job read whole
};

// One thread per cluster (rank 0, thread 0): grouped, solo or exit.
__device__ __forceinline__ unsigned cg_group_join(CgGroupSync* s, unsigned groups, unsigned join_ns) {
    const unsigned old = atomicAdd(&s->state, 1u);
    if (old >> 16) return kCgExit;  // decided without this cluster
    const std::uint64_t t0 = cg_globaltimer();
    for (;;) {
        const unsigned st = cg_ld_acquire_u32(&s->state);
        if ((st >> 16) == 1u) return kCgGrouped;
        if ((st >> 16) == 2u) return kCgExit;
        if ((st & 0xffffu) == groups) {
            if (atomicCAS(&s->state, st, st | (1u << 16)) == st) return kCgGrouped;
            continue;
        }
        if (cg_globaltimer() - t0 > join_ns) {
            if (atomicCAS(&s->state, st, st | (2u << 16)) == st) return kCgSolo;
            continue;
        }
    }
}

// After a cluster-wide barrier: the cluster's rank 0 publishes `target`
// for its group, then every CTA waits until all groups have. The barrier
// before made the whole cluster's global writes visible to rank 0; its
// fence and release store carry them to the other groups.
__device__ __forceinline__ void cg_group_barrier(CgGroupSync* s, unsigned groups, unsigned gidx,
                                                 unsigned rank, unsigned target) {
    if (threadIdx.x == 0) {
        if (rank == 0) {
            __threadfence();
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(&s->seq[gidx]), "r"(target) : "memory");
        }
        for (unsigned g = 0; g < groups; ++g)
            while (cg_ld_acquire_u32(&s->seq[g]) < target) {
            }
    }
    __syncthreads();
}

// The group steps as separate (non-inlined) functions, called at CG phase
// boundaries: inlined, their code made the scheduler interleave the SpMV's
// loads with its gathers and FMAs one chain at a time (3.6x slower).
//
// v[0..W) holds the cluster's total (identical in every CTA): the job's
// total over the groups, summed in group order (the partials are loaded at
// once, then added in that order).
template <int W>
__device__ __noinline__ void cg_group_sum_fn(CgGroupCtx* gx, double* v, unsigned rank) {
    CgGroupSync* const gs = gx->gs;
    const unsigned slot = gx->gseq & 1u, ng = gx->groups, target = gx->gseq + 1;
    if (rank == 0 && threadIdx.x == 0)
        for (int w = 0; w < W; ++w) gs->part[slot][gx->gidx][w] = v[w];
    cg_group_barrier(gs, ng, gx->gidx, rank, target);  // ends in __syncthreads
    if (threadIdx.x == 0) gx->gseq = target;
    double part[kCgMaxGroups][W];
#pragma unroll
    for (int g = 0; g < kCgMaxGroups; ++g)
#pragma unroll
        for (int w = 0; w < W; ++w) part[g][w] = g < static_cast<int>(ng) ? __ldcg(&gs->part[slot][g][w]) : 0.0;
#pragma unroll
    for (int w = 0; w < W; ++w) {
        double t = 0.0;
#pragma unroll
        for (int g = 0; g < kCgMaxGroups; ++g)
            if (g < static_cast<int>(ng)) t += part[g][w];
        v[w] = t;
    }
}

// The groups' barrier alone (after a cluster barrier that completed this
// cluster's writes to the workspace).
__device__ __noinline__ void cg_group_sync_fn(CgGroupCtx* gx, unsigned rank) {
    const unsigned target = gx->gseq + 1;
    cg_group_barrier(gx->gs, gx->groups, gx->gidx, rank, target);
    if (threadIdx.x == 0) gx->gseq = target;
    __syncthreads();
}

// ps[i] = src[i] (f == nullptr) or fma(beta, ps[i], src[i]) for the whole
// vector: the workspace -> this CTA's full copy, 16-byte loads, eight in
// flight per thread.
__device__ __noinline__ void cg_full_vector_fn(double* ps, const double* src, std::uint32_t n, bool update,
                                               double beta) {
    if ((reinterpret_cast<std::uintptr_t>(src) & 15u) == 0) {
        const double2* s2 = reinterpret_cast<const double2*>(src);
        double2* p2 = reinterpret_cast<double2*>(ps);
        const std::uint32_t n2 = n / 2;
        for (std::uint32_t i0 = threadIdx.x; i0 < n2; i0 += 8 * kCgThreads) {
            double2 t[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const std::uint32_t i = i0 + u * kCgThreads;
                if (i < n2) t[u] = __ldcg(s2 + i);
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const std::uint32_t i = i0 + u * kCgThreads;
                if (i < n2) {
                    if (update) {
                        const double2 o = p2[i];
                        t[u].x = fma(beta, o.x, t[u].x);
                        t[u].y = fma(beta, o.y, t[u].y);
                    }
                    p2[i] = t[u];
                }
            }
        }
        if ((n & 1u) && threadIdx.x == 0) ps[n - 1] = update ? fma(beta, ps[n - 1], __ldcg(src + n - 1)) : __ldcg(src + n - 1);
    } else {
        for (std::uint32_t i = threadIdx.x; i < n; i += kCgThreads)
            ps[i] = update ? fma(beta, ps[i], __ldcg(src + i)) : __ldcg(src + i);
    }
    __syncthreads();
}

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

// Sum W per-thread values over the whole cluster with one fixed tree:
// lanes -> warps (shuffle tree), warps -> CTA (warp 0, shuffle tree over the
// 32 warp partials), CTAs -> cluster (warp 0 of every CTA reads all partials
// over DSMEM and runs the same tree), so every CTA holds the same bits and
// results repeat run to run. The cluster barrier inside also orders every
// global write before it.
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
    if (warp == 0) {
#pragma unroll
        for (int w = 0; w < W; ++w) {
            const double s = cg_warp_sum(red.warp[lane][w]);
            if (lane == 0) red.slot[parity][w] = s;
        }
    }
    cluster.sync();
    if (warp == 0) {
        const double* src = lane < csize ? cluster.map_shared_rank(&red.slot[parity][0], lane) : nullptr;
        double part[W];
#pragma unroll
        for (int w = 0; w < W; ++w) part[w] = src ? src[w] : 0.0;
#pragma unroll
        for (int w = 0; w < W; ++w) {
            const double s = cg_warp_sum(part[w]);
            if (lane == 0) red.total[w] = s;
        }
    }
    __syncthreads();
#pragma unroll
    for (int w = 0; w < W; ++w) v[w] = red.total[w];
    parity ^= 1u;
}

// y[row] = sum_k a[k] * v[colidx[k]] for this CTA's rows. A row belongs to
// a segment of `seg` lanes (8, 16 or 32 by the job's nonzeros per row), so a
// warp works on 32 / seg rows at once; each lane issues kCgChains predicated
// loads of (colidx, a) at once (the SpMV is bound by memory latency x
// parallelism per SM, not by bandwidth). Row bounds come from shared memory (rs: this
// CTA's rowstr slice). The sum order is fixed by (seg, lane), so results
// are deterministic. f(row, sum) runs on the segment's first lane.

struct CgMatrix {  // the hot fields of a job, in registers
    const std::uint32_t* __restrict__ colidx;
    const double* __restrict__ a;
    std::uint32_t nm1;  // n - 1: column clamp
    std::uint32_t nnz;  // row-bound clamp
};

template <unsigned seg, unsigned kCgChains, typename Gather, typename F>
__device__ __forceinline__ void cg_spmv(const CgMatrix& m, const std::uint32_t* rs, std::uint32_t r0,
                                        std::uint32_t r1, Gather gather, F f) {
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned sl = lane & (seg - 1);
    constexpr unsigned per_warp = 32 / seg;
    const std::uint32_t nm1 = m.nm1;
    const std::uint32_t* __restrict__ colidx = m.colidx;
    const double* __restrict__ a = m.a;
    for (std::uint32_t row0 = r0 + warp * per_warp; row0 < r1; row0 += (kCgThreads / 32) * per_warp) {
        const std::uint32_t row = row0 + lane / seg;
        double acc[kCgChains];
#pragma unroll
        for (unsigned c = 0; c < kCgChains; ++c) acc[c] = 0.0;
        if (row < r1) {
            // a malformed rowstr (only its ends are checked on the host)
            // cannot send the loads outside the matrix
            const std::uint32_t k1 = min(rs[row - r0 + 1], m.nnz);
            for (std::uint32_t k = rs[row - r0] + sl; k < k1; k += kCgChains * seg) {
                std::uint32_t col[kCgChains];
                double av[kCgChains];
                // one 64-bit address per array and iteration; the chains
                // are immediate offsets from it (a 32-bit k + c * seg per
                // chain cost a wide multiply-add and a register pair each)
                const std::uint32_t* __restrict__ pc = colidx + k;
                const double* __restrict__ pa = a + k;
#pragma unroll
                for (unsigned c = 0; c < kCgChains; ++c) {
                    const bool in = k + c * seg < k1;
                    // malformed column indices are clamped into bounds
                    col[c] = in ? min(__ldg(pc + c * seg), nm1) : 0u;
                    av[c] = in ? __ldg(pa + c * seg) : 0.0;
                }
#pragma unroll
                for (unsigned c = 0; c < kCgChains; ++c) acc[c] = fma(av[c], gather(col[c]), acc[c]);
            }
        }
        // fixed pairwise order over the chains
#pragma unroll
        for (unsigned w = kCgChains / 2; w > 0; w /= 2)
#pragma unroll
            for (unsigned c = 0; c < w; ++c) acc[c] += acc[c + w];
        double s = acc[0];
#pragma unroll
        for (unsigned o = seg / 2; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o, seg);
        if (sl == 0 && row < r1) f(row, s);
    }
}

// Lanes per row segment for a job (measured on B200: S, W and A all run
// best at 16 with four chains per lane).
__host__ __device__ __forceinline__ unsigned cg_segment(std::uint32_t n, std::uint32_t nnz) {
    const std::uint32_t per_row = nnz / (n ? n : 1);
    return per_row >= 256 ? 32u : per_row >= 40 ? 16u : 8u;
}

// Vector placement (kMode, chosen per launch on the host by what fits in
// shared memory):
//   kCgGlobal    all vectors in the job's HBM workspace; p gathered via L2
//   kCgStaged    p re-staged into shared memory after every update
//   kCgResident  everything in shared memory: this CTA's x, z, r, q slices,
//                the whole p; each CTA PUSHES its new p slice into every
//                peer's copy over DSMEM (st.shared::cluster) and the cluster
//                barrier that NPB's dependences need anyway publishes it, so
//                no staging pass and no HBM round trip for vectors at all
//                (classes S..A at the widths the batch allows).
enum CgMode { kCgGlobal = 0, kCgStaged = 1, kCgResident = 2 };

// The CG body of one CTA: kG = the grouped row split (G clusters per job,
// this cluster group gidx), else the plain one (the job over this cluster).
template <int kMode, unsigned kSeg, bool kG>
__device__ __forceinline__ void cg_body(const CgTable& table, unsigned jid, unsigned gidx_in, unsigned G) {
    // dynamic shared memory: p (stage_n doubles) | x z r q slices (own_rows
    // doubles each, kCgResident) | this CTA's rowstr slice (srow_words)
    extern __shared__ double ps[];
    __shared__ CgReduce red;
    __shared__ CgGroupCtx gx;  // group mode only
    cgx::cluster_group cluster = cgx::this_cluster();
    const unsigned csize = cluster.num_blocks();
    const unsigned rank = cluster.block_rank();
    const CgJob& job = table.job[jid];
    const std::uint32_t n = job.n;
    const unsigned groups = kG ? G : 1u, gidx = kG ? gidx_in : 0u;
    const std::uint32_t parts = groups * csize, part = gidx * csize + rank;
    const std::uint32_t r0 = static_cast<std::uint32_t>((static_cast<std::uint64_t>(n) * part) / parts);
    const std::uint32_t r1 = static_cast<std::uint32_t>((static_cast<std::uint64_t>(n) * (part + 1)) / parts);
    if (kG && threadIdx.x == 0) {
        // this cluster's rows (the rest of p / z arrives through the workspace)
        gx.groups = groups;
        gx.gidx = gidx;
        gx.gseq = 0;  // group barriers passed
        gx.gs = job.gsync;
        gx.gp = job.p;
        gx.gz = job.z;
    }
    unsigned parity = 0;
    const CgMatrix mat{job.colidx, job.a, n - 1, job.nnz};
    constexpr bool kStage = kMode != kCgGlobal;
    constexpr bool kRes = kMode == kCgResident;
    // load chains per lane (measured on B200: 4 beats 8 at every class,
    // even where 8 fit the 64-register budget without spilling)
    constexpr unsigned kChains = 4;
    const std::uint32_t own = kRes ? table.own_rows : 0;
    double* const own0 = ps + (kStage ? table.stage_n : 0);
    std::uint32_t* const srow = reinterpret_cast<std::uint32_t*>(own0 + 4ull * own);
    const bool rs_smem = r1 - r0 + 1 <= table.srow_words;
    if (rs_smem)
        for (std::uint32_t i = threadIdx.x; i <= r1 - r0; i += kCgThreads) srow[i] = __ldg(job.rowstr + r0 + i);
    const std::uint32_t* const rs = rs_smem ? srow : job.rowstr + r0;
    // every CTA of the cluster must be running before anyone writes into its
    // shared memory (the first p push below); also orders the srow loads
    cluster.sync();
    // vector element of global row i: own slices rebased to r0 when resident
    double* const x = kRes ? own0 - r0 : job.x;
    double* const z = kRes ? own0 + own - r0 : job.z;
    double* const r = kRes ? own0 + 2ull * own - r0 : job.r;
    double* const q = kRes ? own0 + 3ull * own - r0 : job.q;
    double* const p = kRes ? ps : job.p;  // own rows of p (resident: the local full copy)

    // whole p into shared memory: 16-byte loads, two in flight per thread
    auto stage_p = [&]() {
        if constexpr (kMode == kCgStaged) {
            const double2* p2 = reinterpret_cast<const double2*>(job.p);
            double2* s2 = reinterpret_cast<double2*>(ps);
            const std::uint32_t n2 = n / 2;
            for (std::uint32_t i0 = threadIdx.x; i0 < n2; i0 += 2 * kCgThreads) {
                double2 t[2];
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const std::uint32_t i = i0 + u * kCgThreads;
                    if (i < n2) t[u] = __ldcg(p2 + i);
                }
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const std::uint32_t i = i0 + u * kCgThreads;
                    if (i < n2) s2[i] = t[u];
                }
            }
            if ((n & 1u) && threadIdx.x == 0) ps[n - 1] = __ldcg(job.p + n - 1);
            __syncthreads();
        }
    };
    auto gather_p = [&](std::uint32_t c) -> double {
        if constexpr (kStage) return ps[c];
        else return __ldcg(job.p + c);
    };
    // resident: element i of the full vector in every CTA's copy (own too).
    // Group mode never pushes: every CTA computes the whole p itself from
    // the full r the groups publish (below).
    auto push = [&](std::uint32_t i, double v) {
        if constexpr (kRes) {
            for (unsigned c = 0; c < csize; ++c) cluster.map_shared_rank(ps, c)[i] = v;
        } else {
            p[i] = v;
        }
    };
    // dot product over the job: the cluster's fixed tree, then (group mode)
    // the clusters' partials in group order, the same bits in every CTA
    auto job_sum = [&](auto& v) {
        cg_cluster_sum(v, red, parity, cluster, csize);
        if constexpr (kG) cg_group_sum_fn<sizeof(v) / sizeof(double)>(&gx, v, rank);
    };

    for (std::uint32_t i = r0 + threadIdx.x; i < r1; i += kCgThreads) x[i] = 1.0;
    double zeta = 0.0, rnorm = 0.0, scale = 1.0;
    const std::uint32_t niter = job.niter, cgitmax = job.cgitmax;
    for (std::uint32_t it = 0; it < niter; ++it) {
        // conj_grad: q = z = 0, r = p = x, rho = r . r
        double v1[1] = {0.0};
        if constexpr (kG) {
            // p = x over the whole vector, from what every CTA holds: x = 1
            // at first, then scale * z (the full z the residual gathered)
            for (std::uint32_t i = threadIdx.x; i < n; i += kCgThreads) ps[i] = it == 0 ? 1.0 : scale * ps[i];
        }
        for (std::uint32_t i = r0 + threadIdx.x; i < r1; i += kCgThreads) {
            const double xi = x[i];
            z[i] = 0.0;
            r[i] = xi;
            if constexpr (!kG) push(i, xi);
            v1[0] = fma(xi, xi, v1[0]);
        }
        job_sum(v1);  // also publishes p (and orders the group-mode p writes)
        double rho = v1[0];
        stage_p();
        for (std::uint32_t cgit = 0; cgit < cgitmax; ++cgit) {
            // q = A p, d = p . q
            double d[1] = {0.0};
            cg_spmv<kSeg, kChains>(mat, rs, r0, r1, gather_p, [&](std::uint32_t row, double s) {
                q[row] = s;
                d[0] = fma(gather_p(row), s, d[0]);
            });
            job_sum(d);
            const double alpha = rho / d[0];
            const double rho0 = rho;
            // z += alpha p, r -= alpha q, rho = r . r
            double rr[1] = {0.0};
            for (std::uint32_t i = r0 + threadIdx.x; i < r1; i += kCgThreads) {
                const double pi = p[i];
                z[i] = fma(alpha, pi, z[i]);
                const double ri = fma(-alpha, q[i], r[i]);
                r[i] = ri;
                if constexpr (kG) gx.gp[i] = ri;  // the groups' copy of r
                rr[0] = fma(ri, ri, rr[0]);
            }
            job_sum(rr);  // group mode: its barrier also publishes r
            rho = rr[0];
            const double beta = rho / rho0;
            if constexpr (kG) {
                // p = r + beta p over the whole vector in every CTA (the same
                // bits as the owner's), no push and no barrier of its own
                cg_full_vector_fn(ps, gx.gp, n, true, beta);
            } else {
                for (std::uint32_t i = r0 + threadIdx.x; i < r1; i += kCgThreads) push(i, fma(beta, p[i], r[i]));
                cluster.sync();  // p complete before anyone gathers it
            }
            stage_p();
        }
        // ||x - A z||, x . z, z . z: the residual SpMV gathers z — resident:
        // pushed into every CTA's (now unused) p copy; else from HBM
        if constexpr (kG) {
            // z to the workspace, the groups' barrier, the whole z back
            for (std::uint32_t i = r0 + threadIdx.x; i < r1; i += kCgThreads) gx.gz[i] = z[i];
            cluster.sync();
            cg_group_sync_fn(&gx, rank);
            cg_full_vector_fn(ps, gx.gz, n, false, 0.0);
        } else if constexpr (kRes) {
            for (std::uint32_t i = r0 + threadIdx.x; i < r1; i += kCgThreads) push(i, z[i]);
            cluster.sync();
        }
        double s3[3] = {0.0, 0.0, 0.0};
        cg_spmv<kSeg, kChains>(mat, rs, r0, r1,
                      [&](std::uint32_t c) {
                          if constexpr (kRes) return ps[c];
                          else return __ldcg(job.z + c);
                      },
                      [&](std::uint32_t row, double s) {
                          const double xi = x[row], zi = z[row];
                          const double e = xi - s;
                          s3[0] = fma(e, e, s3[0]);
                          s3[1] = fma(xi, zi, s3[1]);
                          s3[2] = fma(zi, zi, s3[2]);
                      });
        job_sum(s3);
        rnorm = sqrt(s3[0]);
        zeta = job.shift + 1.0 / s3[1];
        scale = 1.0 / sqrt(s3[2]);
        for (std::uint32_t i = r0 + threadIdx.x; i < r1; i += kCgThreads) x[i] = scale * z[i];
    }
    if (gidx == 0 && rank == 0 && threadIdx.x == 0) {
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

// The group-mode instance runs its body as a separate function: inlined
// after the join (atomics, a timed spin, cluster barriers), the scheduler
// interleaved the SpMV's loads with its gathers and FMAs one chain at a time
// instead of issuing all chains' loads first.
template <int kMode, unsigned kSeg, bool kG>
__device__ __noinline__ void cg_body_call(const CgTable& table, unsigned jid, unsigned gidx, unsigned G) {
    cg_body<kMode, kSeg, kG>(table, jid, gidx, G);
}

// kGroups: the group-mode instance (kCgResident only); the plain instance
// compiles without any of its code, so the SpMV keeps its registers
template <int kMode, unsigned kSeg, bool kGroups = false>
__global__ void __launch_bounds__(kCgThreads, 1) cg_kernel(const __grid_constant__ CgTable table) {
    static_assert(!kGroups || kMode == kCgResident, "group mode needs the resident placement");
    cgx::cluster_group cluster = cgx::this_cluster();
    const unsigned csize = cluster.num_blocks();
    const unsigned cid = blockIdx.x / csize;
    if constexpr (!kGroups) {
        cg_body<kMode, kSeg, false>(table, cid, 0, 1);
    } else {
        const unsigned G = table.groups;
        const unsigned jid = G == 1 ? cid : G == 2 ? cid >> 1 : G == 4 ? cid >> 2 : cid / 3u;
        const CgJob& job = table.job[jid];
        const unsigned rank = cluster.block_rank();
        // join the job's other clusters, or run it alone, or leave
        __shared__ unsigned s_mode;
        if (rank == 0 && threadIdx.x == 0) s_mode = G > 1 ? cg_group_join(job.gsync, G, table.join_ns) : kCgSolo;
        cluster.sync();
        const unsigned m = *cluster.map_shared_rank(&s_mode, 0);
        cluster.sync();  // rank 0's word is read before any CTA leaves
        if (m == kCgExit) return;
        if (m == kCgGrouped) cg_body_call<kMode, kSeg, true>(table, jid, cid - jid * G, G);
        else cg_body_call<kMode, kSeg, false>(table, jid, 0, 1);
    }
}

// ---- grid variant: a job spans plain CTAs on any SMs ------------------------
// Clusters live inside one GPC (16-CTA clusters: 7 co-resident on a B200),
// so a batch of 8 class-A jobs gets only 80 SMs as clusters. The grid
// variant gives each job an equal share of ALL SMs (one 1024-thread CTA per
// SM, the launch co-resident by construction: cooperative launch) and
// replaces the cluster barrier and DSMEM with a global-memory barrier and
// partials in L2; p is re-staged into shared memory from L2 after every
// update (n <= kCgStageMax). Same arithmetic, same fixed reduction trees
// (CTA partials summed in CTA order), so results are deterministic too.

struct CgGridSync {            // per job, zeroed before every launch
    unsigned count;
    unsigned gen;
    unsigned pad[2];
    double part[2][kCgMaxGridCtas][4];  // [parity][cta][value]
};

struct CgGridTable {
    CgJob job[kMaxCgJobs];
    CgGridSync* sync[kMaxCgJobs];
    std::uint32_t njobs;
    std::uint32_t ctas_per_job;
    std::uint32_t srow_words;
};

__device__ __forceinline__ unsigned cg_ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// barrier over the job's CTAs (generation counting); orders global memory
__device__ __forceinline__ void cg_grid_barrier(CgGridSync* sy, unsigned nctas, unsigned& gen) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned g = gen;
        __threadfence();
        if (atomicAdd(&sy->count, 1u) == nctas - 1) {
            sy->count = 0;
            __threadfence();
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(&sy->gen), "r"(g + 1) : "memory");
        } else {
            while (cg_ld_acquire(&sy->gen) == g) {
            }
        }
    }
    gen += 1;
    __syncthreads();
}

template <int W>
__device__ __forceinline__ void cg_grid_sum(double (&v)[W], CgReduce& red, unsigned& parity, CgGridSync* sy,
                                            unsigned cta, unsigned nctas, unsigned& gen) {
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int w = 0; w < W; ++w) {
        const double s = cg_warp_sum(v[w]);
        if (lane == 0) red.warp[warp][w] = s;
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int w = 0; w < W; ++w) {
            const double s = cg_warp_sum(red.warp[lane][w]);
            if (lane == 0) sy->part[parity][cta][w] = s;
        }
    }
    cg_grid_barrier(sy, nctas, gen);
    if (warp == 0) {
        double part[W];
#pragma unroll
        for (int w = 0; w < W; ++w) part[w] = lane < nctas ? __ldcg(&sy->part[parity][lane][w]) : 0.0;
#pragma unroll
        for (int w = 0; w < W; ++w) {
            const double s = cg_warp_sum(part[w]);
            if (lane == 0) red.total[w] = s;
        }
    }
    __syncthreads();
#pragma unroll
    for (int w = 0; w < W; ++w) v[w] = red.total[w];
    parity ^= 1u;
}

template <unsigned kSeg>
__global__ void __launch_bounds__(kCgThreads, 1) cg_grid_kernel(const __grid_constant__ CgGridTable table) {
    extern __shared__ double ps[];  // p (n doubles) | rowstr slice
    __shared__ CgReduce red;
    const unsigned nctas = table.ctas_per_job;
    const unsigned jid = blockIdx.x / nctas, cta = blockIdx.x % nctas;
    const CgJob& job = table.job[jid];
    CgGridSync* const sy = table.sync[jid];
    const std::uint32_t n = job.n;
    const std::uint32_t r0 = static_cast<std::uint32_t>((static_cast<std::uint64_t>(n) * cta) / nctas);
    const std::uint32_t r1 = static_cast<std::uint32_t>((static_cast<std::uint64_t>(n) * (cta + 1)) / nctas);
    unsigned parity = 0, gen = 0;
    const CgMatrix mat{job.colidx, job.a, n - 1, job.nnz};
    std::uint32_t* const srow = reinterpret_cast<std::uint32_t*>(ps + n);
    const bool rs_smem = r1 - r0 + 1 <= table.srow_words;
    if (rs_smem)
        for (std::uint32_t i = threadIdx.x; i <= r1 - r0; i += kCgThreads) srow[i] = __ldg(job.rowstr + r0 + i);
    const std::uint32_t* const rs = rs_smem ? srow : job.rowstr + r0;
    __syncthreads();
    double* const x = job.x;
    double* const z = job.z;
    double* const p = job.p;
    double* const q = job.q;
    double* const r = job.r;
    auto stage = [&](const double* src) {
        const double2* s2 = reinterpret_cast<const double2*>(src);
        double2* d2 = reinterpret_cast<double2*>(ps);
        const std::uint32_t n2 = n / 2;
        for (std::uint32_t i0 = threadIdx.x; i0 < n2; i0 += 2 * kCgThreads) {
            double2 t[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const std::uint32_t i = i0 + u * kCgThreads;
                if (i < n2) t[u] = __ldcg(s2 + i);
            }
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const std::uint32_t i = i0 + u * kCgThreads;
                if (i < n2) d2[i] = t[u];
            }
        }
        if ((n & 1u) && threadIdx.x == 0) ps[n - 1] = __ldcg(src + n - 1);
        __syncthreads();
    };
    auto gather = [&](std::uint32_t c) -> double { return ps[c]; };

    for (std::uint32_t i = r0 + threadIdx.x; i < r1; i += kCgThreads) x[i] = 1.0;
    double zeta = 0.0, rnorm = 0.0;
    const std::uint32_t niter = job.niter, cgitmax = job.cgitmax;
    for (std::uint32_t it = 0; it < niter; ++it) {
        double v1[1] = {0.0};
        for (std::uint32_t i = r0 + threadIdx.x; i < r1; i += kCgThreads) {
            const double xi = x[i];
            z[i] = 0.0;
            r[i] = xi;
            p[i] = xi;
            v1[0] = fma(xi, xi, v1[0]);
        }
        cg_grid_sum(v1, red, parity, sy, cta, nctas, gen);  // also publishes p
        double rho = v1[0];
        stage(p);
        for (std::uint32_t cgit = 0; cgit < cgitmax; ++cgit) {
            double d[1] = {0.0};
            cg_spmv<kSeg, 4>(mat, rs, r0, r1, gather, [&](std::uint32_t row, double s) {
                q[row] = s;
                d[0] = fma(ps[row], s, d[0]);
            });
            cg_grid_sum(d, red, parity, sy, cta, nctas, gen);
            const double alpha = rho / d[0];
            const double rho0 = rho;
            double rr[1] = {0.0};
            for (std::uint32_t i = r0 + threadIdx.x; i < r1; i += kCgThreads) {
                z[i] = fma(alpha, ps[i], z[i]);
                const double ri = fma(-alpha, q[i], r[i]);
                r[i] = ri;
                rr[0] = fma(ri, ri, rr[0]);
            }
            cg_grid_sum(rr, red, parity, sy, cta, nctas, gen);
            rho = rr[0];
            const double beta = rho / rho0;
            for (std::uint32_t i = r0 + threadIdx.x; i < r1; i += kCgThreads) p[i] = fma(beta, ps[i], r[i]);
            cg_grid_barrier(sy, nctas, gen);  // p complete before anyone stages it
            stage(p);
        }
        stage(z);  // the residual gathers z (complete since the last barriers)
        double s3[3] = {0.0, 0.0, 0.0};
        cg_spmv<kSeg, 4>(mat, rs, r0, r1, gather, [&](std::uint32_t row, double s) {
            const double xi = x[row], zi = z[row];
            const double e = xi - s;
            s3[0] = fma(e, e, s3[0]);
            s3[1] = fma(xi, zi, s3[1]);
            s3[2] = fma(zi, zi, s3[2]);
        });
        cg_grid_sum(s3, red, parity, sy, cta, nctas, gen);
        rnorm = sqrt(s3[0]);
        zeta = job.shift + 1.0 / s3[1];
        const double scale = 1.0 / sqrt(s3[2]);
        for (std::uint32_t i = r0 + threadIdx.x; i < r1; i += kCgThreads) x[i] = scale * z[i];
    }
    if (cta == 0 && threadIdx.x == 0) {
        vgpu_cg_result res;
        res.zeta = zeta;
        res.rnorm = rnorm;
        res.niter = job.niter;
        res.n = n;
        res.nnz = job.nnz;
        *job.out = res;
    }
}

}  // namespace vgk
