// NAS MG payload ("nas-mg"): the timed part of NPB 3.x MG (mg.f) — nit
// V-cycles of the 3-D periodic Poisson problem on an nx^3 grid — the
// paper's MG benchmark (class S: 32^3, 4 iterations; no
// reference kernel: proj/src/bench/profiles.cpp:37 is a timing profile).
//
// Every grid operator of mg.f (resid, psinv, rprj3, interp, comm3, zero3)
// is a per-point device function. Two schedules run them: for small grids
// (nx <= 64) mg_cluster_kernel, one thread-block cluster per job running
// the whole timed sequence in one launch (comm3 / zero3 fused into the
// writing operator, coarse levels on one CTA; below); for larger grids one
// launch per operator over all jobs of a batch (blockIdx.y = job), one
// thread per output point, with comm3 as a separate pass. Each point
// evaluates mg.f's expression in its order with explicitly rounded binary64
// operations (__dadd_rn / __dsub_rn / __dmul_rn: no FMA contraction), the
// order the oracle restates (oracle/vgpu_oracle.c vo_mg_run), so both
// schedules match the oracle bit for bit. In the per-operator schedule the
// ghost layer (comm3) is a separate pass over the six faces: an in-place
// resid (r = r - A u on the coarse levels) reads its own point only, so a
// thread may overwrite its point, but filling a ghost from the wrapped
// interior inside the same pass would race with that point's thread (the
// fused form writes each ghost from the thread that owns its interior
// mirror instead). norm2u3 is a fixed-order reduction shared with the oracle: per
// i3 plane, lane l of 256 sums the plane's points l, l + 256, ... in order,
// the lanes combine by the stride-doubling tree (warp shuffles, then the 8
// warp sums), the planes add in i3 order.
//
// Layout per job (its slot workspace): for k = 1..lt, u_k then r_k, each
// (2^k + 2)^3 doubles, i1 fastest (Fortran order, ghosts at 1 and n); then
// the norm's per-plane sums and maxima. v stays in the input buffer, the
// interior only.
#pragma once

#include <cstdint>

#include "vgpu_cuda.h"

namespace vgk {

constexpr int kMgThreads = 256;
constexpr int kMaxMgJobs = 16;
constexpr int kMgMaxLevels = 10;  // nx <= 512

struct MgJob {
    const double* v;                 // nx^3 interior values (input buffer)
    double* u[kMgMaxLevels + 1];     // [k], k = 1..lt
    double* r[kMgMaxLevels + 1];
    double* plane_sum;               // nx
    double* plane_max;               // nx
    vgpu_mg_result* out;
};

struct MgTable {
    MgJob job[kMaxMgJobs];
    std::uint32_t njobs, nx, lt, nit;
    double a[4], c[4];
};

__device__ __forceinline__ std::size_t mg_idx(int n, int i1, int i2, int i3) {
    return static_cast<std::size_t>(i1 - 1) +
           static_cast<std::size_t>(n) * (static_cast<std::size_t>(i2 - 1) +
                                          static_cast<std::size_t>(n) * static_cast<std::size_t>(i3 - 1));
}

// interior point number p (0-based) of an m^3 interior -> 1-based coords 2..m+1
__device__ __forceinline__ void mg_interior(std::uint64_t p, int m, int* i1, int* i2, int* i3) {
    // m is a power of two and p < 2^32 (nx <= 512): shifts, no 64-bit division
    const std::uint32_t q = static_cast<std::uint32_t>(p), lg = __ffs(m) - 1, mask = m - 1;
    *i1 = 2 + static_cast<int>(q & mask);
    *i2 = 2 + static_cast<int>((q >> lg) & mask);
    *i3 = 2 + static_cast<int>(q >> (2 * lg));
}

__device__ __forceinline__ double add4(double a, double b, double c, double d) {
    return __dadd_rn(__dadd_rn(__dadd_rn(a, b), c), d);
}

// all points of u_k (or r_k) = 0
__device__ __forceinline__ void mg_zero(const MgTable& t, const MgJob& j, int k,
                                                             int which,
        std::uint64_t p0, std::uint64_t ps) {
    const int n = (1 << k) + 2;
    const std::uint64_t total = static_cast<std::uint64_t>(n) * n * n;
    double* a = which ? j.r[k] : j.u[k];
    for (std::uint64_t p = p0; p < total; p += ps)
        a[p] = 0.0;
}

// comm3: the ghost layer of u_k / r_k from the wrapped interior (the serial
// comm3's three sweeps end with exactly these copies, corners included)
__device__ __forceinline__ void mg_comm3(const MgTable& t, const MgJob& j, int k,
                                                              int which,
        std::uint64_t p0, std::uint64_t ps) {
    const int n = (1 << k) + 2;
    double* a = which ? j.r[k] : j.u[k];
    const std::uint64_t face = static_cast<std::uint64_t>(n) * n;
    for (std::uint64_t p = p0; p < 6 * face; p += ps) {
        // 32-bit index arithmetic (6 n^2 < 2^32)
        const std::uint32_t q = static_cast<std::uint32_t>(p), fc = static_cast<std::uint32_t>(face);
        const int f = static_cast<int>(q / fc);
        const std::uint32_t in_face = q - static_cast<std::uint32_t>(f) * fc;
        const int y = 1 + static_cast<int>(in_face / static_cast<std::uint32_t>(n));
        const int x = 1 + static_cast<int>(in_face - static_cast<std::uint32_t>(y - 1) * n);
        int c[3];
        c[f >> 1] = (f & 1) ? n : 1;
        c[(f >> 1) == 0 ? 1 : 0] = x;
        c[(f >> 1) == 2 ? 1 : 2] = y;
        auto wrap = [n](int i) { return i == 1 ? n - 1 : (i == n ? 2 : i); };
        a[mg_idx(n, c[0], c[1], c[2])] = a[mg_idx(n, wrap(c[0]), wrap(c[1]), wrap(c[2]))];
    }
}

// Store an interior point (coordinates 2..n-1) and, with Ghosts, every ghost
// point comm3 would copy from it: along each axis, interior n-1 is also
// ghost 1 and interior 2 is also ghost n, so a point has up to 7 mirrors
// (comm3's three sweeps end with exactly these copies, corners included).
// The fused operators below need no separate comm3 pass: no operator reads
// the ghosts of the grid it writes.
template <bool Ghosts>
__device__ __forceinline__ void mg_store(double* a, int n, int i1, int i2, int i3, double val) {
    a[mg_idx(n, i1, i2, i3)] = val;
    if constexpr (Ghosts) {
        const int g1 = i1 == n - 1 ? 1 : (i1 == 2 ? n : 0);
        const int g2 = i2 == n - 1 ? 1 : (i2 == 2 ? n : 0);
        const int g3 = i3 == n - 1 ? 1 : (i3 == 2 ? n : 0);
        if (g1) a[mg_idx(n, g1, i2, i3)] = val;
        if (g2) a[mg_idx(n, i1, g2, i3)] = val;
        if (g3) a[mg_idx(n, i1, i2, g3)] = val;
        if (g1 && g2) a[mg_idx(n, g1, g2, i3)] = val;
        if (g1 && g3) a[mg_idx(n, g1, i2, g3)] = val;
        if (g2 && g3) a[mg_idx(n, i1, g2, g3)] = val;
        if (g1 && g2 && g3) a[mg_idx(n, g1, g2, g3)] = val;
    }
}

// resid: r_k = v - A u_k on the interior. top: v is the job's input
// (interior-only layout); else v is r_k itself (in place: each thread reads
// and writes only its own point of r_k).
template <bool Ghosts = false>
__device__ __forceinline__ void mg_resid(const MgTable& t, const MgJob& j, int k, int top,
                                         std::uint64_t p0, std::uint64_t ps) {
    const int m = 1 << k, n = m + 2;
    const std::uint64_t total = static_cast<std::uint64_t>(m) * m * m;
    const double* __restrict__ u = j.u[k];
    double* r = j.r[k];
    const double a0 = t.a[0], a2 = t.a[2], a3 = t.a[3];
    for (std::uint64_t p = p0; p < total; p += ps) {
        int i1, i2, i3;
        mg_interior(p, m, &i1, &i2, &i3);
        auto U = [&](int x, int y, int z) { return u[mg_idx(n, x, y, z)]; };
        auto u1 = [&](int x) { return add4(U(x, i2 - 1, i3), U(x, i2 + 1, i3), U(x, i2, i3 - 1), U(x, i2, i3 + 1)); };
        auto u2 = [&](int x) {
            return add4(U(x, i2 - 1, i3 - 1), U(x, i2 + 1, i3 - 1), U(x, i2 - 1, i3 + 1), U(x, i2 + 1, i3 + 1));
        };
        const double v = top ? j.v[p] : r[mg_idx(n, i1, i2, i3)];
        const double s1 = __dsub_rn(v, __dmul_rn(a0, U(i1, i2, i3)));
        const double s2 = __dsub_rn(s1, __dmul_rn(a2, __dadd_rn(__dadd_rn(u2(i1), u1(i1 - 1)), u1(i1 + 1))));
        mg_store<Ghosts>(r, n, i1, i2, i3, __dsub_rn(s2, __dmul_rn(a3, __dadd_rn(u2(i1 - 1), u2(i1 + 1)))));
    }
}

// psinv: u_k = u_k + C r_k on the interior (Fresh: u_k was just zeroed, so
// its value is the literal 0.0 in the same addition)
template <bool Ghosts = false, bool Fresh = false>
__device__ __forceinline__ void mg_psinv(const MgTable& t, const MgJob& j, int k,
                                         std::uint64_t p0, std::uint64_t ps) {
    const int m = 1 << k, n = m + 2;
    const std::uint64_t total = static_cast<std::uint64_t>(m) * m * m;
    const double* __restrict__ r = j.r[k];
    double* u = j.u[k];
    const double c0 = t.c[0], c1 = t.c[1], c2 = t.c[2];
    for (std::uint64_t p = p0; p < total; p += ps) {
        int i1, i2, i3;
        mg_interior(p, m, &i1, &i2, &i3);
        auto R = [&](int x, int y, int z) { return r[mg_idx(n, x, y, z)]; };
        auto r1 = [&](int x) { return add4(R(x, i2 - 1, i3), R(x, i2 + 1, i3), R(x, i2, i3 - 1), R(x, i2, i3 + 1)); };
        auto r2 = [&](int x) {
            return add4(R(x, i2 - 1, i3 - 1), R(x, i2 + 1, i3 - 1), R(x, i2 - 1, i3 + 1), R(x, i2 + 1, i3 + 1));
        };
        const double u0 = Fresh ? 0.0 : u[mg_idx(n, i1, i2, i3)];
        const double s1 = __dadd_rn(u0, __dmul_rn(c0, R(i1, i2, i3)));
        const double s2 =
            __dadd_rn(s1, __dmul_rn(c1, __dadd_rn(__dadd_rn(R(i1 - 1, i2, i3), R(i1 + 1, i2, i3)), r1(i1))));
        mg_store<Ghosts>(u, n, i1, i2, i3,
                         __dadd_rn(s2, __dmul_rn(c2, __dadd_rn(__dadd_rn(r2(i1), r1(i1 - 1)), r1(i1 + 1)))));
    }
}

// rprj3: r_{k-1} (coarse interior) = restriction of r_k
template <bool Ghosts = false>
__device__ __forceinline__ void mg_rprj3(const MgTable& t, const MgJob& j, int k,
                                         std::uint64_t p0, std::uint64_t ps) {
    const int mf = 1 << k, nf = mf + 2, mc = mf / 2, nc = mc + 2;
    const std::uint64_t total = static_cast<std::uint64_t>(mc) * mc * mc;
    const double* __restrict__ r = j.r[k];
    double* s = j.r[k - 1];
    for (std::uint64_t p = p0; p < total; p += ps) {
        int j1, j2, j3;
        mg_interior(p, mc, &j1, &j2, &j3);
        const int i1 = 2 * j1 - 1, i2 = 2 * j2 - 1, i3 = 2 * j3 - 1;
        auto R = [&](int x, int y, int z) { return r[mg_idx(nf, x, y, z)]; };
        auto x1 = [&](int x) { return add4(R(x, i2 - 1, i3), R(x, i2 + 1, i3), R(x, i2, i3 - 1), R(x, i2, i3 + 1)); };
        auto y1 = [&](int x) {
            return add4(R(x, i2 - 1, i3 - 1), R(x, i2 - 1, i3 + 1), R(x, i2 + 1, i3 - 1), R(x, i2 + 1, i3 + 1));
        };
        const double y2 = y1(i1);
        const double x2 = x1(i1);
        const double t1 = __dmul_rn(0.5, R(i1, i2, i3));
        const double t2 = __dmul_rn(0.25, __dadd_rn(__dadd_rn(R(i1 - 1, i2, i3), R(i1 + 1, i2, i3)), x2));
        const double t3 = __dmul_rn(0.125, __dadd_rn(__dadd_rn(x1(i1 - 1), x1(i1 + 1)), y2));
        const double t4 = __dmul_rn(0.0625, __dadd_rn(y1(i1 - 1), y1(i1 + 1)));
        mg_store<Ghosts>(s, nc, j1, j2, j3, __dadd_rn(__dadd_rn(__dadd_rn(t1, t2), t3), t4));
    }
}

// interp: u_k (every point, ghosts included) += prolongation of u_{k-1};
// each fine point takes exactly one term of mg.f's interp loops
template <bool Fresh = false>
__device__ __forceinline__ void mg_interp(const MgTable& t, const MgJob& j, int k,
                                          std::uint64_t p0, std::uint64_t ps) {
    const int nf = (1 << k) + 2, mm = (1 << (k - 1)) + 2;
    const std::uint64_t total = static_cast<std::uint64_t>(nf) * nf * nf;
    const double* __restrict__ z = j.u[k - 1];
    double* u = j.u[k];
    for (std::uint64_t p = p0; p < total; p += ps) {
        // 32-bit index arithmetic (nf^3 < 2^32)
        const std::uint32_t q = static_cast<std::uint32_t>(p), un = static_cast<std::uint32_t>(nf);
        const std::uint32_t q1 = q / un, q2 = q1 / un;
        const int f1 = 1 + static_cast<int>(q - q1 * un), f2 = 1 + static_cast<int>(q1 - q2 * un),
                  f3 = 1 + static_cast<int>(q2);
        const int i1 = (f1 + 1) / 2, i2 = (f2 + 1) / 2, i3 = (f3 + 1) / 2;
        const bool e1 = !(f1 & 1), e2 = !(f2 & 1), e3 = !(f3 & 1);
        auto Z = [&](int x, int y, int zz) { return z[mg_idx(mm, x, y, zz)]; };
        auto z1 = [&](int x) { return __dadd_rn(Z(x, i2 + 1, i3), Z(x, i2, i3)); };
        auto z2 = [&](int x) { return __dadd_rn(Z(x, i2, i3 + 1), Z(x, i2, i3)); };
        auto z3 = [&](int x) { return __dadd_rn(__dadd_rn(Z(x, i2 + 1, i3 + 1), Z(x, i2, i3 + 1)), z1(x)); };
        double v;
        if (!e2 && !e3) v = e1 ? __dmul_rn(0.5, __dadd_rn(Z(i1 + 1, i2, i3), Z(i1, i2, i3))) : Z(i1, i2, i3);
        else if (e2 && !e3) v = e1 ? __dmul_rn(0.25, __dadd_rn(z1(i1), z1(i1 + 1))) : __dmul_rn(0.5, z1(i1));
        else if (!e2 && e3) v = e1 ? __dmul_rn(0.25, __dadd_rn(z2(i1), z2(i1 + 1))) : __dmul_rn(0.5, z2(i1));
        else v = e1 ? __dmul_rn(0.125, __dadd_rn(z3(i1), z3(i1 + 1))) : __dmul_rn(0.25, z3(i1));
        u[p] = __dadd_rn(Fresh ? 0.0 : u[p], v);
    }
}


// one launch per operator and level over every job (blockIdx.y = job)
__global__ void __launch_bounds__(kMgThreads) mg_zero_kernel(const __grid_constant__ MgTable t, int k, int which) {
    mg_zero(t, t.job[blockIdx.y], k, which, blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x,
           static_cast<std::uint64_t>(gridDim.x) * blockDim.x);
}

__global__ void __launch_bounds__(kMgThreads) mg_comm3_kernel(const __grid_constant__ MgTable t, int k, int which) {
    mg_comm3(t, t.job[blockIdx.y], k, which, blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x,
           static_cast<std::uint64_t>(gridDim.x) * blockDim.x);
}

__global__ void __launch_bounds__(kMgThreads) mg_resid_kernel(const __grid_constant__ MgTable t, int k, int top) {
    mg_resid(t, t.job[blockIdx.y], k, top, blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x,
           static_cast<std::uint64_t>(gridDim.x) * blockDim.x);
}

__global__ void __launch_bounds__(kMgThreads) mg_psinv_kernel(const __grid_constant__ MgTable t, int k) {
    mg_psinv(t, t.job[blockIdx.y], k, blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x,
           static_cast<std::uint64_t>(gridDim.x) * blockDim.x);
}

__global__ void __launch_bounds__(kMgThreads) mg_rprj3_kernel(const __grid_constant__ MgTable t, int k) {
    mg_rprj3(t, t.job[blockIdx.y], k, blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x,
           static_cast<std::uint64_t>(gridDim.x) * blockDim.x);
}

__global__ void __launch_bounds__(kMgThreads) mg_interp_kernel(const __grid_constant__ MgTable t, int k) {
    mg_interp(t, t.job[blockIdx.y], k, blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x,
           static_cast<std::uint64_t>(gridDim.x) * blockDim.x);
}

// norm2u3, stage 1: per i3 plane of r_lt, the fixed-order sum of squares
// and the maximum magnitude (one CTA per plane)
// (threads 0..kMgThreads-1 of the CTA take part; Named: they sync on named
// barrier 1 so a larger CTA's other threads need not)
template <bool Named = false>
__device__ __forceinline__ void mg_norm_plane(const MgTable& t, const MgJob& j, unsigned plane) {
    const int nx = static_cast<int>(t.nx), n = nx + 2, i3 = 2 + static_cast<int>(plane);
    const double* r = j.r[t.lt];
    const std::uint32_t points = static_cast<std::uint32_t>(nx) * nx;
    double acc = 0.0, mx = 0.0;
    for (std::uint32_t q = threadIdx.x; q < points; q += kMgThreads) {
        const double x = r[mg_idx(n, 2 + static_cast<int>(q % nx), 2 + static_cast<int>(q / nx), i3)];
        acc = __dadd_rn(acc, __dmul_rn(x, x));
        mx = fmax(mx, fabs(x));
    }
    // stride-doubling tree over the 256 lanes: shuffles inside each warp...
#pragma unroll
    for (int st = 1; st < 32; st *= 2) {
        acc = __dadd_rn(acc, __shfl_down_sync(0xffffffffu, acc, st));
        mx = fmax(mx, __shfl_down_sync(0xffffffffu, mx, st));
    }
    __shared__ double ws[kMgThreads / 32], wm[kMgThreads / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) {
        ws[warp] = acc;
        wm[warp] = mx;
    }
    if constexpr (Named) asm volatile("bar.sync 1, %0;" ::"n"(kMgThreads) : "memory");
    else __syncthreads();
    // ... then over the 8 warp sums (strides 32, 64, 128 in lane terms)
    if (threadIdx.x == 0) {
        for (int st = 1; st < kMgThreads / 32; st *= 2)
            for (int w = 0; w + st < kMgThreads / 32; w += 2 * st) {
                ws[w] = __dadd_rn(ws[w], ws[w + st]);
                wm[w] = fmax(wm[w], wm[w + st]);
            }
        j.plane_sum[plane] = ws[0];
        j.plane_max[plane] = wm[0];
    }
    // ws / wm are reused by the CTA's next plane
    if constexpr (Named) asm volatile("bar.sync 1, %0;" ::"n"(kMgThreads) : "memory");
    else __syncthreads();
}

__global__ void __launch_bounds__(kMgThreads) mg_norm_kernel(const __grid_constant__ MgTable t) {
    mg_norm_plane(t, t.job[blockIdx.y], blockIdx.x);
}

// norm2u3, stage 2: planes in i3 order -> rnm2 = sqrt(sum / nx^3), rnmu
__device__ __forceinline__ void mg_norm_fold(const MgTable& t, const MgJob& j) {
    double s = 0.0, mx = 0.0;
    for (std::uint32_t p = 0; p < t.nx; ++p) {
        s = __dadd_rn(s, j.plane_sum[p]);
        mx = fmax(mx, j.plane_max[p]);
    }
    const double dn = static_cast<double>(t.nx) * t.nx * t.nx;
    vgpu_mg_result res{};
    res.rnm2 = __dsqrt_rn(__ddiv_rn(s, dn));
    res.rnmu = mx;
    res.nx = t.nx;
    res.nit = t.nit;
    *j.out = res;
}

__global__ void mg_norm_fold_kernel(const __grid_constant__ MgTable t) {
    if (threadIdx.x == 0) mg_norm_fold(t, t.job[blockIdx.x]);
}

// ---- one cluster per job: the whole timed sequence in one launch --------------
//
// For small grids (classes S..W) every operator above is a few microseconds
// of work and the launch-per-operator sequence (149 launches for class S) is
// launch-bound. Here one thread-block cluster of kMgCluster CTAs runs the
// job's whole sequence: the same per-point operators (same arithmetic, same
// bits) over the cluster's threads, a cluster barrier (release / acquire at
// cluster scope: the grids live in global memory, L2-resident at these
// sizes) between operators where the launch boundary was, and the norm's
// planes spread over the CTAs with the same per-plane tree, folded in plane
// order by CTA 0. Clusters of different jobs run independently.
constexpr int kMgCluster = 8;

__device__ __forceinline__ void mg_cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// Threads per CTA: 1024 (8 K threads per job) while every job's cluster is
// co-resident, else 512 (two CTAs per SM; backend.cu picks by occupancy).
template <int Threads>
__global__ void __cluster_dims__(kMgCluster, 1, 1) __launch_bounds__(Threads, 1024 / Threads)
    mg_cluster_kernel(const __grid_constant__ MgTable t) {
    constexpr int kMgClusterThreads = Threads;
    std::uint32_t rank;
    asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    const MgJob& j = t.job[blockIdx.x / kMgCluster];
    const std::uint64_t p0 = rank * static_cast<std::uint64_t>(kMgClusterThreads) + threadIdx.x;
    constexpr std::uint64_t ps = static_cast<std::uint64_t>(kMgCluster) * kMgClusterThreads;
    const int lt = static_cast<int>(t.lt);
    // mg.f's timed sequence with comm3 fused into the operator that writes
    // the grid (mg_store<true>) and each zero3 fused into the operator that
    // then adds into the zeroed grid (Fresh). The coarse levels k <= kLocal
    // (at most 10^3 points) run on CTA 0 alone with CTA barriers (its L1
    // keeps them; a cluster barrier costs microseconds, a CTA barrier tens
    // of ns); the other CTAs go straight to the next cluster barrier. For
    // class S: 38 cluster barriers + 40 CTA barriers per job instead of 74
    // cluster barriers (and 149 launches on the per-operator path).
    // Measured, class S x 8: kLocal 3 0.209 ms, 2 0.223, 4 0.269 (one SM
    // is too slow for the 18^3 level), all operators cluster-wide 0.241.
    constexpr int kLocal = 3;
    const bool lead = rank == 0;
    const std::uint64_t l0 = threadIdx.x, ls = Threads;  // CTA 0's own threads
    mg_zero(t, j, lt, 0, p0, ps);
    mg_cluster_sync();
    mg_resid<true>(t, j, lt, 1, p0, ps);
    mg_cluster_sync();
    for (std::uint32_t it = 0; it < t.nit; ++it) {
        for (int k = lt; k >= 2; --k) {  // restrict down to level 1 (ghosts included)
            if (k - 1 > kLocal) {
                mg_rprj3<true>(t, j, k, p0, ps);
                mg_cluster_sync();
            } else if (lead) {
                mg_rprj3<true>(t, j, k, l0, ls);
                __syncthreads();
            }
        }
        if (lead) {
            mg_psinv<true, true>(t, j, 1, l0, ls);  // zero3 + psinv + comm3 on the coarsest level
            __syncthreads();
        }
        for (int k = 2; k <= lt - 1; ++k) {
            if (k <= kLocal) {
                if (lead) {
                    mg_interp<true>(t, j, k, l0, ls);  // zero3 + interp
                    __syncthreads();
                    mg_resid<true>(t, j, k, 0, l0, ls);
                    __syncthreads();
                    mg_psinv<true>(t, j, k, l0, ls);
                    __syncthreads();
                }
                continue;
            }
            if (k - 1 <= kLocal) mg_cluster_sync();  // CTA 0's coarse levels are done
            mg_interp<true>(t, j, k, p0, ps);
            mg_cluster_sync();
            mg_resid<true>(t, j, k, 0, p0, ps);
            mg_cluster_sync();
            mg_psinv<true>(t, j, k, p0, ps);
            mg_cluster_sync();
        }
        if (lt - 1 <= kLocal) mg_cluster_sync();  // the finest level reads u_{lt-1}
        mg_interp(t, j, lt, p0, ps);
        mg_cluster_sync();
        mg_resid<true>(t, j, lt, 1, p0, ps);
        mg_cluster_sync();
        mg_psinv<true>(t, j, lt, p0, ps);
        mg_cluster_sync();
        mg_resid<true>(t, j, lt, 1, p0, ps);
        mg_cluster_sync();
    }
    if (threadIdx.x < kMgThreads)
        for (unsigned plane = rank; plane < t.nx; plane += kMgCluster) mg_norm_plane<true>(t, j, plane);
    mg_cluster_sync();
    if (rank == 0 && threadIdx.x == 0) mg_norm_fold(t, j);
}

}  // namespace vgk
