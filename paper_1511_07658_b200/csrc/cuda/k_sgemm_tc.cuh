// SGEMM on the 5th-generation tensor cores: 3xTF32 with tcgen05.mma.
//
// Precision contract (stated tolerance): every fp32 operand x is
// split into x_hi = x rounded to nearest TF32 and x_lo = x - x_hi (exact in
// fp32, |x_lo| <= 2^-11 |x|; the MMA keeps its top 10 mantissa bits).
// C = A_hi B_hi + A_hi B_lo + A_lo B_hi. The dropped A_lo B_lo term and the
// lo-part truncation are ~2^-22 per product. The tensor core's fp32
// accumulation is NOT round-to-nearest (measured on B200: one TMEM
// accumulator over K = 2048 gives 1.4e-5 relative Frobenius), so the K loop
// is cut into chunks of chunk_kb * 32: each chunk accumulates into one of
// two TMEM accumulators (ping-pong) and the CUDA cores add the finished
// chunk into registers in IEEE fp32 while the tensor core runs the next
// chunk. Checked at relative Frobenius <= 1e-5 against the binary64 oracle
// (the SIMT kernel's bar). VGPU_SGEMM=simt selects the FP32 SIMT kernel.
//
// Three GEMM kernels (backend.cu launch_jobs picks one per batch):
//   tc_gemm2_tma_kernel  default when every n % 256 == 0: CTA pair
//                        (cta_group::2, 256 x 256 tiles), TMA operand loads
//   tc_gemm2_kernel      the same pair with cp.async loads (VGPU_SGEMM_TMA=0)
//   tc_gemm_kernel       one CTA, 128 x 128 tiles (n % 128 == 0; VGPU_SGEMM=tc)
//
// Pre-pass (tc_split_kernel): A -> A_lo (row-major M x K = K-major; A_hi is
// A itself, which the MMA reads truncated to TF32, so A_lo = A - trunc(A);
// with raw_ahi = 0, A_hi rounded to nearest is written too); B -> B_hi^T,
// B_lo^T (N x K, K-major) through a 64x64 shared-memory transpose, so both
// UMMA operands are K-major.
//
// 1-CTA kernel (tc_gemm_kernel), one 128 x 128 output tile per CTA, 256
// threads, tiles of every task of a batch in one launch (blockIdx.z = task):
//   * 3-stage cp.async pipeline; each stage holds the four 128 x 32 fp32
//     operand tiles (A_hi, A_lo, B_hi, B_lo; 16 KiB each) in the canonical
//     K-major 128-byte-swizzled layout (16-byte chunk c of row r lands at
//     chunk c ^ (r & 7) inside its 1024-byte 8-row group);
//   * fence.proxy.async makes the staged bytes visible to the tensor core;
//     one elected thread issues 4 k-steps x 3 products of
//     tcgen05.mma.cta_group::1.kind::tf32 (M=128, N=128, K=8) into a
//     128-column fp32 TMEM accumulator, then tcgen05.commit arrives on the
//     stage's mbarrier so the stage can be refilled;
//   * chunk drain: warp w reads TMEM lanes 32 (w % 4) .. +31 (= C rows),
//     columns 64 (w / 4) .. +63 of the finished chunk's accumulator with
//     tcgen05.ld.32x32b.x32 and adds them into 64 fp32 registers; the
//     epilogue stores those registers.
#pragma once

#include <cuda.h>

#include <cstdint>

namespace vgk {

constexpr int kTcBM = 128, kTcBN = 128, kTcBK = 32;  // BK in fp32 elements (128 bytes)
constexpr int kTcStages = 3;
constexpr int kTcThreads = 256;
constexpr int kTcTmemCols = 2 * kTcBN;                 // two accumulators (ping-pong)
constexpr int kTcTileBytes = kTcBM * kTcBK * 4;       // 16 KiB
constexpr int kTcStageBytes = 4 * kTcTileBytes;       // 64 KiB
constexpr int kTcSmemBytes = kTcStages * kTcStageBytes + 1024 + 256;  // + barriers / TMEM slot
constexpr int kMaxTcJobs = 64;

struct TcJob {
    const float* A;   // n x n row-major (split source)
    const float* B;
    float* C;
    float* ahi;       // workspace: n*n each
    float* alo;
    float* bthi;      // B^T hi / lo, n x n (row = column of B)
    float* btlo;
    std::uint32_t n;
    std::uint32_t pad;
};

struct TcTable {
    TcJob job[kMaxTcJobs];
    std::uint32_t njobs;
    std::uint32_t chunk_kb;  // k-blocks (of kTcBK) per TMEM accumulation chunk
    std::uint32_t raw_ahi;   // A_hi is A itself (the MMA truncates): the pre-pass writes A_lo only
};

// ---- pre-pass: split + transpose ---------------------------------------------

// hi = x rounded to nearest TF32 (|lo| <= 2^-11 |x|); lo = x - hi is exact
// in fp32. Rounding instead of truncating quarters both neglected terms.
__device__ __forceinline__ void tf32_split(float x, float& hi, float& lo) {
    std::uint32_t h;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(x));
    hi = __uint_as_float(h);
    lo = __fsub_rn(x, hi);
}

// grid (n/64, n/64, jobs), 256 threads; n % 128 == 0 for this path. A 64x64
// tile per CTA, 128-bit loads and stores throughout (the pass is HBM-bound:
// 4 bytes read, 8 written per element of A and of B).
__device__ __forceinline__ void tc_split_tile(const TcJob& job, int bx, int by, bool raw_ahi);

__global__ void __launch_bounds__(256) tc_split_kernel(const __grid_constant__ TcTable table) {
    const TcJob& job = table.job[blockIdx.z];
    const int n = static_cast<int>(job.n);
    const int bx = blockIdx.x * 64, by = blockIdx.y * 64;
    if (bx >= n || by >= n) return;
    tc_split_tile(job, bx, by, table.raw_ahi != 0);
}

// lo = x - trunc_tf32(x): exact; the remainder the MMA drops when it reads x itself
__device__ __forceinline__ float tf32_trunc_lo(float x) {
    return __fsub_rn(x, __uint_as_float(__float_as_uint(x) & 0xffffe000u));
}

__device__ __forceinline__ void tc_split_tile(const TcJob& job, int bx, int by, bool raw_ahi) {
    const int n = static_cast<int>(job.n);
    const int t = threadIdx.x;
    const int c4 = (t & 15) * 4;  // 16 threads x 4 columns = 64 columns
    const int r0 = t >> 4;        // 16 rows per pass, 4 passes
    // A: straight split, rows by.., cols bx..
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const std::size_t idx = static_cast<std::size_t>(by + r0 + 16 * k) * n + bx + c4;
        const float4 v = __ldcs(reinterpret_cast<const float4*>(job.A + idx));
        float4 h, l;
        if (raw_ahi) {
            l = make_float4(tf32_trunc_lo(v.x), tf32_trunc_lo(v.y), tf32_trunc_lo(v.z), tf32_trunc_lo(v.w));
        } else {
            tf32_split(v.x, h.x, l.x);
            tf32_split(v.y, h.y, l.y);
            tf32_split(v.z, h.z, l.z);
            tf32_split(v.w, h.w, l.w);
            *reinterpret_cast<float4*>(job.ahi + idx) = h;
        }
        *reinterpret_cast<float4*>(job.alo + idx) = l;
    }
    // B: transpose through shared memory; Bt[c][r] = B[r][c]
    __shared__ float tile[64][65];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int r = r0 + 16 * k;
        const float4 v = __ldcs(reinterpret_cast<const float4*>(
            job.B + static_cast<std::size_t>(by + r) * n + bx + c4));
        tile[r][c4] = v.x;
        tile[r][c4 + 1] = v.y;
        tile[r][c4 + 2] = v.z;
        tile[r][c4 + 3] = v.w;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int c = r0 + 16 * k;  // column of B = row of Bt
        float4 h, l;
        tf32_split(tile[c4][c], h.x, l.x);
        tf32_split(tile[c4 + 1][c], h.y, l.y);
        tf32_split(tile[c4 + 2][c], h.z, l.z);
        tf32_split(tile[c4 + 3][c], h.w, l.w);
        const std::size_t idx = static_cast<std::size_t>(bx + c) * n + by + c4;
        *reinterpret_cast<float4*>(job.bthi + idx) = h;
        *reinterpret_cast<float4*>(job.btlo + idx) = l;
    }
}

// ---- PTX helpers ---------------------------------------------------------------

__device__ __forceinline__ std::uint32_t smem_u32(const void* p) {
    return static_cast<std::uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void cp_async16(std::uint32_t dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src));
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }

template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N));
}

__device__ __forceinline__ void mbar_init(std::uint64_t* bar, std::uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_wait(std::uint64_t* bar, std::uint32_t phase) {
    asm volatile(
        "{\n"
        ".reg .pred done;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n"
        "@!done bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(phase));
}

// K-major, 128-byte swizzle, 8-row groups 1024 B apart (CuTe canonical
// layout Swizzle<3,4,3> o ((8,m),2):((8,SBO),1) in 16-byte units)
__device__ __forceinline__ std::uint64_t umma_desc_k_sw128(std::uint32_t saddr) {
    std::uint64_t d = 0;
    d |= static_cast<std::uint64_t>((saddr >> 4) & 0x3FFFu);  // start address
    d |= static_cast<std::uint64_t>(1u) << 16;                // LBO (unused for SW128 K-major)
    d |= static_cast<std::uint64_t>(1024u >> 4) << 32;        // SBO: next 8-row group
    d |= static_cast<std::uint64_t>(1u) << 46;                // version (sm_100)
    d |= static_cast<std::uint64_t>(2u) << 61;                // SWIZZLE_128B
    return d;
}

// instruction descriptor: kind::tf32, D f32, A/B tf32, both K-major, M=128, N=128
constexpr std::uint32_t kTcIdesc = (1u << 4)          // c_format F32
                                   | (2u << 7)        // a_format TF32
                                   | (2u << 10)       // b_format TF32
                                   | ((kTcBN >> 3) << 17)
                                   | ((kTcBM >> 4) << 24);

__device__ __forceinline__ void umma_tf32(std::uint32_t tmem_d, std::uint64_t a, std::uint64_t b,
                                          std::uint32_t accumulate) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(kTcIdesc), "r"(accumulate));
}

__device__ __forceinline__ void umma_commit(std::uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
        smem_u32(bar)));
}

// ---- main kernel -----------------------------------------------------------------

__device__ __forceinline__ void tmem_ld32(std::uint32_t taddr, float* out) {
    std::uint32_t v[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
          "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]),
          "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
          "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]),
          "=r"(v[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
    for (int j = 0; j < 32; ++j) out[j] = __uint_as_float(v[j]);
}

__global__ void __launch_bounds__(kTcThreads, 1) tc_gemm_kernel(const __grid_constant__ TcTable table) {
    const TcJob& job = table.job[blockIdx.z];
    const int n = static_cast<int>(job.n);
    const int m0 = blockIdx.y * kTcBM, n0 = blockIdx.x * kTcBN;
    if (m0 >= n || n0 >= n) return;

    extern __shared__ __align__(1024) std::uint8_t smem_raw[];
    std::uint8_t* smem = reinterpret_cast<std::uint8_t*>(
        (reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) & ~std::uintptr_t{1023});
    // bars[0..S-1]: stage free; bars[S], bars[S+1]: accumulator 0/1 chunk done
    std::uint64_t* bars = reinterpret_cast<std::uint64_t*>(smem + kTcStages * kTcStageBytes);
    std::uint32_t* tmem_slot = reinterpret_cast<std::uint32_t*>(bars + kTcStages + 2);

    const int tid = threadIdx.x, warp = tid >> 5;
    if (tid == 0) {
        for (int s = 0; s < kTcStages + 2; ++s) mbar_init(&bars[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "n"(kTcTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const std::uint32_t tmem = *tmem_slot;

    const float* srcs[4] = {job.ahi + static_cast<std::size_t>(m0) * n,
                            job.alo + static_cast<std::size_t>(m0) * n,
                            job.bthi + static_cast<std::size_t>(n0) * n,
                            job.btlo + static_cast<std::size_t>(n0) * n};
    // stage k-block kb into stage s: 4 tiles x 128 rows x 8 chunks, 16 per thread
    auto load_stage = [&](int kb, int s) {
        const std::uint32_t sbase = smem_u32(smem + s * kTcStageBytes);
#pragma unroll
        for (int i = 0; i < (4 * kTcBM * 8) / kTcThreads; ++i) {
            const int chunk = tid + i * kTcThreads;  // 0..4095
            const int tile = chunk >> 10;
            const int r = (chunk >> 3) & 127;
            const int c = chunk & 7;
            const float* g = srcs[tile] + static_cast<std::size_t>(r) * n + kb * kTcBK + c * 4;
            const std::uint32_t d = sbase + tile * kTcTileBytes + (r >> 3) * 1024 + (r & 7) * 128 +
                                    ((c ^ (r & 7)) << 4);
            cp_async16(d, g);
        }
    };

    // this thread's share of the tile: TMEM lane quadrant (warp % 4) = 32 C
    // rows, 64 of the 128 columns (warp / 4)
    const int quad = warp & 3, half = warp >> 2;
    float acc[64];
#pragma unroll
    for (int j = 0; j < 64; ++j) acc[j] = 0.0f;
    auto drain = [&](int chunk) {
        mbar_wait(&bars[kTcStages + (chunk & 1)], (chunk >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const std::uint32_t base = tmem + (static_cast<std::uint32_t>(quad * 32) << 16) +
                                   (chunk & 1) * kTcBN + half * 64;
        float v[32];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            tmem_ld32(base + h * 32, v);
#pragma unroll
            for (int j = 0; j < 32; ++j) acc[h * 32 + j] = __fadd_rn(acc[h * 32 + j], v[j]);
        }
        asm volatile("tcgen05.fence::before_thread_sync;");
    };

    const int kblocks = n / kTcBK;
    const int ckb = static_cast<int>(table.chunk_kb);
#pragma unroll
    for (int s = 0; s < kTcStages - 1; ++s) {
        if (s < kblocks) load_stage(s, s);
        cp_async_commit();
    }
    for (int kb = 0; kb < kblocks; ++kb) {
        const int s = kb % kTcStages;
        const int chunk = kb / ckb;
        const bool chunk_first = kb % ckb == 0;
        const bool chunk_last = (kb + 1) % ckb == 0 || kb + 1 == kblocks;
        cp_async_wait<kTcStages - 2>();
        asm volatile("fence.proxy.async.shared::cta;");  // generic-proxy writes -> tensor core
        __syncthreads();
        if (tid == 0) {
            asm volatile("tcgen05.fence::after_thread_sync;");
            const std::uint32_t sbase = smem_u32(smem + s * kTcStageBytes);
            const std::uint32_t dacc = tmem + (chunk & 1) * kTcBN;
#pragma unroll
            for (int k = 0; k < kTcBK / 8; ++k) {
                const std::uint32_t off = k * 32;  // 8 tf32 = 32 bytes along K
                const std::uint64_t ahi = umma_desc_k_sw128(sbase + 0 * kTcTileBytes + off);
                const std::uint64_t alo = umma_desc_k_sw128(sbase + 1 * kTcTileBytes + off);
                const std::uint64_t bhi = umma_desc_k_sw128(sbase + 2 * kTcTileBytes + off);
                const std::uint64_t blo = umma_desc_k_sw128(sbase + 3 * kTcTileBytes + off);
                // small terms first, then the large one
                umma_tf32(dacc, ahi, blo, (chunk_first && k == 0) ? 0u : 1u);
                umma_tf32(dacc, alo, bhi, 1u);
                umma_tf32(dacc, ahi, bhi, 1u);
            }
            umma_commit(&bars[s]);  // stage s free once these MMAs have read it
            if (chunk_last) umma_commit(&bars[kTcStages + (chunk & 1)]);  // chunk done
        }
        // refill the stage consumed one iteration ago with k-block kb + S - 1
        const int next = kb + kTcStages - 1;
        if (next < kblocks) {
            const int ns = next % kTcStages;
            if (kb >= 1) mbar_wait(&bars[ns], ((kb - 1) / kTcStages) & 1);
            load_stage(next, ns);
        }
        cp_async_commit();
        // fold the previous chunk while the tensor core runs this one; the
        // next MMA into that accumulator comes after a later __syncthreads
        if (chunk_first && chunk > 0) drain(chunk - 1);
    }
    drain((kblocks - 1) / ckb);

    // epilogue: 64 consecutive columns of one C row per thread
    const int row = m0 + quad * 32 + (tid & 31);
    float* crow = job.C + static_cast<std::size_t>(row) * n + n0 + half * 64;
#pragma unroll
    for (int j = 0; j < 64; j += 4)
        *reinterpret_cast<float4*>(crow + j) = make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                     "n"(kTcTmemCols));
}


// ---- CTA-pair variant (cta_group::2) ---------------------------------------------
//
// Two CTAs of a cluster (the two SMs of a TPC) compute a 256 x 256 tile with
// tcgen05.mma.cta_group::2 (M = 256, N = 256, K = 8): each CTA stages its
// own 128 rows of A (hi, lo) and its own 128 columns of B (hi, lo) in the
// same SW128 K-major layout as above, and the leader CTA's single issuing
// thread runs the MMA over both CTAs' operands. Per SM that is half the
// shared-memory operand traffic of the 1-CTA 128 x 128 kernel for the same
// MMA work (the 1-CTA kernel is shared-memory-bandwidth bound at ~60 % of
// the TF32 peak). Each CTA's TMEM holds its 128 rows x 256 columns; the
// same ping-pong chunked accumulation (512 TMEM columns) keeps the FP32
// accuracy. Synchronisation: one cluster barrier per k-block (both CTAs'
// stage is in shared memory), tcgen05.commit multicast to both CTAs'
// mbarriers (stage free / chunk done).
constexpr int kTc2BN = 256;  // pair tile N (each CTA stages 128 columns)
constexpr std::uint32_t kTc2Idesc = (1u << 4) | (2u << 7) | (2u << 10) |
                                    ((kTc2BN >> 3) << 17) | ((256 >> 4) << 24);

__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::
                     : "memory");
}

__device__ __forceinline__ void umma2_tf32(std::uint32_t tmem_d, std::uint64_t a, std::uint64_t b,
                                           std::uint32_t accumulate) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(kTc2Idesc), "r"(accumulate));
}

__device__ __forceinline__ void umma2_commit_both(std::uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
        "[%0], %1;" ::"r"(smem_u32(bar)),
        "h"(static_cast<unsigned short>(3)));
}

// arrive on the mbarrier at the same shared-memory offset in CTA 0 of the
// cluster (release at cluster scope)
__device__ __forceinline__ void mbar_arrive_leader(std::uint64_t* bar) {
    asm volatile(
        "{\n"
        ".reg .b32 remote;\n"
        "mapa.shared::cluster.u32 remote, %0, 0;\n"
        "mbarrier.arrive.release.cluster.shared::cluster.b64 _, [remote];\n"
        "}\n" ::"r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void mbar_wait_cluster(std::uint64_t* bar, std::uint32_t phase) {
    asm volatile(
        "{\n"
        ".reg .pred done;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 done, [%0], %1;\n"
        "@!done bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kTcThreads, 1)
    tc_gemm2_kernel(const __grid_constant__ TcTable table) {
    const TcJob& job = table.job[blockIdx.z];
    const int n = static_cast<int>(job.n);
    std::uint32_t rank;
    asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    const int pair = blockIdx.x >> 1, pairs_n = n / kTc2BN;
    const int pm = pair / max(1, pairs_n), pn = pair % max(1, pairs_n);
    // whole pairs leave together (n % 256 == 0 for every job of this kernel)
    if (pairs_n == 0 || pm * kTc2BN >= n) return;
    const int m0 = pm * kTc2BN + static_cast<int>(rank) * kTcBM;   // my A rows = my C rows
    const int nb = pn * kTc2BN + static_cast<int>(rank) * kTcBM;   // my B columns
    const int c0 = pn * kTc2BN;                                     // C columns (all 256)
    const bool leader = rank == 0;

    extern __shared__ __align__(1024) std::uint8_t smem_raw[];
    std::uint8_t* smem = reinterpret_cast<std::uint8_t*>(
        (reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) & ~std::uintptr_t{1023});
    // bars[0..S-1]: stage free, bars[S], bars[S+1]: accumulator 0/1 chunk
    // done (both multicast by the leader's tcgen05.commit); full[s]: this
    // CTA's copies of stage s landed (every thread's cp.async arrive);
    // peer[s] (leader): the peer CTA's copies landed (relayed arrive)
    std::uint64_t* bars = reinterpret_cast<std::uint64_t*>(smem + kTcStages * kTcStageBytes);
    std::uint64_t* full = bars + kTcStages + 2;
    std::uint64_t* peer = full + kTcStages;
    std::uint32_t* tmem_slot = reinterpret_cast<std::uint32_t*>(peer + kTcStages);

    const int tid = threadIdx.x, warp = tid >> 5;
    if (tid == 0) {
        for (int s = 0; s < kTcStages + 2; ++s) mbar_init(&bars[s], 1);
        for (int s = 0; s < kTcStages; ++s) {
            mbar_init(&full[s], kTcThreads);
            mbar_init(&peer[s], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "n"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    cluster_sync_all();  // barriers of both CTAs initialised, TMEM allocated
    asm volatile("tcgen05.fence::after_thread_sync;");
    const std::uint32_t tmem = *tmem_slot;

    const float* srcs[4] = {job.ahi + static_cast<std::size_t>(m0) * n,
                            job.alo + static_cast<std::size_t>(m0) * n,
                            job.bthi + static_cast<std::size_t>(nb) * n,
                            job.btlo + static_cast<std::size_t>(nb) * n};
    auto load_stage = [&](int kb, int s) {
        const std::uint32_t sbase = smem_u32(smem + s * kTcStageBytes);
#pragma unroll
        for (int i = 0; i < (4 * kTcBM * 8) / kTcThreads; ++i) {
            const int chunk = tid + i * kTcThreads;
            const int tile = chunk >> 10;
            const int r = (chunk >> 3) & 127;
            const int c = chunk & 7;
            const float* g = srcs[tile] + static_cast<std::size_t>(r) * n + kb * kTcBK + c * 4;
            const std::uint32_t d = sbase + tile * kTcTileBytes + (r >> 3) * 1024 + (r & 7) * 128 +
                                    ((c ^ (r & 7)) << 4);
            cp_async16(d, g);
        }
    };

    // warp w: TMEM lanes 32 (w % 4) .. +31 (= my C rows), columns 128 (w / 4) .. +127
    const int quad = warp & 3, half = warp >> 2;
    float acc[128];
#pragma unroll
    for (int j = 0; j < 128; ++j) acc[j] = 0.0f;
    auto drain = [&](int chunk) {
        mbar_wait(&bars[kTcStages + (chunk & 1)], (chunk >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const std::uint32_t base = tmem + (static_cast<std::uint32_t>(quad * 32) << 16) +
                                   (chunk & 1) * kTc2BN + half * 128;
        float v[32];
#pragma unroll
        for (int h = 0; h < 4; ++h) {
            tmem_ld32(base + h * 32, v);
#pragma unroll
            for (int j = 0; j < 32; ++j) acc[h * 32 + j] = __fadd_rn(acc[h * 32 + j], v[j]);
        }
        asm volatile("tcgen05.fence::before_thread_sync;");
    };

    const int kblocks = n / kTcBK;
    // >= 2: the copies that feed chunk c+2 are issued after the drain of
    // chunk c (program order below), which frees its TMEM accumulator
    const int ckb = max(2, static_cast<int>(table.chunk_kb));
    // stage s for k-block kb: this thread's 16 copies, tracked by full[s]
    auto fill = [&](int kb, int s) {
        load_stage(kb, s);
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&full[s]))
                     : "memory");
    };
#pragma unroll
    for (int s = 0; s < kTcStages - 1; ++s)
        if (s < kblocks) fill(s, s);
    // No CTA- or cluster-wide barrier in the loop: mbarriers only. The
    // leader's thread 0 issues MMA(kb) once both CTAs' copies of k-block kb
    // landed (own full[s] + the peer's relayed arrive), so MMAs stay queued
    // ahead of the tensor core while the other threads drain and refill.
    for (int kb = 0; kb < kblocks; ++kb) {
        const int s = kb % kTcStages;
        const std::uint32_t ph = (kb / kTcStages) & 1;
        const int chunk = kb / ckb;
        const bool chunk_first = kb % ckb == 0;
        const bool chunk_last = (kb + 1) % ckb == 0 || kb + 1 == kblocks;
        if (tid == 0) {
            mbar_wait(&full[s], ph);  // this CTA's stage s (acquire: copies visible)
            asm volatile("fence.proxy.async.shared::cta;");  // -> tensor core (async proxy)
            if (leader) {
                mbar_wait_cluster(&peer[s], ph);  // the peer's stage s
                asm volatile("tcgen05.fence::after_thread_sync;");
                const std::uint32_t sbase = smem_u32(smem + s * kTcStageBytes);
                const std::uint32_t dacc = tmem + (chunk & 1) * kTc2BN;
#pragma unroll
                for (int k = 0; k < kTcBK / 8; ++k) {
                    const std::uint32_t off = k * 32;
                    const std::uint64_t ahi = umma_desc_k_sw128(sbase + 0 * kTcTileBytes + off);
                    const std::uint64_t alo = umma_desc_k_sw128(sbase + 1 * kTcTileBytes + off);
                    const std::uint64_t bhi = umma_desc_k_sw128(sbase + 2 * kTcTileBytes + off);
                    const std::uint64_t blo = umma_desc_k_sw128(sbase + 3 * kTcTileBytes + off);
                    umma2_tf32(dacc, ahi, blo, (chunk_first && k == 0) ? 0u : 1u);
                    umma2_tf32(dacc, alo, bhi, 1u);
                    umma2_tf32(dacc, ahi, bhi, 1u);
                }
                umma2_commit_both(&bars[s]);
                if (chunk_last) umma2_commit_both(&bars[kTcStages + (chunk & 1)]);
            } else {
                mbar_arrive_leader(&peer[s]);  // relay: my stage s is ready
            }
        }
        __syncwarp();
        // fold the previous chunk while the tensor core runs this one
        if (chunk_first && chunk > 0) drain(chunk - 1);
        // refill the stage MMA(kb-1) read with k-block kb + S - 1
        const int next = kb + kTcStages - 1;
        if (next < kblocks) {
            const int ns = next % kTcStages;
            if (kb >= 1) mbar_wait(&bars[ns], ((kb - 1) / kTcStages) & 1);
            fill(next, ns);
        }
    }
    drain((kblocks - 1) / ckb);

    const int row = m0 + quad * 32 + (tid & 31);
    float* crow = job.C + static_cast<std::size_t>(row) * n + c0 + half * 128;
#pragma unroll
    for (int j = 0; j < 128; j += 4)
        *reinterpret_cast<float4*>(crow + j) = make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
    asm volatile("tcgen05.fence::before_thread_sync;");
    cluster_sync_all();  // both CTAs done with the pair's TMEM
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
}


// ---- CTA pair with TMA operand loads ------------------------------------------------
//
// Same pair / chunking / accumulation as tc_gemm2_kernel, but each CTA's
// thread 0 fetches a stage with four TMA tile loads (cp.async.bulk.tensor,
// 128 rows x 128 bytes, SWIZZLE_128B: the canonical K-major layout the UMMA
// descriptors expect) on a 64 KiB expect_tx mbarrier, instead of 256
// threads issuing 4096 16-byte cp.async copies. The other threads only
// drain accumulators. Tensor maps (4 per job: A_hi, A_lo, B^T_hi, B^T_lo)
// travel in the kernel's parameter space.
constexpr int kMaxTc2TmaJobs = 16;

struct alignas(64) TcTmaTable {
    CUtensorMap maps[kMaxTc2TmaJobs][4];
    TcJob job[kMaxTc2TmaJobs];
    std::uint32_t njobs;
    std::uint32_t chunk_kb;
};

__device__ __forceinline__ void tma_load_2d(std::uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                            std::uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
        "l"(reinterpret_cast<std::uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kTcThreads, 1)
    tc_gemm2_tma_kernel(const __grid_constant__ TcTmaTable table) {
    const TcJob& job = table.job[blockIdx.z];
    const CUtensorMap* maps = table.maps[blockIdx.z];
    const int n = static_cast<int>(job.n);
    std::uint32_t rank;
    asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    const int pair = blockIdx.x >> 1, pairs_n = n / kTc2BN;
    const int pm = pair / max(1, pairs_n), pn = pair % max(1, pairs_n);
    if (pairs_n == 0 || pm * kTc2BN >= n) return;
    const int m0 = pm * kTc2BN + static_cast<int>(rank) * kTcBM;
    const int nb = pn * kTc2BN + static_cast<int>(rank) * kTcBM;
    const int c0 = pn * kTc2BN;
    const bool leader = rank == 0;

    extern __shared__ __align__(1024) std::uint8_t smem_raw[];
    std::uint8_t* smem = reinterpret_cast<std::uint8_t*>(
        (reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) & ~std::uintptr_t{1023});
    std::uint64_t* bars = reinterpret_cast<std::uint64_t*>(smem + kTcStages * kTcStageBytes);
    std::uint64_t* full = bars + kTcStages + 2;
    std::uint64_t* peer = full + kTcStages;
    std::uint32_t* tmem_slot = reinterpret_cast<std::uint32_t*>(peer + kTcStages);

    const int tid = threadIdx.x, warp = tid >> 5;
    if (tid == 0) {
        for (int s = 0; s < kTcStages + 2; ++s) mbar_init(&bars[s], 1);
        for (int s = 0; s < kTcStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&peer[s], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
        for (int t = 0; t < 4; ++t)
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<std::uint64_t>(&maps[t])));
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "n"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    cluster_sync_all();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const std::uint32_t tmem = *tmem_slot;

    const int quad = warp & 3, half = warp >> 2;
    float acc[128];
#pragma unroll
    for (int j = 0; j < 128; ++j) acc[j] = 0.0f;
    auto drain = [&](int chunk) {
        mbar_wait(&bars[kTcStages + (chunk & 1)], (chunk >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const std::uint32_t base = tmem + (static_cast<std::uint32_t>(quad * 32) << 16) +
                                   (chunk & 1) * kTc2BN + half * 128;
        float v[32];
#pragma unroll
        for (int h = 0; h < 4; ++h) {
            tmem_ld32(base + h * 32, v);
#pragma unroll
            for (int j = 0; j < 32; ++j) acc[h * 32 + j] = __fadd_rn(acc[h * 32 + j], v[j]);
        }
        asm volatile("tcgen05.fence::before_thread_sync;");
    };

    const int kblocks = n / kTcBK;
    // >= 4: a chunk-opening refill (issued right after the MMAs, before
    // this iteration's drain) then targets an accumulator whose drain ran
    // two or more iterations earlier; the __syncthreads below covers it
    const int ckb = max(4, static_cast<int>(table.chunk_kb));
    // stage s <- k-block kb (A rows m0.., B^T rows nb..), 64 KiB
    auto fill = [&](int kb, int s) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])),
                     "r"(kTcStageBytes)
                     : "memory");
        const std::uint32_t sbase = smem_u32(smem + s * kTcStageBytes);
        tma_load_2d(sbase + 0 * kTcTileBytes, &maps[0], kb * kTcBK, m0, &full[s]);
        tma_load_2d(sbase + 1 * kTcTileBytes, &maps[1], kb * kTcBK, m0, &full[s]);
        tma_load_2d(sbase + 2 * kTcTileBytes, &maps[2], kb * kTcBK, nb, &full[s]);
        tma_load_2d(sbase + 3 * kTcTileBytes, &maps[3], kb * kTcBK, nb, &full[s]);
    };
    if (tid == 0)
        for (int s = 0; s < kTcStages - 1; ++s)
            if (s < kblocks) fill(s, s);
    for (int kb = 0; kb < kblocks; ++kb) {
        const int s = kb % kTcStages;
        const std::uint32_t ph = (kb / kTcStages) & 1;
        const int chunk = kb / ckb;
        const bool chunk_first = kb % ckb == 0;
        const bool chunk_last = (kb + 1) % ckb == 0 || kb + 1 == kblocks;
        if (tid == 0) {
            mbar_wait(&full[s], ph);  // TMA bytes of my stage s landed
            if (leader) {
                mbar_wait_cluster(&peer[s], ph);  // the peer's stage s
                asm volatile("tcgen05.fence::after_thread_sync;");
                const std::uint32_t sbase = smem_u32(smem + s * kTcStageBytes);
                const std::uint32_t dacc = tmem + (chunk & 1) * kTc2BN;
#pragma unroll
                for (int k = 0; k < kTcBK / 8; ++k) {
                    const std::uint32_t off = k * 32;
                    const std::uint64_t ahi = umma_desc_k_sw128(sbase + 0 * kTcTileBytes + off);
                    const std::uint64_t alo = umma_desc_k_sw128(sbase + 1 * kTcTileBytes + off);
                    const std::uint64_t bhi = umma_desc_k_sw128(sbase + 2 * kTcTileBytes + off);
                    const std::uint64_t blo = umma_desc_k_sw128(sbase + 3 * kTcTileBytes + off);
                    umma2_tf32(dacc, ahi, blo, (chunk_first && k == 0) ? 0u : 1u);
                    umma2_tf32(dacc, alo, bhi, 1u);
                    umma2_tf32(dacc, ahi, bhi, 1u);
                }
                umma2_commit_both(&bars[s]);
                if (chunk_last) umma2_commit_both(&bars[kTcStages + (chunk & 1)]);
            } else {
                mbar_arrive_leader(&peer[s]);
            }
        }
        __syncwarp();
        // refill the stage MMA(kb-1) read with k-block kb + S - 1 (warp 1's
        // lane 0, so the MMA issue in warp 0 never waits behind it). When
        // that k-block opens chunk c', chunk c'-2's accumulator must be
        // drained by every thread first: drain(c'-2) ran at iteration
        // next - ckb <= kb - 2, and this barrier gathers the CTA.
        const int next = kb + kTcStages - 1;
        if (next < kblocks) {
            if (next % ckb == 0 && next / ckb >= 2) __syncthreads();
            if (tid == 32) {
                if (kb >= 1) mbar_wait(&bars[next % kTcStages], ((kb - 1) / kTcStages) & 1);
                fill(next, next % kTcStages);
            }
            __syncwarp();
        }
        // all threads: fold the previous chunk while the tensor core runs this one
        if (chunk_first && chunk > 0) drain(chunk - 1);
    }
    drain((kblocks - 1) / ckb);

    const int row = m0 + quad * 32 + (tid & 31);
    float* crow = job.C + static_cast<std::size_t>(row) * n + c0 + half * 128;
#pragma unroll
    for (int j = 0; j < 128; j += 4)
        *reinterpret_cast<float4*>(crow + j) = make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
    asm volatile("tcgen05.fence::before_thread_sync;");
    cluster_sync_all();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
}

}  // namespace vgk
