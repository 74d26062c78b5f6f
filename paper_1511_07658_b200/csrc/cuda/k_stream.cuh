// Streaming payload kernels: vector-add, vector-mul and vector-scale over a
// TASK TABLE.
//
// Reference arithmetic: kernels::vector_add / vector_scale
// (proj/src/payload_kernels.cpp:7-22): out[i] = a[i] + b[i], out[i] = x[i]*f,
// one IEEE fp32 operation per element, so results are bit-identical to the
// serial CPU loop (no FTZ, no fast-math in this translation unit).
// vector-mul (out[i] = a[i] * b[i]) is the paper's VecMul benchmark
// (proj/src/bench/profiles.cpp:33 timing profile; no reference kernel), with
// vector-add's layout.
//
// B200 design: one launch covers every task of a PS-1 batch (each client's
// slice is a row of the table passed by value in the parameter space), so a
// batch of N small tasks costs one launch instead of N. Each CTA streams a
// contiguous 16 KiB chunk of one task: 256 threads x 4 x 128-bit loads per
// operand in flight, evict-first loads/stores (__ldcs/__stcs) because every
// byte is touched exactly once. HBM-bound: 12 B/element for add and mul, 8 for scale.
// The b operand starts at byte 4n of the client's input, which is only
// 16-byte aligned when n % 4 == 0; such tasks take a scalar path (uniform
// per CTA, decided on the host).
#pragma once

#include <cstdint>

namespace vgk {

constexpr int kStreamThreads = 256;
constexpr int kStreamVecPerThread = 4;                               // float4 per thread per operand
constexpr int kStreamChunk = kStreamThreads * kStreamVecPerThread * 4;  // floats per CTA
constexpr int kMaxTableJobs = 64;

struct StreamJob {
    const float* a;
    const float* b;   // nullptr for scale
    float* out;
    std::uint64_t n;
    std::uint32_t cta_begin;
    std::uint32_t vec_ok;
    float factor;
    std::uint32_t pad;
};

struct StreamTable {
    StreamJob job[kMaxTableJobs];
    std::uint32_t njobs;
};

__device__ __forceinline__ int find_job(const StreamTable& t, std::uint32_t cta) {
    int j = 0;
#pragma unroll 1
    for (int k = 1; k < static_cast<int>(t.njobs); ++k)
        if (t.job[k].cta_begin <= cta) j = k;
    return j;
}

enum StreamOp { kOpScale = 0, kOpAdd = 1, kOpMul = 2 };

template <int kOp>
__device__ __forceinline__ float stream_op(float a, float b, float f) {
    if constexpr (kOp == kOpAdd) return __fadd_rn(a, b);
    else if constexpr (kOp == kOpMul) return __fmul_rn(a, b);
    else return __fmul_rn(a, f);
}

template <int kOp>
__global__ void __launch_bounds__(kStreamThreads)
stream_table_kernel(const __grid_constant__ StreamTable table) {
    // lets an independent follow-up launch (PDL) ramp up under this one's tail
    asm volatile("griddepcontrol.launch_dependents;");
    const int j = find_job(table, blockIdx.x);
    const StreamJob& job = table.job[j];
    const std::uint64_t chunk = blockIdx.x - job.cta_begin;
    const std::uint64_t base = chunk * kStreamChunk;
    const std::uint64_t n = job.n;
    constexpr bool kAdd = kOp != kOpScale;  // two operands
    if (job.vec_ok) {
        const float4* a4 = reinterpret_cast<const float4*>(job.a);
        const float4* b4 = reinterpret_cast<const float4*>(job.b);
        float4* o4 = reinterpret_cast<float4*>(job.out);
        const std::uint64_t nv = n >> 2;
        const std::uint64_t v0 = (base >> 2) + threadIdx.x;
        float4 x[kStreamVecPerThread], y[kStreamVecPerThread];
#pragma unroll
        for (int k = 0; k < kStreamVecPerThread; ++k) {
            const std::uint64_t v = v0 + static_cast<std::uint64_t>(k) * kStreamThreads;
            if (v < nv) {
                x[k] = __ldcs(a4 + v);
                if (kAdd) y[k] = __ldcs(b4 + v);
            }
        }
#pragma unroll
        for (int k = 0; k < kStreamVecPerThread; ++k) {
            const std::uint64_t v = v0 + static_cast<std::uint64_t>(k) * kStreamThreads;
            if (v < nv) {
                float4 r;
                if (!kAdd) y[k] = x[k];  // unused operand
                r.x = stream_op<kOp>(x[k].x, y[k].x, job.factor);
                r.y = stream_op<kOp>(x[k].y, y[k].y, job.factor);
                r.z = stream_op<kOp>(x[k].z, y[k].z, job.factor);
                r.w = stream_op<kOp>(x[k].w, y[k].w, job.factor);
                __stcs(o4 + v, r);
            }
        }
        // n % 4 tail (vector-scale with ragged n; handled by the last CTA)
        const std::uint64_t tail0 = nv << 2;
        if (tail0 < n && base + kStreamChunk >= n && threadIdx.x < n - tail0) {
            const std::uint64_t i = tail0 + threadIdx.x;
            job.out[i] = stream_op<kOp>(job.a[i], kAdd ? job.b[i] : 0.0f, job.factor);
        }
    } else {
#pragma unroll
        for (int k = 0; k < kStreamVecPerThread * 4; ++k) {
            const std::uint64_t i = base + threadIdx.x + static_cast<std::uint64_t>(k) * kStreamThreads;
            if (i < n)
                job.out[i] = stream_op<kOp>(__ldcs(job.a + i), kAdd ? __ldcs(job.b + i) : 0.0f, job.factor);
        }
    }
}

}  // namespace vgk
