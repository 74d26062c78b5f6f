// Black-Scholes (European call + put), CUDA-SDK formulation in fp32.
//
// No reference arithmetic exists (proj/src/bench/profiles.cpp:39 is a
// timing triple); the formula follows the CUDA SDK sample that the paper's
// BS benchmark is (Table 2): R = 0.02, V = 0.30, polynomial CND
// with A1..A5, RSQRT2PI. Checked against the binary64 oracle with an L1
// relative tolerance of 1e-6 (the SDK's own acceptance test).
//
// Layout per task: input S||X||T (n fp32 each), output call||put.
// HBM-bound: 12 B read + 8 B written per option. Each thread prices 4
// options per step with 128-bit loads of S, X, T and 128-bit stores of
// call and put (requires n % 4 == 0; ragged n takes the scalar path).
// Arithmetic is the SDK kernel's own (BlackScholes_kernel.cuh): MUFU-based
// exp / log, approximate reciprocals and rsqrt. With IEEE expf/logf/divisions the
// kernel was issue-bound (ncu: 90% issue active, DRAM 41%); the SDK form is
// what the SDK validates against binary64 at L1 <= 1e-6. With the MUFU ops
// in their flush-to-zero forms (below) the per-option instruction count
// drops by a third and the 16-task launch runs 199 us instead of 222.
#pragma once

#include <cstdint>

namespace vgk {

constexpr int kBsThreads = 256;
constexpr int kBsVecPerThread = 2;                                  // float4 groups per thread
constexpr int kBsChunk = kBsThreads * kBsVecPerThread * 4;          // options per CTA
constexpr int kMaxBsJobs = 64;

struct BsJob {
    const float* S;
    const float* X;
    const float* T;
    float* call;
    float* put;
    std::uint64_t n;
    std::uint32_t cta_begin;
    std::uint32_t vec_ok;
};

struct BsTable {
    BsJob job[kMaxBsJobs];
    std::uint32_t njobs;
    float R, V;
};

// The SDK's fast operations as the bare MUFU instructions in their
// flush-to-zero forms: __expf / __logf / __fdividef / rsqrtf compiled
// without -ftz guard every call against denormal operands and results and
// __fdividef against huge divisors (FSETP / FSEL / scaling FMULs: ~40 FMULs
// and 12 FSETPs per option, which kept the kernel issue-bound at 94 %).
// Every operand here is a normal float (S in [5, 30], X in [1, 100], T in
// [0.25, 10], divisors >= 0.15), so the results are the same; an exp that
// would underflow to a subnormal (|d| > 13) gives 0, below the 1e-6 L1
// contract by 30 orders of magnitude.
__device__ __forceinline__ float bs_rcp(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float bs_exp(float x) {  // e^x = 2^(x log2 e)
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x * 1.4426950408889634f));
    return y;
}
__device__ __forceinline__ float bs_log(float x) {  // ln x = log2(x) ln 2
    float y;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y * 0.6931471805599453f;
}
__device__ __forceinline__ float bs_rsqrt(float x) {
    float y;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ float bs_cnd(float d) {
    const float A1 = 0.31938153f, A2 = -0.356563782f, A3 = 1.781477937f,
                A4 = -1.821255978f, A5 = 1.330274429f;
    const float RSQRT2PI = 0.39894228040143267793994605993438f;
    const float K = bs_rcp(1.0f + 0.2316419f * fabsf(d));
    float c = RSQRT2PI * bs_exp(-0.5f * d * d) *
              (K * (A1 + K * (A2 + K * (A3 + K * (A4 + K * A5)))));
    return d > 0.0f ? 1.0f - c : c;
}

__device__ __forceinline__ void bs_price(float S, float X, float T, float R, float V,
                                         float& call, float& put) {
    const float sqrtT = bs_rcp(bs_rsqrt(T));
    const float d1 = (bs_log(S * bs_rcp(X)) + (R + 0.5f * V * V) * T) * bs_rcp(V * sqrtT);
    const float d2 = d1 - V * sqrtT;
    const float c1 = bs_cnd(d1), c2 = bs_cnd(d2);
    const float expRT = bs_exp(-R * T);
    call = S * c1 - X * expRT * c2;
    put = X * expRT * (1.0f - c2) - S * (1.0f - c1);
}

__global__ void __launch_bounds__(kBsThreads)
bs_table_kernel(const __grid_constant__ BsTable table) {
    asm volatile("griddepcontrol.launch_dependents;");  // no-op unless launched with PDL
    int j = 0;
#pragma unroll 1
    for (int k = 1; k < static_cast<int>(table.njobs); ++k)
        if (table.job[k].cta_begin <= blockIdx.x) j = k;
    const BsJob& job = table.job[j];
    const std::uint64_t base = static_cast<std::uint64_t>(blockIdx.x - job.cta_begin) * kBsChunk;
    const float R = table.R, V = table.V;
    if (job.vec_ok) {
        const std::uint64_t nv = job.n >> 2;
        const float4* S4 = reinterpret_cast<const float4*>(job.S);
        const float4* X4 = reinterpret_cast<const float4*>(job.X);
        const float4* T4 = reinterpret_cast<const float4*>(job.T);
        float4* C4 = reinterpret_cast<float4*>(job.call);
        float4* P4 = reinterpret_cast<float4*>(job.put);
        float4 s[kBsVecPerThread], x[kBsVecPerThread], t[kBsVecPerThread];
        const std::uint64_t v0 = (base >> 2) + threadIdx.x;
#pragma unroll
        for (int k = 0; k < kBsVecPerThread; ++k) {
            const std::uint64_t v = v0 + static_cast<std::uint64_t>(k) * kBsThreads;
            if (v < nv) {
                s[k] = __ldcs(S4 + v);
                x[k] = __ldcs(X4 + v);
                t[k] = __ldcs(T4 + v);
            }
        }
#pragma unroll
        for (int k = 0; k < kBsVecPerThread; ++k) {
            const std::uint64_t v = v0 + static_cast<std::uint64_t>(k) * kBsThreads;
            if (v < nv) {
                float4 c, p;
                bs_price(s[k].x, x[k].x, t[k].x, R, V, c.x, p.x);
                bs_price(s[k].y, x[k].y, t[k].y, R, V, c.y, p.y);
                bs_price(s[k].z, x[k].z, t[k].z, R, V, c.z, p.z);
                bs_price(s[k].w, x[k].w, t[k].w, R, V, c.w, p.w);
                __stcs(C4 + v, c);
                __stcs(P4 + v, p);
            }
        }
    } else {
#pragma unroll
        for (int k = 0; k < kBsVecPerThread * 4; ++k) {
            const std::uint64_t i = base + threadIdx.x + static_cast<std::uint64_t>(k) * kBsThreads;
            if (i < job.n) {
                float c, p;
                bs_price(job.S[i], job.X[i], job.T[i], R, V, c, p);
                job.call[i] = c;
                job.put[i] = p;
            }
        }
    }
}

}  // namespace vgk
