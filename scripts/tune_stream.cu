// Tuning harness for the streaming add kernel shape (not part of the product).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tune_stream scripts/tune_stream.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#define CK(x)                                                              \
    do {                                                                   \
        cudaError_t e = (x);                                               \
        if (e != cudaSuccess) {                                            \
            std::printf("%s: %s\n", #x, cudaGetErrorString(e));            \
            return 1;                                                      \
        }                                                                  \
    } while (0)

// one CTA per chunk of T*V float4
template <int T, int V>
__global__ void __launch_bounds__(T) chunked(const float4* a, const float4* b, float4* o, size_t nv) {
    const size_t base = (size_t)blockIdx.x * T * V + threadIdx.x;
    float4 x[V], y[V];
#pragma unroll
    for (int k = 0; k < V; ++k) {
        const size_t i = base + (size_t)k * T;
        if (i < nv) {
            x[k] = __ldcs(a + i);
            y[k] = __ldcs(b + i);
        }
    }
#pragma unroll
    for (int k = 0; k < V; ++k) {
        const size_t i = base + (size_t)k * T;
        if (i < nv) __stcs(o + i, make_float4(x[k].x + y[k].x, x[k].y + y[k].y, x[k].z + y[k].z, x[k].w + y[k].w));
    }
}

// persistent grid-stride, U chunks of T float4 per iteration
template <int T, int U>
__global__ void __launch_bounds__(T) strided(const float4* a, const float4* b, float4* o, size_t nv) {
    const size_t step = (size_t)gridDim.x * T * U;
    for (size_t base = (size_t)blockIdx.x * T * U + threadIdx.x; base < nv; base += step) {
        float4 x[U], y[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
            const size_t i = base + (size_t)k * T;
            if (i < nv) {
                x[k] = __ldcs(a + i);
                y[k] = __ldcs(b + i);
            }
        }
#pragma unroll
        for (int k = 0; k < U; ++k) {
            const size_t i = base + (size_t)k * T;
            if (i < nv) __stcs(o + i, make_float4(x[k].x + y[k].x, x[k].y + y[k].y, x[k].z + y[k].z, x[k].w + y[k].w));
        }
    }
}

template <class F>
int timeit(const char* name, F launch, size_t nfloats, std::vector<float*>& A, std::vector<float*>& B,
           std::vector<float*>& O) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int sets = (int)A.size();
    for (int w = 0; w < 5; ++w) launch(A[w % sets], B[w % sets], O[w % sets]);
    cudaDeviceSynchronize();
    float best = 1e9, sum = 0;
    const int iters = 40;
    for (int it = 0; it < iters; ++it) {
        const int s = it % sets;
        cudaEventRecord(e0);
        launch(A[s], B[s], O[s]);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
        sum += ms;
    }
    const double bytes = 12.0 * nfloats;
    std::printf("%-28s n=%9zu  avg %7.2f us (%6.0f GB/s)  best %7.2f us (%6.0f GB/s)\n", name, nfloats,
                1e3 * sum / iters, bytes / (sum / iters * 1e-3) / 1e9, 1e3 * best, bytes / (best * 1e-3) / 1e9);
    return 0;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (size_t nf : {(size_t)1 << 20, (size_t)4 << 20, (size_t)16 << 20, (size_t)64 << 20}) {
        const int sets = (int)std::max<size_t>(2, (512ull << 20) / (12 * nf) + 1);
        std::vector<float*> A(sets), B(sets), O(sets);
        for (int s = 0; s < sets; ++s) {
            CK(cudaMalloc(&A[s], 4 * nf));
            CK(cudaMalloc(&B[s], 4 * nf));
            CK(cudaMalloc(&O[s], 4 * nf));
            cudaMemset(A[s], 0, 4 * nf);
            cudaMemset(B[s], 0, 4 * nf);
        }
        const size_t nv = nf / 4;
        auto C = [&](auto kern, int T, int V) {
            return [=](float* a, float* b, float* o) {
                const unsigned g = (unsigned)((nv + (size_t)T * V - 1) / ((size_t)T * V));
                kern<<<g, T>>>((const float4*)a, (const float4*)b, (float4*)o, nv);
            };
        };
        auto S = [&](auto kern, int T, int ctas_per_sm) {
            return [=](float* a, float* b, float* o) {
                kern<<<sms * ctas_per_sm, T>>>((const float4*)a, (const float4*)b, (float4*)o, nv);
            };
        };
        timeit("chunked<256,4> (current)", C(chunked<256, 4>, 256, 4), nf, A, B, O);
        timeit("chunked<256,2>", C(chunked<256, 2>, 256, 2), nf, A, B, O);
        timeit("chunked<256,1>", C(chunked<256, 1>, 256, 1), nf, A, B, O);
        timeit("chunked<128,4>", C(chunked<128, 4>, 128, 4), nf, A, B, O);
        timeit("chunked<512,2>", C(chunked<512, 2>, 512, 2), nf, A, B, O);
        timeit("strided<256,2> x8/SM", S(strided<256, 2>, 256, 8), nf, A, B, O);
        timeit("strided<256,4> x4/SM", S(strided<256, 4>, 256, 4), nf, A, B, O);
        timeit("strided<256,4> x6/SM", S(strided<256, 4>, 256, 6), nf, A, B, O);
        timeit("strided<512,2> x4/SM", S(strided<512, 2>, 512, 4), nf, A, B, O);
        timeit("strided<1024,2> x2/SM", S(strided<1024, 2>, 1024, 2), nf, A, B, O);
        timeit("strided<256,1> x8/SM", S(strided<256, 1>, 256, 8), nf, A, B, O);
        // reference point: cudaMemcpy D2D of the same traffic (8 MB read+write per 4 MB copy)
        for (int s = 0; s < sets; ++s) {
            cudaFree(A[s]);
            cudaFree(B[s]);
            cudaFree(O[s]);
        }
    }
    return 0;
}
