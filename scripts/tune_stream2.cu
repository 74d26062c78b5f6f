// Tuning harness #2 for the streaming step (not part of the product):
// back-to-back launches (no per-launch events), one event pair over K steps.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tune_stream2 scripts/tune_stream2.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

__device__ __forceinline__ float4 ld_l2_256(const float4* p) {
    float4 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(p));
    return r;
}

template <int T, int V, int MODE, bool PDL>
__global__ void __launch_bounds__(T, MODE == 2 ? 8 : 1)
kern(const float4* a, const float4* b, float4* o, size_t nv) {
    if (PDL) asm volatile("griddepcontrol.launch_dependents;");
    const size_t base = (size_t)blockIdx.x * T * V + threadIdx.x;
    float4 x[V], y[V];
#pragma unroll
    for (int k = 0; k < V; ++k) {
        const size_t i = base + (size_t)k * T;
        if (i < nv) {
            if (MODE == 1) {
                x[k] = ld_l2_256(a + i);
                y[k] = ld_l2_256(b + i);
            } else {
                x[k] = __ldcs(a + i);
                y[k] = __ldcs(b + i);
            }
        }
    }
#pragma unroll
    for (int k = 0; k < V; ++k) {
        const size_t i = base + (size_t)k * T;
        if (i < nv)
            __stcs(o + i, make_float4(x[k].x + y[k].x, x[k].y + y[k].y, x[k].z + y[k].z, x[k].w + y[k].w));
    }
}

template <int T, int V, int MODE, bool PDL>
void launch(cudaStream_t s, const float* a, const float* b, float* o, size_t nf) {
    const size_t nv = nf / 4;
    const unsigned g = (unsigned)((nv + (size_t)T * V - 1) / ((size_t)T * V));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(g);
    cfg.blockDim = dim3(T);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = PDL ? 1 : 0;
    cudaLaunchKernelEx(&cfg, kern<T, V, MODE, PDL>, (const float4*)a, (const float4*)b, (float4*)o, nv);
}

template <int T, int V, int MODE, bool PDL>
void bench(const char* name, size_t nf, std::vector<float*>& A, std::vector<float*>& B,
           std::vector<float*>& O, int streams) {
    cudaStream_t st[2];
    cudaStreamCreateWithFlags(&st[0], cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&st[1], cudaStreamNonBlocking);
    cudaEvent_t e0, e1, j;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventCreate(&j);
    const int sets = (int)A.size(), K = 50;
    for (int w = 0; w < 5; ++w) launch<T, V, MODE, PDL>(st[0], A[w % sets], B[w % sets], O[w % sets], nf);
    cudaStreamSynchronize(st[0]);
    cudaEventRecord(e0, st[0]);
    cudaStreamWaitEvent(st[1], e0, 0);
    for (int k = 0; k < K; ++k)
        launch<T, V, MODE, PDL>(st[k % streams], A[k % sets], B[k % sets], O[k % sets], nf);
    cudaEventRecord(j, st[1]);
    cudaStreamWaitEvent(st[0], j, 0);
    cudaEventRecord(e1, st[0]);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double per = ms / K;
    std::printf("%-34s streams=%d n=%9zu  %7.2f us/launch  %6.0f GB/s  (%.3f of 6550.7)\n", name, streams, nf,
                1e3 * per, 12.0 * nf / (per * 1e-3) / 1e9, 12.0 * nf / (per * 1e-3) / 1e9 / 6550.7);
    cudaStreamDestroy(st[0]);
    cudaStreamDestroy(st[1]);
}

int main() {
    for (size_t nf : {(size_t)4 << 20, (size_t)16 << 20}) {
        const int sets = (int)std::max<size_t>(3, (600ull << 20) / (12 * nf) + 1);
        std::vector<float*> A(sets), B(sets), O(sets);
        for (int s = 0; s < sets; ++s) {
            cudaMalloc(&A[s], 4 * nf);
            cudaMalloc(&B[s], 4 * nf);
            cudaMalloc(&O[s], 4 * nf);
            cudaMemset(A[s], 0, 4 * nf);
            cudaMemset(B[s], 0, 4 * nf);
        }
        for (int streams : {1, 2}) {
            bench<256, 4, 0, false>("chunked<256,4> ldcs", nf, A, B, O, streams);
            bench<256, 4, 1, false>("chunked<256,4> L2::256B", nf, A, B, O, streams);
            bench<256, 2, 2, false>("chunked<256,2> 8 CTA/SM", nf, A, B, O, streams);
            bench<256, 1, 0, false>("chunked<256,1> ldcs", nf, A, B, O, streams);
            bench<256, 4, 0, true>("chunked<256,4> ldcs PDL", nf, A, B, O, streams);
            bench<256, 4, 1, true>("chunked<256,4> L2::256B PDL", nf, A, B, O, streams);
            bench<256, 1, 1, true>("chunked<256,1> L2::256B PDL", nf, A, B, O, streams);
        }
        for (int s = 0; s < sets; ++s) {
            cudaFree(A[s]);
            cudaFree(B[s]);
            cudaFree(O[s]);
        }
    }
    cudaError_t e = cudaGetLastError();
    std::printf("last error: %s\n", cudaGetErrorString(e));
    return 0;
}
