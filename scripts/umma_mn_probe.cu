// Probe: tcgen05.mma.cta_group::1.kind::tf32 with B in the MN-major SW128
// layout. One CTA, M = 128, N = 128, K = 32 (4 MMAs of K = 8). A K-major
// SW128 (128 rows x 128 B), B MN-major SW128 as 4 column atoms (32 N x 32 K
// rows each, 4 KiB) placed either "atoms apart" (atom j at j*4096, K groups
// 1 KiB apart inside) or "groups apart" (K group g at g*4096, atom j at
// j*1024 inside). Variants try (LBO, SBO) both ways and compare with the
// host product. Build: nvcc -gencode arch=compute_100a,code=sm_100a -o
// scripts/umma_mn_probe scripts/umma_mn_probe.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

__device__ __forceinline__ std::uint32_t smem_u32(const void* p) {
    return static_cast<std::uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ std::uint64_t desc(std::uint32_t saddr, std::uint32_t lbo, std::uint32_t sbo) {
    std::uint64_t d = 0;
    d |= static_cast<std::uint64_t>((saddr >> 4) & 0x3FFFu);
    d |= static_cast<std::uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
    d |= static_cast<std::uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
    d |= static_cast<std::uint64_t>(1u) << 46;
    d |= static_cast<std::uint64_t>(2u) << 61;
    return d;
}

// layout 0: atom j at j*4096, K row k at (k>>3)*1024 + (k&7)*128
// layout 1: atom j at j*1024, K row k at (k>>3)*4096 + (k&7)*128
__device__ __forceinline__ std::uint32_t b_off(int layout, int k, int nn) {
    const int j = nn >> 5, c = (nn & 31) >> 2, e = nn & 3;
    const int row = k & 7;
    const std::uint32_t base = layout == 0 ? j * 4096 + (k >> 3) * 1024 : j * 1024 + (k >> 3) * 4096;
    return base + row * 128 + ((c ^ row) << 4) + e * 4;
}

__global__ void probe(const float* A, const float* B, float* C, int layout, std::uint32_t lbo,
                      std::uint32_t sbo, int bmajor, std::uint32_t kstep) {
    extern __shared__ __align__(1024) std::uint8_t smem_raw[];
    std::uint8_t* sm = reinterpret_cast<std::uint8_t*>(
        (reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) & ~std::uintptr_t{1023});
    std::uint8_t* sa = sm;            // 16 KiB
    std::uint8_t* sb = sm + 16384;    // 16 KiB
    std::uint64_t* bar = reinterpret_cast<std::uint64_t*>(sm + 32768);
    std::uint32_t* slot = reinterpret_cast<std::uint32_t*>(bar + 1);
    const int tid = threadIdx.x;
    // A: 128 rows x 32 K, K-major SW128
    for (int i = tid; i < 128 * 32; i += blockDim.x) {
        const int r = i / 32, k = i % 32;
        const std::uint32_t off = (r >> 3) * 1024 + (r & 7) * 128 + (((k >> 2) ^ (r & 7)) << 4) + (k & 3) * 4;
        *reinterpret_cast<float*>(sa + off) = A[r * 32 + k];
    }
    // B: K = 32 x N = 128 (B[k][n])
    for (int i = tid; i < 32 * 128; i += blockDim.x) {
        const int k = i / 128, nn = i % 128;
        std::uint32_t off;
        if (bmajor) {
            off = b_off(layout, k, nn);
        } else {  // K-major control: row = n
            off = (nn >> 3) * 1024 + (nn & 7) * 128 + (((k >> 2) ^ (nn & 7)) << 4) + (k & 3) * 4;
        }
        *reinterpret_cast<float*>(sb + off) = B[k * 128 + nn];
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (tid < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const std::uint32_t tmem = *slot;
    const std::uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<std::uint32_t>(bmajor) << 16) |
                                ((128 >> 3) << 17) | ((128 >> 4) << 24);
    if (tid == 0) {
        for (int k = 0; k < 4; ++k) {
            const std::uint64_t da = desc(smem_u32(sa) + k * 32, 16, 1024);
            const std::uint64_t db = bmajor ? desc(smem_u32(sb) + k * kstep, lbo, sbo)
                                            : desc(smem_u32(sb) + k * 32, 16, 1024);
            asm volatile(
                "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                "l"(da), "l"(db), "r"(idesc), "r"(k > 0 ? 1u : 0u));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(bar)));
    }
    __syncwarp();
    asm volatile(
        "{\n.reg .pred done;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 done, [%0], 0;\n@!done bra W;\n}\n" ::"r"(
            smem_u32(bar)));
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (tid < 128) {
        const int w = tid >> 5;
        for (int c = 0; c < 128; ++c) {
            std::uint32_t v;
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];"
                         : "=r"(v)
                         : "r"(tmem + (static_cast<std::uint32_t>(w * 32) << 16) + c));
            asm volatile("tcgen05.wait::ld.sync.aligned;");
            C[tid * 128 + c] = __uint_as_float(v);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
}

int main() {
    std::vector<float> A(128 * 32), B(32 * 128), C(128 * 128), R(128 * 128);
    std::srand(3);
    for (auto& x : A) x = static_cast<float>(std::rand() % 9 - 4);
    for (auto& x : B) x = static_cast<float>(std::rand() % 9 - 4);
    for (int i = 0; i < 128; ++i)
        for (int j = 0; j < 128; ++j) {
            double s = 0;
            for (int k = 0; k < 32; ++k) s += double(A[i * 32 + k]) * B[k * 128 + j];
            R[i * 128 + j] = static_cast<float>(s);
        }
    float *dA, *dB, *dC;
    cudaMalloc(&dA, A.size() * 4);
    cudaMalloc(&dB, B.size() * 4);
    cudaMalloc(&dC, C.size() * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024);
    struct V {
        int layout, bmajor;
        std::uint32_t lbo, sbo, kstep;
        const char* name;
    } vs[] = {
        {0, 0, 0, 0, 0, "K-major control"},
        {0, 1, 4096, 1024, 1024, "atoms 4K apart: LBO=4096 SBO=1024"},
        {0, 1, 1024, 4096, 1024, "atoms 4K apart: LBO=1024 SBO=4096"},
        {1, 1, 1024, 4096, 4096, "groups 4K apart: LBO=1024 SBO=4096"},
        {1, 1, 4096, 1024, 4096, "groups 4K apart: LBO=4096 SBO=1024"},
    };
    for (const auto& v : vs) {
        cudaMemset(dC, 0, C.size() * 4);
        probe<<<1, 128, 40 * 1024>>>(dA, dB, dC, v.layout, v.lbo, v.sbo, v.bmajor, v.kstep);
        const cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost);
        double err = 0;
        int nz = 0;
        for (size_t i = 0; i < C.size(); ++i) {
            err = std::max(err, static_cast<double>(std::abs(C[i] - R[i])));
            nz += C[i] != 0.0f;
        }
        std::printf("%-40s err=%s maxabs=%g nonzero=%d C[0][0..3]=%g %g %g %g ref=%g %g %g %g\n", v.name,
                    cudaGetErrorString(e), err, nz, C[0], C[1], C[2], C[3], R[0], R[1], R[2], R[3]);
        if (e != cudaSuccess) return 1;
    }
    return 0;
}
