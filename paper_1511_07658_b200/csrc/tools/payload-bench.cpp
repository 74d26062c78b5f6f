// payload-bench — device throughput of every payload kernel, the B200
// counterpart of the reference's CPU payload-bench
// (proj/tools/payload_bench.cpp:28-58): inputs resident in HBM, rotating
// input sets larger than L2, CUDA-event timing, GB/s and GFLOP/s.
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "vgpu/npb_mg.hpp"
#include "vgpu_cuda.h"
#include "workloads.hpp"

int main(int argc, char** argv) {
    // payload-bench [device] [kind|all] [tasks|0=1,4,16] [steps]   (mg: NPB class S)
    int device = argc > 1 ? std::atoi(argv[1]) : 0;
    const std::string only = argc > 2 ? argv[2] : "all";
    const std::uint32_t only_tasks = argc > 3 ? std::atoi(argv[3]) : 0;
    const std::uint32_t steps = argc > 4 ? std::atoi(argv[4]) : 20;
    vgpu::wl::mg_builder() = [](char cls) {
        const vgpu::npb::MgClass c = vgpu::npb::mg_class(cls);
        return vgpu::npb::make_mg_input(c.nx, c.nit, c.coeffs);
    };
    const char* kinds[] = {"vecadd", "ep", "bs", "mm", "mg"};
    const std::uint32_t kernels[] = {VGPU_CU_K_VADD, VGPU_CU_K_EP, VGPU_CU_K_BS, VGPU_CU_K_SGEMM,
                                     VGPU_CU_K_MG};
    for (int k = 0; k < 5; ++k) {
        if (only != "all" && only != kinds[k]) continue;
        const std::vector<std::uint32_t> counts =
            only_tasks ? std::vector<std::uint32_t>{only_tasks} : std::vector<std::uint32_t>{1, 4, 16};
        for (std::uint32_t tasks : counts) {
            std::vector<vgpu::wl::Job> jobs;
            std::vector<const void*> ptrs;
            std::vector<std::uint64_t> sizes;
            for (std::uint32_t w = 0; w < tasks; ++w)
                jobs.push_back(vgpu::wl::make_job(kinds[k], w, tasks));
            std::uint64_t set_bytes = 0;
            for (auto& j : jobs) {
                ptrs.push_back(j.input.data());
                sizes.push_back(j.input.size());
                set_bytes += j.input.size() + j.output_bytes;
            }
            const std::uint32_t sets =
                static_cast<std::uint32_t>(std::min<std::uint64_t>(16, 1 + (512ull << 20) / (set_bytes + 1)));
            vgpu_cu_resident_result r{};
            const int rc = vgpu_cu_resident_bench(device, kernels[k], 2.0f, tasks, ptrs.data(),
                                                  sizes.data(), sets, 3, steps, 0, &r);
            if (rc) {
                std::printf("%-7s tasks=%2u  error %s: %s\n", kinds[k], tasks, vgpu_cu_strerror(rc),
                            vgpu_cu_last_error());
                return 1;
            }
            const double s = r.kernel_ms_per_launch * 1e-3;
            std::printf("%-7s tasks=%2u launches/step=%u  kernel %.3f ms  %.1f GB/s  %.2f G(FL)OP/s  "
                        "step %.3f ms (sets=%u)\n",
                        kinds[k], tasks, r.launches_per_step, r.kernel_ms_per_launch,
                        r.algo_bytes_per_launch / s / 1e9, r.algo_flops_per_launch / s / 1e9,
                        r.ms_per_step, r.sets);
        }
    }
    return 0;
}
