// vgpu::kernels (include/vgpu/payload_kernels.hpp): the builtin payloads'
// element-wise kernels. The reference runs them as OpenMP loops
// (proj/src/payload_kernels.cpp); here the data-parallel versions are the
// sm_100a stream kernels through vgpu_cu_execute (this process's own
// context, device 0 or $VGPU_DEVICE), checked bit for bit against the
// serial loops by the reference's own test_payload.cpp.
#include "vgpu/payload_kernels.hpp"

#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "vgpu/payload.hpp"
#include "vgpu_cuda.h"

namespace vgpu::kernels {

namespace {

int device() {
    const char* e = std::getenv("VGPU_DEVICE");
    return e ? std::atoi(e) : 0;
}

void run(std::uint32_t kernel, float param, const std::vector<float>& in, float* out, std::size_t n) {
    std::uint64_t written = 0;
    const int rc = vgpu_cu_execute(device(), kernel, param, in.data(), in.size() * sizeof(float), out,
                                   n * sizeof(float), &written);
    if (rc != VGPU_CU_OK || written != n * sizeof(float))
        throw PayloadError(PayloadError::Kind::MalformedInput,
                           std::string("kernels: CUDA device path failed: ") + vgpu_cu_strerror(rc) + ": " +
                               vgpu_cu_last_error());
}

}  // namespace

void vector_add(float* out, const float* a, const float* b, std::size_t n) {
    if (n == 0) return;
    std::vector<float> in(2 * n);  // the payload's input layout: a || b
    std::memcpy(in.data(), a, n * sizeof(float));
    std::memcpy(in.data() + n, b, n * sizeof(float));
    run(VGPU_CU_K_VADD, 0.0f, in, out, n);
}

void vector_add_serial(float* out, const float* a, const float* b, std::size_t n) {
    for (std::size_t i = 0; i < n; ++i) out[i] = a[i] + b[i];
}

void vector_scale(float* out, const float* in, float factor, std::size_t n) {
    if (n == 0) return;
    run(VGPU_CU_K_VSCALE, factor, std::vector<float>(in, in + n), out, n);
}

void vector_scale_serial(float* out, const float* in, float factor, std::size_t n) {
    for (std::size_t i = 0; i < n; ++i) out[i] = factor * in[i];
}

}  // namespace vgpu::kernels
