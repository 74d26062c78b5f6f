// Payload registry. Contract from the reference (proj/src/payload.cpp:
// 49-73, SPEC.md register_payload/execute_payload): ids are unique, unknown
// ids and malformed inputs raise PayloadError, outputs are deterministic.
//
// The builtin ids are DEVICE bindings to sm_100a kernels in
// libvgpu_cuda.so; there is no CPU implementation of them in the product.
#include <cstdlib>
#include <string>

#include "vgpu/payload.hpp"
#include "vgpu_cuda.h"

namespace vgpu {

namespace {

int default_device() {
    const char* env = std::getenv("VGPU_CUDA_DEVICE");
    return env && *env ? std::atoi(env) : 0;
}

const char* kBuiltinIds[VGPU_CU_K_COUNT] = {
    "identity", "vector-add", "vector-scale", "nas-ep",         "black-scholes",
    "sgemm",    "vector-mul", "nas-cg",       "electrostatics", "nas-mg"};

}  // namespace

namespace detail {

Bytes DeviceKernelFn::operator()(ByteView input) const {
    std::uint64_t out_bytes = 0;
    int rc = vgpu_cu_output_size(k.kernel, input.data(), input.size(), &out_bytes);
    if (rc == VGPU_CU_EPAYLOAD)
        throw PayloadError(PayloadError::Kind::MalformedInput,
                           std::string(kBuiltinIds[k.kernel < VGPU_CU_K_COUNT ? k.kernel : 0]) +
                               ": " + vgpu_cu_last_error());
    if (rc != VGPU_CU_OK)
        throw std::runtime_error(std::string("payload: ") + vgpu_cu_strerror(rc));
    Bytes out(out_bytes);
    std::uint64_t written = 0;
    rc = vgpu_cu_execute(default_device(), k.kernel, k.param, input.data(),
                         input.size(), out.data(), out.size(), &written);
    if (rc == VGPU_CU_EPAYLOAD)
        throw PayloadError(PayloadError::Kind::MalformedInput, vgpu_cu_last_error());
    if (rc != VGPU_CU_OK)
        throw std::runtime_error(std::string("payload on CUDA device failed: ") +
                                 vgpu_cu_strerror(rc) + ": " + vgpu_cu_last_error());
    out.resize(written);
    return out;
}

}  // namespace detail

void PayloadRegistry::register_payload(std::string id, PayloadFn fn) {
    Entry e;
    if (const auto* dk = fn.target<detail::DeviceKernelFn>()) {
        e.on_device = true;
        e.dk = dk->k;
    }
    e.fn = std::move(fn);
    auto [it, fresh] = fns_.emplace(std::move(id), std::move(e));
    if (!fresh)
        throw PayloadError(PayloadError::Kind::DuplicateId,
                           "payload id already registered: " + it->first);
}

bool PayloadRegistry::contains(std::string_view id) const {
    return fns_.find(id) != fns_.end();
}

Bytes PayloadRegistry::execute(std::string_view id, ByteView input) const {
    const auto it = fns_.find(id);
    if (it == fns_.end())
        throw PayloadError(PayloadError::Kind::UnknownId,
                           "unknown payload id: " + std::string(id));
    return it->second.fn(input);
}

const DeviceKernel* PayloadRegistry::device_kernel(std::string_view id) const {
    const auto it = fns_.find(id);
    if (it == fns_.end() || !it->second.on_device) return nullptr;
    return &it->second.dk;
}

bool PayloadRegistry::needs_device() const {
    for (const auto& [id, e] : fns_)
        if (e.on_device) return true;
    return false;
}

PayloadFn make_vector_scale(float factor) {
    return detail::DeviceKernelFn{DeviceKernel{VGPU_CU_K_VSCALE, factor}};
}

PayloadRegistry PayloadRegistry::with_builtins() {
    PayloadRegistry r;
    for (std::uint32_t k = 0; k < VGPU_CU_K_COUNT; ++k) {
        const float param = k == VGPU_CU_K_VSCALE ? 2.0f : 0.0f;
        r.register_payload(kBuiltinIds[k], detail::DeviceKernelFn{DeviceKernel{k, param}});
    }
    return r;
}

const PayloadRegistry& PayloadRegistry::builtins() {
    static const PayloadRegistry r = with_builtins();
    return r;
}

}  // namespace vgpu
