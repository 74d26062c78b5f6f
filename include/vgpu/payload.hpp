// vgpu-b200 — payload registry: the ids a KernelDescriptor may name.
//
// API-identical to the reference (proj/include/vgpu/payload.hpp:15-46):
// PayloadFn is a bytes->bytes function and the registry maps ids to them.
//
// B200 difference (the point of the port): the builtin ids are bound to
// hand-written sm_100a kernels, not to CPU loops. A binding is either
//   * a DEVICE binding — the GVM batches it onto per-client CUDA streams
//     (libvgpu_cuda.so, include/vgpu_cuda.h), or
//   * a HOST binding — an arbitrary user PayloadFn, run on the dispatcher
//     thread exactly as the reference runs every payload (daemon.cpp:413).
// execute() on a device binding runs the kernel synchronously on the GPU and
// throws std::runtime_error when no CUDA device is usable: there is no CPU
// fallback for the builtin kernels.
//
// Builtin ids (input layout -> output layout):
//   identity       bytes -> the same bytes
//   vector-add     a||b, n fp32 each        -> a+b, n fp32     (reference)
//   vector-scale   n fp32                   -> 2*x, n fp32     (reference)
//   nas-ep         EpParams (32 B)          -> EpResult (112 B)  (new)
//   black-scholes  S||X||T, n fp32 each     -> call||put, n fp32 (new)
//   sgemm          A||B, n*n fp32 each      -> A*B, n*n fp32     (new)
//   vector-mul     a||b, n fp32 each        -> a*b, n fp32       (new)
//   nas-cg         CgHeader + CSR matrix    -> CgResult (32 B)   (new)
//   electrostatics EsHeader + atoms (x,y,z,q) -> lattice potential fp32 (new)
#ifndef VGPU_PAYLOAD_HPP
#define VGPU_PAYLOAD_HPP

#include <cstdint>
#include <functional>
#include <map>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

namespace vgpu {

using Bytes = std::vector<std::uint8_t>;
using ByteView = std::span<const std::uint8_t>;
using PayloadFn = std::function<Bytes(ByteView)>;

struct PayloadError : std::runtime_error {
    enum class Kind { UnknownId, DuplicateId, MalformedInput };
    PayloadError(Kind k, const std::string& what)
        : std::runtime_error(what), kind(k) {}
    Kind kind;
};

// A device kernel a payload id can be bound to (values = vgpu_cu_kernel in
// include/vgpu_cuda.h).
struct DeviceKernel {
    std::uint32_t kernel = 0;
    float param = 0.0f;  // vector-scale factor; unused by the others
};

namespace detail {
// Callable stored inside a PayloadFn built by make_vector_scale() or the
// builtins; the registry recovers it with std::function::target<>() so the
// GVM can batch the kernel instead of calling it synchronously.
struct DeviceKernelFn {
    DeviceKernel k;
    Bytes operator()(ByteView input) const;
};
}  // namespace detail

class PayloadRegistry {
public:
    void register_payload(std::string id, PayloadFn fn);
    bool contains(std::string_view id) const;
    Bytes execute(std::string_view id, ByteView input) const;

    static const PayloadRegistry& builtins();
    static PayloadRegistry with_builtins();

    // ---- B200 extensions -------------------------------------------------
    // Device binding of `id`, or nullptr for host payloads / unknown ids.
    const DeviceKernel* device_kernel(std::string_view id) const;
    // True when any id is bound to a device kernel (the GVM then needs CUDA).
    bool needs_device() const;

private:
    struct Entry {
        PayloadFn fn;
        bool on_device = false;
        DeviceKernel dk;
    };
    std::map<std::string, Entry, std::less<>> fns_;
};

PayloadFn make_vector_scale(float factor);

}  // namespace vgpu

#endif  // VGPU_PAYLOAD_HPP
