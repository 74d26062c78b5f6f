// NVTX ranges for the GVM's verbs and device stages (nsys / ncu timelines).
// NVTX3 is header-only: without a profiler attached a range costs a branch.
#pragma once

#include <nvtx3/nvToolsExt.h>

namespace vgpu::trace {

inline nvtxDomainHandle_t domain() {
    static nvtxDomainHandle_t d = nvtxDomainCreateA("vgpu");
    return d;
}

// RAII: one range on the calling thread, named with a string literal
class Range {
public:
    explicit Range(const char* name) {
        nvtxEventAttributes_t a{};
        a.version = NVTX_VERSION;
        a.size = NVTX_EVENT_ATTRIB_STRUCT_SIZE;
        a.messageType = NVTX_MESSAGE_TYPE_ASCII;
        a.message.ascii = name;
        nvtxDomainRangePushEx(domain(), &a);
    }
    ~Range() { nvtxDomainRangePop(domain()); }
    Range(const Range&) = delete;
    Range& operator=(const Range&) = delete;
};

}  // namespace vgpu::trace
