// C-ABI over the C++ host stack (include/vgpu_c.h). Exceptions never cross
// the boundary: each entry point maps them to a status code and keeps the
// detail in a thread-local string.
#include <cstring>
#include <sstream>
#include <string>

#include "vgpu/client.hpp"
#include "vgpu/daemon.hpp"
#include "vgpu/device.hpp"
#include "vgpu/model.hpp"
#include "vgpu/multigpu.hpp"
#include "vgpu/npb_cg.hpp"
#include "vgpu/npb_mg.hpp"
#include "vgpu_c.h"
#include "vgpu_cuda.h"

using namespace vgpu;

struct vgpu_gvm {
    std::unique_ptr<GvmDaemon> daemon;
};

struct vgpu_client {
    VgpuHandle handle;
};

namespace {

thread_local std::string t_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return VGPU_OK;
    } catch (const VgpuError& e) {
        t_err = e.what();
        return static_cast<int>(e.code());
    } catch (const TransportError& e) {
        t_err = e.what();
        return VGPU_E_TRANSPORT;
    } catch (const PayloadError& e) {
        t_err = e.what();
        return VGPU_E_PAYLOAD;
    } catch (const std::invalid_argument& e) {
        t_err = e.what();
        return VGPU_E_INVALID;
    } catch (const std::exception& e) {
        t_err = e.what();
        return VGPU_E_RUNTIME;
    }
}

GvmConfig to_cfg(const vgpu_gvm_config& c) {
    GvmConfig g;
    if (c.instance) g.instance = c.instance;
    g.max_clients = c.max_clients;
    g.barrier_size = c.barrier_size;
    g.per_client_shm_bytes = c.per_client_shm_bytes;
    g.barrier_window = c.barrier_window_us;
    g.t_init = c.t_init_us;
    g.t_ctx_switch = c.t_ctx_switch_us;
    g.clock = c.clock ? ClockMode::Real : ClockMode::Virtual;
    g.cuda_device = c.cuda_device;
    g.data_plane = c.data_plane ? DataPlane::Snapshot : DataPlane::ZeroCopy;
    g.device.num_sms = c.device_sms;
    g.device.max_concurrent_kernels = c.device_max_kernels;
    g.device.block_slots_per_sm = c.device_slots_per_sm;
    g.scale = c.scale;
    return g;
}

KernelDescriptor to_desc(const vgpu_descriptor* d) {
    KernelDescriptor k;
    if (!d) throw std::invalid_argument("null descriptor");
    k.payload_id = d->payload_id ? d->payload_id : "identity";
    k.t_data_in = d->t_data_in;
    k.t_comp = d->t_comp;
    k.t_data_out = d->t_data_out;
    k.grid_size = d->grid_size;
    k.output_bytes = d->output_bytes;
    return k;
}

void copy_out(const Bytes& b, void* out, std::uint64_t cap, std::uint64_t* len) {
    if (len) *len = b.size();
    if (b.size() > cap) throw VgpuError(ErrCode::Size, "output buffer too small");
    if (!b.empty()) std::memcpy(out, b.data(), b.size());
}

}  // namespace

extern "C" {

int vgpu_gvm_fold(vgpu_gvm* g, double* out16) {
    if (!g || !out16) return VGPU_E_INVALID;
    return guarded([&] {
        const auto rec = g->daemon->fold_record();
        std::memcpy(out16, rec.data(), sizeof(double) * rec.size());
    });
}

int vgpu_rendezvous_publish(const char* path, const void* data, uint64_t n) {
    if (!path || (!data && n)) return VGPU_E_INVALID;
    return guarded([&] {
        multigpu::publish_id(path, {static_cast<const std::uint8_t*>(data), static_cast<std::size_t>(n)});
    });
}

int vgpu_rendezvous_fetch(const char* path, void* out, uint64_t n, int64_t timeout_ms) {
    if (!path || (!out && n)) return VGPU_E_INVALID;
    return guarded([&] {
        const auto id = multigpu::fetch_id(path, n, std::chrono::milliseconds(std::max<int64_t>(0, timeout_ms)));
        std::memcpy(out, id.data(), id.size());
    });
}

int vgpu_fold_in_rank_order(const double* all, uint32_t nranks, double* out16) {
    if (!all || !out16 || nranks == 0) return VGPU_E_INVALID;
    return guarded([&] {
        const auto rec = multigpu::fold_in_rank_order({all, static_cast<std::size_t>(nranks) * 16}, nranks);
        std::memcpy(out16, rec.data(), sizeof(double) * rec.size());
    });
}

int vgpu_local_cpus(const char* pci_bus_id, int32_t* out, uint32_t cap, uint32_t* n) {
    if (!pci_bus_id || !n || (!out && cap)) return VGPU_E_INVALID;
    return guarded([&] {
        const auto cpus = multigpu::local_cpus(pci_bus_id);
        *n = static_cast<uint32_t>(cpus.size());
        for (uint32_t i = 0; i < std::min<uint32_t>(cap, *n); ++i) out[i] = cpus[i];
    });
}

int vgpu_mg_class(char cls, uint32_t* nx, uint32_t* nit, uint32_t* coeffs, double* rnm2_verify) {
    if (!nx || !nit || !coeffs || !rnm2_verify) return VGPU_E_INVALID;
    return guarded([&] {
        const npb::MgClass c = npb::mg_class(cls);
        *nx = c.nx;
        *nit = c.nit;
        *coeffs = c.coeffs;
        *rnm2_verify = c.rnm2_verify;
    });
}

int vgpu_mg_make_input(uint32_t nx, uint32_t nit, uint32_t coeffs, uint8_t* out, uint64_t cap,
                       uint64_t* len) {
    if (!len) return VGPU_E_INVALID;
    return guarded([&] {
        *len = vgpu_mg_input_bytes(nx);
        if (!out) return;
        if (cap < *len) throw VgpuError(ErrCode::Size, "nas-mg input exceeds the buffer");
        const auto b = npb::make_mg_input(nx, nit, coeffs);
        std::memcpy(out, b.data(), b.size());
    });
}

const char* vgpu_last_error(void) { return t_err.c_str(); }

void vgpu_gvm_config_default(vgpu_gvm_config* c) {
    if (!c) return;
    const GvmConfig g;
    std::memset(c, 0, sizeof *c);
    c->instance = nullptr;
    c->max_clients = g.max_clients;
    c->barrier_size = g.barrier_size;
    c->per_client_shm_bytes = g.per_client_shm_bytes;
    c->barrier_window_us = g.barrier_window;
    c->t_init_us = g.t_init;
    c->t_ctx_switch_us = g.t_ctx_switch;
    c->clock = 0;
    c->cuda_device = g.cuda_device;
    c->data_plane = 0;
    c->device_sms = g.device.num_sms;
    c->device_max_kernels = g.device.max_concurrent_kernels;
    c->device_slots_per_sm = g.device.block_slots_per_sm;
    c->scale = g.scale;
}

int vgpu_gvm_start_os(const vgpu_gvm_config* cfg, vgpu_gvm** out) {
    if (!cfg || !out) return VGPU_E_INVALID;
    *out = nullptr;
    return guarded([&] {
        auto g = std::make_unique<vgpu_gvm>();
        g->daemon = GvmDaemon::start_os(to_cfg(*cfg));
        *out = g.release();
    });
}

int vgpu_gvm_stop(vgpu_gvm* g) {
    if (!g) return VGPU_E_INVALID;
    return guarded([&] { g->daemon->stop(); });
}

void vgpu_gvm_destroy(vgpu_gvm* g) {
    if (!g) return;
    try {
        delete g;
    } catch (...) {
    }
}

int vgpu_gvm_summary_get(vgpu_gvm* g, vgpu_gvm_summary* out) {
    if (!g || !out) return VGPU_E_INVALID;
    return guarded([&] {
        const MetricsSnapshot m = g->daemon->metrics();
        out->tasks = m.tasks.size();
        out->batches_flushed = m.batches_flushed;
        out->uptime_us = m.uptime_us;
        out->busy_us = m.busy_us;
        out->t_init_us = m.t_init_us;
        out->kernel_launches = m.kernel_launches;
        out->device_tasks = m.device_tasks;
    });
}

int vgpu_gvm_tasks(vgpu_gvm* g, vgpu_task_metrics* out, uint32_t cap, uint32_t* n) {
    if (!g || !n) return VGPU_E_INVALID;
    return guarded([&] {
        const MetricsSnapshot m = g->daemon->metrics();
        *n = static_cast<uint32_t>(m.tasks.size());
        for (uint32_t i = 0; i < std::min<uint32_t>(cap, *n); ++i) {
            const auto& t = m.tasks[i];
            out[i] = vgpu_task_metrics{t.task_id, t.client_id, 0, t.queue_wait_us,
                                       t.pure_gpu_us, t.end_to_end_us, t.h2d_us, t.comp_us,
                                       t.d2h_us};
        }
    });
}

int vgpu_gvm_batches(vgpu_gvm* g, vgpu_batch_metrics* out, uint32_t cap, uint32_t* n) {
    if (!g || !n) return VGPU_E_INVALID;
    return guarded([&] {
        const MetricsSnapshot m = g->daemon->metrics();
        *n = static_cast<uint32_t>(m.batches.size());
        for (uint32_t i = 0; i < std::min<uint32_t>(cap, *n); ++i) {
            const auto& b = m.batches[i];
            out[i] = vgpu_batch_metrics{b.batch_id, b.style == ProgrammingStyle::PS2 ? 1 : 0,
                                        b.task_count, b.model_makespan_us,
                                        b.measured_makespan_us};
        }
    });
}

int vgpu_gvm_metrics_csv(vgpu_gvm* g, char* buf, uint64_t cap, uint64_t* len) {
    if (!g || !len) return VGPU_E_INVALID;
    return guarded([&] {
        std::ostringstream os;
        write_metrics_csv(g->daemon->metrics(), os);
        const std::string s = os.str();
        *len = s.size();
        if (buf && cap) {
            const std::size_t k = std::min<std::size_t>(cap - 1, s.size());
            std::memcpy(buf, s.data(), k);
            buf[k] = '\0';
        }
    });
}

int vgpu_gvm_timeline_csv(vgpu_gvm* g, char* buf, uint64_t cap, uint64_t* len) {
    if (!g || !len) return VGPU_E_INVALID;
    return guarded([&] {
        std::ostringstream os;
        write_timeline_csv(g->daemon->metrics().device_timeline, os);
        const std::string s = os.str();
        *len = s.size();
        if (buf && cap) {
            const std::size_t k = std::min<std::size_t>(cap - 1, s.size());
            std::memcpy(buf, s.data(), k);
            buf[k] = '\0';
        }
    });
}

int vgpu_unlink_instance(const char* instance, uint32_t max_clients) {
    if (!instance) return VGPU_E_INVALID;
    return guarded([&] { unlink_os_instance(instance, max_clients); });
}

int vgpu_client_req(const char* instance, vgpu_client** out) {
    if (!out) return VGPU_E_INVALID;
    *out = nullptr;
    return guarded([&] {
        auto c = new vgpu_client{req(instance ? std::string(instance) : std::string())};
        *out = c;
    });
}

void vgpu_client_free(vgpu_client* c) { delete c; }

uint32_t vgpu_client_id(const vgpu_client* c) { return c ? c->handle.client_id() : 0; }
uint64_t vgpu_client_shm_bytes(const vgpu_client* c) { return c ? c->handle.lease().shm_bytes : 0; }
int vgpu_client_phase(const vgpu_client* c) {
    return c ? static_cast<int>(c->handle.phase()) : -1;
}

int vgpu_client_snd(vgpu_client* c, const void* data, uint64_t bytes) {
    if (!c || (!data && bytes)) return VGPU_E_INVALID;
    return guarded([&] {
        c->handle.snd({static_cast<const std::uint8_t*>(data), static_cast<std::size_t>(bytes)});
    });
}

int vgpu_client_str(vgpu_client* c, const vgpu_descriptor* d) {
    if (!c) return VGPU_E_INVALID;
    return guarded([&] { c->handle.str(to_desc(d)); });
}

int vgpu_client_stp(vgpu_client* c, int* done) {
    if (!c || !done) return VGPU_E_INVALID;
    return guarded([&] { *done = c->handle.stp() ? 1 : 0; });
}

int vgpu_client_stp_wait(vgpu_client* c) {
    if (!c) return VGPU_E_INVALID;
    return guarded([&] { c->handle.stp_wait(); });
}

int vgpu_client_rcv(vgpu_client* c, void* out, uint64_t cap, uint64_t* len) {
    if (!c || !len) return VGPU_E_INVALID;
    return guarded([&] {
        *len = c->handle.rcv_into({static_cast<std::uint8_t*>(out), static_cast<std::size_t>(cap)});
    });
}

int vgpu_client_rls(vgpu_client* c) {
    if (!c) return VGPU_E_INVALID;
    return guarded([&] { c->handle.rls(); });
}

int vgpu_client_run_task(vgpu_client* c, const void* in, uint64_t in_bytes,
                         const vgpu_descriptor* d, void* out, uint64_t cap, uint64_t* len) {
    if (!c || !len || (!in && in_bytes)) return VGPU_E_INVALID;
    return guarded([&] {
        c->handle.snd({static_cast<const std::uint8_t*>(in), static_cast<std::size_t>(in_bytes)});
        c->handle.str(to_desc(d));
        c->handle.stp_wait();
        *len = c->handle.rcv_into({static_cast<std::uint8_t*>(out), static_cast<std::size_t>(cap)});
    });
}

int vgpu_client_region(vgpu_client* c, void** base, uint64_t* bytes) {
    if (!c || !base || !bytes) return VGPU_E_INVALID;
    return guarded([&] {
        const auto r = c->handle.region();
        *base = r.data();
        *bytes = r.size();
    });
}

int vgpu_client_snd_region(vgpu_client* c, uint64_t bytes) {
    if (!c) return VGPU_E_INVALID;
    return guarded([&] { c->handle.snd_region(bytes); });
}

int vgpu_client_snd_region_at(vgpu_client* c, uint64_t offset, uint64_t bytes) {
    if (!c) return VGPU_E_INVALID;
    return guarded([&] { c->handle.snd_region_at(offset, bytes); });
}

int vgpu_client_rcv_region(vgpu_client* c, const void** data, uint64_t* len) {
    if (!c || !data || !len) return VGPU_E_INVALID;
    return guarded([&] {
        const auto r = c->handle.rcv_region();
        *data = r.data();
        *len = r.size();
    });
}

int vgpu_client_run_task_region(vgpu_client* c, uint64_t in_bytes, const vgpu_descriptor* d,
                                const void** data, uint64_t* len) {
    if (!c || !data || !len) return VGPU_E_INVALID;
    return guarded([&] {
        const auto r = c->handle.run_task_region(in_bytes, to_desc(d));
        *data = r.data();
        *len = r.size();
    });
}

int vgpu_native_run_task(int cuda_device, const vgpu_descriptor* d, const void* in,
                         uint64_t in_bytes, void* out, uint64_t cap, uint64_t* len) {
    if (!len || (!in && in_bytes)) return VGPU_E_INVALID;
    return guarded([&] {
        NativeConfig nc;
        nc.cuda_device = cuda_device;
        NativeVgpu h{nc};
        const Bytes r = h.run_task(
            {static_cast<const std::uint8_t*>(in), static_cast<std::size_t>(in_bytes)}, to_desc(d));
        copy_out(r, out, cap, len);
    });
}

uint64_t vgpu_model_simulate(int style, uint32_t n, uint64_t t_in, uint64_t t_comp,
                             uint64_t t_out, uint32_t grid, uint32_t sms, uint32_t max_kernels,
                             uint32_t slots_per_sm) {
    try {
        KernelProfile p;
        p.t_data_in = t_in;
        p.t_comp = t_comp;
        p.t_data_out = t_out;
        p.grid_size = grid;
        std::vector<KernelProfile> ps(n, p);
        DeviceSpec dev;
        dev.num_sms = sms;
        dev.max_concurrent_kernels = max_kernels;
        dev.block_slots_per_sm = slots_per_sm;
        return simulate(build_work_queue(style ? ProgrammingStyle::PS2 : ProgrammingStyle::PS1, ps),
                        dev)
            .makespan;
    } catch (const std::exception& e) {
        t_err = e.what();
        return 0;
    }
}

uint64_t vgpu_model_simulate_fluid(int style, uint32_t n, uint64_t t_in, uint64_t t_comp,
                                   uint64_t t_out, uint32_t grid, uint32_t sms,
                                   uint32_t ctas_per_sm, uint64_t launch_us, int shared) {
    try {
        KernelProfile p;
        p.t_data_in = t_in;
        p.t_comp = t_comp;
        p.t_data_out = t_out;
        p.grid_size = grid;
        std::vector<KernelProfile> ps(n, p);
        DeviceSpec dev = DeviceSpec::b200();
        dev.num_sms = sms;
        dev.block_slots_per_sm = ctas_per_sm;
        dev.fluid_blocks = shared ? 2 : 1;
        dev.kernel_launch_us = static_cast<std::uint16_t>(std::min<uint64_t>(launch_us, 65535));
        return simulate(build_work_queue(style ? ProgrammingStyle::PS2 : ProgrammingStyle::PS1, ps),
                        dev)
            .makespan;
    } catch (const std::exception& e) {
        t_err = e.what();
        return 0;
    }
}

int vgpu_model_classify(uint64_t t_in, uint64_t t_comp, uint64_t t_out) {
    KernelProfile p;
    p.t_data_in = t_in;
    p.t_comp = t_comp;
    p.t_data_out = t_out;
    return static_cast<int>(classify_kernel(p));
}

uint64_t vgpu_model_no_vt(uint32_t n, uint64_t t_init, uint64_t t_ctx, uint64_t t_in,
                          uint64_t t_comp, uint64_t t_out) {
    try {
        ModelParams m;
        m.n_process = n;
        m.t_init = t_init;
        m.t_ctx_switch = t_ctx;
        m.profile.t_data_in = t_in;
        m.profile.t_comp = t_comp;
        m.profile.t_data_out = t_out;
        return t_total_no_vt(m);
    } catch (const std::exception& e) {
        t_err = e.what();
        return 0;
    }
}

int vgpu_cg_class(char cls, uint32_t* n, uint32_t* nonzer, uint32_t* niter, double* shift,
                  double* zeta_verify) {
    if (!n || !nonzer || !niter || !shift || !zeta_verify) return VGPU_E_INVALID;
    return guarded([&] {
        const npb::CgClass c = npb::cg_class(cls);
        *n = c.n;
        *nonzer = c.nonzer;
        *niter = c.niter;
        *shift = c.shift;
        *zeta_verify = c.zeta_verify;
    });
}

int vgpu_cg_make_input(uint32_t n, uint32_t nonzer, uint32_t niter, double shift, uint8_t* out,
                       uint64_t cap, uint64_t* len) {
    if (!len) return VGPU_E_INVALID;
    return guarded([&] {
        const std::vector<std::uint8_t> b = npb::make_cg_input(n, nonzer, niter, shift);
        *len = b.size();
        if (!out) return;
        if (cap < b.size()) throw std::invalid_argument("vgpu_cg_make_input: buffer too small");
        std::memcpy(out, b.data(), b.size());
    });
}

int vgpu_encode_frame(uint8_t opcode, uint32_t client_id, uint64_t task_id, const uint8_t* payload,
                      uint64_t payload_len, uint8_t* out, uint64_t cap, uint64_t* len) {
    if (!len || (!payload && payload_len)) return VGPU_E_INVALID;
    Message m;
    m.opcode = static_cast<Opcode>(opcode);
    m.client_id = client_id;
    m.task_id = task_id;
    if (payload_len) m.payload.assign(payload, payload + payload_len);
    const auto f = encode(m);
    *len = f.size();
    if (f.size() > cap || !out) return VGPU_E_INVALID;
    std::memcpy(out, f.data(), f.size());
    return VGPU_OK;
}

int vgpu_decode_frame(const uint8_t* frame, uint64_t len, uint8_t* opcode, uint32_t* client_id,
                      uint64_t* task_id, uint64_t* payload_len) {
    if (!frame && len) return VGPU_E_INVALID;
    const auto r = decode({frame, static_cast<std::size_t>(len)});
    if (const auto* e = std::get_if<DecodeError>(&r)) return 1 + static_cast<int>(*e);
    const Message& m = std::get<Message>(r);
    if (opcode) *opcode = static_cast<uint8_t>(m.opcode);
    if (client_id) *client_id = m.client_id;
    if (task_id) *task_id = m.task_id;
    if (payload_len) *payload_len = m.payload.size();
    return VGPU_OK;
}

}  // extern "C"
