/*
 * vgpu-b200 — C-ABI of the host stack (libvgpu.so), for FFI callers.
 *
 * The reference exposes only a C++ API (proj/include/vgpu/client.hpp:41-113,
 * daemon.hpp:69-96); a ctypes/cgo/JNI binding needs plain C. Each entry
 * point below wraps exactly one reference call:
 *   vgpu_gvm_start_os      GvmDaemon::start_os            daemon.hpp:79  (daemon.cpp:629-634)
 *   vgpu_gvm_stop          GvmDaemon::stop                daemon.hpp:85  (daemon.cpp:638-643)
 *   vgpu_gvm_metrics*      GvmDaemon::metrics + write_metrics_csv  daemon.hpp:68,:86
 *   vgpu_unlink_instance   unlink_os_instance             transport.hpp:173
 *   vgpu_client_req        req(instance)                  client.hpp:69   (client.cpp:146-153)
 *   vgpu_client_snd/str/stp/stp_wait/rcv/rls/run_task
 *                          VgpuHandle::snd .. run_task    client.hpp:41-48 (client.cpp:71-142)
 *   vgpu_client_region/snd_region/rcv_region/run_task_region
 *                          B200 in-place data plane (no reference counterpart;
 *                          same frames as snd/rcv, client.cpp:71-80, :116-127)
 *   vgpu_native_run_task   NativeVgpu::run_task           client.hpp:101  (client.cpp:250-256)
 * Status: 0 ok; 1..8 = vgpu::ErrCode (NACK codes verbatim); VGPU_E_* below.
 * The detail string of the last failure on this thread: vgpu_last_error().
 */
#ifndef VGPU_C_H
#define VGPU_C_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    VGPU_OK = 0,
    /* 1..8: vgpu::ErrCode Phase, NoLease, Size, Pending, Payload, Full, Malformed, Internal */
    VGPU_E_TRANSPORT = 20, /* vgpu::TransportError (endpoint missing, socket failure) */
    VGPU_E_INVALID = 21,   /* std::invalid_argument (bad config / argument)         */
    VGPU_E_RUNTIME = 22,   /* other failures (e.g. CUDA device unavailable)         */
    VGPU_E_PAYLOAD = 23    /* vgpu::PayloadError thrown client-side                 */
};

typedef struct vgpu_gvm_config {
    const char* instance;          /* NULL -> "default"                         */
    uint32_t max_clients;
    uint32_t barrier_size;         /* 0 = max_clients                            */
    uint64_t per_client_shm_bytes;
    uint64_t barrier_window_us;
    uint64_t t_init_us;
    uint64_t t_ctx_switch_us;
    int32_t clock;                 /* 0 virtual, 1 real                          */
    int32_t cuda_device;
    int32_t data_plane;            /* 0 zero-copy, 1 snapshot                    */
    uint32_t device_sms;           /* DeviceSpec for the model prediction        */
    uint32_t device_max_kernels;
    uint32_t device_slots_per_sm;
    double scale;
} vgpu_gvm_config;

typedef struct vgpu_descriptor {
    const char* payload_id;
    uint64_t t_data_in;
    uint64_t t_comp;
    uint64_t t_data_out;
    uint32_t grid_size;
    uint64_t output_bytes;
} vgpu_descriptor;

typedef struct vgpu_gvm_summary {
    uint64_t tasks;
    uint64_t batches_flushed;
    uint64_t uptime_us;
    uint64_t busy_us;
    uint64_t t_init_us;
    uint64_t kernel_launches;
    uint64_t device_tasks;
} vgpu_gvm_summary;

typedef struct vgpu_task_metrics {
    uint64_t task_id;
    uint32_t client_id;
    uint32_t pad;
    uint64_t queue_wait_us;
    uint64_t pure_gpu_us;
    uint64_t end_to_end_us;
    double h2d_us, comp_us, d2h_us;
} vgpu_task_metrics;

typedef struct vgpu_batch_metrics {
    uint64_t batch_id;
    int32_t style; /* 0 PS1, 1 PS2 */
    uint32_t task_count;
    uint64_t model_makespan_us;
    uint64_t measured_makespan_us;
} vgpu_batch_metrics;

typedef struct vgpu_gvm vgpu_gvm;
typedef struct vgpu_client vgpu_client;

void vgpu_gvm_config_default(vgpu_gvm_config* cfg);
int vgpu_gvm_start_os(const vgpu_gvm_config* cfg, vgpu_gvm** out);
int vgpu_gvm_stop(vgpu_gvm* g);
void vgpu_gvm_destroy(vgpu_gvm* g);
int vgpu_gvm_summary_get(vgpu_gvm* g, vgpu_gvm_summary* out);
int vgpu_gvm_tasks(vgpu_gvm* g, vgpu_task_metrics* out, uint32_t cap, uint32_t* n);
int vgpu_gvm_batches(vgpu_gvm* g, vgpu_batch_metrics* out, uint32_t cap, uint32_t* n);
/* write_metrics_csv into buf; *len = full length even when truncated */
int vgpu_gvm_metrics_csv(vgpu_gvm* g, char* buf, uint64_t cap, uint64_t* len);
/* the measured schedule (MetricsSnapshot::device_timeline) in the
 * reference's timeline CSV schema (write_timeline_csv, device.cpp) */
int vgpu_gvm_timeline_csv(vgpu_gvm* g, char* buf, uint64_t cap, uint64_t* len);
int vgpu_unlink_instance(const char* instance, uint32_t max_clients);

int vgpu_client_req(const char* instance, vgpu_client** out);
void vgpu_client_free(vgpu_client* c); /* releases a live lease like ~VgpuHandle */
uint32_t vgpu_client_id(const vgpu_client* c);
uint64_t vgpu_client_shm_bytes(const vgpu_client* c);
int vgpu_client_phase(const vgpu_client* c); /* vgpu::Phase ordinal */
int vgpu_client_snd(vgpu_client* c, const void* data, uint64_t bytes);
int vgpu_client_str(vgpu_client* c, const vgpu_descriptor* d);
int vgpu_client_stp(vgpu_client* c, int* done);
int vgpu_client_stp_wait(vgpu_client* c);
int vgpu_client_rcv(vgpu_client* c, void* out, uint64_t cap, uint64_t* len);
int vgpu_client_rls(vgpu_client* c);
int vgpu_client_run_task(vgpu_client* c, const void* in, uint64_t in_bytes,
                         const vgpu_descriptor* d, void* out, uint64_t cap, uint64_t* len);
/* In-place data plane (B200 extension, VgpuHandle::region / snd_region /
 * rcv_region / run_task_region): the leased region, page-locked by the GVM,
 * holds the input the caller wrote there and, after RCV, the result (a view:
 * valid until the next SND or RLS; it overwrites the region from offset 0). */
int vgpu_client_region(vgpu_client* c, void** base, uint64_t* bytes);
int vgpu_client_snd_region(vgpu_client* c, uint64_t bytes);
int vgpu_client_snd_region_at(vgpu_client* c, uint64_t offset, uint64_t bytes);
int vgpu_client_rcv_region(vgpu_client* c, const void** data, uint64_t* len);
int vgpu_client_run_task_region(vgpu_client* c, uint64_t in_bytes, const vgpu_descriptor* d,
                                const void** data, uint64_t* len);

/* Non-virtualized baseline: this process's own CUDA context. */
int vgpu_native_run_task(int cuda_device, const vgpu_descriptor* d, const void* in,
                         uint64_t in_bytes, void* out, uint64_t cap, uint64_t* len);

/* Paper model (reporting): batch makespan predicted by simulate() for n
 * identical tasks, and the closed forms. */
uint64_t vgpu_model_simulate(int style, uint32_t n, uint64_t t_in, uint64_t t_comp,
                             uint64_t t_out, uint32_t grid, uint32_t sms,
                             uint32_t max_kernels, uint32_t slots_per_sm);
/* simulate() with DeviceSpec::fluid_blocks (B200 block scheduler as a
 * fluid): grid = the task's CTAs, ctas_per_sm = its resident CTAs per SM,
 * launch_us = the fixed part of a kernel's measured span (once per kernel,
 * not per wave; vgpu_cu_launch_probe); shared = 0: queue-order slots,
 * 1: processor sharing among the kernels that run at once */
uint64_t vgpu_model_simulate_fluid(int style, uint32_t n, uint64_t t_in, uint64_t t_comp,
                                   uint64_t t_out, uint32_t grid, uint32_t sms,
                                   uint32_t ctas_per_sm, uint64_t launch_us, int shared);
int vgpu_model_classify(uint64_t t_in, uint64_t t_comp, uint64_t t_out);
uint64_t vgpu_model_no_vt(uint32_t n, uint64_t t_init, uint64_t t_ctx, uint64_t t_in,
                          uint64_t t_comp, uint64_t t_out);

/* Wire codec (FFI-side protocol tests). *len = frame length. */
int vgpu_encode_frame(uint8_t opcode, uint32_t client_id, uint64_t task_id,
                      const uint8_t* payload, uint64_t payload_len, uint8_t* out,
                      uint64_t cap, uint64_t* len);
/* Returns 0 and fills the header fields, or 1+vgpu::DecodeError ordinal. */
int vgpu_decode_frame(const uint8_t* frame, uint64_t len, uint8_t* opcode,
                      uint32_t* client_id, uint64_t* task_id, uint64_t* payload_len);

/* NPB CG problems for the nas-cg payload (client side, NPB's untimed
 * makea; include/vgpu/npb_cg.hpp). vgpu_cg_class: class 'S','W','A','B','C'
 * -> parameters and the published zeta. vgpu_cg_make_input: the nas-cg input
 * bytes into out (cap bytes); *len = bytes needed (call with out = NULL to
 * size the buffer). */
int vgpu_cg_class(char cls, uint32_t* n, uint32_t* nonzer, uint32_t* niter, double* shift,
                  double* zeta_verify);
int vgpu_cg_make_input(uint32_t n, uint32_t nonzer, uint32_t niter, double shift, uint8_t* out,
                       uint64_t cap, uint64_t* len);

/* Multi-GPU (include/vgpu/multigpu.hpp). vgpu_gvm_fold: the
 * GVM's partial record (GvmDaemon::fold_record, 16 doubles). The NCCL id
 * rendezvous: rank 0 publishes `n` bytes in `path` (atomic rename), other
 * ranks fetch them (polling, timeout_ms). vgpu_fold_in_rank_order: fold the
 * all-gathered records (nranks x 16, rank-major) in rank order into out[16].
 * vgpu_local_cpus: host cores local to a PCI device (sysfs), *n = count. */
int vgpu_gvm_fold(vgpu_gvm* g, double* out16);
int vgpu_rendezvous_publish(const char* path, const void* data, uint64_t n);
int vgpu_rendezvous_fetch(const char* path, void* out, uint64_t n, int64_t timeout_ms);
int vgpu_fold_in_rank_order(const double* all, uint32_t nranks, double* out16);
int vgpu_local_cpus(const char* pci_bus_id, int32_t* out, uint32_t cap, uint32_t* n);

/* NPB MG problems for the nas-mg payload (client side, NPB's untimed zran3;
 * include/vgpu/npb_mg.hpp). vgpu_mg_class: class 'S','W','A','B','C' ->
 * nx, nit, smoother set and the published rnm2. vgpu_mg_make_input: the
 * input bytes into out (cap); *len = bytes needed (out = NULL sizes it). */
int vgpu_mg_class(char cls, uint32_t* nx, uint32_t* nit, uint32_t* coeffs, double* rnm2_verify);
int vgpu_mg_make_input(uint32_t nx, uint32_t nit, uint32_t coeffs, uint8_t* out, uint64_t cap,
                       uint64_t* len);

const char* vgpu_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* VGPU_C_H */
