/*
 * vgpu-b200 — thin C-ABI between the GVM host layer (C++) and the B200
 * device backend (libvgpu_cuda.so, nvcc -gencode arch=compute_100a,code=sm_100a).
 *
 * This replaces, in the reference, the two plug points the GVM dispatches
 * through:
 *   - PayloadRegistry::execute / PayloadFn         proj/include/vgpu/payload.hpp:17,:38
 *     (called from flush_barrier, proj/src/daemon.cpp:413)
 *   - simulate() as the executor of the work queue proj/include/vgpu/device.hpp:86
 *     (proj/src/daemon.cpp:384-385; PS-1/PS-2 order proj/src/device.cpp:56-69)
 * and the completion lane that paced sleeps stood in for
 *   - completer_loop / apply_completion            proj/src/daemon.cpp:474-585.
 *
 * Conventions: plain C types only; integer status returns (0 = ok, codes 3/5/8
 * deliberately equal vgpu::ErrCode Size/Payload/Internal); no C++ exception
 * crosses the ABI; host pointers handed to submit stay valid until poll()
 * reports the task. upload/submit/poll/wait are called from the GVM
 * dispatcher thread only; completion is detected by event queries in poll()
 * (no CUDA host callbacks).
 */
#ifndef VGPU_CUDA_H
#define VGPU_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------- */
enum vgpu_cu_status {
    VGPU_CU_OK = 0,
    VGPU_CU_ESIZE = 3,       /* result does not fit / buffer too small       */
    VGPU_CU_EPAYLOAD = 5,    /* unknown payload id or malformed input bytes  */
    VGPU_CU_EINTERNAL = 8,   /* CUDA runtime failure (detail: last_error)     */
    VGPU_CU_ENODEV = 100,    /* no usable CUDA device                         */
    VGPU_CU_EINVAL = 101,    /* bad argument                                  */
    VGPU_CU_ENCCL = 102      /* NCCL missing or failed                        */
};

/* ---- device kernels (payload ids) --------------------------------------- */
enum vgpu_cu_kernel {
    VGPU_CU_K_IDENTITY = 0,  /* "identity"      bytes -> bytes (copy only)     */
    VGPU_CU_K_VADD = 1,      /* "vector-add"    a||b fp32 -> a+b               */
    VGPU_CU_K_VSCALE = 2,    /* "vector-scale"  x fp32 -> param*x              */
    VGPU_CU_K_EP = 3,        /* "nas-ep"        vgpu_ep_params -> vgpu_ep_result */
    VGPU_CU_K_BS = 4,        /* "black-scholes" S||X||T fp32 -> call||put      */
    VGPU_CU_K_SGEMM = 5,     /* "sgemm"         A||B (n*n fp32) -> A*B         */
    VGPU_CU_K_VMUL = 6,      /* "vector-mul"    a||b fp32 -> a*b               */
    VGPU_CU_K_CG = 7,        /* "nas-cg"        vgpu_cg_header + CSR -> vgpu_cg_result */
    VGPU_CU_K_ES = 8,        /* "electrostatics" vgpu_es_header + atoms -> lattice potential */
    VGPU_CU_K_MG = 9,        /* "nas-mg"        vgpu_mg_header + v -> vgpu_mg_result */
    VGPU_CU_K_COUNT = 10
};

/* NAS EP job (input, 32 bytes little-endian). The job computes batches
 * [first_batch, first_batch + n_batches) of the class with 2^m pairs,
 * 2^mk pairs per batch (NPB: mk = 16). */
typedef struct vgpu_ep_params {
    uint32_t m;
    uint32_t mk;
    uint64_t first_batch;
    uint64_t n_batches;
    uint64_t reserved; /* must be 0 */
} vgpu_ep_params;

/* NAS EP job result (output, 112 bytes). sx/sy follow the fixed reduction
 * order documented in DESIGN.md (bit-identical to oracle/vgpu_oracle.c). */
typedef struct vgpu_ep_result {
    uint64_t q[10];
    double sx;
    double sy;
    uint64_t pairs;     /* accepted Gaussian pairs = sum(q) */
    uint64_t n_batches;
} vgpu_ep_result;

/* NAS CG job (input, little-endian): the timed part of NPB CG — `niter`
 * outer iterations of `cgitmax` conjugate-gradient steps on the sparse
 * symmetric matrix the SPMD program built (NPB makea, untimed in NPB
 * too; vgpu_cg_make_input), starting from x = 1. Layout:
 *   vgpu_cg_header | rowstr u32[n+1] | colidx u32[nnz] | pad to 8 | a f64[nnz]
 * rowstr[0] = 0, rowstr[n] = nnz, colidx < n (CSR, zero-based). */
typedef struct vgpu_cg_header {
    uint32_t n;
    uint32_t nnz;
    uint32_t niter;    /* NPB NITER (15 for classes S..A, 75 for B, C) */
    uint32_t cgitmax;  /* NPB: 25 */
    double shift;      /* NPB SHIFT: zeta = shift + 1 / (x . z) */
} vgpu_cg_header;

/* NAS CG job result (output, 32 bytes): zeta and ||x - A z|| after the last
 * outer iteration (the values NPB prints and verifies). */
typedef struct vgpu_cg_result {
    double zeta;
    double rnorm;
    uint32_t niter;
    uint32_t n;
    uint64_t nnz;
} vgpu_cg_result;

/* Bytes of the nas-cg input for a given CSR shape. */
static inline uint64_t vgpu_cg_input_bytes(uint32_t n, uint32_t nnz) {
    uint64_t b = sizeof(vgpu_cg_header) + 4ull * (n + 1ull) + 4ull * nnz;
    b = (b + 7u) & ~7ull;
    return b + 8ull * nnz;
}

/* Electrostatics job (VMD direct Coulomb summation, the paper's ES):
 * input = vgpu_es_header | float atoms[natoms][4] (x, y, z, q); output =
 * float V[nz][ny][nx], V(p) = sum_i q_i / |p - a_i| at p = (x, y, z) * spacing.
 * Atoms must not sit on lattice points (r = 0). */
typedef struct vgpu_es_header {
    uint32_t natoms;
    uint32_t nx, ny, nz;
    float spacing;
    uint32_t reserved[3]; /* must be 0 */
} vgpu_es_header;

/* NAS MG job (NPB 3.x mg.f, the timed part): `nit` V-cycles (mg3P + resid)
 * of the 3-D Poisson problem A u = v on an nx^3 periodic grid from u = 0,
 * then ||r||_2 / sqrt(nx^3) and max |r| (NPB's rnm2, rnmu). The SPMD
 * program builds v with NPB's zran3 (untimed in NPB too): input =
 * vgpu_mg_header | double v[nx][nx][nx] (the interior, i1 fastest).
 * coeffs 0: the smoother of classes S/W/A, 1: of classes B/C/D. */
typedef struct vgpu_mg_header {
    uint32_t nx;       /* power of two, 4 .. 512 */
    uint32_t nit;
    uint32_t coeffs;
    uint32_t reserved; /* must be 0 */
} vgpu_mg_header;

typedef struct vgpu_mg_result {
    double rnm2;
    double rnmu;
    uint32_t nx;
    uint32_t nit;
    uint64_t reserved;
} vgpu_mg_result;

/* Bytes of the nas-mg input, and of the job's device workspace (u and r on
 * every level k = 1..log2(nx), (2^k + 2)^3 doubles each, plus the norm's
 * per-plane partials). */
static inline uint64_t vgpu_mg_input_bytes(uint32_t nx) {
    return sizeof(vgpu_mg_header) + 8ull * nx * nx * nx;
}
static inline uint64_t vgpu_mg_workspace_bytes(uint32_t nx) {
    uint64_t b = 0;
    for (uint32_t m = 2; m <= nx; m *= 2) b += 2ull * 8ull * (m + 2ull) * (m + 2ull) * (m + 2ull);
    return b + 16ull * nx + 256;
}

/* Black-Scholes constants (CUDA SDK formulation). */
#define VGPU_BS_RISKFREE 0.02f
#define VGPU_BS_VOLATILITY 0.30f

/* ---- one task of a dispatch batch --------------------------------------- */
/* task flag: the input already sits in the slot's HBM buffer (uploaded at
 * SND time with vgpu_cu_upload); the task skips its H2D stage */
#define VGPU_CU_TASK_INPUT_RESIDENT 1u

typedef struct vgpu_cu_task {
    uint32_t slot;       /* client slot 1..max_clients: stream + HBM buffers */
    uint32_t kernel;     /* vgpu_cu_kernel                                    */
    float param;         /* vector-scale factor                               */
    uint32_t flags;      /* VGPU_CU_TASK_*                                    */
    const void* h_in;    /* host source (registered region / pinned staging)  */
    uint64_t in_bytes;
    void* h_out;         /* host destination of the result                    */
    uint64_t out_bytes;  /* vgpu_cu_output_size()                             */
    uint64_t tag;        /* echoed in vgpu_cu_done                            */
} vgpu_cu_task;

enum vgpu_cu_done_kind { VGPU_CU_DONE_TASK = 0, VGPU_CU_DONE_UPLOAD = 1 };

typedef struct vgpu_cu_done {
    uint64_t tag;
    uint64_t batch;        /* batch sequence number from submit              */
    int32_t status;        /* VGPU_CU_OK or error                            */
    uint32_t slot;
    float h2d_us;          /* CUDA-event stage durations (a streamed upload:
                              the DMA busy time, summed over its parts)      */
    float comp_us;
    float d2h_us;
    float span_us;         /* this task: H2D start -> D2H end                */
    float batch_span_us;   /* set on the batch's last completion: first H2D
                              start -> last D2H end over the batch; else 0   */
    uint32_t batch_done;   /* 1 on the batch's last completion               */
    uint32_t kind;         /* vgpu_cu_done_kind                              */
    uint32_t reserved;
    /* stage starts in us since the handle's epoch event (vgpu_cu_open), for
     * the measured timeline; -1: the stage did not run on the device       */
    float t_h2d_us;
    float t_comp_us;
    float t_d2h_us;
    uint32_t reserved2;
} vgpu_cu_done;

typedef struct vgpu_cu_stats {
    uint64_t kernel_launches;  /* our kernels launched by this device handle */
    uint64_t tasks;            /* tasks submitted                             */
    uint64_t h2d_bytes;
    uint64_t d2h_bytes;
    uint64_t batches;
} vgpu_cu_stats;

typedef struct vgpu_cu_dev vgpu_cu_dev;

/* Open the GVM's device: primary context on `device`, one non-blocking
 * stream and an in/out HBM buffer pair of slot_bytes per client slot. */
int vgpu_cu_open(int device, uint32_t max_clients, uint64_t slot_bytes,
                 vgpu_cu_dev** out);
void vgpu_cu_close(vgpu_cu_dev* dev);

/* Page-lock a client region (cudaHostRegister) so H2D/D2H DMA it directly. */
int vgpu_cu_register_region(vgpu_cu_dev* dev, uint32_t slot, void* base,
                            uint64_t bytes);
/* Pinned host staging (DataPlane::Snapshot). */
int vgpu_cu_alloc_pinned(vgpu_cu_dev* dev, uint64_t bytes, void** out);
void vgpu_cu_free_pinned(vgpu_cu_dev* dev, void* p);

/* Payload id -> kernel; unknown ids return VGPU_CU_EPAYLOAD. */
int vgpu_cu_payload(const char* id, uint32_t* kernel);
/* Host-side validation before launch: result size for this input, or
 * VGPU_CU_EPAYLOAD when the input is malformed (the reference's
 * PayloadError::MalformedInput). `in` may be NULL except for EP. */
int vgpu_cu_output_size(uint32_t kernel, const void* in, uint64_t in_bytes,
                        uint64_t* out_bytes);
/* Per-task preflight against THIS device's slots: vgpu_cu_output_size plus
 * the slot limits submit enforces (input, result and device workspace must
 * fit the slot). The GVM runs it per task before a batch is submitted, so a
 * task that cannot run fails alone (VGPU_CU_EPAYLOAD / VGPU_CU_ESIZE) and
 * never takes its co-batched clients down with a failed submit. */
int vgpu_cu_task_check(vgpu_cu_dev* dev, uint32_t kernel, const void* in, uint64_t in_bytes,
                       uint64_t* out_bytes);

/* Eager upload (SND time): H2D of `bytes` from h_in into the slot's input
 * buffer on the slot's stream; poll() reports it as VGPU_CU_DONE_UPLOAD with
 * `tag`. Once reported, the bytes are captured in HBM (SND snapshot). */
int vgpu_cu_upload(vgpu_cu_dev* dev, uint32_t slot, const void* h_in, uint64_t bytes,
                   uint64_t tag);

/* Streamed SND upload: the same op as vgpu_cu_upload, issued in parts while
 * the client is still filling its region. flags BEGIN opens the op (records
 * its start event), each call copies [offset, offset + bytes) of the input
 * from h_src into the slot's input buffer on the slot's stream, END closes
 * it; poll() then reports one VGPU_CU_DONE_UPLOAD with `tag` (given with
 * BEGIN). BEGIN|END in one call equals vgpu_cu_upload. */
#define VGPU_CU_UPLOAD_BEGIN 1u
#define VGPU_CU_UPLOAD_END 2u
int vgpu_cu_upload_part(vgpu_cu_dev* dev, uint32_t slot, const void* h_src, uint64_t offset,
                        uint64_t bytes, uint32_t flags, uint64_t tag);

/* Enqueue a batch. style 0 = PS-1 (all H2D, then compute — one launch per
 * kernel kind over the whole batch's task table — then all D2H), 1 = PS-2
 * (per-stream H2D -> kernel -> D2H triples). Returns immediately. */
int vgpu_cu_submit_batch(vgpu_cu_dev* dev, int style, const vgpu_cu_task* tasks,
                         uint32_t n, uint64_t* batch_id);
/* Collect finished tasks (non-blocking). */
int vgpu_cu_poll(vgpu_cu_dev* dev, vgpu_cu_done* out, uint32_t cap,
                 uint32_t* n_out);
/* Operations (tasks and uploads) submitted but not yet reported by poll().
 * poll() detects completion by querying each one's final CUDA event (no
 * callback latency), so a dispatcher with work pending polls it. */
int vgpu_cu_pending(vgpu_cu_dev* dev);
/* Wait (polling events) until an op completed or timeout_us passed. */
int vgpu_cu_wait(vgpu_cu_dev* dev, int64_t timeout_us);
int vgpu_cu_get_stats(vgpu_cu_dev* dev, vgpu_cu_stats* out);

/* Synchronous single task in the CALLING process's own context, pageable
 * host memory, cudaMemcpy + launch + sync: PayloadRegistry::execute() and
 * the NativeVgpu (non-virtualized) baseline. */
int vgpu_cu_execute(int device, uint32_t kernel, float param, const void* in,
                    uint64_t in_bytes, void* out, uint64_t out_cap,
                    uint64_t* out_bytes);
/* Kernel launches issued by vgpu_cu_execute in this process. */
uint64_t vgpu_cu_execute_launches(void);

/* Fault containment. A sticky device fault (illegal address, trap, ...)
 * seen by vgpu_cu_poll reports every op that was in flight with status
 * VGPU_CU_EINTERNAL, resets the context and tries to rebuild it (slot
 * buffers, streams, events, region and staging registrations). The
 * generation counts the resets (inputs uploaded before one are gone);
 * last_fault says what caused the last. When the driver refuses a new
 * context in this process, device_lost turns 1 and every later upload /
 * submit / register fails fast with VGPU_CU_EINTERNAL: the owner restarts
 * in a fresh process (vgpud --respawn). inject_fault (tests; only with
 * VGPU_ENABLE_FAULT_INJECTION=1) queues a trapping kernel as a task op;
 * with the same variable set, an "identity" task whose input is exactly
 * the 13 bytes "VGPU-TRAP-NOW" runs the trapping kernel instead (fault
 * injection through the unchanged client API). */
uint64_t vgpu_cu_generation(vgpu_cu_dev* dev);
int vgpu_cu_device_lost(vgpu_cu_dev* dev);
const char* vgpu_cu_last_fault(vgpu_cu_dev* dev);
int vgpu_cu_inject_fault(vgpu_cu_dev* dev, uint32_t slot, uint64_t tag);

int vgpu_cu_device_count(int* n);
/* One task's launch shape: the CTAs its share of a batched launch gets and
 * the kernel's resident CTAs per SM (cudaOccupancy), for the model's B200
 * block-scheduler spec. Kernels that size their grid to the device report
 * the SM count and 1. */
int vgpu_cu_task_shape(int device, uint32_t kernel, const void* in, uint64_t in_bytes,
                       uint32_t* ctas, uint32_t* ctas_per_sm);
/* PCI bus id of a device ("00000000:1B:00.0"), for NUMA-local placement */
int vgpu_cu_device_pci_bus_id(int device, char* buf, int len);
const char* vgpu_cu_strerror(int code);
const char* vgpu_cu_last_error(void); /* thread-local detail of the last failure */

/* ---- device-resident measurement (bench.py `value` and roofline) ------- */
typedef struct vgpu_cu_resident_result {
    double ms_total;            /* all timed steps, CUDA events              */
    double ms_per_step;
    double kernel_ms_per_launch;/* average duration of the dominant launch  */
    uint32_t launches_per_step;
    uint32_t sets;              /* rotating input sets actually used         */
    uint64_t algo_bytes_per_launch;
    double algo_flops_per_launch;
    uint64_t resident_bytes;    /* HBM held by the rotating sets             */
    uint32_t pdl;               /* 1: steps chained with programmatic
                                   dependent launch (HBM-streaming kernels) */
    uint32_t reserved;
} vgpu_cu_resident_result;

/* Times `steps` batched launches of `kernel` over n_tasks tasks whose inputs
 * (copied once from h_inputs[i], in_bytes[i]) sit in HBM; `sets` rotating
 * copies keep the working set above L2 between steps. */
#define VGPU_CU_RESIDENT_NO_PDL 1u /* flags: serialize steps (per-launch duration) */
#define VGPU_CU_RESIDENT_MAIN_ONLY 2u /* flags: SGEMM: time the tcgen05 GEMM alone
                                         (split pre-pass done before the timed steps) */
int vgpu_cu_resident_bench(int device, uint32_t kernel, float param,
                           uint32_t n_tasks, const void* const* h_inputs,
                           const uint64_t* in_bytes, uint32_t sets,
                           uint32_t warmup, uint32_t steps, uint32_t flags,
                           vgpu_cu_resident_result* out);

/* ---- roofline denominators measured on the device ------------------------ */
/* Dependent-chain FMA microbenchmark (8 independent chains per thread, a
 * few waves of 148 x 8 CTAs): the pipe peak the EP (FP64) and SIMT SGEMM
 * (FP32) rooflines are quoted against, counting 2 FLOP per FMA. */
enum vgpu_cu_peak_kind { VGPU_CU_PEAK_FP64 = 0, VGPU_CU_PEAK_FP32 = 1 };
int vgpu_cu_peak_probe(int device, uint32_t kind, double* tflops);
/* The fixed cost inside a CUDA-event-timed kernel span: median event span of
 * an empty 148-CTA kernel on its own stream (us). The model's B200 spec
 * charges it once per kernel instead of once per wave. */
int vgpu_cu_launch_probe(int device, double* us);

/* Host link (PCIe) probe: the e2e roofline's denominator. `bytes`-sized
 * copies between page-locked host memory (cudaHostAlloc) and HBM, each
 * direction alone and both at once on two streams (the copy engines are
 * full duplex), best of `reps` after a warm-up, CUDA events. GB/s = 1e9 B/s;
 * bidir counts the bytes of both directions. */
typedef struct vgpu_cu_link_result {
    double h2d_gbs;
    double d2h_gbs;
    double bidir_gbs;
    uint64_t bytes;
} vgpu_cu_link_result;
#define VGPU_CU_LINK_SHM 1u /* flags: POSIX shm pages registered in place (the data plane's kind) */
int vgpu_cu_link_probe(int device, uint64_t bytes, uint32_t reps, uint32_t flags,
                       vgpu_cu_link_result* out);

/* ---- multi-GPU: the single final reduction (NCCL over NVLink) --------- */
#define VGPU_CU_NCCL_ID_BYTES 128
int vgpu_cu_nccl_unique_id(void* id_out /* VGPU_CU_NCCL_ID_BYTES */);
int vgpu_cu_comm_init(vgpu_cu_dev* dev, const void* id, int nranks, int rank);
/* All-gather `bytes` of partial record from every rank into all_out
 * (nranks * bytes, rank order). Callers fold in rank order on the host. */
int vgpu_cu_reduce_final(vgpu_cu_dev* dev, const void* partial, uint64_t bytes,
                         void* all_out);

#ifdef __cplusplus
}
#endif

#endif /* VGPU_CUDA_H */
