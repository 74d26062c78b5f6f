// vgpu-b200 — the GPU Virtualization Manager (GVM).
//
// Declarations match proj/include/vgpu/daemon.hpp:15-96. The GVM owns the
// ONE CUDA context of its B200, leases per-client shm regions, gathers
// concurrently arriving STRs behind a barrier and dispatches each batch as
// H2D -> kernel -> D2H on per-client CUDA streams in the PS-1 / PS-2 order
// the paper's model picks. Completion is driven by CUDA events.
//
// Clock modes keep the reference's observable contract:
//   Virtual  metrics are the simulated schedule (vnow advances by the model
//            makespan, measured == model) and every STR of a batch is ACKed
//            only once the batch has really finished on the GPU, so STP right
//            after the STR ACK answers ACK — as in reference daemon.cpp:428-440;
//   Real     STRs are ACKed at enqueue; completion, pure_gpu_us and the
//            measured batch makespan come from CUDA events (the reference's
//            sleep-paced completer, daemon.cpp:532-585, is replaced by the
//            hardware itself).
#ifndef VGPU_DAEMON_HPP
#define VGPU_DAEMON_HPP

#include <iosfwd>
#include <memory>
#include <string>
#include <vector>

#include "vgpu/device.hpp"
#include "vgpu/payload.hpp"
#include "vgpu/transport.hpp"
#include "vgpu/types.hpp"

namespace vgpu {

enum class ClockMode { Virtual, Real };

// B200: how client bytes move between the shm region and HBM.
//   ZeroCopy  the daemon cudaHostRegister()s every region; H2D reads the
//             region at dispatch and D2H writes the result straight into it
//             when the task completes. No host memcpy on the data path.
//   Snapshot  reference-exact timing of the region accesses: SND copies the
//             region into a pinned staging slot (daemon.cpp:248) and RCV
//             copies the result out of pinned staging (daemon.cpp:335).
// The SDK (VgpuHandle) cannot tell the two apart; a raw-protocol client that
// rewrites its region between SND and dispatch can.
enum class DataPlane { ZeroCopy, Snapshot };

struct GvmConfig {
    std::string instance = "default";
    std::uint32_t max_clients = 8;
    std::uint64_t per_client_shm_bytes = 1 << 20;
    Micros barrier_window = 2000;
    std::uint32_t barrier_size = 0;  // 0 = max_clients
    DeviceSpec device;
    Micros t_init = 150000;
    Micros t_ctx_switch = 5000;
    ClockMode clock = ClockMode::Virtual;
    double scale = 1.0;

    // ---- B200 extensions ----
    int cuda_device = 0;                   // ordinal the GVM's context lives on
    DataPlane data_plane = DataPlane::ZeroCopy;
};

enum class Phase { Idle, Leased, DataIn, Queued, Running, Done, Released };
const char* to_string(Phase p);

struct TaskMetrics {
    std::uint64_t task_id = 0;
    std::uint32_t client_id = 0;
    Micros queue_wait_us = 0;
    Micros pure_gpu_us = 0;
    Micros end_to_end_us = 0;
    // B200: CUDA-event stage times of the task (0 for host payloads and
    // under the virtual clock). These are the paper's model inputs.
    double h2d_us = 0.0;
    double comp_us = 0.0;
    double d2h_us = 0.0;
};

struct BatchMetrics {
    std::uint64_t batch_id = 0;
    ProgrammingStyle style = ProgrammingStyle::PS1;
    std::uint32_t task_count = 0;
    Micros model_makespan_us = 0;
    Micros measured_makespan_us = 0;
};

struct MetricsSnapshot {
    std::vector<TaskMetrics> tasks;
    std::vector<BatchMetrics> batches;
    Micros uptime_us = 0;
    Micros busy_us = 0;
    Micros t_init_us = 0;
    std::uint64_t batches_flushed = 0;
    // B200: device work issued so far.
    std::uint64_t kernel_launches = 0;
    std::uint64_t device_tasks = 0;
    // B200: the measured schedule — each device task's H2D / kernel / D2H
    // interval from its CUDA events, in us since the GVM opened the device,
    // stream_id = slot - 1 (write_timeline_csv's schema, device.cpp).
    Timeline device_timeline;
};

void write_metrics_csv(const MetricsSnapshot& m, std::ostream& out);

class GvmDaemon {
public:
    static std::unique_ptr<GvmDaemon> start(
        GvmConfig cfg, std::unique_ptr<DaemonTransport> transport,
        const PayloadRegistry* payloads = nullptr);
    static std::unique_ptr<GvmDaemon> start_loopback(GvmConfig cfg,
                                                     LoopbackHub& hub);
    static std::unique_ptr<GvmDaemon> start_os(GvmConfig cfg);

    ~GvmDaemon();
    GvmDaemon(const GvmDaemon&) = delete;
    GvmDaemon& operator=(const GvmDaemon&) = delete;

    void stop();
    MetricsSnapshot metrics() const;
    const GvmConfig& config() const { return cfg_; }

    // B200: this GVM's partial record of the run, the input of
    // the single cross-GPU reduction (vgpu_cu_reduce_final, folded in rank
    // order). kFoldWidth doubles: [0] device tasks completed, [1..10] NAS EP
    // q[0..9], [11] sx, [12] sy, [13] pairs, [14] EP batches covered, [15]
    // result bytes returned mod 1000003. EP results are kept per slice
    // (keyed by first_batch; a slice computed again must repeat its bits,
    // else [14] is set to -1) and folded in first_batch order, so the
    // floating-point sums do not depend on completion order.
    static constexpr std::size_t kFoldWidth = 16;
    std::array<double, kFoldWidth> fold_record() const;

    // B200 fault containment: a sticky device fault failed every in-flight
    // task (NACK Internal) and the context could not be rebuilt in this
    // process; the GVM must restart in a fresh one (vgpud exits with 3 and,
    // with --respawn, re-executes itself).
    bool device_lost() const;

    struct Impl;

private:
    GvmDaemon(GvmConfig cfg, std::unique_ptr<DaemonTransport> transport,
              const PayloadRegistry* payloads);

    GvmConfig cfg_;
    std::unique_ptr<Impl> impl_;
};

}  // namespace vgpu

#endif  // VGPU_DAEMON_HPP
