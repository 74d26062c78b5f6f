// vgpud — the GVM daemon for one B200. Flag surface of the reference
// (proj/tools/vgpud.cpp:26-55) plus --device / --data-plane; CLI11 is not
// available, so flags are parsed by hand ("--name value" or "--name=value").
// Serves REQ/SND/STR/STP/RCV/RLS until SIGINT/SIGTERM, then writes the
// per-task metrics CSV (reference daemon.cpp:31-39 schema).
//
// Multi-GPU: with --nranks N --rank R --rendezvous PATH this
// GVM is rank R of N per-GPU GVMs. At start rank 0 creates the NCCL unique
// id and publishes it in PATH (the others wait for the file), every rank
// joins the communicator, and only then is the daemon ready. At shutdown
// each rank all-gathers its fold record (GvmDaemon::fold_record) in the one
// ncclAllGather of the run; the records are folded in rank order and rank 0
// writes the result as JSON to --reduce-out (--fold-out: every rank's own
// record, with or without a communicator). --cpus LIST pins the daemon
// (default: the cores local to its GPU, from sysfs).
#include <unistd.h>

#include <cerrno>
#include <csignal>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <map>
#include <string>
#include <thread>

#include <cstring>
#include <iomanip>
#include <sstream>
#include <vector>

#include "vgpu/daemon.hpp"
#include "vgpu/device.hpp"
#include "vgpu/multigpu.hpp"
#include "vgpu/transport.hpp"
#include "vgpu_cuda.h"

namespace {

volatile std::sig_atomic_t g_stop = 0;
void on_signal(int) { g_stop = 1; }

void usage() {
    std::puts(
        "vgpud [--instance NAME] [--clients N] [--shm-bytes B] [--barrier-window US]\n"
        "      [--barrier-size K] [--clock virtual|real] [--scale F] [--device-sms N]\n"
        "      [--device-max-kernels N] [--device-slots-per-sm N] [--t-init US]\n"
        "      [--t-ctx-switch US] [--metrics-out PATH] [--device ORDINAL]\n"
        "      [--data-plane zero-copy|snapshot] [--ready-file PATH]\n"
        "      [--nranks N --rank R --rendezvous PATH [--reduce-out PATH]]\n"
        "      [--fold-out PATH] [--timeline-out PATH] [--cpus LIST|none] [--respawn N]\n"
        "exit status 3: the device context was lost to a sticky fault (every in-flight\n"
        "task was NACKed Internal); with --respawn N the daemon re-executes itself in a\n"
        "fresh process (new context, same instance name) up to N times instead.");
}

}  // namespace

int main(int argc, char** argv) {
    std::map<std::string, std::string> opt;
    for (int i = 1; i < argc; ++i) {
        std::string a = argv[i];
        if (a == "-h" || a == "--help") {
            usage();
            return 0;
        }
        if (a.rfind("--", 0) != 0) {
            std::cerr << "vgpud: unexpected argument " << a << '\n';
            return 2;
        }
        const auto eq = a.find('=');
        if (eq != std::string::npos) {
            opt[a.substr(2, eq - 2)] = a.substr(eq + 1);
        } else if (i + 1 < argc) {
            opt[a.substr(2)] = argv[++i];
        } else {
            std::cerr << "vgpud: " << a << " needs a value\n";
            return 2;
        }
    }
    vgpu::GvmConfig cfg;
    std::string metrics_out, ready_file, rendezvous, reduce_out, fold_out, timeline_out, cpus = "auto";
    int nranks = 0, rank = 0, respawn = 0;
    try {
        for (const auto& [k, v] : opt) {
            if (k == "instance") cfg.instance = v;
            else if (k == "clients") cfg.max_clients = std::stoul(v);
            else if (k == "shm-bytes") cfg.per_client_shm_bytes = std::stoull(v);
            else if (k == "barrier-window") cfg.barrier_window = std::stoull(v);
            else if (k == "barrier-size") cfg.barrier_size = std::stoul(v);
            else if (k == "clock") {
                if (v == "virtual") cfg.clock = vgpu::ClockMode::Virtual;
                else if (v == "real") cfg.clock = vgpu::ClockMode::Real;
                else throw std::invalid_argument("--clock must be virtual or real");
            } else if (k == "scale") cfg.scale = std::stod(v);
            else if (k == "device-sms") cfg.device.num_sms = std::stoul(v);
            else if (k == "device-max-kernels") cfg.device.max_concurrent_kernels = std::stoul(v);
            else if (k == "device-slots-per-sm") cfg.device.block_slots_per_sm = std::stoul(v);
            else if (k == "t-init") cfg.t_init = std::stoull(v);
            else if (k == "t-ctx-switch") cfg.t_ctx_switch = std::stoull(v);
            else if (k == "metrics-out") metrics_out = v;
            else if (k == "ready-file") ready_file = v;
            else if (k == "device") cfg.cuda_device = std::stoi(v);
            else if (k == "nranks") nranks = std::stoi(v);
            else if (k == "rank") rank = std::stoi(v);
            else if (k == "rendezvous") rendezvous = v;
            else if (k == "reduce-out") reduce_out = v;
            else if (k == "fold-out") fold_out = v;
            else if (k == "timeline-out") timeline_out = v;
            else if (k == "cpus") cpus = v;
            else if (k == "respawn") respawn = std::stoi(v);
            else if (k == "data-plane") {
                if (v == "zero-copy") cfg.data_plane = vgpu::DataPlane::ZeroCopy;
                else if (v == "snapshot") cfg.data_plane = vgpu::DataPlane::Snapshot;
                else throw std::invalid_argument("--data-plane must be zero-copy or snapshot");
            } else {
                throw std::invalid_argument("unknown flag --" + k);
            }
        }
    } catch (const std::exception& e) {
        std::cerr << "vgpud: " << e.what() << '\n';
        return 2;
    }

    if (nranks > 0 && (rank < 0 || rank >= nranks || rendezvous.empty())) {
        std::cerr << "vgpud: --nranks needs --rank in [0, nranks) and --rendezvous\n";
        return 2;
    }
    // NUMA-local placement of the daemon (its dispatcher and the CUDA
    // driver threads inherit the mask)
    std::vector<int> cpu_set;
    if (cpus == "auto") {
        char bus[32] = {};
        if (vgpu_cu_device_pci_bus_id(cfg.cuda_device, bus, sizeof bus) == VGPU_CU_OK)
            cpu_set = vgpu::multigpu::local_cpus(bus);
    } else if (cpus != "none") {
        cpu_set = vgpu::multigpu::parse_cpulist(cpus);
    }
    const bool pinned = vgpu::multigpu::pin_to(cpu_set);

    std::unique_ptr<vgpu::GvmDaemon> daemon;
    try {
        daemon = vgpu::GvmDaemon::start_os(cfg);
    } catch (const std::exception& e) {
        std::cerr << "vgpud: " << e.what() << '\n';
        return 1;
    }
    // the cross-GPU communicator: joined before the daemon reports ready
    vgpu_cu_dev* comm_dev = nullptr;
    if (nranks > 0) {
        try {
            if (vgpu_cu_open(cfg.cuda_device, 1, 4096, &comm_dev) != VGPU_CU_OK)
                throw std::runtime_error(std::string("device: ") + vgpu_cu_last_error());
            std::vector<std::uint8_t> id(VGPU_CU_NCCL_ID_BYTES);
            if (rank == 0) {
                if (vgpu_cu_nccl_unique_id(id.data()) != VGPU_CU_OK)
                    throw std::runtime_error(vgpu_cu_last_error());
                vgpu::multigpu::publish_id(rendezvous, id);
            } else {
                id = vgpu::multigpu::fetch_id(rendezvous, id.size(), std::chrono::seconds(300));
            }
            if (vgpu_cu_comm_init(comm_dev, id.data(), nranks, rank) != VGPU_CU_OK)
                throw std::runtime_error(vgpu_cu_last_error());
        } catch (const std::exception& e) {
            std::cerr << "vgpud: rank " << rank << " could not join the communicator: " << e.what()
                      << '\n';
            daemon->stop();
            if (comm_dev) vgpu_cu_close(comm_dev);
            return 1;
        }
    }
    std::signal(SIGINT, on_signal);
    std::signal(SIGTERM, on_signal);
    std::cout << "vgpud: instance '" << cfg.instance << "' serving " << cfg.max_clients
              << " clients on CUDA device " << cfg.cuda_device
              << (nranks > 0 ? " as rank " + std::to_string(rank) + " of " + std::to_string(nranks) : "")
              << (pinned ? " (pinned to " + std::to_string(cpu_set.size()) + " local cores)" : "")
              << std::endl;
    if (!ready_file.empty()) std::ofstream(ready_file) << "ready\n";
    while (!g_stop && !daemon->device_lost()) std::this_thread::sleep_for(std::chrono::milliseconds(20));
    if (daemon->device_lost()) {
        // process-level fault containment: CUDA keeps a faulted process's
        // device unavailable, so a fresh process takes over the instance
        daemon->stop();
        daemon.reset();  // closes the endpoint and the client regions
        vgpu::unlink_os_instance(cfg.instance, cfg.max_clients);
        if (respawn > 0) {
            std::vector<std::string> args;
            for (int i = 0; i < argc; ++i) {
                const std::string a = argv[i];
                if (a == "--respawn") {
                    ++i;
                    continue;
                }
                if (a.rfind("--respawn=", 0) == 0) continue;
                args.push_back(a);
            }
            args.push_back("--respawn");
            args.push_back(std::to_string(respawn - 1));
            std::vector<char*> av;
            for (auto& a : args) av.push_back(a.data());
            av.push_back(nullptr);
            std::cerr << "vgpud: device context lost; restarting instance '" << cfg.instance
                      << "' in a fresh process (" << respawn - 1 << " restart(s) left)" << std::endl;
            if (!ready_file.empty()) std::remove(ready_file.c_str());
            execv("/proc/self/exe", av.data());
            std::cerr << "vgpud: re-exec failed: " << std::strerror(errno) << '\n';
        } else {
            std::cerr << "vgpud: device context lost to a sticky fault; exiting (3)" << std::endl;
        }
        return 3;
    }
    daemon->stop();
    int rc = 0;
    if (!fold_out.empty()) {  // this GVM's own record (also without a communicator)
        const auto rec = daemon->fold_record();
        std::ofstream out(fold_out);
        out << std::setprecision(17) << "{\"rank\": " << rank << ", \"record\": [";
        for (std::size_t i = 0; i < rec.size(); ++i) out << (i ? ", " : "") << rec[i];
        out << "]}\n";
    }
    if (comm_dev) {
        // the run's single cross-GPU collective
        const auto rec = daemon->fold_record();
        std::vector<double> all(static_cast<std::size_t>(nranks) * rec.size());
        const auto t0 = std::chrono::steady_clock::now();
        if (vgpu_cu_reduce_final(comm_dev, rec.data(), sizeof(double) * rec.size(), all.data()) !=
            VGPU_CU_OK) {
            std::cerr << "vgpud: final reduction failed: " << vgpu_cu_last_error() << '\n';
            rc = 1;
        } else if (rank == 0 && !reduce_out.empty()) {
            const double us = std::chrono::duration<double, std::micro>(
                                  std::chrono::steady_clock::now() - t0).count();
            const auto folded = vgpu::multigpu::fold_in_rank_order(all, nranks);
            auto hex = [](double d) {
                std::uint64_t b;
                std::memcpy(&b, &d, 8);
                std::ostringstream o;
                o << std::hex << b;
                return o.str();
            };
            std::ofstream out(reduce_out);
            out << std::setprecision(17) << "{\"nranks\": " << nranks << ", \"collective\": "
                << "\"ncclAllGather of " << sizeof(double) * rec.size() << " B per GVM\", "
                << "\"reduce_us\": " << us << ", \"record\": [";
            for (std::size_t i = 0; i < folded.size(); ++i) out << (i ? ", " : "") << folded[i];
            out << "], \"sx_bits\": \"" << hex(folded[11]) << "\", \"sy_bits\": \""
                << hex(folded[12]) << "\", \"per_rank\": [";
            for (int r = 0; r < nranks; ++r) {
                out << (r ? ", " : "") << "[";
                for (std::size_t i = 0; i < rec.size(); ++i)
                    out << (i ? ", " : "") << all[r * rec.size() + i];
                out << "]";
            }
            out << "]}\n";
        }
        vgpu_cu_close(comm_dev);
    }
    const auto m = daemon->metrics();
    if (!timeline_out.empty()) {  // the measured schedule, reference timeline schema
        std::ofstream out(timeline_out);
        vgpu::write_timeline_csv(m.device_timeline, out);
    }
    if (metrics_out.empty()) {
        vgpu::write_metrics_csv(m, std::cout);
    } else {
        std::ofstream out(metrics_out);
        if (!out) {
            std::cerr << "vgpud: cannot write " << metrics_out << '\n';
            return 1;
        }
        vgpu::write_metrics_csv(m, out);
    }
    return rc;
}
