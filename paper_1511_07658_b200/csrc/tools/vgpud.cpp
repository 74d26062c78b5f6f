// vgpud — the GVM daemon for one B200. Flag surface of the reference
// (proj/tools/vgpud.cpp:26-55) plus --device / --data-plane; CLI11 is not
// available, so flags are parsed by hand ("--name value" or "--name=value").
// Serves REQ/SND/STR/STP/RCV/RLS until SIGINT/SIGTERM, then writes the
// per-task metrics CSV (reference daemon.cpp:31-39 schema).
#include <csignal>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <map>
#include <string>
#include <thread>

#include "vgpu/daemon.hpp"

namespace {

volatile std::sig_atomic_t g_stop = 0;
void on_signal(int) { g_stop = 1; }

void usage() {
    std::puts(
        "vgpud [--instance NAME] [--clients N] [--shm-bytes B] [--barrier-window US]\n"
        "      [--barrier-size K] [--clock virtual|real] [--scale F] [--device-sms N]\n"
        "      [--device-max-kernels N] [--device-slots-per-sm N] [--t-init US]\n"
        "      [--t-ctx-switch US] [--metrics-out PATH] [--device ORDINAL]\n"
        "      [--data-plane zero-copy|snapshot] [--ready-file PATH]");
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
    std::string metrics_out, ready_file;
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

    std::unique_ptr<vgpu::GvmDaemon> daemon;
    try {
        daemon = vgpu::GvmDaemon::start_os(cfg);
    } catch (const std::exception& e) {
        std::cerr << "vgpud: " << e.what() << '\n';
        return 1;
    }
    std::signal(SIGINT, on_signal);
    std::signal(SIGTERM, on_signal);
    std::cout << "vgpud: instance '" << cfg.instance << "' serving " << cfg.max_clients
              << " clients on CUDA device " << cfg.cuda_device << std::endl;
    if (!ready_file.empty()) std::ofstream(ready_file) << "ready\n";
    while (!g_stop) std::this_thread::sleep_for(std::chrono::milliseconds(20));
    daemon->stop();
    const auto m = daemon->metrics();
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
    return 0;
}
