// vgpu-launch — one GVM per GPU, SPMD processes pinned next to it, one
// final reduction (the paper's 4..16 processes per GPU).
//
//   vgpu-launch [--gpus N] [--procs-per-gpu P] [--workload W] [--rounds R]
//               [--warmup K] [--inplace] [--shared-gpu] [--no-affinity]
//               [--tag T] [--out PATH] [--ep-m M --bs-n N ... (vgpu-spmd sizes)]
//
// For g in 0..N-1 it starts `vgpud --instance gpu<g> --device g` (pinned by
// vgpud to the cores sysfs lists as local to that GPU), rank g of N: GVM 0
// publishes the NCCL unique id in a file, every GVM joins the communicator
// before it reports ready. Then it forks P `vgpu-spmd` workers per GPU,
// each pinned to its GPU's local cores with VGPU_INSTANCE=gpu<g> in its
// environment — the SPMD program finds its GVM through the reference's
// unchanged $VGPU_INSTANCE lookup (proj/src/client.cpp:146-151). Worker w
// runs on GPU w / P. When every worker is done the GVMs are stopped; each
// all-gathers its fold record (GvmDaemon::fold_record) in the run's one
// ncclAllGather and rank 0 folds them in rank order.
//
// --shared-gpu (test mode for one-GPU boxes): every GVM drives device 0;
// NCCL cannot put two ranks on one GPU, so the GVMs skip the communicator
// and the launcher folds their records (vgpud --fold-out) in rank order on
// the host. The output says which path ran.
//
// Prints one JSON line: jobs, the timed window (first finish of the last
// warm-up round -> last finish, over all workers), jobs/s, per-GPU jobs/s,
// the reduction result, and where each process was pinned.
#include <fcntl.h>
#include <poll.h>
#include <signal.h>
#include <sys/stat.h>
#include <sys/wait.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iomanip>
#include <iostream>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "vgpu/multigpu.hpp"
#include "vgpu/transport.hpp"
#include "vgpu_cuda.h"
#include "workloads.hpp"

namespace {

namespace mg = vgpu::multigpu;

std::string dir_of(const std::string& path) {
    const auto slash = path.rfind('/');
    return slash == std::string::npos ? "." : path.substr(0, slash);
}

std::string self_dir() {
    char buf[PATH_MAX] = {};
    const ssize_t n = readlink("/proc/self/exe", buf, sizeof buf - 1);
    return n > 0 ? dir_of(std::string(buf, static_cast<std::size_t>(n))) : ".";
}

std::string join_cpus(const std::vector<int>& cpus) {
    std::ostringstream o;
    for (std::size_t i = 0; i < cpus.size(); ++i) o << (i ? "," : "") << cpus[i];
    return o.str();
}

std::string read_file(const std::string& path) {
    std::ifstream in(path);
    std::stringstream ss;
    ss << in.rdbuf();
    return ss.str();
}

// minimal extraction from the one-line JSON objects the tools print
bool json_number(const std::string& s, const std::string& key, double* out) {
    const auto k = s.find("\"" + key + "\":");
    if (k == std::string::npos) return false;
    *out = std::strtod(s.c_str() + k + key.size() + 3, nullptr);
    return true;
}

std::vector<double> json_array(const std::string& s, const std::string& key) {
    std::vector<double> v;
    auto k = s.find("\"" + key + "\": [");
    if (k == std::string::npos) return v;
    const char* p = s.c_str() + k + key.size() + 5;
    while (*p && *p != ']') {
        char* end = nullptr;
        const double d = std::strtod(p, &end);
        if (end == p) break;
        v.push_back(d);
        p = end;
        while (*p == ',' || *p == ' ') ++p;
    }
    return v;
}

struct Child {
    pid_t pid = -1;
    int in = -1, out = -1;  // our ends of its stdin / stdout
    std::string buf;
};

Child spawn(const std::vector<std::string>& argv, const std::vector<int>& cpus,
            const std::string& instance_env, bool pipes) {
    int pin[2] = {-1, -1}, pout[2] = {-1, -1};
    if (pipes && (pipe(pin) != 0 || pipe(pout) != 0)) throw std::runtime_error("pipe");
    const pid_t pid = fork();
    if (pid < 0) throw std::runtime_error("fork");
    if (pid == 0) {
        if (pipes) {
            dup2(pin[0], 0);
            dup2(pout[1], 1);
            close(pin[0]);
            close(pin[1]);
            close(pout[0]);
            close(pout[1]);
        }
        mg::pin_to(cpus);
        if (!instance_env.empty()) setenv("VGPU_INSTANCE", instance_env.c_str(), 1);
        std::vector<char*> a;
        for (const auto& s : argv) a.push_back(const_cast<char*>(s.c_str()));
        a.push_back(nullptr);
        execv(a[0], a.data());
        _exit(127);
    }
    Child c;
    c.pid = pid;
    if (pipes) {
        close(pin[0]);
        close(pout[1]);
        c.in = pin[1];
        c.out = pout[0];
    }
    return c;
}

// read one line from the child's stdout (blocking up to timeout)
bool read_line(Child& c, std::string* line, int timeout_ms) {
    const auto deadline = std::chrono::steady_clock::now() + std::chrono::milliseconds(timeout_ms);
    for (;;) {
        const auto nl = c.buf.find('\n');
        if (nl != std::string::npos) {
            *line = c.buf.substr(0, nl);
            c.buf.erase(0, nl + 1);
            return true;
        }
        const int left = static_cast<int>(std::chrono::duration_cast<std::chrono::milliseconds>(
                                              deadline - std::chrono::steady_clock::now())
                                              .count());
        if (left <= 0) return false;
        pollfd p{c.out, POLLIN, 0};
        if (poll(&p, 1, left) <= 0) continue;
        char tmp[4096];
        const ssize_t n = read(c.out, tmp, sizeof tmp);
        if (n <= 0) return false;
        c.buf.append(tmp, static_cast<std::size_t>(n));
    }
}

}  // namespace

int main(int argc, char** argv) {
    int gpus = 0;
    std::uint32_t procs = 16, rounds = 10, warmup = 2;
    std::string workload = "mixed", tag, out_path;
    bool shared = false, affinity = true, inplace = false;
    std::vector<std::string> size_args;
    vgpu::wl::Sizes sizes;
    try {
        for (int i = 1; i < argc; ++i) {
            const std::string a = argv[i];
            auto val = [&]() -> std::string {
                if (i + 1 >= argc) throw std::invalid_argument(a + " needs a value");
                return argv[++i];
            };
            if (a == "--gpus") gpus = std::stoi(val());
            else if (a == "--procs-per-gpu") procs = std::stoul(val());
            else if (a == "--workload") workload = val();
            else if (a == "--rounds") rounds = std::stoul(val());
            else if (a == "--warmup") warmup = std::stoul(val());
            else if (a == "--inplace") inplace = true;
            else if (a == "--shared-gpu") shared = true;
            else if (a == "--no-affinity") affinity = false;
            else if (a == "--tag") tag = val();
            else if (a == "--out") out_path = val();
            else if (a == "--ep-m" || a == "--ep-batches" || a == "--bs-n" || a == "--mm-n" ||
                     a == "--vecadd-n" || a == "--cg-class" || a == "--es-atoms" || a == "--mg-class") {
                const std::string v = val();
                size_args.push_back(a);
                size_args.push_back(v);
                if (a == "--ep-m") sizes.ep_m = std::stoul(v);
                else if (a == "--ep-batches") sizes.ep_batches = std::stoull(v);
                else if (a == "--bs-n") sizes.bs_n = std::stoull(v);
                else if (a == "--mm-n") sizes.mm_n = std::stoul(v);
                else if (a == "--vecadd-n") sizes.vecadd_n = std::stoull(v);
                else if (a == "--cg-class") sizes.cg_class = v[0];
                else if (a == "--mg-class") sizes.mg_class = v[0];
                else if (a == "--es-atoms") sizes.es_atoms = std::stoul(v);
            } else if (a == "-h" || a == "--help") {
                std::puts("vgpu-launch [--gpus N] [--procs-per-gpu P] [--workload W] [--rounds R]\n"
                          "            [--warmup K] [--inplace] [--shared-gpu] [--no-affinity]\n"
                          "            [--tag T] [--out PATH] [vgpu-spmd size flags]");
                return 0;
            } else {
                throw std::invalid_argument("unknown argument " + a);
            }
        }
    } catch (const std::exception& e) {
        std::fprintf(stderr, "vgpu-launch: %s\n", e.what());
        return 2;
    }
    int devices = 0;
    if (vgpu_cu_device_count(&devices) != VGPU_CU_OK || devices < 1) {
        std::fprintf(stderr, "vgpu-launch: no CUDA device (%s)\n", vgpu_cu_last_error());
        return 1;
    }
    if (gpus <= 0) gpus = shared ? 1 : devices;
    if (!shared && gpus > devices) {
        std::fprintf(stderr, "vgpu-launch: %d GPUs asked, %d visible (use --shared-gpu to test)\n",
                     gpus, devices);
        return 2;
    }
    const std::string bin = self_dir();
    const std::string run = "/tmp/vgpu-launch." + std::to_string(getpid());
    mkdir(run.c_str(), 0700);
    const std::string sfx = tag.empty() ? "" : "." + tag;
    const std::uint64_t shm = vgpu::wl::region_bytes(workload, sizes);
    const std::uint32_t total = procs * static_cast<std::uint32_t>(gpus);

    // ---- per-GPU GVMs ------------------------------------------------------
    std::vector<Child> daemons;
    std::vector<std::vector<int>> gpu_cpus(gpus);
    for (int g = 0; g < gpus; ++g) {
        const int dev = shared ? 0 : g;
        if (affinity) {
            char bus[32] = {};
            if (vgpu_cu_device_pci_bus_id(dev, bus, sizeof bus) == VGPU_CU_OK)
                gpu_cpus[g] = mg::local_cpus(bus);
        }
        const std::string inst = "gpu" + std::to_string(g) + sfx;
        vgpu::unlink_os_instance(inst, procs);
        std::vector<std::string> a = {bin + "/vgpud", "--instance", inst, "--device", std::to_string(dev),
                                      "--clients", std::to_string(procs), "--shm-bytes", std::to_string(shm),
                                      "--clock", "real", "--barrier-size", "1", "--barrier-window", "2000",
                                      "--ready-file", run + "/ready" + std::to_string(g),
                                      "--fold-out", run + "/fold" + std::to_string(g) + ".json",
                                      "--metrics-out", run + "/metrics" + std::to_string(g) + ".csv",
                                      "--cpus", gpu_cpus[g].empty() ? "none" : join_cpus(gpu_cpus[g])};
        if (!shared) {
            a.insert(a.end(), {"--nranks", std::to_string(gpus), "--rank", std::to_string(g),
                               "--rendezvous", run + "/ncclid", "--reduce-out", run + "/reduce.json"});
        }
        daemons.push_back(spawn(a, {}, "", false));
    }
    auto stop_all = [&](int sig) {
        for (auto& d : daemons)
            if (d.pid > 0) kill(d.pid, sig);
    };
    // ready = every GVM serves and (multi-GPU) joined the communicator
    const auto ready_deadline = std::chrono::steady_clock::now() + std::chrono::seconds(300);
    for (int g = 0; g < gpus; ++g) {
        struct stat st {};
        while (stat((run + "/ready" + std::to_string(g)).c_str(), &st) != 0) {
            int status = 0;
            if (waitpid(daemons[g].pid, &status, WNOHANG) == daemons[g].pid) {
                std::fprintf(stderr, "vgpu-launch: vgpud %d exited before it was ready\n", g);
                daemons[g].pid = -1;
                stop_all(SIGTERM);
                return 1;
            }
            if (std::chrono::steady_clock::now() > ready_deadline) {
                std::fprintf(stderr, "vgpu-launch: vgpud %d not ready in time\n", g);
                stop_all(SIGTERM);
                return 1;
            }
            std::this_thread::sleep_for(std::chrono::milliseconds(5));
        }
    }

    // ---- SPMD workers, NUMA-local, found through $VGPU_INSTANCE --------------
    std::vector<Child> workers;
    for (std::uint32_t w = 0; w < total; ++w) {
        const int g = static_cast<int>(w / procs);
        std::vector<std::string> a = {bin + "/vgpu-spmd", "--worker", std::to_string(w), "--workers",
                                      std::to_string(total), "--workload", workload, "--rounds",
                                      std::to_string(rounds + warmup)};
        a.insert(a.end(), size_args.begin(), size_args.end());
        if (inplace) a.push_back("--inplace");
        workers.push_back(spawn(a, gpu_cpus[g], "gpu" + std::to_string(g) + sfx, true));
    }
    bool ok = true;
    std::string line;
    for (auto& c : workers) {
        for (;;) {
            if (!read_line(c, &line, 300000)) {
                ok = false;
                break;
            }
            if (line.rfind("READY", 0) == 0) break;
            if (!line.empty() && line[0] == '{') {
                ok = false;
                std::fprintf(stderr, "vgpu-launch: worker failed: %s\n", line.c_str());
                break;
            }
        }
    }
    for (auto& c : workers)
        if (write(c.in, "g", 1) != 1) ok = false;
    double begin = 1e300, end = 0.0;
    std::vector<double> gpu_begin(gpus, 1e300), gpu_end(gpus, 0.0);
    std::uint32_t failed = 0;
    for (std::uint32_t w = 0; w < workers.size(); ++w) {
        auto& c = workers[w];
        std::string res;
        while (read_line(c, &line, 3600000))
            if (!line.empty() && line[0] == '{') res = line;
        int status = 0;
        waitpid(c.pid, &status, 0);
        close(c.in);
        close(c.out);
        const auto t1 = json_array(res, "t1");
        const bool wok = res.find("\"ok\": true") != std::string::npos && WIFEXITED(status) &&
                         WEXITSTATUS(status) == 0 && t1.size() == rounds + warmup;
        if (!wok) {
            ++failed;
            std::fprintf(stderr, "vgpu-launch: worker %u: %s\n", w, res.c_str());
            continue;
        }
        double t_go = 0.0;
        json_number(res, "t_go", &t_go);
        const double b = warmup ? t1[warmup - 1] : t_go;
        const int g = static_cast<int>(w / procs);
        begin = std::min(begin, b);
        end = std::max(end, t1.back());
        gpu_begin[g] = std::min(gpu_begin[g], b);
        gpu_end[g] = std::max(gpu_end[g], t1.back());
    }
    ok = ok && failed == 0;

    // ---- stop the GVMs: each all-gathers its record, rank 0 folds -----------
    stop_all(SIGTERM);
    int daemon_rc = 0;
    for (auto& d : daemons) {
        int status = 0;
        waitpid(d.pid, &status, 0);
        if (!WIFEXITED(status) || WEXITSTATUS(status) != 0) daemon_rc = 1;
    }
    std::vector<double> all;
    for (int g = 0; g < gpus; ++g) {
        auto rec = json_array(read_file(run + "/fold" + std::to_string(g) + ".json"), "record");
        rec.resize(mg::kRecordWidth, 0.0);
        all.insert(all.end(), rec.begin(), rec.end());
    }
    const auto host_fold = mg::fold_in_rank_order(all, static_cast<std::uint32_t>(gpus));
    std::string reduce = shared ? "" : read_file(run + "/reduce.json");
    while (!reduce.empty() && (reduce.back() == '\n' || reduce.back() == ' ')) reduce.pop_back();
    bool reduce_matches = shared;
    if (!shared) {
        const auto rec = json_array(reduce, "record");
        reduce_matches = rec.size() == mg::kRecordWidth &&
                         std::memcmp(rec.data(), host_fold.data(), sizeof(double) * rec.size()) == 0;
    }

    const double secs = (end - begin) * 1e-9;
    const double jobs = static_cast<double>(total) * rounds;
    std::ostringstream o;
    o << std::setprecision(17) << "{\"ok\": " << (ok && daemon_rc == 0 ? "true" : "false")
      << ", \"gpus\": " << gpus << ", \"procs_per_gpu\": " << procs << ", \"workload\": \""
      << workload << "\", \"rounds\": " << rounds << ", \"warmup\": " << warmup
      << ", \"jobs\": " << jobs << ", \"seconds\": " << secs
      << ", \"jobs_per_s\": " << (secs > 0 ? jobs / secs : 0.0) << ", \"per_gpu_jobs_per_s\": [";
    for (int g = 0; g < gpus; ++g)
        o << (g ? ", " : "")
          << (gpu_end[g] > gpu_begin[g] ? procs * rounds / ((gpu_end[g] - gpu_begin[g]) * 1e-9) : 0.0);
    o << "], \"reduce_path\": \""
      << (shared ? "shared-GPU test mode: per-GVM records (vgpud --fold-out) folded on the host"
                 : "ncclAllGather across the per-GPU GVMs (vgpud rank 0 folds in rank order)")
      << "\", \"record\": [";
    for (std::size_t i = 0; i < host_fold.size(); ++i) o << (i ? ", " : "") << host_fold[i];
    o << "], \"nccl_reduce\": " << (reduce.empty() ? "null" : reduce)
      << ", \"nccl_matches_rank_fold\": " << (reduce_matches ? "true" : "false")
      << ", \"affinity\": [";
    for (int g = 0; g < gpus; ++g) o << (g ? ", " : "") << "\"" << join_cpus(gpu_cpus[g]) << "\"";
    o << "], \"failed_workers\": " << failed << "}";
    std::cout << o.str() << std::endl;
    if (!out_path.empty()) std::ofstream(out_path) << o.str() << "\n";
    // the run directory holds only this run's ids, records and metrics
    for (const char* f : {"/ncclid", "/reduce.json"}) unlink((run + f).c_str());
    for (int g = 0; g < gpus; ++g)
        for (const std::string f : {"/ready", "/fold", "/metrics"}) {
            unlink((run + f + std::to_string(g)).c_str());
            unlink((run + f + std::to_string(g) + ".json").c_str());
            unlink((run + f + std::to_string(g) + ".csv").c_str());
        }
    rmdir(run.c_str());
    return ok && daemon_rc == 0 ? 0 : 1;
}
