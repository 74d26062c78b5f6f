// ORACLE — the reference arm. Links the UNMODIFIED reference library
// (oracle/_ref/libvgpu_ref.a, built from /root/reference/proj/src by
// oracle/Makefile.ref) and drives its own public API the way its harness
// does (proj/src/bench/bench.cpp:186-231; tests/acceptance.cpp:412-479):
// N forked SPMD clients lease a VGPU over the OS transport from
// GvmDaemon::start(cfg, open_os_daemon_transport(...), &registry) and run
// `rounds` tasks each with VgpuHandle::run_task; the clock is Virtual so no
// pacing sleeps are timed.
//
// Registry: the reference builtins (vector-add is the reference's own CPU
// arithmetic, OpenMP-parallel) plus, for workloads the reference has no
// arithmetic for, the oracle restatements (nas-ep, black-scholes, sgemm,
// nas-cg, nas-mg, vector-mul, electrostatics)
// registered through the reference's register_payload (payload.hpp:36).
//
// --native: SURVEY.md §8(d)(ii), the reference's per-process CPU path: the
// same N forked workers each run the reference's NativeVgpu (virtual clock:
// the payload executes in the calling process, no daemon) with
// OMP_NUM_THREADS = max(1, cores / N) so the processes do not oversubscribe
// the host (proj/include/vgpu/client.hpp:87-113, proj/src/client.cpp:196-232).
//
// Output: one JSON line {jobs_per_s, per-round timestamps summary, ...}.
#include <omp.h>
#include <sys/mman.h>
#include <sys/wait.h>
#include <unistd.h>

#include <chrono>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "vgpu/client.hpp"
#include "vgpu/daemon.hpp"
#include "vgpu_oracle.h"
#include "../paper_1511_07658_b200/csrc/tools/workloads.hpp"

namespace {

std::int64_t now_ns() {
    return std::chrono::duration_cast<std::chrono::nanoseconds>(
               std::chrono::steady_clock::now().time_since_epoch())
        .count();
}

vgpu::Bytes ep_payload(vgpu::ByteView in) {
    if (in.size() != sizeof(vgpu_ep_params))
        throw vgpu::PayloadError(vgpu::PayloadError::Kind::MalformedInput, "nas-ep input");
    vgpu_ep_params p;
    std::memcpy(&p, in.data(), sizeof p);
    vgpu_ep_result r;
    if (vo_ep_job(&p, &r) != 0)
        throw vgpu::PayloadError(vgpu::PayloadError::Kind::MalformedInput, "nas-ep params");
    vgpu::Bytes out(sizeof r);
    std::memcpy(out.data(), &r, sizeof r);
    return out;
}

vgpu::Bytes bs_payload(vgpu::ByteView in) {
    if (in.size() % 12)
        throw vgpu::PayloadError(vgpu::PayloadError::Kind::MalformedInput, "black-scholes input");
    const std::size_t n = in.size() / 12;
    const float* f = reinterpret_cast<const float*>(in.data());
    std::vector<double> c(n), p(n);
    vo_black_scholes(f, f + n, f + 2 * n, n, VGPU_BS_RISKFREE, VGPU_BS_VOLATILITY, c.data(), p.data());
    vgpu::Bytes out(8 * n);
    float* o = reinterpret_cast<float*>(out.data());
    for (std::size_t i = 0; i < n; ++i) {
        o[i] = static_cast<float>(c[i]);
        o[n + i] = static_cast<float>(p[i]);
    }
    return out;
}

vgpu::Bytes mm_payload(vgpu::ByteView in) {
    const std::size_t n = static_cast<std::size_t>(std::llround(std::sqrt(in.size() / 8.0)));
    if (in.size() != 8 * n * n)
        throw vgpu::PayloadError(vgpu::PayloadError::Kind::MalformedInput, "sgemm input");
    const float* f = reinterpret_cast<const float*>(in.data());
    std::vector<double> c(n * n);
    vo_sgemm(f, f + n * n, n, c.data());
    vgpu::Bytes out(4 * n * n);
    float* o = reinterpret_cast<float*>(out.data());
    for (std::size_t i = 0; i < n * n; ++i) o[i] = static_cast<float>(c[i]);
    return out;
}

vgpu::Bytes cg_payload(vgpu::ByteView in) {
    vgpu_cg_result r;
    if (vo_cg_run(in.data(), in.size(), &r) != 0)
        throw vgpu::PayloadError(vgpu::PayloadError::Kind::MalformedInput, "nas-cg input");
    vgpu::Bytes out(sizeof r);
    std::memcpy(out.data(), &r, sizeof r);
    return out;
}

vgpu::Bytes vmul_payload(vgpu::ByteView in) {
    if (in.size() % 8)
        throw vgpu::PayloadError(vgpu::PayloadError::Kind::MalformedInput, "vector-mul input");
    const std::size_t n = in.size() / 8;
    const float* f = reinterpret_cast<const float*>(in.data());
    vgpu::Bytes out(4 * n);
    vo_vector_mul(reinterpret_cast<float*>(out.data()), f, f + n, n);
    return out;
}

vgpu::Bytes es_payload(vgpu::ByteView in) {
    if (in.size() < sizeof(vgpu_es_header))
        throw vgpu::PayloadError(vgpu::PayloadError::Kind::MalformedInput, "electrostatics input");
    vgpu_es_header h;
    std::memcpy(&h, in.data(), sizeof h);
    const std::size_t pts = static_cast<std::size_t>(h.nx) * h.ny * h.nz;
    std::vector<double> v(pts);
    if (vo_es(in.data(), in.size(), v.data()) != 0)
        throw vgpu::PayloadError(vgpu::PayloadError::Kind::MalformedInput, "electrostatics input");
    vgpu::Bytes out(4 * pts);
    float* o = reinterpret_cast<float*>(out.data());
    for (std::size_t i = 0; i < pts; ++i) o[i] = static_cast<float>(v[i]);
    return out;
}

// the CG program's makea: the oracle's NPB restatement
vgpu::Bytes cg_makea(char cls) {
    static const struct { char c; std::uint32_t n, nonzer, niter; double shift; } kClasses[] = {
        {'S', 1400, 7, 15, 10.0}, {'W', 7000, 8, 15, 12.0}, {'A', 14000, 11, 15, 20.0},
        {'B', 75000, 13, 75, 60.0}, {'C', 150000, 15, 75, 110.0}};
    for (const auto& k : kClasses)
        if (k.c == cls) {
            vgpu::Bytes b(vo_cg_makea(k.n, k.nonzer, k.niter, k.shift, nullptr, 0));
            vo_cg_makea(k.n, k.nonzer, k.niter, k.shift, b.data(), b.size());
            return b;
        }
    throw std::invalid_argument("unknown NPB CG class");
}

vgpu::Bytes mg_payload(vgpu::ByteView in) {
    vgpu_mg_result r;
    if (vo_mg_run(in.data(), in.size(), &r, nullptr) != 0)
        throw vgpu::PayloadError(vgpu::PayloadError::Kind::MalformedInput, "nas-mg input");
    vgpu::Bytes out(sizeof r);
    std::memcpy(out.data(), &r, sizeof r);
    return out;
}

// the MG program's zran3: the oracle's NPB restatement
vgpu::Bytes mg_make(char cls) {
    static const struct { char c; std::uint32_t nx, nit, coeffs; } kClasses[] = {
        {'S', 32, 4, 0}, {'W', 128, 4, 0}, {'A', 256, 4, 0}, {'B', 256, 20, 1}, {'C', 512, 20, 1}};
    for (const auto& k : kClasses)
        if (k.c == cls) {
            vgpu::Bytes b(vo_mg_make_input(k.nx, k.nit, k.coeffs, nullptr, 0));
            vo_mg_make_input(k.nx, k.nit, k.coeffs, b.data(), b.size());
            return b;
        }
    throw std::invalid_argument("unknown NPB MG class");
}

}  // namespace

int main(int argc, char** argv) {
    vgpu::wl::cg_builder() = cg_makea;
    vgpu::wl::mg_builder() = mg_make;
    std::string workload = "vecadd", instance = "refbench" + std::to_string(getpid());
    std::uint32_t procs = 4, rounds = 3, warmup = 1;
    bool native = false;
    vgpu::wl::Sizes sizes;
    for (int i = 1; i < argc; ++i)
        if (std::string(argv[i]) == "--native") {
            native = true;
            for (int j = i; j + 1 < argc; ++j) argv[j] = argv[j + 1];
            --argc;
            break;
        }
    for (int i = 1; i + 1 < argc; i += 2) {
        const std::string a = argv[i], v = argv[i + 1];
        if (a == "--workload") workload = v;
        else if (a == "--procs") procs = std::stoul(v);
        else if (a == "--rounds") rounds = std::stoul(v);
        else if (a == "--warmup") warmup = std::stoul(v);
        else if (a == "--instance") instance = v;
        else if (a == "--vecadd-n") sizes.vecadd_n = std::stoull(v);
        else if (a == "--ep-m") sizes.ep_m = std::stoul(v);
        else if (a == "--ep-batches") sizes.ep_batches = std::stoull(v);
        else if (a == "--bs-n") sizes.bs_n = std::stoull(v);
        else if (a == "--mm-n") sizes.mm_n = std::stoul(v);
        else if (a == "--cg-class") sizes.cg_class = v[0];
        else if (a == "--mg-class") sizes.mg_class = v[0];
        else if (a == "--es-atoms") sizes.es_atoms = std::stoul(v);
    }
    const std::uint32_t total = warmup + rounds;
    // per-worker timestamps live in a shared anonymous mapping
    const std::size_t slots = static_cast<std::size_t>(procs) * total * 2;
    auto* ts = static_cast<std::int64_t*>(mmap(nullptr, slots * 8 + 64 * procs, PROT_READ | PROT_WRITE,
                                               MAP_SHARED | MAP_ANONYMOUS, -1, 0));
    auto* status = reinterpret_cast<std::int32_t*>(ts + slots);
    int go_pipe[2];
    if (pipe(go_pipe) != 0) return 1;
    vgpu::unlink_os_instance(instance, procs);

    vgpu::PayloadRegistry reg = vgpu::PayloadRegistry::with_builtins();
    reg.register_payload("nas-ep", ep_payload);
    reg.register_payload("black-scholes", bs_payload);
    reg.register_payload("sgemm", mm_payload);
    reg.register_payload("nas-cg", cg_payload);
    reg.register_payload("vector-mul", vmul_payload);
    reg.register_payload("electrostatics", es_payload);
    reg.register_payload("nas-mg", mg_payload);
    const unsigned cores = std::max(1u, std::thread::hardware_concurrency());
    const unsigned omp_threads = native ? std::max(1u, cores / procs) : cores;

    std::vector<pid_t> kids;
    for (std::uint32_t w = 0; w < procs; ++w) {
        const pid_t pid = fork();
        if (pid == 0) {
            close(go_pipe[1]);
            int st = 1;
            try {
                const vgpu::wl::Job job = vgpu::wl::make_job(workload, w, procs, sizes);
                vgpu::KernelDescriptor d;
                d.payload_id = job.desc.payload_id;
                d.t_data_in = job.desc.t_data_in;
                d.t_comp = job.desc.t_comp;
                d.t_data_out = job.desc.t_data_out;
                d.grid_size = job.desc.grid_size;
                char go = 0;
                if (read(go_pipe[0], &go, 1) != 1) _exit(2);
                if (native) {
                    omp_set_num_threads(static_cast<int>(omp_threads));
                    vgpu::NativeVgpu nv({}, &reg);  // virtual clock: no pacing sleeps
                    st = 0;
                    for (std::uint32_t r = 0; r < total; ++r) {
                        ts[(w * total + r) * 2] = now_ns();
                        const vgpu::Bytes out = nv.run_task(job.input, d);
                        ts[(w * total + r) * 2 + 1] = now_ns();
                        if (out.size() != job.output_bytes) st = 3;
                    }
                    nv.rls();
                    status[w] = st;
                    _exit(st);
                }
                std::unique_ptr<vgpu::VgpuHandle> h;
                for (int attempt = 0; !h; ++attempt) {
                    try {
                        h = std::make_unique<vgpu::VgpuHandle>(vgpu::req(instance));
                    } catch (const vgpu::TransportError&) {
                        if (attempt > 2000) throw;
                        usleep(2000);
                    }
                }
                st = 0;
                for (std::uint32_t r = 0; r < total; ++r) {
                    ts[(w * total + r) * 2] = now_ns();
                    const vgpu::Bytes out = h->run_task(job.input, d);
                    ts[(w * total + r) * 2 + 1] = now_ns();
                    if (out.size() != job.output_bytes) st = 3;
                }
                h->rls();
            } catch (...) {
                st = 4;
            }
            status[w] = st;
            _exit(st);
        }
        kids.push_back(pid);
    }
    close(go_pipe[0]);

    vgpu::GvmConfig g;
    g.instance = instance;
    g.max_clients = procs;
    g.barrier_size = procs;
    g.barrier_window = 1'000'000;
    g.per_client_shm_bytes = vgpu::wl::region_bytes(workload, sizes);
    g.clock = vgpu::ClockMode::Virtual;
    std::unique_ptr<vgpu::GvmDaemon> daemon;
    if (!native)
        daemon = vgpu::GvmDaemon::start(
            g, vgpu::open_os_daemon_transport(instance, procs, g.per_client_shm_bytes), &reg);
    std::vector<char> go(procs, 1);
    if (write(go_pipe[1], go.data(), procs) != static_cast<ssize_t>(procs)) return 1;
    bool ok = true;
    for (pid_t k : kids) {
        int st = 0;
        waitpid(k, &st, 0);
        ok &= WIFEXITED(st) && WEXITSTATUS(st) == 0;
    }
    if (daemon) daemon->stop();
    // timed region: first finish of the warm-up rounds -> last finish
    std::int64_t t_begin = INT64_MAX, t_end = 0;
    for (std::uint32_t w = 0; w < procs; ++w) {
        const std::int64_t start = warmup ? ts[(w * total + warmup - 1) * 2 + 1]
                                          : ts[(w * total) * 2];
        t_begin = std::min(t_begin, start);
        t_end = std::max(t_end, ts[(w * total + total - 1) * 2 + 1]);
    }
    const double secs = (t_end - t_begin) * 1e-9;
    const double jobs = static_cast<double>(procs) * rounds;
    std::printf("{\"ok\": %s, \"workload\": \"%s\", \"procs\": %u, \"rounds\": %u, \"warmup\": %u, "
                "\"seconds\": %.6f, \"jobs_per_s\": %.3f, \"ms_per_round\": %.3f, \"threads\": %u, "
                "\"mode\": \"%s\", \"omp_threads_per_proc\": %u}\n",
                ok ? "true" : "false", workload.c_str(), procs, rounds, warmup, secs, jobs / secs,
                1e3 * secs / rounds, cores, native ? "native" : "gvm", omp_threads);
    return ok ? 0 : 1;
}
