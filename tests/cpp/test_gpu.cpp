// [gpu] parity of the sm_100a payload kernels against the CPU oracle,
// through every path a client can reach them: the GVM (loopback and OS
// transports, PS-1 batched launches and PS-2 triples, both data planes),
// PayloadRegistry::execute and the NativeVgpu baseline.
// Bars: bit-exact for vector-add / vector-scale / identity / nas-ep;
// black-scholes L1-relative <= 1e-6 vs binary64; sgemm relative
// Frobenius <= 1e-5 vs binary64 accumulation.
#include <sys/wait.h>
#include <unistd.h>

#include <cmath>
#include <cstring>
#include <thread>

#include "minitest.hpp"
#include "vgpu/client.hpp"
#include "vgpu/npb_cg.hpp"
#include "vgpu_cuda.h"
#include "vgpu_oracle.h"

using namespace vgpu;
using namespace std::chrono_literals;

namespace {

GvmConfig gcfg(std::uint32_t clients, std::uint64_t shm = 16 << 20, Micros window = 2000) {
    GvmConfig g;
    g.max_clients = clients;
    g.barrier_size = clients;
    g.barrier_window = window;
    g.per_client_shm_bytes = shm;
    g.t_init = 100;
    return g;
}

KernelDescriptor desc(const std::string& id, bool compute_intensive = true) {
    KernelDescriptor d;
    d.payload_id = id;
    d.t_data_in = compute_intensive ? 20 : 60;
    d.t_comp = compute_intensive ? 50 : 20;
    d.t_data_out = compute_intensive ? 20 : 40;
    return d;
}

template <class T>
Bytes pack(const std::vector<T>& v) {
    Bytes b(v.size() * sizeof(T));
    if (!b.empty()) std::memcpy(b.data(), v.data(), b.size());
    return b;
}

template <class T>
std::vector<T> unpack(const Bytes& b) {
    std::vector<T> v(b.size() / sizeof(T));
    if (!b.empty()) std::memcpy(v.data(), b.data(), b.size());
    return v;
}

Bytes vadd_input(std::size_t n, std::uint64_t seed) {
    std::vector<float> v(2 * n);
    std::uint64_t s = seed;
    for (auto& x : v) x = vo_rng_uniform(&s, -1000.f, 1000.f);
    return pack(v);
}

Bytes vadd_expect(const Bytes& in) {
    const std::size_t n = in.size() / 8;
    std::vector<float> out(n);
    const float* a = reinterpret_cast<const float*>(in.data());
    vo_vector_add(out.data(), a, a + n, n);
    return pack(out);
}

Bytes ep_input(std::uint32_t m, std::uint64_t first, std::uint64_t count) {
    vgpu_ep_params p{m, 16, first, count, 0};
    Bytes b(sizeof p);
    std::memcpy(b.data(), &p, sizeof p);
    return b;
}

Bytes ep_expect(const Bytes& in) {
    vgpu_ep_params p;
    std::memcpy(&p, in.data(), sizeof p);
    vgpu_ep_result r;
    vo_ep_job(&p, &r);
    Bytes b(sizeof r);
    std::memcpy(b.data(), &r, sizeof r);
    return b;
}

Bytes bs_input(std::size_t n, std::uint64_t seed) {
    std::vector<float> v(3 * n);
    std::uint64_t s = seed;
    for (std::size_t i = 0; i < n; ++i) {
        v[i] = vo_rng_uniform(&s, 5.f, 30.f);
        v[n + i] = vo_rng_uniform(&s, 1.f, 100.f);
        v[2 * n + i] = vo_rng_uniform(&s, 0.25f, 10.f);
    }
    return pack(v);
}

double bs_l1_error(const Bytes& in, const Bytes& out) {
    const std::size_t n = in.size() / 12;
    const float* f = reinterpret_cast<const float*>(in.data());
    std::vector<double> call(n), put(n);
    vo_black_scholes(f, f + n, f + 2 * n, n, VGPU_BS_RISKFREE, VGPU_BS_VOLATILITY, call.data(),
                     put.data());
    const auto got = unpack<float>(out);
    double num = 0.0, den = 0.0;
    for (std::size_t i = 0; i < n; ++i) {
        num += std::fabs(call[i] - got[i]) + std::fabs(put[i] - got[n + i]);
        den += std::fabs(call[i]) + std::fabs(put[i]);
    }
    return den > 0 ? num / den : num;
}

Bytes mm_input(std::size_t n, std::uint64_t seed) {
    std::vector<float> v(2 * n * n);
    std::uint64_t s = seed;
    for (auto& x : v) x = vo_rng_uniform(&s, -1.f, 1.f);
    return pack(v);
}

double mm_rel_error(const Bytes& in, const Bytes& out) {
    const std::size_t n = static_cast<std::size_t>(std::llround(std::sqrt(in.size() / 8.0)));
    const float* f = reinterpret_cast<const float*>(in.data());
    std::vector<double> c(n * n);
    vo_sgemm(f, f + n * n, n, c.data());
    const auto got = unpack<float>(out);
    double num = 0.0, den = 0.0;
    for (std::size_t i = 0; i < n * n; ++i) {
        num += (c[i] - got[i]) * (c[i] - got[i]);
        den += c[i] * c[i];
    }
    return den > 0 ? std::sqrt(num / den) : std::sqrt(num);
}

}  // namespace

TEST_CASE("[gpu] device is a B200-class part") {
    int n = 0;
    REQUIRE(vgpu_cu_device_count(&n) == VGPU_CU_OK);
    REQUIRE(n >= 1);
}

TEST_CASE("[gpu] reference goldens through PayloadRegistry::execute") {
    const auto& reg = PayloadRegistry::builtins();
    const Bytes data{1, 2, 3, 4, 5};
    CHECK(reg.execute("identity", data) == data);
    CHECK(unpack<float>(reg.execute("vector-add", pack<float>({1.f, 2.f, 3.f, 4.f}))) ==
          std::vector<float>({4.f, 6.f}));
    CHECK(unpack<float>(reg.execute("vector-scale", pack<float>({1.5f}))) ==
          std::vector<float>({3.0f}));
    CHECK_THROWS_AS((void)reg.execute("vector-add", Bytes{1, 2, 3}), PayloadError);
    CHECK_THROWS_AS((void)reg.execute("vector-scale", Bytes{1, 2, 3}), PayloadError);
    CHECK_THROWS_AS((void)reg.execute("no-such", Bytes{}), PayloadError);
    // custom factor still lands on the device kernel
    auto r2 = PayloadRegistry::with_builtins();
    r2.register_payload("scale-3.25", make_vector_scale(3.25f));
    REQUIRE(r2.device_kernel("scale-3.25") != nullptr);
    CHECK(unpack<float>(r2.execute("scale-3.25", pack<float>({2.f}))) == std::vector<float>({6.5f}));
}

TEST_CASE("[gpu] vector-add / vector-scale bit-exact vs serial oracle (test_payload sizes)") {
    const auto& reg = PayloadRegistry::builtins();
    auto scaled = PayloadRegistry::with_builtins();
    scaled.register_payload("scale-3.25", make_vector_scale(3.25f));
    for (std::size_t n : {1u, 7u, 1024u, 100003u, 1u << 20}) {
        const Bytes in = vadd_input(n, 41 + n);
        CHECK(reg.execute("vector-add", in) == vadd_expect(in));
        const Bytes a(in.begin(), in.begin() + 4 * n);
        std::vector<float> want(n);
        vo_vector_scale(want.data(), reinterpret_cast<const float*>(a.data()), 3.25f, n);
        CHECK(scaled.execute("scale-3.25", a) == pack(want));
        vo_vector_scale(want.data(), reinterpret_cast<const float*>(a.data()), 2.0f, n);
        CHECK(reg.execute("vector-scale", a) == pack(want));
    }
    CHECK(reg.execute("vector-add", Bytes{}).empty());
}

TEST_CASE("[gpu] two-client flow with the real kernels (virtual clock)") {
    LoopbackHub hub;
    auto d = GvmDaemon::start_loopback(gcfg(2, 1 << 16, 1'000'000'000), hub);
    VgpuHandle a = req(hub);
    VgpuHandle b = req(hub);
    a.snd(pack<float>({1, 2, 3, 4}));
    b.snd(pack<float>({10, 20, 30, 40}));
    std::thread tb([&] { b.str(desc("vector-add")); });
    a.str(desc("vector-add"));
    tb.join();
    CHECK(a.stp());  // virtual clock: done by the time STR is acked
    CHECK(b.stp());
    CHECK(unpack<float>(a.rcv()) == std::vector<float>({4, 6}));
    CHECK(unpack<float>(b.rcv()) == std::vector<float>({40, 60}));
    const auto m = d->metrics();
    CHECK(m.batches_flushed == 1);
    CHECK(m.kernel_launches == 1);  // one batched launch for both clients
    CHECK(m.batches.at(0).model_makespan_us == 130);  // PS-1 form at N = 2: 2(20+20)+50
}

TEST_CASE("[gpu] GVM parity for every payload, PS-1 and PS-2, both data planes") {
    for (DataPlane plane : {DataPlane::ZeroCopy, DataPlane::Snapshot})
        for (bool ci : {true, false}) {
            LoopbackHub hub;
            auto g = gcfg(4, 16 << 20);
            g.data_plane = plane;
            g.clock = ClockMode::Real;
            auto d = GvmDaemon::start_loopback(g, hub);
            std::vector<std::string> err(4);
            std::vector<std::thread> ts;
            for (int w = 0; w < 4; ++w)
                ts.emplace_back([&, w] {
                    try {
                        VgpuHandle h = req(hub);
                        for (int rep = 0; rep < 3; ++rep) {
                            const std::size_t n = rep == 0 ? 100003 : (1u << 18) + 4 * w;
                            const Bytes in = vadd_input(n, 1000 * w + rep);
                            if (h.run_task(in, desc("vector-add", ci)) != vadd_expect(in))
                                err[w] += "vadd ";
                            const Bytes ep = ep_input(20, 3 * w, 2 + w % 2);
                            if (h.run_task(ep, desc("nas-ep", ci)) != ep_expect(ep)) err[w] += "ep ";
                            const Bytes bs = bs_input(4096 + w, 7 + w);
                            if (bs_l1_error(bs, h.run_task(bs, desc("black-scholes", ci))) > 1e-6)
                                err[w] += "bs ";
                            const Bytes mm = mm_input(w == 3 ? 100 : 128, 11 + w);
                            if (mm_rel_error(mm, h.run_task(mm, desc("sgemm", ci))) > 1e-5)
                                err[w] += "mm ";
                            const Bytes id{1, 2, 3, static_cast<std::uint8_t>(w)};
                            if (h.run_task(id, desc("identity", ci)) != id) err[w] += "id ";
                        }
                        h.rls();
                    } catch (const std::exception& e) {
                        err[w] += e.what();
                    }
                });
            for (auto& t : ts) t.join();
            for (int w = 0; w < 4; ++w) {
                if (!err[w].empty()) MESSAGE("worker " + std::to_string(w) + ": " + err[w]);
                CHECK(err[w].empty());
            }
            const auto m = d->metrics();
            CHECK(m.device_tasks == 4 * 3 * 5);
            bool style_ok = true;
            for (const auto& b : m.batches)
                style_ok &= b.style == (ci ? ProgrammingStyle::PS1 : ProgrammingStyle::PS2);
            CHECK(style_ok);
            bool timed = true;
            for (const auto& t : m.tasks) timed &= t.pure_gpu_us > 0 || t.end_to_end_us > 0;
            CHECK(timed);
        }
}

TEST_CASE("[gpu] mixed-kernel batch and EP slices fold to the whole class") {
    LoopbackHub hub;
    auto d = GvmDaemon::start_loopback(gcfg(5, 4 << 20), hub);
    std::vector<Bytes> outs(5);
    std::vector<Bytes> ins = {ep_input(22, 0, 16), ep_input(22, 16, 16), ep_input(22, 32, 32),
                              vadd_input(5000, 3), mm_input(64, 5)};
    const char* ids[] = {"nas-ep", "nas-ep", "nas-ep", "vector-add", "sgemm"};
    std::vector<std::thread> ts;
    for (int w = 0; w < 5; ++w)
        ts.emplace_back([&, w] {
            VgpuHandle h = req(hub);
            outs[w] = h.run_task(ins[w], desc(ids[w]));
        });
    for (auto& t : ts) t.join();
    CHECK(outs[3] == vadd_expect(ins[3]));
    CHECK(mm_rel_error(ins[4], outs[4]) <= 1e-5);
    vgpu_ep_result parts[3], folded, whole;
    for (int i = 0; i < 3; ++i) {
        CHECK(outs[i] == ep_expect(ins[i]));
        std::memcpy(&parts[i], outs[i].data(), sizeof parts[i]);
    }
    vo_ep_fold(parts, 3, &folded);
    vgpu_ep_params p{22, 16, 0, 64, 0};
    vo_ep_job(&p, &whole);
    CHECK(folded.pairs == whole.pairs);
    for (int i = 0; i < 10; ++i) CHECK(folded.q[i] == whole.q[i]);
    CHECK(std::fabs(folded.sx - whole.sx) <= 1e-9 * std::fabs(whole.sx));
    CHECK(d->metrics().batches_flushed == 1);
}

TEST_CASE("[gpu] NAS EP class S on the GPU equals NPB's verification sums") {
    const Bytes in = ep_input(24, 0, 256);
    const Bytes out = PayloadRegistry::builtins().execute("nas-ep", in);
    CHECK(out == ep_expect(in));
    vgpu_ep_result r;
    std::memcpy(&r, out.data(), sizeof r);
    CHECK(r.pairs == 13176389ull);
    CHECK(std::fabs((r.sx - -3.247834652034740e3) / 3.247834652034740e3) < 1e-8);
    CHECK(std::fabs((r.sy - -6.958407078382297e3) / 6.958407078382297e3) < 1e-8);
}

TEST_CASE("[gpu] NAS CG class S through the C++ API meets NPB's verification") {
    const npb::CgClass c = npb::cg_class('S');
    const Bytes in = npb::make_cg_input(c.n, c.nonzer, c.niter, c.shift);
    const Bytes out = PayloadRegistry::builtins().execute("nas-cg", in);
    REQUIRE(out.size() == sizeof(vgpu_cg_result));
    vgpu_cg_result r;
    std::memcpy(&r, out.data(), sizeof r);
    CHECK(std::fabs(r.zeta - c.zeta_verify) / c.zeta_verify <= 1e-10);
    vgpu_cg_result o;
    REQUIRE(vo_cg_run(in.data(), in.size(), &o) == 0);
    CHECK(std::fabs(r.zeta - o.zeta) / o.zeta <= 1e-12);
    CHECK(r.nnz == o.nnz);
    // the oracle's NPB makea builds the same bytes
    Bytes ref(vo_cg_makea(c.n, c.nonzer, c.niter, c.shift, nullptr, 0));
    vo_cg_makea(c.n, c.nonzer, c.niter, c.shift, ref.data(), ref.size());
    CHECK(ref == in);
}

TEST_CASE("[gpu] vector-mul and electrostatics through the C++ API") {
    std::vector<float> v(2 * 1001);
    for (std::size_t i = 0; i < v.size(); ++i) v[i] = 0.25f * static_cast<float>(i % 97) - 7.0f;
    Bytes out = PayloadRegistry::builtins().execute("vector-mul", pack<float>(v));
    std::vector<float> want(1001);
    vo_vector_mul(want.data(), v.data(), v.data() + 1001, 1001);
    CHECK(out == pack<float>(want));
    // one charge: V = q / r exactly up to rsqrt.approx
    vgpu_es_header h{};
    h.natoms = 1;
    h.nx = 5;
    h.ny = 3;
    h.nz = 2;
    h.spacing = 0.5f;
    Bytes in(sizeof h + 16);
    const float atom[4] = {0.3f, 0.4f, 0.1f, -2.0f};
    std::memcpy(in.data(), &h, sizeof h);
    std::memcpy(in.data() + sizeof h, atom, 16);
    out = PayloadRegistry::builtins().execute("electrostatics", in);
    REQUIRE(out.size() == 4u * 30u);
    std::vector<double> ref(30);
    REQUIRE(vo_es(in.data(), in.size(), ref.data()) == 0);
    const float* got = reinterpret_cast<const float*>(out.data());
    for (int i = 0; i < 30; ++i) CHECK(std::fabs(got[i] - ref[i]) <= 1e-6 * std::fabs(ref[i]));
}

TEST_CASE("[gpu] malformed inputs fail through STP with Payload, slot stays usable after RLS") {
    LoopbackHub hub;
    auto d = GvmDaemon::start_loopback(gcfg(1, 1 << 16), hub);
    const std::pair<const char*, Bytes> bad[] = {
        {"vector-add", Bytes{1, 2, 3}},
        {"vector-scale", Bytes{1, 2}},
        {"black-scholes", Bytes(13)},
        {"sgemm", Bytes(24)},
        {"nas-ep", Bytes(31)},
        {"nas-ep", ep_input(30, 1ull << 14, 1)},
        {"vector-mul", Bytes{1, 2, 3}},
        {"nas-cg", Bytes(23)},
        {"nas-cg", Bytes(64)},  // header says n = 0
        {"electrostatics", Bytes(31)},
        {"electrostatics", Bytes(48)},  // header says 0 x 0 x 0, spacing 0
    };
    for (const auto& [id, in] : bad) {
        VgpuHandle h = req(hub);
        h.snd(in);
        h.str(desc(id));
        try {
            h.stp_wait();
            FAIL(std::string("accepted malformed ") + id);
        } catch (const VgpuError& e) {
            CHECK(e.code() == ErrCode::Payload);
        }
        h.rls();
    }
    VgpuHandle h = req(hub);
    CHECK(h.run_task(pack<float>({1, 2, 3, 4}), desc("vector-add")) == pack<float>({4, 6}));
    // empty input (n = 0 is valid: no launch) and a 64-byte input, both on
    // the inline SND path (<= 64 B snapshotted at SND, no DMA round trip)
    CHECK(h.run_task(Bytes{}, desc("vector-add")).empty());
    std::vector<float> v(16);
    for (int i = 0; i < 16; ++i) v[i] = 0.5f * static_cast<float>(i);
    const Bytes out = h.run_task(pack<float>(v), desc("vector-add"));
    std::vector<float> want(8);
    for (int i = 0; i < 8; ++i) want[i] = v[i] + v[8 + i];
    CHECK(out == pack<float>(want));
}

TEST_CASE("[gpu] OS transport: forked SPMD clients through one GVM (real clock)") {
    GvmConfig g = gcfg(4, 8 << 20, 20000);
    g.clock = ClockMode::Real;
    g.instance = "gt" + std::to_string(getpid());
    unlink_os_instance(g.instance, g.max_clients);
    std::vector<pid_t> kids;
    for (std::uint32_t w = 0; w < 4; ++w) {
        const pid_t pid = fork();
        if (pid == 0) {
            for (int attempt = 0; attempt < 2000; ++attempt) {
                try {
                    VgpuHandle h = req(g.instance);
                    for (int rep = 0; rep < 10; ++rep) {
                        // >= 4 MiB inputs: streamed SNDs (parts uploaded while
                        // the copy runs), odd lengths included
                        const Bytes in = vadd_input((1u << 20) - 5u * (rep % 3), w * 100 + rep);
                        if (h.run_task(in, desc("vector-add", false)) != vadd_expect(in)) _exit(3);
                    }
                    h.rls();
                    _exit(0);
                } catch (const TransportError&) {
                    usleep(5000);
                } catch (...) {
                    _exit(5);
                }
            }
            _exit(6);
        }
        kids.push_back(pid);
    }
    auto d = GvmDaemon::start_os(g);
    for (pid_t k : kids) {
        int st = 0;
        waitpid(k, &st, 0);
        CHECK(WIFEXITED(st));
        CHECK(WEXITSTATUS(st) == 0);
    }
    const auto m = d->metrics();
    CHECK(m.tasks.size() == 40);
    bool measured = true;
    for (const auto& t : m.tasks) measured &= t.h2d_us > 0 && t.d2h_us > 0 && t.pure_gpu_us > 0;
    CHECK(measured);
    for (const auto& b : m.batches) CHECK(b.measured_makespan_us > 0);
    d->stop();
}

TEST_CASE("[gpu] NativeVgpu (own context, pageable copies) matches the GVM") {
    const Bytes in = vadd_input(123457, 99);
    NativeVgpu n{NativeConfig{}};
    CHECK(n.run_task(in, desc("vector-add")) == vadd_expect(in));
    const Bytes ep = ep_input(20, 5, 3);
    CHECK(n.run_task(ep, desc("nas-ep")) == ep_expect(ep));
    const Bytes mm = mm_input(256, 17);
    CHECK(mm_rel_error(mm, n.run_task(mm, desc("sgemm"))) <= 1e-5);
    const Bytes bs = bs_input(1 << 16, 23);
    CHECK(bs_l1_error(bs, n.run_task(bs, desc("black-scholes"))) <= 1e-6);
}

TEST_CASE("[gpu] fault containment: a trapping task fails alone, the handle rebuilds or fails fast") {
    if (!std::getenv("VGPU_FAULT_CHILD")) {
        // a sticky fault can poison this process's device for good: run the
        // case in a fresh process (this binary, filtered to this case)
        const pid_t pid = fork();
        REQUIRE(pid >= 0);
        if (pid == 0) {
            setenv("VGPU_FAULT_CHILD", "1", 1);
            execl("/proc/self/exe", "vgpu-tests", "fault containment", static_cast<char*>(nullptr));
            _exit(127);
        }
        int st = 0;
        REQUIRE(waitpid(pid, &st, 0) == pid);
        CHECK(WIFEXITED(st));
        CHECK(WEXITSTATUS(st) == 0);
        return;
    }
    setenv("VGPU_ENABLE_FAULT_INJECTION", "1", 1);
    vgpu_cu_dev* dev = nullptr;
    REQUIRE(vgpu_cu_open(0, 2, 1 << 20, &dev) == VGPU_CU_OK);
    void* host = nullptr;
    REQUIRE(vgpu_cu_alloc_pinned(dev, 2 << 20, &host) == VGPU_CU_OK);
    auto* in = static_cast<std::uint8_t*>(host);
    auto* out = in + (1 << 20);
    auto run_vadd = [&](std::uint64_t seed, std::uint64_t tag) {
        const Bytes data = vadd_input(4096, seed);
        std::memcpy(in, data.data(), data.size());
        vgpu_cu_task t{};
        t.slot = 1;
        t.kernel = VGPU_CU_K_VADD;
        t.h_in = in;
        t.in_bytes = data.size();
        t.h_out = out;
        t.out_bytes = data.size() / 2;
        t.tag = tag;
        std::uint64_t bid = 0;
        const int rc = vgpu_cu_submit_batch(dev, 1, &t, 1, &bid);
        if (rc != VGPU_CU_OK)
            std::fprintf(stderr, "submit after %llu reset(s): %s: %s\n",
                         (unsigned long long)vgpu_cu_generation(dev), vgpu_cu_strerror(rc), vgpu_cu_last_error());
        REQUIRE(rc == VGPU_CU_OK);
        vgpu_cu_done d{};
        std::uint32_t n = 0;
        for (int i = 0; i < 100000 && n == 0; ++i) {
            REQUIRE(vgpu_cu_poll(dev, &d, 1, &n) == VGPU_CU_OK);
            if (!n) usleep(50);
        }
        REQUIRE(n == 1);
        CHECK(d.tag == tag);
        CHECK(d.status == VGPU_CU_OK);
        CHECK(Bytes(out, out + data.size() / 2) == vadd_expect(data));
    };
    run_vadd(1, 1);
    CHECK(vgpu_cu_generation(dev) == 0);
    // slot 2's task traps: the op is reported failed, the context is rebuilt
    REQUIRE(vgpu_cu_inject_fault(dev, 2, 77) == VGPU_CU_OK);
    vgpu_cu_done d{};
    std::uint32_t n = 0;
    for (int i = 0; i < 100000 && n == 0; ++i) {
        REQUIRE(vgpu_cu_poll(dev, &d, 1, &n) == VGPU_CU_OK);
        if (!n) usleep(50);
    }
    REQUIRE(n == 1);
    CHECK(d.tag == 77);
    CHECK(d.status == VGPU_CU_EINTERNAL);
    CHECK(vgpu_cu_generation(dev) == 1);
    CHECK(std::string(vgpu_cu_last_fault(dev)).size() > 0);
    std::fprintf(stderr, "contained fault: %s (device %s)\n", vgpu_cu_last_fault(dev),
                 vgpu_cu_device_lost(dev) ? "lost: the owner restarts" : "rebuilt");
    if (vgpu_cu_device_lost(dev)) {
        // the driver refused a new context in this process: every later call
        // fails at once with a clear error (no hang); vgpud then re-executes
        vgpu_cu_task t{};
        t.slot = 1;
        t.kernel = VGPU_CU_K_IDENTITY;
        t.h_in = in;
        t.in_bytes = 16;
        t.h_out = out;
        t.out_bytes = 16;
        std::uint64_t bid = 0;
        CHECK(vgpu_cu_submit_batch(dev, 1, &t, 1, &bid) == VGPU_CU_EINTERNAL);
        CHECK(std::string(vgpu_cu_last_error()).find("context lost") != std::string::npos);
        CHECK(vgpu_cu_upload(dev, 1, in, 16, 9) == VGPU_CU_EINTERNAL);
    } else {
        // the same handle and the same staging buffer serve the next tasks
        run_vadd(2, 2);
        run_vadd(3, 3);
    }
    vgpu_cu_free_pinned(dev, host);
    vgpu_cu_close(dev);
}
