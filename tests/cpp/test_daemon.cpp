// GVM protocol and session semantics on CPU. The daemon is given a test
// registry whose "vector-add" is a HOST test double (so no CUDA device is
// opened); the same flows run against the real sm_100a kernels in
// test_gpu.cpp. Expectations follow proj/tests/test_daemon.cpp:114-430,
// test_client.cpp:42-195 and acceptance criteria 8-9.
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <sys/wait.h>
#include <unistd.h>

#include <cmath>
#include <cstring>
#include <thread>

#include <random>

#include "minitest.hpp"
#include "vgpu/client.hpp"
#include "vgpu/multigpu.hpp"

using namespace vgpu;
using namespace std::chrono_literals;

namespace {

Bytes host_add(ByteView in) {  // test double of the vector-add contract
    if (in.size() % 8) throw PayloadError(PayloadError::Kind::MalformedInput, "odd input");
    const std::size_t n = in.size() / 8;
    Bytes out(4 * n);
    const float* a = reinterpret_cast<const float*>(in.data());
    float* o = reinterpret_cast<float*>(out.data());
    for (std::size_t i = 0; i < n; ++i) o[i] = a[i] + a[n + i];
    return out;
}

const PayloadRegistry& host_registry() {
    static const PayloadRegistry r = [] {
        PayloadRegistry p;
        p.register_payload("vector-add", host_add);
        p.register_payload("reverse", [](ByteView b) { return Bytes(b.rbegin(), b.rend()); });
        p.register_payload("huge", [](ByteView) { return Bytes(1 << 20); });
        return p;
    }();
    return r;
}

GvmConfig cfg(std::uint32_t clients, std::uint32_t barrier, Micros window = 1'000'000'000) {
    GvmConfig g;
    g.max_clients = clients;
    g.barrier_size = barrier;
    g.barrier_window = window;
    g.per_client_shm_bytes = 1 << 16;
    g.t_init = 100;
    g.t_ctx_switch = 10;
    return g;
}

std::unique_ptr<GvmDaemon> start(LoopbackHub& hub, GvmConfig g) {
    return GvmDaemon::start(g, hub.bind_daemon(g.max_clients, g.per_client_shm_bytes),
                            &host_registry());
}

KernelDescriptor descr(Micros in, Micros comp, Micros out, std::string id = "vector-add",
                       std::uint32_t grid = 1) {
    KernelDescriptor d;
    d.payload_id = std::move(id);
    d.t_data_in = in;
    d.t_comp = comp;
    d.t_data_out = out;
    d.grid_size = grid;
    return d;
}
const KernelDescriptor kCIdesc = descr(20, 50, 20);
const KernelDescriptor kIOIdesc = descr(60, 20, 40);

Bytes pair(float a0, float a1, float b0, float b1) {
    Bytes b(16);
    const float v[4] = {a0, a1, b0, b1};
    std::memcpy(b.data(), v, 16);
    return b;
}

struct Raw {
    std::unique_ptr<ClientChannel> ch;
    LeaseInfo lease;
    std::vector<Opcode> seen;
    explicit Raw(LoopbackHub& hub) : ch(hub.connect()) {}
    Message call(Message m, std::chrono::microseconds t = 2s) {
        ch->send(m);
        auto r = ch->recv(t);
        if (!r) throw std::runtime_error("no reply");
        seen.push_back(r->opcode);
        return *r;
    }
    Message await(std::chrono::microseconds t = 2s) {
        auto r = ch->recv(t);
        if (!r) throw std::runtime_error("no reply");
        seen.push_back(r->opcode);
        return *r;
    }
    Message req() {
        Message r = call({Opcode::Req, 0, 0, {}});
        if (r.opcode == Opcode::Ack) {
            lease = *parse_lease(r.payload);
            ch->attach_lease(lease);
        }
        return r;
    }
    Message snd(ByteView d) {
        std::memcpy(ch->region().data(), d.data(), d.size());
        return call({Opcode::Snd, lease.client_id, 0, encode_u64(d.size())});
    }
    Message snd_claim(std::uint64_t n) { return call({Opcode::Snd, lease.client_id, 0, encode_u64(n)}); }
    void str(std::uint64_t task, const KernelDescriptor& d) {
        ch->send({Opcode::Str, lease.client_id, task, encode_descriptor(d)});
    }
    Message stp(std::uint64_t t) { return call({Opcode::Stp, lease.client_id, t, {}}); }
    Message rcv(std::uint64_t t) { return call({Opcode::Rcv, lease.client_id, t, {}}); }
    Message rls() { return call({Opcode::Rls, lease.client_id, 0, {}}); }
};

ErrCode code(const Message& m) {
    if (m.opcode != Opcode::Nack) throw std::runtime_error("expected NACK");
    return parse_nack(m.payload)->code;
}

float f32(const std::uint8_t* p, int i) {
    float v;
    std::memcpy(&v, p + 4 * i, 4);
    return v;
}

}  // namespace

TEST_CASE("gvm: REQ leases distinct slots, Full when exhausted") {
    LoopbackHub hub;
    auto d = start(hub, cfg(2, 2));
    Raw a(hub), b(hub), c(hub);
    CHECK(a.req().opcode == Opcode::Ack);
    CHECK(a.lease.client_id == 1);
    CHECK(a.lease.shm_bytes == (1 << 16));
    CHECK(a.lease.stream_hint == 0);
    CHECK(a.lease.shm_name == IpcNames::region(hub.instance(), 1));
    b.req();
    CHECK(b.lease.client_id == 2);
    CHECK(code(c.req()) == ErrCode::Full);
}

TEST_CASE("gvm: phase violations, NoLease after RLS, Size on SND") {
    LoopbackHub hub;
    auto d = start(hub, cfg(1, 1));
    Raw a(hub);
    a.req();
    CHECK(code(a.stp(1)) == ErrCode::Phase);
    CHECK(code(a.rcv(1)) == ErrCode::Phase);
    a.str(1, kCIdesc);
    CHECK(code(a.await()) == ErrCode::Phase);
    CHECK(code(a.snd_claim(1 << 20)) == ErrCode::Size);
    a.snd(pair(1, 2, 3, 4));
    CHECK(a.rls().opcode == Opcode::Ack);
    CHECK(code(a.snd_claim(4)) == ErrCode::NoLease);
}

TEST_CASE("gvm: STR validates descriptor, payload id, sizes, grid") {
    LoopbackHub hub;
    auto d = start(hub, cfg(1, 1));
    Raw a(hub);
    a.req();
    a.snd(pair(1, 2, 3, 4));
    a.ch->send({Opcode::Str, a.lease.client_id, 9, {1, 2, 3}});
    CHECK(code(a.await()) == ErrCode::Malformed);
    a.str(9, descr(20, 50, 20, "no-such-payload"));
    CHECK(code(a.await()) == ErrCode::Payload);
    auto big = kCIdesc;
    big.output_bytes = 1 << 30;
    a.str(9, big);
    CHECK(code(a.await()) == ErrCode::Size);
    auto zero = kCIdesc;
    zero.grid_size = 0;
    a.str(9, zero);
    CHECK(code(a.await()) == ErrCode::Malformed);
    auto huge = kCIdesc;
    huge.t_comp = 2'000'000'000'000ull;
    a.str(9, huge);
    CHECK(code(a.await()) == ErrCode::Malformed);
}

TEST_CASE("gvm: two-client flow, barrier, exact sums and ACK sequence") {
    LoopbackHub hub;
    auto d = start(hub, cfg(2, 2));
    Raw a(hub), b(hub);
    CHECK(a.req().opcode == Opcode::Ack);
    CHECK(b.req().opcode == Opcode::Ack);
    CHECK(a.snd(pair(1, 2, 3, 4)).opcode == Opcode::Ack);
    CHECK(b.snd(pair(10, 20, 30, 40)).opcode == Opcode::Ack);
    a.str(1, kCIdesc);
    CHECK_FALSE(a.ch->recv(50ms).has_value());  // held at the barrier
    b.str(1, kCIdesc);
    CHECK(a.await().opcode == Opcode::Ack);
    CHECK(b.await().opcode == Opcode::Ack);
    CHECK(a.stp(1).opcode == Opcode::Ack);
    CHECK(b.stp(1).opcode == Opcode::Ack);
    const Message ra = a.rcv(1);
    CHECK(parse_u64(ra.payload) == 8);
    CHECK(f32(a.ch->region().data(), 0) == 4.f);
    CHECK(f32(a.ch->region().data(), 1) == 6.f);
    const Message rb = b.rcv(1);
    CHECK(parse_u64(rb.payload) == 8);
    CHECK(f32(b.ch->region().data(), 0) == 40.f);
    CHECK(f32(b.ch->region().data(), 1) == 60.f);
    CHECK(a.rls().opcode == Opcode::Ack);
    CHECK(b.rls().opcode == Opcode::Ack);
    const std::vector<Opcode> six(6, Opcode::Ack);
    CHECK(a.seen == six);
    CHECK(b.seen == six);
    const auto m = d->metrics();
    CHECK(m.batches_flushed == 1);
    CHECK(m.tasks.size() == 2);
}

TEST_CASE("gvm: batch style and model makespan 210 / 300 / 90") {
    struct Case {
        KernelDescriptor d;
        std::uint32_t n;
        ProgrammingStyle style;
        Micros span;
    };
    for (const Case& c : {Case{kCIdesc, 4, ProgrammingStyle::PS1, 210},
                          Case{kIOIdesc, 4, ProgrammingStyle::PS2, 300},
                          Case{kCIdesc, 1, ProgrammingStyle::PS1, 90}}) {
        LoopbackHub hub;
        auto d = start(hub, cfg(c.n, c.n));
        std::vector<std::unique_ptr<Raw>> cl;
        for (std::uint32_t i = 0; i < c.n; ++i) {
            cl.push_back(std::make_unique<Raw>(hub));
            cl.back()->req();
            cl.back()->snd(pair(1, 2, 3, 4));
        }
        for (auto& r : cl) r->str(1, c.d);
        for (auto& r : cl) r->await();
        const auto m = d->metrics();
        REQUIRE(m.batches.size() == 1);
        CHECK(m.batches[0].style == c.style);
        CHECK(m.batches[0].model_makespan_us == c.span);
        CHECK(m.batches[0].measured_makespan_us == c.span);
    }
}

TEST_CASE("gvm: mixed batch — majority class, ties go to PS1") {
    LoopbackHub hub;
    auto d = start(hub, cfg(3, 3));
    std::vector<std::unique_ptr<Raw>> cl;
    for (int i = 0; i < 3; ++i) {
        cl.push_back(std::make_unique<Raw>(hub));
        cl.back()->req();
        cl.back()->snd(pair(1, 2, 3, 4));
    }
    cl[0]->str(1, kIOIdesc);
    cl[1]->str(1, kIOIdesc);
    cl[2]->str(1, kCIdesc);
    for (auto& r : cl) r->await();
    CHECK(d->metrics().batches.at(0).style == ProgrammingStyle::PS2);

    LoopbackHub hub2;
    auto d2 = start(hub2, cfg(2, 2));
    Raw x(hub2), y(hub2);
    x.req();
    y.req();
    x.snd(pair(1, 2, 3, 4));
    y.snd(pair(1, 2, 3, 4));
    x.str(1, kIOIdesc);
    y.str(1, kCIdesc);
    x.await();
    y.await();
    CHECK(d2->metrics().batches.at(0).style == ProgrammingStyle::PS1);
}

TEST_CASE("gvm: partial batch flushes after the window") {
    LoopbackHub hub;
    auto d = start(hub, cfg(4, 4, 5000));
    Raw a(hub);
    a.req();
    a.snd(pair(1, 2, 3, 4));
    a.str(1, kCIdesc);
    CHECK(a.await(2s).opcode == Opcode::Ack);
    CHECK(a.stp(1).opcode == Opcode::Ack);
}

TEST_CASE("gvm: one t_init charge, no context switches") {
    LoopbackHub hub;
    auto d = start(hub, cfg(3, 1));
    std::vector<std::unique_ptr<Raw>> cl;
    for (int i = 0; i < 3; ++i) {
        cl.push_back(std::make_unique<Raw>(hub));
        cl.back()->req();
        cl.back()->snd(pair(1, 2, 3, 4));
        cl.back()->str(1, kCIdesc);
        cl.back()->await();
    }
    const auto m = d->metrics();
    CHECK(m.t_init_us == 100);
    CHECK(m.busy_us == 270);
    CHECK(m.uptime_us == 370);
    CHECK(m.batches_flushed == 3);
    for (const auto& t : m.tasks) {
        CHECK(t.pure_gpu_us <= t.end_to_end_us);
    }
}

TEST_CASE("gvm: payload failures surface through STP, RCV stays illegal") {
    LoopbackHub hub;
    auto d = start(hub, cfg(1, 1));
    Raw a(hub);
    a.req();
    a.snd(Bytes{1, 2, 3});
    a.str(1, kCIdesc);
    a.await();
    CHECK(code(a.stp(1)) == ErrCode::Payload);
    CHECK(code(a.rcv(1)) == ErrCode::Phase);
    CHECK(a.rls().opcode == Opcode::Ack);
    // output larger than the region
    Raw b(hub);
    b.req();
    b.snd(pair(1, 2, 3, 4));
    b.str(1, descr(20, 50, 20, "huge"));
    b.await();
    CHECK(code(b.stp(1)) == ErrCode::Size);
}

TEST_CASE("gvm: config validation and double start") {
    LoopbackHub hub;
    CHECK_THROWS_AS((void)GvmDaemon::start_loopback(cfg(2, 3), hub), std::invalid_argument);
    auto bad = cfg(2, 2);
    bad.scale = 0.0;
    CHECK_THROWS_AS((void)GvmDaemon::start_loopback(bad, hub), std::invalid_argument);
    auto bad2 = cfg(0, 0);
    CHECK_THROWS_AS((void)GvmDaemon::start_loopback(bad2, hub), std::invalid_argument);
    auto d = start(hub, cfg(1, 1));
    CHECK_THROWS_AS((void)start(hub, cfg(1, 1)), TransportError);
}

TEST_CASE("gvm: snapshot data plane keeps reference SND timing") {
    for (DataPlane plane : {DataPlane::ZeroCopy, DataPlane::Snapshot}) {
        LoopbackHub hub;
        auto g = cfg(1, 1);
        g.data_plane = plane;
        auto d = start(hub, g);
        Raw a(hub);
        a.req();
        a.snd(pair(1, 2, 3, 4));
        // a raw client rewriting its region after SND ACK (the SDK never does)
        const Bytes late = pair(100, 200, 300, 400);
        std::memcpy(a.ch->region().data(), late.data(), late.size());
        a.str(1, kCIdesc);
        a.await();
        a.stp(1);
        a.rcv(1);
        const float got = f32(a.ch->region().data(), 0);
        if (plane == DataPlane::Snapshot) CHECK(got == 4.f);   // bytes at SND
        else CHECK(got == 400.f);                               // bytes at dispatch
    }
}

TEST_CASE("client: run_task, reuse, release") {
    LoopbackHub hub;
    auto d = start(hub, cfg(1, 1));
    VgpuHandle h = req(hub);
    CHECK(h.client_id() == 1);
    CHECK(h.phase() == Phase::Leased);
    Bytes out = h.run_task(pair(1, 2, 3, 4), kCIdesc);
    CHECK(f32(out.data(), 0) == 4.f);
    CHECK(f32(out.data(), 1) == 6.f);
    out = h.run_task(pair(5, 6, 7, 8), kCIdesc);
    CHECK(f32(out.data(), 0) == 12.f);
    h.rls();
    CHECK(h.phase() == Phase::Released);
}

TEST_CASE("client: large SND/RCV through the streaming copy, odd sizes and offsets") {
    // >= 256 KiB payloads take the non-temporal AVX2 copy into the region
    // (client.cpp stream_copy): unaligned heads and 128-byte tails included
    LoopbackHub hub;
    GvmConfig g = cfg(1, 1);
    g.per_client_shm_bytes = 2 << 20;
    auto d = start(hub, g);
    VgpuHandle h = req(hub);
    std::mt19937 rng(7);
    for (std::size_t n : {std::size_t{256} << 10, (std::size_t{1} << 20) + 37, (std::size_t{2} << 20) - 5}) {
        Bytes in(n + 3);
        for (auto& b : in) b = static_cast<std::uint8_t>(rng());
        const std::span<const std::uint8_t> view(in.data() + 3, n);  // misaligned source
        const Bytes out = h.run_task(view, descr(1, 1, 1, "reverse"));
        REQUIRE(out.size() == n);
        CHECK(std::equal(out.rbegin(), out.rend(), view.begin()));
    }
    h.rls();
}

TEST_CASE("client: illegal orders fail locally; oversize SND; second SND wins") {
    LoopbackHub hub;
    auto d = start(hub, cfg(1, 1));
    VgpuHandle h = req(hub);
    CHECK_THROWS_AS((void)h.rcv(), VgpuError);
    CHECK_THROWS_AS((void)h.stp(), VgpuError);
    CHECK_THROWS_AS(h.str(kCIdesc), VgpuError);
    try {
        (void)h.rcv();
    } catch (const VgpuError& e) {
        CHECK(e.code() == ErrCode::Phase);
    }
    const Bytes big((1 << 16) + 1);
    try {
        h.snd(big);
        FAIL("oversize SND accepted");
    } catch (const VgpuError& e) {
        CHECK(e.code() == ErrCode::Size);
    }
    h.snd(pair(9, 9, 9, 9));
    h.snd(pair(1, 1, 2, 2));
    h.str(kCIdesc);
    h.stp_wait();
    const Bytes out = h.rcv();
    CHECK(f32(out.data(), 0) == 3.f);
    h.rls();
    CHECK_THROWS_AS(h.snd(Bytes{1}), VgpuError);
}

TEST_CASE("client: Full and NACK codes verbatim") {
    LoopbackHub hub;
    auto d = start(hub, cfg(1, 1));
    VgpuHandle h = req(hub);
    CHECK_THROWS_AS((void)req(hub), VgpuError);
    h.snd(Bytes{1, 2, 3});
    h.str(kCIdesc);
    try {
        h.stp_wait();
        FAIL("expected the payload failure");
    } catch (const VgpuError& e) {
        CHECK(e.code() == ErrCode::Payload);
    }
}

TEST_CASE("client: concurrent handles stay isolated (real clock, doorbell)") {
    LoopbackHub hub;
    auto g = cfg(4, 4, 2000);
    g.clock = ClockMode::Real;
    auto d = start(hub, g);
    std::vector<std::thread> ts;
    std::vector<std::string> err(4);
    for (int i = 0; i < 4; ++i)
        ts.emplace_back([&, i] {
            try {
                VgpuHandle h = req(hub);
                for (int rep = 0; rep < 20; ++rep) {
                    const float base = static_cast<float>(i + 1) + rep;
                    const Bytes out = h.run_task(pair(base, base * 2, 10, 20), kCIdesc);
                    if (f32(out.data(), 0) != base + 10 || f32(out.data(), 1) != base * 2 + 20)
                        err[i] = "wrong result";
                }
                h.rls();
            } catch (const std::exception& e) {
                err[i] = e.what();
            }
        });
    for (auto& t : ts) t.join();
    for (auto& e : err) CHECK(e.empty());
    const auto m = d->metrics();
    CHECK(m.tasks.size() == 80);
}

TEST_CASE("client: one worker body drives daemon and a user host payload natively") {
    LoopbackHub hub;
    auto d = start(hub, cfg(1, 1));
    VgpuHandle v = req(hub);
    const Bytes input = pair(2, 4, 1, 1);
    auto body = [&](auto& h) {
        h.snd(input);
        h.str(kCIdesc);
        h.stp_wait();
        return h.rcv();
    };
    const Bytes a = body(v);
    NativeVgpu n{NativeConfig{}, &host_registry()};
    const Bytes b = body(n);
    CHECK(a == b);
    CHECK_THROWS_AS((void)n.rcv(), VgpuError);
    n.rls();
    CHECK_THROWS_AS(n.snd(Bytes{1}), VgpuError);
}

TEST_CASE("gvm os: start creates endpoint, regions, doorbell; 8 processes x 100 reps") {
    GvmConfig g = cfg(8, 8, 20000);
    g.instance = "mtd" + std::to_string(getpid());
    g.per_client_shm_bytes = 4096;
    unlink_os_instance(g.instance, g.max_clients);
    // children first (single-threaded at fork); they retry until the daemon is up
    std::vector<pid_t> kids;
    for (std::uint32_t w = 0; w < 8; ++w) {
        const pid_t pid = fork();
        if (pid == 0) {
            for (int attempt = 0; attempt < 1000; ++attempt) {
                try {
                    VgpuHandle h = req(g.instance);
                    for (int rep = 0; rep < 100; ++rep) {
                        float in[128];
                        for (int j = 0; j < 64; ++j) {
                            in[j] = float(w * 1000 + j);
                            in[64 + j] = float(rep * 10 + j);
                        }
                        Bytes input(sizeof in);
                        std::memcpy(input.data(), in, sizeof in);
                        const Bytes out = h.run_task(input, kIOIdesc);
                        if (out.size() != 256) _exit(3);
                        for (int j = 0; j < 64; ++j)
                            if (f32(out.data(), j) != in[j] + in[64 + j]) _exit(4);
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
    auto d = GvmDaemon::start(g, open_os_daemon_transport(g.instance, 8, g.per_client_shm_bytes),
                              &host_registry());
    struct stat st {};
    CHECK(stat(IpcNames::endpoint(g.instance).c_str(), &st) == 0);
    for (std::uint32_t s = 1; s <= 8; ++s) {
        const int fd = shm_open(IpcNames::region(g.instance, s).c_str(), O_RDWR, 0600);
        CHECK(fd >= 0);
        if (fd >= 0) close(fd);
    }
    const int bell = shm_open(IpcNames::doorbell(g.instance).c_str(), O_RDWR, 0600);
    CHECK(bell >= 0);
    if (bell >= 0) close(bell);
    CHECK_THROWS_AS((void)open_os_daemon_transport(g.instance, 8, 4096), TransportError);
    for (pid_t k : kids) {
        int status = 0;
        waitpid(k, &status, 0);
        CHECK(WIFEXITED(status));
        CHECK(WEXITSTATUS(status) == 0);
    }
    CHECK(d->metrics().tasks.size() == 800);
    d->stop();
}

TEST_CASE("gvm: a dead client's lease is reclaimed by the next REQ") {
    LoopbackHub hub;
    auto d = start(hub, cfg(1, 1));
    {
        Raw a(hub);
        CHECK(a.req().opcode == Opcode::Ack);
        Raw b(hub);
        CHECK(code(b.req()) == ErrCode::Full);  // a is alive: no reclaim
    }  // both connections drop without RLS
    Raw c(hub);
    CHECK(c.req().opcode == Opcode::Ack);
    CHECK(c.lease.client_id == 1);
    c.snd(pair(1, 2, 3, 4));
    c.str(1, kCIdesc);
    CHECK(c.await().opcode == Opcode::Ack);
    CHECK(c.stp(1).opcode == Opcode::Ack);
}

TEST_CASE("gvm os: streamed SND — the ACK waits for the fill, odd sizes, copy threads") {
    // The SDK streams SNDs >= 4 MiB to a daemon that advertises it on its
    // doorbell page: frame first, then the (multi-threaded) copy publishes
    // the filled prefix. Host payloads: the daemon waits for the fill and
    // takes the plain SND path (the device path uploads the parts as they fill).
    GvmConfig g = cfg(2, 1, 1000);
    g.instance = "stream" + std::to_string(getpid());
    g.per_client_shm_bytes = 16 << 20;
    unlink_os_instance(g.instance, g.max_clients);
    auto d = GvmDaemon::start(g, open_os_daemon_transport(g.instance, 2, g.per_client_shm_bytes),
                              &host_registry());
    {
        VgpuHandle h = req(g.instance);
        std::mt19937 rng(11);
        for (std::size_t n : {std::size_t{4} << 20, (std::size_t{4} << 20) + 37,
                              (std::size_t{13} << 20) - 5, std::size_t{3} << 20}) {
            Bytes in(n + 5);
            for (auto& b : in) b = static_cast<std::uint8_t>(rng());
            const std::span<const std::uint8_t> view(in.data() + 5, n);  // misaligned source
            const Bytes out = h.run_task(view, descr(1, 1, 1, "reverse"));
            REQUIRE(out.size() == n);
            CHECK(std::equal(out.rbegin(), out.rend(), view.begin()));
        }
        // second SND wins, also when both are streamed
        Bytes a(5 << 20, 1), b(6 << 20, 2);
        h.snd(a);
        h.snd(b);
        h.str(descr(1, 1, 1, "reverse"));
        h.stp_wait();
        const Bytes out = h.rcv();
        CHECK(out.size() == b.size());
        CHECK(out.front() == 2);
        h.rls();
    }
    {
        // raw protocol: SND flagged streamed before the region is filled
        auto ch = open_os_client_channel(g.instance);
        ch->send({Opcode::Req, 0, 0, {}});
        auto lease_msg = ch->recv(2s);
        REQUIRE(lease_msg.has_value());
        const LeaseInfo lease = *parse_lease(lease_msg->payload);
        ch->attach_lease(lease);
        std::uint64_t* fill = ch->stream_fill();
        REQUIRE(fill != nullptr);
        CHECK(ch->leased_clients() == 1);
        const std::size_t n = 8 << 20;
        __atomic_store_n(fill, 0, __ATOMIC_RELEASE);
        std::memset(ch->region().data(), 7, n / 2);
        __atomic_store_n(fill, n / 2, __ATOMIC_RELEASE);
        ch->send({Opcode::Snd, lease.client_id, 0, encode_snd(n, kSndStreamed)});
        CHECK(!ch->recv(50ms).has_value());  // half filled: no answer yet
        // a frame sent meanwhile is answered after the SND, in order
        ch->send({Opcode::Str, lease.client_id, 1, encode_descriptor(descr(1, 1, 1, "reverse"))});
        CHECK(!ch->recv(20ms).has_value());
        std::memset(ch->region().data() + n / 2, 9, n / 2);
        __atomic_store_n(fill, n, __ATOMIC_RELEASE);
        auto ack = ch->recv(2s);
        REQUIRE(ack.has_value());
        CHECK(ack->opcode == Opcode::Ack);
        CHECK(ack->task_id == 0);
        auto str_ack = ch->recv(2s);
        REQUIRE(str_ack.has_value());
        CHECK(str_ack->opcode == Opcode::Ack);
        CHECK(str_ack->task_id == 1);
        for (int i = 0; i < 200; ++i) {
            ch->send({Opcode::Stp, lease.client_id, 1, {}});
            auto r = ch->recv(2s);
            REQUIRE(r.has_value());
            if (r->opcode == Opcode::Ack) break;
            std::this_thread::sleep_for(1ms);
        }
        ch->send({Opcode::Rcv, lease.client_id, 1, {}});
        auto rcv = ch->recv(2s);
        REQUIRE(rcv.has_value());
        CHECK(parse_u64(rcv->payload).value_or(0) == n);
        CHECK(ch->region().data()[0] == 9);      // reversed: the second half first
        CHECK(ch->region().data()[n - 1] == 7);
        ch->send({Opcode::Rls, lease.client_id, 0, {}});
        CHECK(ch->recv(2s).has_value());
    }
    d->stop();
}

TEST_CASE("multi-GPU: NCCL id rendezvous through a file, across processes") {
    namespace mg = vgpu::multigpu;
    const std::string path = "/tmp/vgpu-test-rdv." + std::to_string(getpid());
    unlink(path.c_str());
    std::vector<std::uint8_t> id(128);
    for (std::size_t i = 0; i < id.size(); ++i) id[i] = static_cast<std::uint8_t>(i * 37 + 5);
    // ranks 1..3 start first and wait for the file
    std::vector<pid_t> kids;
    for (int r = 1; r < 4; ++r) {
        const pid_t pid = fork();
        if (pid == 0) {
            try {
                const auto got = mg::fetch_id(path, id.size(), std::chrono::seconds(10));
                _exit(got == id ? 0 : 3);
            } catch (...) {
                _exit(4);
            }
        }
        kids.push_back(pid);
    }
    std::this_thread::sleep_for(30ms);
    mg::publish_id(path, id);
    for (pid_t k : kids) {
        int st = 0;
        waitpid(k, &st, 0);
        CHECK(WIFEXITED(st));
        CHECK(WEXITSTATUS(st) == 0);
    }
    // a short or foreign file is never taken for an id
    CHECK_THROWS_AS((void)mg::fetch_id(path, 64, std::chrono::milliseconds(20)), std::runtime_error);
    unlink(path.c_str());
    CHECK_THROWS_AS((void)mg::fetch_id(path, 128, std::chrono::milliseconds(20)), std::runtime_error);
}

TEST_CASE("multi-GPU: records fold in rank order; placement helpers") {
    namespace mg = vgpu::multigpu;
    std::vector<double> all(3 * mg::kRecordWidth, 0.0);
    const double sx[3] = {0.1, 1e16, -1e16};  // order-sensitive in binary64
    for (int r = 0; r < 3; ++r) {
        double* rec = all.data() + r * mg::kRecordWidth;
        rec[0] = 16;
        rec[1] = 1000 + r;
        rec[11] = sx[r];
        rec[14] = 4096;
        rec[15] = 1000000;
    }
    const auto f = mg::fold_in_rank_order(all, 3);
    CHECK(f[0] == 48);
    CHECK(f[1] == 3003);
    CHECK(f[11] == ((0.0 + 0.1) + 1e16) + -1e16);  // left to right, not 0.1
    CHECK(f[14] == 3 * 4096);
    CHECK(f[15] == std::fmod(3000000.0, 1000003.0));
    all[mg::kRecordWidth + 14] = -1.0;  // rank 1 saw a slice change bits
    CHECK(mg::fold_in_rank_order(all, 3)[14] == -1.0);
    CHECK_THROWS_AS((void)mg::fold_in_rank_order(std::span<const double>(all).first(20), 3),
                    std::invalid_argument);
    CHECK(mg::parse_cpulist("0-3,8,10-11\n") == std::vector<int>({0, 1, 2, 3, 8, 10, 11}));
    CHECK(mg::parse_cpulist("5, 2-3,x,3").size() == 3);
    CHECK(mg::local_cpus("0000:ff:1f.7").empty());  // no such device: no placement
}

TEST_CASE("gvm os: the doorbell page publishes the lease count") {
    GvmConfig g = cfg(3, 1, 1000);
    g.instance = "leases" + std::to_string(getpid());
    g.per_client_shm_bytes = 4096;
    unlink_os_instance(g.instance, g.max_clients);
    auto d = GvmDaemon::start(g, open_os_daemon_transport(g.instance, 3, g.per_client_shm_bytes),
                              &host_registry());
    {
        VgpuHandle a = req(g.instance);
        VgpuHandle b = req(g.instance);
        auto ch = open_os_client_channel(g.instance);
        ch->send({Opcode::Req, 0, 0, {}});
        auto r = ch->recv(2s);
        REQUIRE(r.has_value());
        ch->attach_lease(*parse_lease(r->payload));
        CHECK(ch->leased_clients() == 3);
        b.rls();
        ch->send({Opcode::Stp, parse_lease(r->payload)->client_id, 0, {}});  // any round trip
        (void)ch->recv(2s);
        CHECK(ch->leased_clients() == 2);
    }
    d->stop();
}
