// Wire codec and transports. Cases mirror the reference's
// proj/tests/test_message.cpp:26-116 and test_transport.cpp:11-148
// (same expectations, independent code), plus the B200 doorbell.
#include <unistd.h>

#include <random>
#include <thread>

#include "minitest.hpp"
#include "vgpu/message.hpp"
#include "vgpu/payload.hpp"
#include "vgpu/transport.hpp"

using namespace vgpu;
using namespace std::chrono_literals;

namespace {

Message random_frame(std::mt19937_64& g) {
    static const Opcode all[] = {Opcode::Req, Opcode::Snd, Opcode::Str, Opcode::Stp,
                                 Opcode::Rcv, Opcode::Rls, Opcode::Ack, Opcode::Nack};
    Message m;
    m.opcode = all[g() % 8];
    m.client_id = static_cast<std::uint32_t>(g());
    m.task_id = g();
    m.payload.resize(g() % 300);
    for (auto& b : m.payload) b = static_cast<std::uint8_t>(g());
    return m;
}

}  // namespace

TEST_CASE("codec: 26-byte little-endian header, bit-exact") {
    const auto f = encode({Opcode::Req, 7, 0, {}});
    REQUIRE(f.size() == 26);
    const std::uint8_t head[] = {0x56, 0x47, 0x50, 0x55, 0x01, 0x01, 7, 0, 0, 0};
    for (int i = 0; i < 10; ++i) CHECK(f[i] == head[i]);
    for (int i = 10; i < 26; ++i) CHECK(f[i] == 0);

    const auto g = encode({Opcode::Str, 0x01020304u, 0x1122334455667788ull, {0xAB}});
    CHECK(g.size() == 27);
    CHECK(g[5] == 0x03);
    CHECK(g[6] == 0x04);
    CHECK(g[9] == 0x01);
    CHECK(g[10] == 0x88);
    CHECK(g[17] == 0x11);
    CHECK(g[18] == 1);
    for (int i = 19; i < 26; ++i) CHECK(g[i] == 0);
    CHECK(g[26] == 0xAB);
}

TEST_CASE("codec: 100k random frames round-trip (acceptance criterion 8)") {
    std::mt19937_64 g(8);
    int bad = 0;
    for (int i = 0; i < 100000; ++i) {
        const Message m = random_frame(g);
        const auto r = decode(encode(m));
        if (!std::holds_alternative<Message>(r) || std::get<Message>(r) != m) ++bad;
    }
    CHECK(bad == 0);
}

TEST_CASE("codec: corrupt frames are classified, never crash") {
    const auto good = encode({Opcode::Req, 1, 2, {9, 9}});
    auto mutate = [&](auto fn) {
        auto f = good;
        fn(f);
        return decode(f);
    };
    auto err = [](const DecodeResult& r) { return std::get<DecodeError>(r); };
    CHECK(err(mutate([](auto& f) { f[0] = 'X'; })) == DecodeError::BadMagic);
    CHECK(err(mutate([](auto& f) { f[4] = 9; })) == DecodeError::BadVersion);
    CHECK(err(mutate([](auto& f) { f[5] = 0x7F; })) == DecodeError::BadOpcode);
    CHECK(err(mutate([](auto& f) { f[5] = 0x00; })) == DecodeError::BadOpcode);
    CHECK(err(mutate([](auto& f) { f.resize(10); })) == DecodeError::Truncated);
    CHECK(err(mutate([](auto& f) { f.resize(27); })) == DecodeError::Truncated);
    CHECK(err(mutate([](auto& f) { f.push_back(0); })) == DecodeError::Truncated);
    CHECK(err(decode({})) == DecodeError::Truncated);
    CHECK(std::string(to_string(DecodeError::BadMagic)) == "bad magic");
}

TEST_CASE("codec: structured payloads round-trip and reject truncation") {
    const LeaseInfo lease{3, 1 << 20, 2, "/vgpu.test.3", "/vgpu.test.rsp.3"};
    CHECK(parse_lease(encode_lease(lease)) == lease);
    const KernelDescriptor d{"vector-add", 100, 200, 300, 16, 4096};
    CHECK(parse_descriptor(encode_descriptor(d)) == d);
    CHECK(parse_u64(encode_u64(0xDEADBEEFull)) == 0xDEADBEEFull);
    const auto nack = parse_nack(encode_nack(ErrCode::Size, "too big"));
    REQUIRE(nack.has_value());
    CHECK(nack->code == ErrCode::Size);
    CHECK(nack->detail == "too big");
    auto cut = encode_descriptor(d);
    for (std::size_t n = 0; n < cut.size(); ++n) {
        std::vector<std::uint8_t> part(cut.begin(), cut.begin() + n);
        CHECK_FALSE(parse_descriptor(part).has_value());
    }
    auto extra = cut;
    extra.push_back(0);
    CHECK_FALSE(parse_descriptor(extra).has_value());
    CHECK_FALSE(parse_lease(Bytes{1, 2, 3}).has_value());
    CHECK_FALSE(parse_u64(Bytes{1, 2, 3}).has_value());
    // descriptor byte layout: u32 len + id + 3 x u64 + u32 + u64
    CHECK(encode_descriptor(d).size() == 4 + 10 + 24 + 4 + 8);
}

TEST_CASE("ipc names match the reference") {
    CHECK(IpcNames::endpoint("gpu0") == "/tmp/vgpu.gpu0.sock");
    CHECK(IpcNames::region("gpu0", 3) == "/vgpu.gpu0.3");
    CHECK(IpcNames::doorbell("gpu0") == "/vgpu.gpu0.bell");
}

TEST_CASE("loopback: identical frames in FIFO order") {
    LoopbackHub hub;
    auto daemon = hub.bind_daemon(2, 4096);
    auto client = hub.connect();
    const Message m{Opcode::Req, 0, 42, {1, 2, 3}};
    client->send(m);
    auto got = daemon->recv(100ms);
    REQUIRE(got.has_value());
    CHECK(got->msg == m);
    for (std::uint64_t i = 0; i < 20; ++i) client->send({Opcode::Stp, 1, i, {}});
    for (std::uint64_t i = 0; i < 20; ++i) {
        auto n = daemon->recv(100ms);
        REQUIRE(n.has_value());
        CHECK(n->msg.task_id == i);
    }
    CHECK_FALSE(daemon->recv(1ms).has_value());
}

TEST_CASE("loopback: responses are routed per connection") {
    LoopbackHub hub;
    auto daemon = hub.bind_daemon(2, 4096);
    auto a = hub.connect();
    auto b = hub.connect();
    a->send({Opcode::Req, 0, 7, {}});
    b->send({Opcode::Req, 0, 8, {}});
    auto fa = daemon->recv(100ms);
    auto fb = daemon->recv(100ms);
    REQUIRE(fa.has_value());
    REQUIRE(fb.has_value());
    CHECK(fa->origin != fb->origin);
    daemon->reply_origin(fa->origin, {Opcode::Ack, 1, 7, {}});
    daemon->reply_origin(fb->origin, {Opcode::Ack, 2, 8, {}});
    CHECK(a->recv(100ms)->task_id == 7);
    CHECK(b->recv(100ms)->task_id == 8);
    daemon->bind(1, fa->origin);
    daemon->bind(2, fb->origin);
    for (std::uint64_t i = 0; i < 10; ++i) {
        daemon->send(1, {Opcode::Ack, 1, i, {}});
        daemon->send(2, {Opcode::Ack, 2, 100 + i, {}});
    }
    for (std::uint64_t i = 0; i < 10; ++i) {
        CHECK(a->recv(100ms)->task_id == i);
        CHECK(b->recv(100ms)->task_id == 100 + i);
    }
}

TEST_CASE("loopback: regions exist before any client and are shared") {
    LoopbackHub hub;
    auto daemon = hub.bind_daemon(3, 512);
    for (std::uint32_t c = 1; c <= 3; ++c) {
        CHECK(daemon->region(c).size() == 512);
        CHECK(daemon->region_name(c) == IpcNames::region(hub.instance(), c));
        // page aligned so the GVM can page-lock each slot separately
        CHECK((reinterpret_cast<std::uintptr_t>(daemon->region(c).data()) & 4095) == 0);
    }
    auto client = hub.connect();
    LeaseInfo lease;
    lease.client_id = 2;
    lease.shm_bytes = 512;
    lease.shm_name = daemon->region_name(2);
    client->attach_lease(lease);
    client->region().data()[0] = 0xEE;
    CHECK(daemon->region(2).data()[0] == 0xEE);
}

TEST_CASE("loopback: second daemon rejected; sender blocks at depth 64 then drains") {
    LoopbackHub hub;
    auto daemon = hub.bind_daemon(1, 64);
    CHECK_THROWS_AS((void)hub.bind_daemon(1, 64), TransportError);
    auto client = hub.connect();
    const std::uint64_t total = ProtocolLimits::kQueueDepth + 16;
    std::thread producer([&] {
        for (std::uint64_t i = 0; i < total; ++i) client->send({Opcode::Stp, 1, i, {}});
    });
    std::uint64_t seen = 0;
    while (seen < total)
        if (daemon->recv(200ms)) ++seen;
    producer.join();
    CHECK(seen == total);
}

TEST_CASE("loopback: wake() cuts a blocking recv short; doorbell counts") {
    LoopbackHub hub;
    auto daemon = hub.bind_daemon(1, 64);
    auto client = hub.connect();
    LeaseInfo lease;
    lease.client_id = 1;
    lease.shm_bytes = 64;
    lease.shm_name = daemon->region_name(1);
    client->attach_lease(lease);
    const auto t0 = std::chrono::steady_clock::now();
    std::thread waker([&] {
        std::this_thread::sleep_for(20ms);
        daemon->wake();
    });
    CHECK_FALSE(daemon->recv(5s).has_value());
    waker.join();
    CHECK(std::chrono::steady_clock::now() - t0 < 2s);

    const auto seq = client->notify_seq();
    REQUIRE(seq.has_value());
    std::thread ringer([&] {
        std::this_thread::sleep_for(20ms);
        daemon->notify(1);
    });
    client->wait_notify(*seq, 5s);
    ringer.join();
    CHECK(client->notify_seq().value() == *seq + 1);
}

TEST_CASE("os transport: connect without a daemon fails") {
    CHECK_THROWS_AS((void)open_os_client_channel("no-such-instance-xyz"), TransportError);
}

TEST_CASE("os transport: end to end, regions, doorbell, double start") {
    const std::string inst = "mt" + std::to_string(getpid());
    unlink_os_instance(inst, 2);
    auto daemon = open_os_daemon_transport(inst, 2, 4096);
    CHECK_THROWS_AS((void)open_os_daemon_transport(inst, 2, 4096), TransportError);
    auto client = open_os_client_channel(inst);
    const Message request{Opcode::Req, 0, 5, {'x'}};
    client->send(request);
    auto got = daemon->recv(2s);
    REQUIRE(got.has_value());
    CHECK(got->msg == request);
    daemon->reply_origin(got->origin, {Opcode::Ack, 1, 5, {}});
    auto reply = client->recv(2s);
    REQUIRE(reply.has_value());
    CHECK(reply->opcode == Opcode::Ack);

    LeaseInfo lease;
    lease.client_id = 1;
    lease.shm_bytes = 4096;
    lease.shm_name = daemon->region_name(1);
    client->attach_lease(lease);
    client->region().data()[100] = 0x5A;
    CHECK(daemon->region(1).data()[100] == 0x5A);

    daemon->bind(1, got->origin);
    daemon->send(1, {Opcode::Ack, 1, 6, {}});
    auto routed = client->recv(2s);
    REQUIRE(routed.has_value());
    CHECK(routed->task_id == 6);

    // doorbell across the process boundary (same mechanism, one process here)
    const auto seq = client->notify_seq();
    REQUIRE(seq.has_value());
    std::thread ringer([&] {
        std::this_thread::sleep_for(20ms);
        daemon->notify(1);
    });
    client->wait_notify(*seq, 5s);
    ringer.join();
    CHECK(client->notify_seq().value() == *seq + 1);

    // wake
    std::thread waker([&] {
        std::this_thread::sleep_for(20ms);
        daemon->wake();
    });
    const auto t0 = std::chrono::steady_clock::now();
    CHECK_FALSE(daemon->recv(5s).has_value());
    waker.join();
    CHECK(std::chrono::steady_clock::now() - t0 < 2s);
}
