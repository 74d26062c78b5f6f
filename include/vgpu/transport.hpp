// vgpu-b200 — control plane (framed message queues) and data plane (one
// fixed-size byte region per client slot).
//
// Source-compatible with proj/include/vgpu/transport.hpp:22-176: same
// classes, same virtual methods, same IPC names, same factory functions.
// Two loopback/OS realizations are provided:
//   * LoopbackHub — in-process FIFOs, frames still cross encoded (tests);
//   * OS          — one SOCK_SEQPACKET endpoint /tmp/vgpu.<inst>.sock and
//                   POSIX shm regions /vgpu.<inst>.<slot>, created up front.
//
// B200 additions (all virtual with defaults, so reference-style transports
// still compile): a daemon-side wake() so the CUDA completion path can cut
// a blocking recv short, and a per-slot completion doorbell that lets
// VgpuHandle::stp_wait() sleep on a futex instead of polling STP on a
// 100 us -> 10 ms backoff (reference client.cpp:108-114). The wire protocol
// is unchanged; a client without a doorbell falls back to the backoff.
// The doorbell page also carries the streamed-SND fill counters: a client
// that sees the capability copies its input into the region chunk by chunk
// while the GVM already DMAs the filled part (SND frame sent first, flagged).
#ifndef VGPU_TRANSPORT_HPP
#define VGPU_TRANSPORT_HPP

#include <chrono>
#include <cstdint>
#include <memory>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "vgpu/message.hpp"

namespace vgpu {

struct TransportError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

struct IpcNames {
    // "/tmp/vgpu.<instance>.sock"
    static std::string endpoint(std::string_view instance);
    // "/vgpu.<instance>.<client_id>"
    static std::string region(std::string_view instance,
                              std::uint32_t client_id);
    // B200: "/vgpu.<instance>.bell" — per-slot completion counters.
    static std::string doorbell(std::string_view instance);
};

struct ProtocolLimits {
    static constexpr std::size_t kQueueDepth = 64;
    static constexpr std::size_t kMaxControlFrame = 8192;
};

class DataRegion {
public:
    virtual ~DataRegion() = default;
    virtual std::uint8_t* data() = 0;
    virtual std::size_t size() const = 0;

    std::span<std::uint8_t> bytes() { return {data(), size()}; }
    std::span<const std::uint8_t> bytes() const {
        return {const_cast<DataRegion*>(this)->data(), size()};
    }
};

class ClientChannel {
public:
    virtual ~ClientChannel() = default;
    virtual void send(const Message& m) = 0;
    virtual std::optional<Message> recv(std::chrono::microseconds timeout) = 0;
    virtual void attach_lease(const LeaseInfo& lease) = 0;
    virtual DataRegion& region() = 0;

    // B200 doorbell: current completion count of the attached lease, or
    // nullopt when the daemon offers none.
    virtual std::optional<std::uint64_t> notify_seq() { return std::nullopt; }
    // Block until the count moves past `seen` or the timeout passes.
    virtual void wait_notify(std::uint64_t /*seen*/,
                             std::chrono::microseconds /*timeout*/) {}
    // B200 streamed SND: the attached slot's fill counter in shared memory
    // (bytes of the current SND already in the region), or nullptr when the
    // daemon does not take streamed SNDs.
    virtual std::uint64_t* stream_fill() { return nullptr; }
    // B200: leases the daemon holds right now (sizes the SDK's copy
    // threads), 0 when unknown.
    virtual std::uint32_t leased_clients() { return 0; }
};

struct Inbound {
    Message msg;
    std::string origin;
};

class DaemonTransport {
public:
    virtual ~DaemonTransport() = default;
    virtual std::optional<Inbound> recv(std::chrono::microseconds timeout) = 0;
    virtual void reply_origin(const std::string& origin, const Message& m) = 0;
    virtual void bind(std::uint32_t client_id, const std::string& origin) = 0;
    virtual void send(std::uint32_t client_id, const Message& m) = 0;
    virtual DataRegion& region(std::uint32_t client_id) = 0;
    virtual std::string region_name(std::uint32_t client_id) const = 0;
    virtual std::uint32_t max_clients() const = 0;

    // B200: make a blocked recv() return early (thread-safe).
    virtual void wake() {}
    // B200: bump the slot's completion doorbell (thread-safe).
    virtual void notify(std::uint32_t /*client_id*/) {}
    // B200: false once the peer bound to this slot has disconnected (client
    // death); the GVM then reclaims the slot instead of leaking the lease.
    virtual bool route_alive(std::uint32_t /*client_id*/) const { return true; }
    // B200 streamed SND: the slot's fill counter the client advances while
    // it copies (nullptr: this transport has none, clients never stream).
    virtual const std::uint64_t* stream_fill(std::uint32_t /*client_id*/) { return nullptr; }
    // B200: publish how many slots are leased (clients size copy threads).
    virtual void publish_leases(std::uint32_t /*leased*/) {}
};

// ---- in-process loopback --------------------------------------------------

class LoopbackHub {
public:
    explicit LoopbackHub(std::string instance = "loopback");
    ~LoopbackHub();
    LoopbackHub(const LoopbackHub&) = delete;
    LoopbackHub& operator=(const LoopbackHub&) = delete;

    std::unique_ptr<ClientChannel> connect();
    std::unique_ptr<DaemonTransport> bind_daemon(std::uint32_t max_clients,
                                                 std::uint64_t region_bytes);
    const std::string& instance() const;

    struct State;  // implementation detail (transport.cpp)

private:
    std::shared_ptr<State> state_;
};

// ---- OS transport -----------------------------------------------------------

std::unique_ptr<DaemonTransport> open_os_daemon_transport(
    const std::string& instance, std::uint32_t max_clients,
    std::uint64_t region_bytes);

std::unique_ptr<ClientChannel> open_os_client_channel(
    const std::string& instance);

void unlink_os_instance(const std::string& instance,
                        std::uint32_t max_clients);

}  // namespace vgpu

#endif  // VGPU_TRANSPORT_HPP
