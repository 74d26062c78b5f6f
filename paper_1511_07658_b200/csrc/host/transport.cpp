// IPC names and the in-process loopback transport.
//
// Behavioural contract from the reference (proj/src/transport.cpp:7-249):
// one FIFO request queue into the daemon with per-connection origins, one
// FIFO response queue per connection, queue depth 64 with blocking senders,
// regions created by bind_daemon before any client, a second daemon on the
// same hub rejected. Frames cross the queues encoded so the wire codec is
// exercised. Implementation here: a small bounded queue template plus
// page-aligned anonymous mappings for the regions (so the CUDA backend can
// page-lock them without sharing pages between slots).
#include <sys/mman.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <deque>
#include <map>
#include <mutex>

#include "vgpu/transport.hpp"

namespace vgpu {

std::string IpcNames::endpoint(std::string_view instance) {
    std::string s = "/tmp/vgpu.";
    s.append(instance);
    s.append(".sock");
    return s;
}

std::string IpcNames::region(std::string_view instance,
                             std::uint32_t client_id) {
    std::string s = "/vgpu.";
    s.append(instance);
    s.push_back('.');
    s.append(std::to_string(client_id));
    return s;
}

std::string IpcNames::doorbell(std::string_view instance) {
    std::string s = "/vgpu.";
    s.append(instance);
    s.append(".bell");
    return s;
}

namespace {

using Frame = std::vector<std::uint8_t>;

template <class T>
class Bounded {
public:
    explicit Bounded(std::size_t depth) : depth_(depth) {}

    void push(T v) {
        std::unique_lock lk(mu_);
        can_push_.wait(lk, [&] { return q_.size() < depth_ || closed_; });
        if (closed_) throw TransportError("loopback queue closed");
        q_.push_back(std::move(v));
        can_pop_.notify_one();
    }

    // Returns nullopt on timeout, on close, or when interrupt() was called.
    std::optional<T> pop(std::chrono::microseconds timeout) {
        std::unique_lock lk(mu_);
        can_pop_.wait_for(lk, timeout,
                          [&] { return !q_.empty() || closed_ || kicked_; });
        kicked_ = false;
        if (q_.empty()) return std::nullopt;
        T v = std::move(q_.front());
        q_.pop_front();
        can_push_.notify_one();
        return v;
    }

    void interrupt() {
        std::lock_guard lk(mu_);
        kicked_ = true;
        can_pop_.notify_all();
    }

    void close() {
        std::lock_guard lk(mu_);
        closed_ = true;
        can_pop_.notify_all();
        can_push_.notify_all();
    }

private:
    std::mutex mu_;
    std::condition_variable can_push_, can_pop_;
    std::deque<T> q_;
    std::size_t depth_;
    bool closed_ = false;
    bool kicked_ = false;
};

Message must_decode(std::span<const std::uint8_t> f) {
    auto r = decode(f);
    if (const auto* e = std::get_if<DecodeError>(&r))
        throw TransportError(std::string("loopback frame rejected: ") +
                             to_string(*e));
    return std::get<Message>(std::move(r));
}

// Page-aligned zeroed bytes shared by the daemon and client views.
struct Store {
    void* base = MAP_FAILED;
    std::size_t bytes = 0;
    explicit Store(std::size_t n) : bytes(n) {
        const std::size_t map_len = std::max<std::size_t>(n, 1);
        base = mmap(nullptr, map_len, PROT_READ | PROT_WRITE,
                    MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
        if (base == MAP_FAILED) throw TransportError("loopback region mmap failed");
    }
    ~Store() {
        if (base != MAP_FAILED) munmap(base, std::max<std::size_t>(bytes, 1));
    }
};

class StoreRegion final : public DataRegion {
public:
    explicit StoreRegion(std::shared_ptr<Store> s) : s_(std::move(s)) {}
    std::uint8_t* data() override { return static_cast<std::uint8_t*>(s_->base); }
    std::size_t size() const override { return s_->bytes; }

private:
    std::shared_ptr<Store> s_;
};

struct Bell {
    std::mutex mu;
    std::condition_variable cv;
    std::uint64_t seq = 0;
};

}  // namespace

struct LoopbackHub::State {
    explicit State(std::string inst) : instance(std::move(inst)) {}

    struct Conn {
        std::uint64_t id = 0;
        Bounded<Frame> to_client{ProtocolLimits::kQueueDepth};
    };
    struct Routed {
        std::uint64_t conn = 0;
        Frame frame;
    };

    std::string instance;
    std::mutex mu;
    bool daemon_bound = false;
    std::uint64_t next_conn = 1;
    std::map<std::uint64_t, std::shared_ptr<Conn>> conns;
    std::map<std::string, std::shared_ptr<Store>> regions;
    std::map<std::uint32_t, std::shared_ptr<Bell>> bells;
    Bounded<Routed> requests{ProtocolLimits::kQueueDepth};

    std::shared_ptr<Conn> conn(std::uint64_t id) {
        std::lock_guard lk(mu);
        auto it = conns.find(id);
        return it == conns.end() ? nullptr : it->second;
    }
    std::shared_ptr<Bell> bell(std::uint32_t slot) {
        std::lock_guard lk(mu);
        auto& b = bells[slot];
        if (!b) b = std::make_shared<Bell>();
        return b;
    }
};

namespace {

std::uint64_t conn_of(const std::string& origin) {
    constexpr std::string_view pfx = "conn:";
    if (origin.compare(0, pfx.size(), pfx) != 0)
        throw TransportError("malformed loopback origin: " + origin);
    return std::stoull(origin.substr(pfx.size()));
}

class LoopbackClient final : public ClientChannel {
public:
    LoopbackClient(std::shared_ptr<LoopbackHub::State> st,
                   std::shared_ptr<LoopbackHub::State::Conn> c)
        : st_(std::move(st)), conn_(std::move(c)) {}

    ~LoopbackClient() override {
        conn_->to_client.close();
        std::lock_guard lk(st_->mu);
        st_->conns.erase(conn_->id);
    }

    void send(const Message& m) override {
        st_->requests.push({conn_->id, encode(m)});
    }

    std::optional<Message> recv(std::chrono::microseconds timeout) override {
        auto f = conn_->to_client.pop(timeout);
        if (!f) return std::nullopt;
        return must_decode(*f);
    }

    void attach_lease(const LeaseInfo& lease) override {
        std::shared_ptr<Store> s;
        {
            std::lock_guard lk(st_->mu);
            auto it = st_->regions.find(lease.shm_name);
            if (it != st_->regions.end()) s = it->second;
        }
        if (!s) throw TransportError("leased region not found: " + lease.shm_name);
        region_ = std::make_unique<StoreRegion>(std::move(s));
        bell_ = st_->bell(lease.client_id);
    }

    DataRegion& region() override {
        if (!region_) throw TransportError("no lease attached");
        return *region_;
    }

    std::optional<std::uint64_t> notify_seq() override {
        if (!bell_) return std::nullopt;
        std::lock_guard lk(bell_->mu);
        return bell_->seq;
    }

    void wait_notify(std::uint64_t seen,
                     std::chrono::microseconds timeout) override {
        if (!bell_) return;
        std::unique_lock lk(bell_->mu);
        bell_->cv.wait_for(lk, timeout, [&] { return bell_->seq != seen; });
    }

private:
    std::shared_ptr<LoopbackHub::State> st_;
    std::shared_ptr<LoopbackHub::State::Conn> conn_;
    std::unique_ptr<StoreRegion> region_;
    std::shared_ptr<Bell> bell_;
};

class LoopbackDaemon final : public DaemonTransport {
public:
    LoopbackDaemon(std::shared_ptr<LoopbackHub::State> st, std::uint32_t n,
                   std::uint64_t bytes)
        : st_(std::move(st)) {
        for (std::uint32_t slot = 1; slot <= n; ++slot) {
            auto name = IpcNames::region(st_->instance, slot);
            auto store = std::make_shared<Store>(bytes);
            {
                std::lock_guard lk(st_->mu);
                st_->regions[name] = store;
            }
            regions_.push_back(std::make_unique<StoreRegion>(store));
            names_.push_back(std::move(name));
            bells_.push_back(st_->bell(slot));
        }
    }

    ~LoopbackDaemon() override {
        std::lock_guard lk(st_->mu);
        st_->daemon_bound = false;
    }

    std::optional<Inbound> recv(std::chrono::microseconds timeout) override {
        auto r = st_->requests.pop(timeout);
        if (!r) return std::nullopt;
        return Inbound{must_decode(r->frame), "conn:" + std::to_string(r->conn)};
    }

    void reply_origin(const std::string& origin, const Message& m) override {
        if (auto c = st_->conn(conn_of(origin))) c->to_client.push(encode(m));
    }

    void bind(std::uint32_t client_id, const std::string& origin) override {
        routes_[client_id] = conn_of(origin);
    }

    bool route_alive(std::uint32_t client_id) const override {
        auto it = routes_.find(client_id);
        return it != routes_.end() && st_->conn(it->second) != nullptr;
    }

    void send(std::uint32_t client_id, const Message& m) override {
        auto it = routes_.find(client_id);
        if (it == routes_.end()) return;
        if (auto c = st_->conn(it->second)) c->to_client.push(encode(m));
    }

    DataRegion& region(std::uint32_t client_id) override {
        return *regions_.at(client_id - 1);
    }
    std::string region_name(std::uint32_t client_id) const override {
        return names_.at(client_id - 1);
    }
    std::uint32_t max_clients() const override {
        return static_cast<std::uint32_t>(regions_.size());
    }

    void wake() override { st_->requests.interrupt(); }

    void notify(std::uint32_t client_id) override {
        if (client_id < 1 || client_id > bells_.size()) return;
        auto& b = bells_[client_id - 1];
        {
            std::lock_guard lk(b->mu);
            ++b->seq;
        }
        b->cv.notify_all();
    }

private:
    std::shared_ptr<LoopbackHub::State> st_;
    std::vector<std::unique_ptr<StoreRegion>> regions_;
    std::vector<std::string> names_;
    std::vector<std::shared_ptr<Bell>> bells_;
    std::map<std::uint32_t, std::uint64_t> routes_;
};

}  // namespace

LoopbackHub::LoopbackHub(std::string instance)
    : state_(std::make_shared<State>(std::move(instance))) {}

LoopbackHub::~LoopbackHub() = default;

const std::string& LoopbackHub::instance() const { return state_->instance; }

std::unique_ptr<ClientChannel> LoopbackHub::connect() {
    auto c = std::make_shared<State::Conn>();
    {
        std::lock_guard lk(state_->mu);
        c->id = state_->next_conn++;
        state_->conns[c->id] = c;
    }
    return std::make_unique<LoopbackClient>(state_, std::move(c));
}

std::unique_ptr<DaemonTransport> LoopbackHub::bind_daemon(
    std::uint32_t max_clients, std::uint64_t region_bytes) {
    {
        std::lock_guard lk(state_->mu);
        if (state_->daemon_bound)
            throw TransportError("loopback instance '" + state_->instance +
                                 "' already has a daemon");
        state_->daemon_bound = true;
    }
    return std::make_unique<LoopbackDaemon>(state_, max_clients, region_bytes);
}

}  // namespace vgpu
