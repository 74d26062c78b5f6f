// Multi-GPU plumbing: NCCL id rendezvous through a file, rank-order fold,
// NUMA-local placement (include/vgpu/multigpu.hpp).
#include "vgpu/multigpu.hpp"

#include <fcntl.h>
#include <sched.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cctype>
#include <cerrno>
#include <cmath>
#include <cstring>
#include <fstream>
#include <sstream>
#include <stdexcept>
#include <thread>

namespace vgpu::multigpu {

namespace {

// file layout: magic "VGID", u32 byte count, the id
constexpr char kMagic[4] = {'V', 'G', 'I', 'D'};

std::runtime_error io_error(const std::string& what) {
    return std::runtime_error(what + ": " + std::strerror(errno));
}

}  // namespace

void publish_id(const std::string& path, std::span<const std::uint8_t> id) {
    const std::string tmp = path + ".tmp." + std::to_string(getpid());
    const int fd = ::open(tmp.c_str(), O_CREAT | O_TRUNC | O_WRONLY | O_CLOEXEC, 0600);
    if (fd < 0) throw io_error("rendezvous: create " + tmp);
    std::vector<std::uint8_t> buf(8 + id.size());
    std::memcpy(buf.data(), kMagic, 4);
    const std::uint32_t n = static_cast<std::uint32_t>(id.size());
    std::memcpy(buf.data() + 4, &n, 4);
    std::memcpy(buf.data() + 8, id.data(), id.size());
    const bool ok = ::write(fd, buf.data(), buf.size()) == static_cast<ssize_t>(buf.size()) &&
                    ::fsync(fd) == 0;
    ::close(fd);
    if (!ok || ::rename(tmp.c_str(), path.c_str()) != 0) {
        const int e = errno;
        ::unlink(tmp.c_str());
        errno = e;
        throw io_error("rendezvous: publish " + path);
    }
}

std::vector<std::uint8_t> fetch_id(const std::string& path, std::size_t bytes,
                                   std::chrono::milliseconds timeout) {
    const auto deadline = std::chrono::steady_clock::now() + timeout;
    for (;;) {
        std::ifstream in(path, std::ios::binary);
        if (in) {
            std::vector<char> buf(8 + bytes);
            in.read(buf.data(), static_cast<std::streamsize>(buf.size()));
            std::uint32_t n = 0;
            std::memcpy(&n, buf.data() + 4, 4);
            if (in.gcount() == static_cast<std::streamsize>(buf.size()) &&
                std::memcmp(buf.data(), kMagic, 4) == 0 && n == bytes)
                return {buf.begin() + 8, buf.end()};
        }
        if (std::chrono::steady_clock::now() >= deadline)
            throw std::runtime_error("rendezvous: no id in " + path + " before the timeout");
        std::this_thread::sleep_for(std::chrono::milliseconds(1));
    }
}

std::array<double, kRecordWidth> fold_in_rank_order(std::span<const double> all,
                                                    std::uint32_t nranks) {
    if (all.size() < static_cast<std::size_t>(nranks) * kRecordWidth)
        throw std::invalid_argument("fold: fewer records than ranks");
    std::array<double, kRecordWidth> out{};
    bool mismatch = false;
    for (std::uint32_t r = 0; r < nranks; ++r) {
        const double* rec = all.data() + static_cast<std::size_t>(r) * kRecordWidth;
        for (std::size_t i = 0; i + 1 < kRecordWidth; ++i) out[i] = out[i] + rec[i];
        mismatch |= rec[14] < 0.0;
        out[15] = std::fmod(out[15] + rec[15], 1000003.0);
    }
    if (mismatch) out[14] = -1.0;
    return out;
}

std::vector<int> parse_cpulist(const std::string& list) {
    std::vector<int> cpus;
    std::stringstream ss(list);
    std::string part;
    while (std::getline(ss, part, ',')) {
        part.erase(std::remove_if(part.begin(), part.end(), [](unsigned char c) { return std::isspace(c); }),
                   part.end());
        if (part.empty()) continue;
        try {
            const auto dash = part.find('-');
            const int lo = std::stoi(part.substr(0, dash));
            const int hi = dash == std::string::npos ? lo : std::stoi(part.substr(dash + 1));
            for (int c = lo; c <= hi && c - lo < 4096; ++c) cpus.push_back(c);
        } catch (const std::exception&) {
            // skip a malformed part
        }
    }
    std::sort(cpus.begin(), cpus.end());
    cpus.erase(std::unique(cpus.begin(), cpus.end()), cpus.end());
    return cpus;
}

std::vector<int> local_cpus(const std::string& bus_id) {
    std::string id = bus_id;
    for (auto& c : id) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
    // CUDA prints an 8-digit domain ("00000000:1B:00.0"); sysfs uses 4
    if (auto colon = id.find(':'); colon == 8 && id.compare(0, 4, "0000") == 0) id = id.substr(4);
    std::ifstream in("/sys/bus/pci/devices/" + id + "/local_cpulist");
    std::string list;
    if (!in || !std::getline(in, list)) return {};
    return parse_cpulist(list);
}

bool pin_to(const std::vector<int>& cpus) {
    if (cpus.empty()) return false;
    cpu_set_t set;
    CPU_ZERO(&set);
    for (int c : cpus)
        if (c >= 0 && c < CPU_SETSIZE) CPU_SET(c, &set);
    return sched_setaffinity(0, sizeof set, &set) == 0;
}

}  // namespace vgpu::multigpu
