// vgpu-b200 — multi-GPU plumbing around the per-GPU GVMs.
//
// One GVM process per B200 (`vgpud --device g --instance gpu<g>`), clients
// pinned to their GPU's NUMA-local cores and routed by the unchanged
// $VGPU_INSTANCE lookup (reference client.cpp:146-151). The only cross-GPU
// traffic is the single final reduction: GVM 0 creates the NCCL unique id
// and publishes it in a file (no MPI, no torch), every GVM joins the
// communicator, all-gathers its fold record (GvmDaemon::fold_record) and
// folds the records in rank order, so floating-point sums are deterministic.
#ifndef VGPU_MULTIGPU_HPP
#define VGPU_MULTIGPU_HPP

#include <array>
#include <chrono>
#include <cstdint>
#include <span>
#include <string>
#include <vector>

namespace vgpu::multigpu {

inline constexpr std::size_t kRecordWidth = 16;  // == GvmDaemon::kFoldWidth

// Rank 0: write `id` to `path` atomically (temp file + rename), so a reader
// never sees a partial id. Throws std::runtime_error on I/O failure.
void publish_id(const std::string& path, std::span<const std::uint8_t> id);

// Ranks > 0: wait until `path` holds a complete id of `bytes` bytes (polls
// every millisecond), then return it. Throws std::runtime_error on timeout.
std::vector<std::uint8_t> fetch_id(const std::string& path, std::size_t bytes,
                                   std::chrono::milliseconds timeout);

// The all-gathered records (rank-major, nranks x kRecordWidth) folded in
// rank order: [0..14] summed left to right, [15] summed mod 1000003. Any
// rank's EP coverage of -1 (a slice that changed bits) makes [14] -1.
std::array<double, kRecordWidth> fold_in_rank_order(std::span<const double> all,
                                                    std::uint32_t nranks);

// "0-3,8,10-11" -> {0,1,2,3,8,10,11}; malformed parts are skipped.
std::vector<int> parse_cpulist(const std::string& list);

// The host cores local to the PCI device `bus_id` ("0000:1b:00.0"; case and
// an 8-digit domain accepted), from sysfs local_cpulist; empty when unknown.
std::vector<int> local_cpus(const std::string& bus_id);

// Pin the calling thread/process to `cpus` (sched_setaffinity); false when
// the set is empty or the call fails.
bool pin_to(const std::vector<int>& cpus);

}  // namespace vgpu::multigpu

#endif  // VGPU_MULTIGPU_HPP
