// Synthetic SPMD workloads of BASELINE.json configs C1-C5.
//
// Each worker of an SPMD run builds ONE job: its payload id, a kernel
// descriptor (the timing triple is the client's declared estimate — the
// GVM uses it only to pick PS-1/PS-2 and to report the model prediction)
// and its private input bytes:
//   vecadd  C1  n = 2^20 fp32 per operand; a[j] = (w+1)*1000 + j%512,
//               b[j] = (j%512)*0.25 — the reference bench pattern
//               (proj/src/bench/bench.cpp:34-49), every sum exact in fp32;
//   ep      C2  NAS EP class A (m = 28) split over the EP workers in equal
//               contiguous batch ranges (NPB-MPI decomposition);
//   bs      C3  4 Mi options, S~U[5,30], X~U[1,100], T~U[0.25,10], seed 5347+w;
//   mm      C4  2048 x 2048 fp32, A,B ~ U[-1,1], seed 1000+w;
//   mixed   C5  worker w runs kind w % 4 (vecadd, ep, bs, mm);
// and the paper's remaining payloads (not BASELINE
// configs):
//   cg      NAS CG, every worker runs the whole NPB class (default A): the
//           program builds its matrix with NPB's makea (untimed in NPB) —
//           through cg_builder(), which the program sets (vgpu-spmd: the
//           product's vgpu::npb::make_cg_input; ref-bench: the oracle's);
//   vmul    VecMul, vecadd's shapes and values, payload vector-mul;
//   es      Electrostatics (VMD direct Coulomb summation): 100K atoms,
//           64 x 64 lattice x 25 slices (the paper's "100K atoms / 25
//           iterations"), atoms ~ U(box), q ~ U[-1,1], seed 777+w;
//   mg      NAS MG, every worker runs the whole NPB class (default S, the
//           paper's 32^3 / 4 iterations): the program builds v with NPB's
//           zran3 (untimed in NPB) through mg_builder().
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "vgpu/message.hpp"
#include "vgpu/payload.hpp"
#include "vgpu_cuda.h"

namespace vgpu::wl {

enum class Kind { VecAdd, Ep, Bs, Mm, Cg, VecMul, Es, Mg };

struct Sizes {
    std::uint64_t vecadd_n = 1ull << 20;
    std::uint32_t ep_m = 28;
    std::uint64_t ep_batches = 0;  // batches of the whole run's problem; 0 = 2^(ep_m-16)
    std::uint64_t bs_n = 4ull << 20;
    std::uint32_t mm_n = 2048;
    char cg_class = 'A';
    char mg_class = 'S';
    std::uint32_t es_atoms = 100000;
    std::uint32_t es_nx = 64, es_ny = 64, es_nz = 25;
    float es_h = 0.5f;
};

// NPB CG shapes (cg.f): rows, nonzeros per generated vector
struct CgShape {
    std::uint32_t n, nonzer;
};

inline CgShape cg_shape(char cls) {
    switch (cls) {
        case 'S': return {1400, 7};
        case 'W': return {7000, 8};
        case 'A': return {14000, 11};
        case 'B': return {75000, 13};
        case 'C': return {150000, 15};
        default: throw std::invalid_argument(std::string("unknown NPB CG class ") + cls);
    }
}

// The program's NPB zran3: nas-mg input bytes for a class
using MgBuilder = Bytes (*)(char cls);
inline MgBuilder& mg_builder() {
    static MgBuilder b = nullptr;
    return b;
}

// NPB MG classes (mg.f): grid points per dimension
inline std::uint32_t mg_nx(char cls) {
    switch (cls) {
        case 'S': return 32;
        case 'W': return 128;
        case 'A': case 'B': return 256;
        case 'C': return 512;
        default: throw std::invalid_argument("unknown NPB MG class");
    }
}

// The program's NPB makea: nas-cg input bytes for a class
using CgBuilder = Bytes (*)(char cls);
inline CgBuilder& cg_builder() {
    static CgBuilder b = nullptr;
    return b;
}

struct Job {
    Kind kind;
    KernelDescriptor desc;
    Bytes input;
    std::uint64_t output_bytes = 0;
};

inline Kind kind_of(const std::string& workload, std::uint32_t worker) {
    if (workload == "vecadd") return Kind::VecAdd;
    if (workload == "ep") return Kind::Ep;
    if (workload == "bs") return Kind::Bs;
    if (workload == "mm") return Kind::Mm;
    if (workload == "cg") return Kind::Cg;
    if (workload == "vmul") return Kind::VecMul;
    if (workload == "es") return Kind::Es;
    if (workload == "mg") return Kind::Mg;
    if (workload == "mixed") return static_cast<Kind>(worker % 4);
    throw std::invalid_argument("unknown workload: " + workload);
}

inline std::uint64_t xorshift(std::uint64_t& s) {
    s ^= s >> 12;
    s ^= s << 25;
    s ^= s >> 27;
    return s * 0x2545F4914F6CDD1Dull;
}

inline float uniform(std::uint64_t& s, float lo, float hi) {
    const double u = static_cast<double>(xorshift(s) >> 11) * (1.0 / 9007199254740992.0);
    return static_cast<float>(lo + (hi - lo) * u);
}

inline std::uint64_t fnv1a(const std::uint8_t* p, std::size_t n) {
    std::uint64_t h = 0xcbf29ce484222325ull;
    for (std::size_t i = 0; i < n; ++i) {
        h ^= p[i];
        h *= 0x100000001b3ull;
    }
    return h;
}

// declared stage estimates (us): PCIe ~50 GB/s, HBM ~6.5 TB/s, FP32 ~50 TF/s
inline Micros pcie_us(std::uint64_t bytes) { return bytes / 50'000 + 1; }

inline Job make_job(const std::string& workload, std::uint32_t worker, std::uint32_t workers,
                    const Sizes& sz = {}) {
    Job j;
    j.kind = kind_of(workload, worker);
    switch (j.kind) {
        case Kind::VecMul:
        case Kind::VecAdd: {
            const std::uint64_t n = sz.vecadd_n;
            std::vector<float> v(2 * n);
            for (std::uint64_t i = 0; i < n; ++i) {
                v[i] = static_cast<float>(worker + 1) * 1000.0f + static_cast<float>(i % 512);
                v[n + i] = static_cast<float>(i % 512) * 0.25f;
            }
            j.input.resize(8 * n);
            std::memcpy(j.input.data(), v.data(), j.input.size());
            j.desc.payload_id = j.kind == Kind::VecAdd ? "vector-add" : "vector-mul";
            j.desc.t_data_in = pcie_us(8 * n);
            j.desc.t_comp = (12 * n) / 6'500'000 + 1;
            j.desc.t_data_out = pcie_us(4 * n);
            j.desc.grid_size = static_cast<std::uint32_t>((n + 4095) / 4096);
            j.output_bytes = 4 * n;
            break;
        }
        case Kind::Ep: {
            // EP workers share the class: rank among EP workers, count of EP workers
            std::uint32_t rank = worker, count = workers;
            if (workload == "mixed") {
                rank = worker / 4;
                count = (workers + 2) / 4;  // workers w with w % 4 == 1
            }
            const std::uint64_t total = sz.ep_batches ? sz.ep_batches : 1ull << (sz.ep_m - 16);
            const std::uint64_t per = total / count, extra = total % count;
            vgpu_ep_params p{};
            p.m = sz.ep_m;
            p.mk = 16;
            p.first_batch = rank * per + std::min<std::uint64_t>(rank, extra);
            p.n_batches = per + (rank < extra ? 1 : 0);
            j.input.resize(sizeof p);
            std::memcpy(j.input.data(), &p, sizeof p);
            j.desc.payload_id = "nas-ep";
            j.desc.t_data_in = 1;
            j.desc.t_comp = p.n_batches / 4 + 1;  // ~0.25 us per 2^16-pair batch
            j.desc.t_data_out = 1;
            j.desc.grid_size = static_cast<std::uint32_t>(p.n_batches);
            j.output_bytes = sizeof(vgpu_ep_result);
            break;
        }
        case Kind::Bs: {
            const std::uint64_t n = sz.bs_n;
            std::vector<float> v(3 * n);
            std::uint64_t s = 5347 + worker;
            for (std::uint64_t i = 0; i < n; ++i) {
                v[i] = uniform(s, 5.0f, 30.0f);
                v[n + i] = uniform(s, 1.0f, 100.0f);
                v[2 * n + i] = uniform(s, 0.25f, 10.0f);
            }
            j.input.resize(12 * n);
            std::memcpy(j.input.data(), v.data(), j.input.size());
            j.desc.payload_id = "black-scholes";
            j.desc.t_data_in = pcie_us(12 * n);
            j.desc.t_comp = (20 * n) / 6'500'000 + 1;
            j.desc.t_data_out = pcie_us(8 * n);
            j.desc.grid_size = static_cast<std::uint32_t>((n + 2047) / 2048);
            j.output_bytes = 8 * n;
            break;
        }
        case Kind::Es: {
            vgpu_es_header h{};
            h.natoms = sz.es_atoms;
            h.nx = sz.es_nx;
            h.ny = sz.es_ny;
            h.nz = sz.es_nz;
            h.spacing = sz.es_h;
            std::vector<float> at(4ull * h.natoms);
            std::uint64_t s = 777 + worker;
            for (std::uint32_t i = 0; i < h.natoms; ++i) {
                at[4 * i] = uniform(s, 0.0f, h.nx * h.spacing);
                at[4 * i + 1] = uniform(s, 0.0f, h.ny * h.spacing);
                at[4 * i + 2] = uniform(s, 0.0f, h.nz * h.spacing);
                at[4 * i + 3] = uniform(s, -1.0f, 1.0f);
            }
            j.input.resize(sizeof h + 16ull * h.natoms);
            std::memcpy(j.input.data(), &h, sizeof h);
            std::memcpy(j.input.data() + sizeof h, at.data(), 16ull * h.natoms);
            const std::uint64_t pts = static_cast<std::uint64_t>(h.nx) * h.ny * h.nz;
            j.desc.payload_id = "electrostatics";
            j.desc.t_data_in = pcie_us(j.input.size());
            j.desc.t_comp = static_cast<Micros>(pts * h.natoms / 4.6e6) + 1;  // ~4.6e12 rsqrt/s
            j.desc.t_data_out = pcie_us(4 * pts);
            j.desc.grid_size = static_cast<std::uint32_t>((h.nx + 63) / 64 * ((h.ny + 7) / 8) * h.nz);
            j.output_bytes = 4 * pts;
            break;
        }
        case Kind::Mg: {
            if (!mg_builder()) throw std::logic_error("mg workload: no NPB zran3 set (mg_builder)");
            j.input = mg_builder()(sz.mg_class);
            vgpu_mg_header h;
            std::memcpy(&h, j.input.data(), sizeof h);
            j.desc.payload_id = "nas-mg";
            j.desc.t_data_in = pcie_us(j.input.size());
            // ~100 B per finest point per V-cycle at ~2 TB/s, plus ~150
            // launches of ~3 us per cycle set
            const double pts = static_cast<double>(h.nx) * h.nx * h.nx;
            j.desc.t_comp = static_cast<Micros>(h.nit * (pts * 115.0 / 2e6 + 110.0)) + 1;
            j.desc.t_data_out = 1;
            j.desc.grid_size = 64;  // the paper's MG grid
            j.output_bytes = sizeof(vgpu_mg_result);
            break;
        }
        case Kind::Cg: {
            if (!cg_builder()) throw std::logic_error("cg workload: no NPB makea set (cg_builder)");
            j.input = cg_builder()(sz.cg_class);
            vgpu_cg_header h;
            std::memcpy(&h, j.input.data(), sizeof h);
            j.desc.payload_id = "nas-cg";
            j.desc.t_data_in = pcie_us(j.input.size());
            // niter x 26 SpMVs of 12 B per nonzero at ~2 TB/s
            j.desc.t_comp = static_cast<Micros>(h.niter * 26.0 * 12.0 * h.nnz / 2e6) + 1;
            j.desc.t_data_out = 1;
            j.desc.grid_size = 16;
            j.output_bytes = sizeof(vgpu_cg_result);
            break;
        }
        case Kind::Mm: {
            const std::uint64_t n = sz.mm_n;
            std::vector<float> v(2 * n * n);
            std::uint64_t s = 1000 + worker;
            for (auto& x : v) x = uniform(s, -1.0f, 1.0f);
            j.input.resize(8 * n * n);
            std::memcpy(j.input.data(), v.data(), j.input.size());
            j.desc.payload_id = "sgemm";
            j.desc.t_data_in = pcie_us(8 * n * n);
            j.desc.t_comp = static_cast<Micros>(2.0 * n * n * n / 50e6) + 1;
            j.desc.t_data_out = pcie_us(4 * n * n);
            j.desc.grid_size = static_cast<std::uint32_t>((n / 128) * (n / 128));
            j.output_bytes = 4 * n * n;
            break;
        }
    }
    return j;
}

// ---- the SPMD program's own result check (sampled, binary64) -------------
//
// What a worker verifies about its result after the timed rounds, the way
// NPB programs verify themselves: Black-Scholes prices of every `stride`-th
// option recomputed in binary64 with the SDK formulation (polynomial CND,
// R = 0.02, V = 0.30), L1-relative over the sample; SGEMM rows i = 0,
// stride, 2 stride, ... of C recomputed with binary64 accumulation,
// relative Frobenius over those rows. Tolerances are the GPU parity bars
// (BS 1e-6, SGEMM 1e-5).
struct SampleCheck {
    bool ok = true;
    double err = 0.0;        // L1-relative (BS) / relative Frobenius (SGEMM)
    std::uint64_t samples = 0;
};

inline double bs_cnd64(double d) {
    const double k = 1.0 / (1.0 + 0.2316419 * std::fabs(d));
    const double poly =
        k * (0.31938153 + k * (-0.356563782 + k * (1.781477937 + k * (-1.821255978 + k * 1.330274429))));
    const double c = 0.39894228040143267793994605993438 * std::exp(-0.5 * d * d) * poly;
    return d > 0.0 ? 1.0 - c : c;
}

inline SampleCheck check_bs_sample(const Bytes& in, const Bytes& out, std::uint64_t stride) {
    SampleCheck r;
    const std::uint64_t n = in.size() / 12;
    if (out.size() != 8 * n || n == 0) return {false, 1.0, 0};
    const float* S = reinterpret_cast<const float*>(in.data());
    const float* call = reinterpret_cast<const float*>(out.data());
    const double R = VGPU_BS_RISKFREE, V = VGPU_BS_VOLATILITY;
    double num = 0.0, den = 0.0;
    for (std::uint64_t i = 0; i < n; i += stride) {
        const double s = S[i], x = S[n + i], t = S[2 * n + i];
        const double vt = V * std::sqrt(t);
        const double d1 = (std::log(s / x) + (R + 0.5 * V * V) * t) / vt, d2 = d1 - vt;
        const double disc = x * std::exp(-R * t);
        const double c = s * bs_cnd64(d1) - disc * bs_cnd64(d2);
        const double p = disc * (1.0 - bs_cnd64(d2)) - s * (1.0 - bs_cnd64(d1));
        num += std::fabs(call[i] - c) + std::fabs(call[n + i] - p);
        den += std::fabs(c) + std::fabs(p);
        ++r.samples;
    }
    r.err = den > 0.0 ? num / den : 0.0;
    r.ok = r.err <= 1e-6;
    return r;
}

inline SampleCheck check_mm_sample(const Bytes& in, const Bytes& out, std::uint64_t row_stride) {
    SampleCheck r;
    const std::uint64_t nn = in.size() / 8;
    std::uint64_t n = static_cast<std::uint64_t>(std::sqrt(static_cast<double>(nn)));
    while (n * n > nn) --n;
    if (n == 0 || n * n != nn || out.size() != 4 * nn) return {false, 1.0, 0};
    const float* A = reinterpret_cast<const float*>(in.data());
    const float* B = A + nn;
    const float* C = reinterpret_cast<const float*>(out.data());
    std::vector<double> row(n);
    double num = 0.0, den = 0.0;
    for (std::uint64_t i = 0; i < n; i += row_stride) {
        std::fill(row.begin(), row.end(), 0.0);
        for (std::uint64_t k = 0; k < n; ++k) {
            const double a = A[i * n + k];
            const float* b = B + k * n;
            for (std::uint64_t j = 0; j < n; ++j) row[j] += a * b[j];
        }
        for (std::uint64_t j = 0; j < n; ++j) {
            const double dlt = C[i * n + j] - row[j];
            num += dlt * dlt;
            den += row[j] * row[j];
        }
        r.samples += n;
    }
    r.err = den > 0.0 ? std::sqrt(num / den) : 0.0;
    r.ok = r.err <= 1e-5;
    return r;
}

// Largest region any worker of `workload` needs.
inline std::uint64_t region_bytes(const std::string& workload, const Sizes& sz = {}) {
    const std::uint64_t va = 8 * sz.vecadd_n, bs = 12 * sz.bs_n,
                        mm = 8ull * sz.mm_n * sz.mm_n, ep = sizeof(vgpu_ep_result);
    if (workload == "vecadd") return va;
    if (workload == "ep") return ep;
    if (workload == "bs") return bs;
    if (workload == "mm") return mm;
    if (workload == "vmul") return va;
    if (workload == "es")
        return std::max<std::uint64_t>(sizeof(vgpu_es_header) + 16ull * sz.es_atoms,
                                       4ull * sz.es_nx * sz.es_ny * sz.es_nz);
    if (workload == "mg") {  // the input, or half the grids' workspace (slot ws = 2 x region)
        const std::uint32_t nx = mg_nx(sz.mg_class);
        return std::max<std::uint64_t>(vgpu_mg_input_bytes(nx), (vgpu_mg_workspace_bytes(nx) + 1) / 2);
    }
    if (workload == "cg") {  // upper bound: nnz <= n (nonzer + 1)^2
        const CgShape c = cg_shape(sz.cg_class);
        return vgpu_cg_input_bytes(c.n, c.n * (c.nonzer + 1) * (c.nonzer + 1));
    }
    return std::max({va, bs, mm, ep});
}

}  // namespace vgpu::wl
