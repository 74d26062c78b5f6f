// Paper model (Eqs. 1-11) and the work-queue simulator. Expectations are
// those of proj/tests/test_model.cpp:62-216, test_device.cpp:62-253 and
// acceptance criteria 1-4 (tests/acceptance.cpp:58-199), checked against
// brute-force stage walks written here from the definitions.
#include <algorithm>
#include <cmath>
#include <random>
#include <sstream>

#include "minitest.hpp"
#include "vgpu/device.hpp"
#include "vgpu/model.hpp"

using namespace vgpu;

namespace {

struct Tri {
    Micros in, comp, out;
};
constexpr Tri kCI{20, 50, 20};
constexpr Tri kIOI{60, 20, 40};

KernelProfile prof(Tri t, std::uint32_t grid = 1) {
    KernelProfile p;
    p.t_data_in = t.in;
    p.t_comp = t.comp;
    p.t_data_out = t.out;
    p.grid_size = grid;
    return p;
}

ModelParams par(std::uint32_t n, Tri t, Micros init = 100, Micros ctx = 10) {
    return ModelParams{n, init, ctx, prof(t)};
}

// brute-force walks of the three issue disciplines (idealized regime)
Micros walk_native(Micros n, Micros init, Micros ctx, Tri t) {
    Micros total = 0;
    for (Micros i = 0; i < n; ++i) total += (i ? ctx : 0) + init + t.in + t.comp + t.out;
    return total;
}
Micros walk_ps1(Micros n, Tri t) {
    Micros last_comp = 0;
    for (Micros i = 1; i <= n; ++i) last_comp = std::max(last_comp, i * t.in + t.comp);
    return std::max(n * t.in, last_comp + n * t.out);
}
Micros walk_ps2(Micros n, Tri t) {
    Micros h2d = 0, d2h = 0, comp = 0, span = 0;
    for (Micros i = 0; i < n; ++i) {
        h2d += t.in;
        const Micros c = std::max(h2d, comp) + t.comp;
        d2h = std::max(c, d2h) + t.out;
        comp = c;
        span = std::max(span, d2h);
    }
    return span;
}

}  // namespace

TEST_CASE("model: classification and style choice") {
    CHECK(classify_kernel(prof({20, 50, 20})) == KernelClass::ComputeIntensive);
    CHECK(classify_kernel(prof({60, 20, 40})) == KernelClass::IOIntensive);
    CHECK(classify_kernel(prof({50, 50, 50})) == KernelClass::ComputeIntensive);
    CHECK(classify_kernel(prof({60, 50, 10})) == KernelClass::Intermediate);
    CHECK(classify_kernel(prof({10, 50, 60})) == KernelClass::Intermediate);
    CHECK(recommend_style(KernelClass::ComputeIntensive) == ProgrammingStyle::PS1);
    CHECK(recommend_style(KernelClass::IOIntensive) == ProgrammingStyle::PS2);
    CHECK(recommend_style(KernelClass::Intermediate) == ProgrammingStyle::PS1);
    std::mt19937_64 g(7);
    for (int i = 0; i < 2000; ++i) {
        const Tri t{g() % 101, g() % 101, g() % 101};
        const auto c = classify_kernel(prof(t));
        if (t.in <= t.comp && t.out <= t.comp) CHECK(c == KernelClass::ComputeIntensive);
        else if (t.in > t.comp && t.out > t.comp) CHECK(c == KernelClass::IOIntensive);
        else CHECK(c == KernelClass::Intermediate);
    }
}

TEST_CASE("model: equation values (acceptance criterion 1)") {
    CHECK(t_total_no_vt(par(1, kCI)) == 190);
    CHECK(t_total_no_vt(par(4, kCI)) == 790);
    CHECK(t_total_no_vt(par(8, kCI)) == 1590);
    CHECK(t_total_ci_ps1(par(1, kCI)) == 90);
    CHECK(t_total_ci_ps1(par(4, kCI)) == 210);
    CHECK(t_total_ci_ps1(par(8, kCI)) == 370);
    CHECK(t_total_ci_ps2(par(4, kCI)) == 240);
    CHECK(t_total_ci_ps2(par(8, kCI)) == 440);
    CHECK(t_total_ioi_ps1(par(1, kIOI)) == 120);
    CHECK(t_total_ioi_ps1(par(4, kIOI)) == 420);
    CHECK(t_total_ioi_ps1(par(8, kIOI)) == 820);
    CHECK(t_total_ioi_ps2(par(4, kIOI)) == 300);
    CHECK(t_total_ioi_ps2(par(4, {40, 20, 60})) == 300);
    CHECK(std::abs(speedup_ci(par(4, kCI)) - 790.0 / 210.0) < 1e-12);
    CHECK(std::abs(speedup_ci(par(4, kCI)) - 3.762) < 0.001);
    CHECK(std::abs(speedup_limit_ci(par(4, kCI)) - 5.0) < 0.001);
    CHECK(std::abs(speedup_limit_ioi(par(4, kIOI)) - 230.0 / 60.0) < 0.001);
    CHECK(std::abs(speedup_ci(par(1, kCI, 0, 0)) - 1.0) < 1e-12);
    CHECK(std::abs(speedup_ioi(par(1, kIOI, 0, 0)) - 1.0) < 1e-12);
    const auto tie = compare_styles(par(1, {60, 50, 10}, 0, 0));
    CHECK(tie.ps1_total == tie.ps2_total);
    CHECK(tie.preferred == ProgrammingStyle::PS1);
    const auto mm = compare_styles(par(4, {60, 50, 10}, 0, 0));
    CHECK(mm.ps1_total == walk_ps1(4, {60, 50, 10}));
    CHECK(mm.ps2_total == walk_ps2(4, {60, 50, 10}));
    CHECK(mm.preferred == ProgrammingStyle::PS2);
    ModelParams zero = par(1, kCI);
    zero.n_process = 0;
    CHECK_THROWS_AS((void)t_total_no_vt(zero), std::invalid_argument);
}

TEST_CASE("model: closed forms equal brute-force walks; speedups converge") {
    std::mt19937_64 g(20260810);
    for (int i = 0; i < 1000; ++i) {
        const Tri t{1 + g() % 100000, 1 + g() % 100000, 1 + g() % 100000};
        for (std::uint32_t n = 1; n <= 16; ++n) {
            const auto m = par(n, t);
            CHECK(t_total_no_vt(m) == walk_native(n, 100, 10, t));
            CHECK(t_total_ps1(m) == walk_ps1(n, t));
            CHECK(t_total_ps2(m) == walk_ps2(n, t));
        }
    }
    for (const Tri t : {kCI, kIOI}) {
        double prev = 0.0;
        for (std::uint32_t n = 1; n <= 64; ++n) {
            const double s = t.comp >= t.in ? speedup_ci(par(n, t)) : speedup_ioi(par(n, t));
            CHECK(s >= prev - 1e-12);
            prev = s;
        }
        const auto big = par(10000, t);
        const double lim = t.comp >= t.in ? speedup_limit_ci(big) : speedup_limit_ioi(big);
        const double s = t.comp >= t.in ? speedup_ci(big) : speedup_ioi(big);
        CHECK(std::abs(s / lim - 1.0) < 0.01);
    }
}

TEST_CASE("device: work-queue layout per style") {
    const std::vector<KernelProfile> ps{prof(kCI), prof(kCI), prof(kCI)};
    const auto q1 = build_work_queue(ProgrammingStyle::PS1, ps);
    REQUIRE(q1.commands.size() == 9);
    for (int i = 0; i < 3; ++i) {
        CHECK(q1.commands[i].kind == CommandKind::SendData);
        CHECK(q1.commands[3 + i].kind == CommandKind::Compute);
        CHECK(q1.commands[6 + i].kind == CommandKind::RtrvData);
        CHECK(q1.commands[i].stream_id == static_cast<std::uint32_t>(i));
    }
    const auto q2 = build_work_queue(ProgrammingStyle::PS2, ps);
    for (int i = 0; i < 3; ++i) {
        CHECK(q2.commands[3 * i].kind == CommandKind::SendData);
        CHECK(q2.commands[3 * i + 1].kind == CommandKind::Compute);
        CHECK(q2.commands[3 * i + 2].kind == CommandKind::RtrvData);
        CHECK(q2.commands[3 * i].stream_id == static_cast<std::uint32_t>(i));
    }
    const std::vector<std::uint64_t> ids{11, 12, 13};
    const auto q3 = build_work_queue(ProgrammingStyle::PS1, ps, ids);
    CHECK(q3.commands[4].task_id == 12);
    CHECK_THROWS_AS((void)build_work_queue(ProgrammingStyle::PS1, std::vector<KernelProfile>{}),
                    std::invalid_argument);
    CHECK_THROWS_AS((void)build_work_queue(ProgrammingStyle::PS1, ps,
                                           std::vector<std::uint64_t>{1}),
                    std::invalid_argument);
}

TEST_CASE("device: canonical makespans 210 / 240 / 300 / 120") {
    const DeviceSpec dev;
    auto span = [&](ProgrammingStyle s, Tri t, std::uint32_t n) {
        return simulate(build_work_queue(s, std::vector<KernelProfile>(n, prof(t))), dev).makespan;
    };
    CHECK(span(ProgrammingStyle::PS1, kCI, 4) == 210);
    CHECK(span(ProgrammingStyle::PS2, kCI, 4) == 240);
    CHECK(span(ProgrammingStyle::PS2, kIOI, 4) == 300);
    CHECK(span(ProgrammingStyle::PS1, kIOI, 1) == 120);
    CHECK(span(ProgrammingStyle::PS1, kCI, 1) == 90);
}

TEST_CASE("device: simulate equals the closed forms (acceptance criterion 2)") {
    std::mt19937_64 g(20260810);
    const DeviceSpec dev;
    int bad = 0;
    for (int i = 0; i < 1000; ++i) {
        const Tri t{1 + g() % 100000, 1 + g() % 100000, 1 + g() % 100000};
        for (std::uint32_t n = 1; n <= 16; ++n) {
            const std::vector<KernelProfile> ps(n, prof(t));
            const auto m = par(n, t);
            if (simulate(build_work_queue(ProgrammingStyle::PS1, ps), dev).makespan != t_total_ps1(m)) ++bad;
            if (simulate(build_work_queue(ProgrammingStyle::PS2, ps), dev).makespan != t_total_ps2(m)) ++bad;
            if (simulate_native(ps, 100, 10).makespan != t_total_no_vt(m)) ++bad;
        }
    }
    CHECK(bad == 0);
}

TEST_CASE("device: capacity waves, determinism, timeline csv") {
    DeviceSpec dev;  // 14 x 8 = 112 slots
    const std::vector<KernelProfile> one{prof(kCI, 224)};
    const auto t = simulate(build_work_queue(ProgrammingStyle::PS1, one), dev);
    CHECK(t.makespan == 20 + 2 * 50 + 20);  // two waves
    const std::vector<KernelProfile> four(4, prof(kCI, 112));
    const auto full = simulate(build_work_queue(ProgrammingStyle::PS1, four), dev);
    CHECK(full.makespan > 210);  // capacity degradation vs Eq. (2)
    const auto again = simulate(build_work_queue(ProgrammingStyle::PS1, four), dev);
    CHECK(again.makespan == full.makespan);
    CHECK(again.entries.size() == full.entries.size());
    std::ostringstream os;
    write_timeline_csv(simulate(build_work_queue(ProgrammingStyle::PS2,
                                                 std::vector<KernelProfile>{prof(kIOI)}),
                                dev),
                       os);
    CHECK(os.str() ==
          "task_id,stream_id,kind,start_us,end_us\n0,0,SendData,0,60\n0,0,Compute,60,80\n"
          "0,0,RtrvData,80,120\n");
    const auto nat = simulate_native(std::vector<KernelProfile>(2, prof(kIOI)), 100, 10);
    CHECK(nat.makespan == 2 * (100 + 120) + 10);
    CHECK(nat.task_start(1) == 100 + 120 + 10 + 100);
    CHECK(DeviceSpec::b200().num_sms == 148);
    CHECK_THROWS_AS((void)simulate(WorkQueue{}, dev), std::invalid_argument);
}

TEST_CASE("device: B200 fluid block scheduler (DeviceSpec::fluid_blocks)") {
    // 148 SMs x 4 resident CTAs = 592 slots; a NAS EP slice = 512 CTAs
    DeviceSpec dev = DeviceSpec::b200();
    dev.block_slots_per_sm = 4;
    dev.fluid_blocks = true;
    KernelProfile p;
    p.t_data_in = 0;
    p.t_comp = 100;
    p.t_data_out = 0;
    p.grid_size = 512;
    auto span = [&](std::size_t n) {
        std::vector<KernelProfile> ps(n, p);
        return simulate(build_work_queue(ProgrammingStyle::PS1, ps), dev).makespan;
    };
    CHECK(span(1) == 100);
    // the second kernel runs on the 80 free slots, then on 512 once the first
    // is done: 512*100 work, 8000 by t = 100, the rest at 512 per us
    CHECK(span(2) == 100 + static_cast<Micros>(std::ceil(43200.0 / 512)));
    // n kernels saturate the device: total work / 592 slots, to within a
    // kernel's tail (the last one cannot use more than 512 slots)
    const Micros s8 = span(8);
    CHECK(s8 >= static_cast<Micros>(8 * 512 * 100 / 592));
    CHECK(s8 <= static_cast<Micros>(8 * 512 * 100 / 592) + 20);
    // the reference's rule charges the late kernel whole waves on its 80 slots
    dev.fluid_blocks = false;
    CHECK(span(2) == 700);
    // a grid larger than the device: its solo time already holds its waves
    dev.fluid_blocks = true;
    p.grid_size = 2 * 592;
    CHECK(span(1) == 100);
    CHECK(span(2) == 200);
    // the fixed part of a kernel span (launch probe) is paid once per kernel,
    // concurrently, not per wave: two full-device kernels of 110 us with 10 us
    // fixed take 10 + 2 x 100, not 2 x 110
    p.grid_size = 592;
    p.t_comp = 110;
    dev.kernel_launch_us = 10;
    CHECK(span(1) == 110);
    CHECK(span(2) == 210);
    // shared slots (processor sharing): two 512-CTA kernels on 592 slots run
    // side by side and end together at 2 x 512 x 100 / 592, where queue order
    // leaves the second one a tail on 512 slots
    dev.kernel_launch_us = 0;
    p.grid_size = 512;
    p.t_comp = 100;
    dev.fluid_blocks = 2;
    CHECK(span(1) == 100);
    CHECK(span(2) == static_cast<Micros>(std::ceil(2.0 * 512 * 100 / 592)));
    const Micros shared8 = span(8);
    CHECK(shared8 == static_cast<Micros>(std::ceil(8.0 * 512 * 100 / 592)));
    dev.fluid_blocks = 1;
    CHECK(span(8) > shared8);
}

TEST_CASE("DeviceSpec keeps the reference's layout (it sits inside GvmConfig)") {
    // the reference's DeviceSpec: five uint32 fields (20 bytes); B200 fields
    // live in its tail padding so reference-built programs keep GvmConfig's
    // layout when they link libvgpu
    CHECK(sizeof(vgpu::DeviceSpec) <= 24);
    CHECK(alignof(vgpu::DeviceSpec) == 4);
}
