// NPB CG problem builder (include/vgpu/npb_cg.hpp). Client-side input
// generation, the untimed makea phase of NPB CG; the timed iterations run in
// the nas-cg kernel (csrc/cuda/k_cg.cuh).
//
// Assembly: NPB's sparse() inserts each outer product's entries into
// per-row sorted lists, summing duplicates as they arrive (increasing outer
// index i). Here every contribution is bucketed by row in arrival order,
// each row is stably sorted by column, and runs of one column are summed
// left to right from 0.0: the same additions in the same order, so the same
// bits, without the insertion shifting.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <stdexcept>

#include "vgpu/npb_cg.hpp"
#include "vgpu_cuda.h"

namespace vgpu::npb {

namespace {

constexpr std::uint64_t kMask46 = (1ull << 46) - 1;
constexpr std::uint64_t kMult = 1220703125ull;  // 5^13
constexpr double kRcond = 0.1;

struct Lcg {
    std::uint64_t x;
    double next() {  // NPB randlc: x <- 5^13 x mod 2^46, returns x / 2^46
        x = (x * kMult) & kMask46;
        return static_cast<double>(x) * 0x1p-46;
    }
};

}  // namespace

CgClass cg_class(char cls) {
    switch (cls) {
        case 'S': return {1400, 7, 15, 10.0, 8.5971775078648};
        case 'W': return {7000, 8, 15, 12.0, 10.362595087124};
        case 'A': return {14000, 11, 15, 20.0, 17.130235054029};
        case 'B': return {75000, 13, 75, 60.0, 22.712745482631};
        case 'C': return {150000, 15, 75, 110.0, 28.973605592845};
        default: throw std::invalid_argument(std::string("NPB CG class must be S, W, A, B or C, got ") + cls);
    }
}

std::vector<std::uint8_t> make_cg_input(std::uint32_t n, std::uint32_t nonzer, std::uint32_t niter,
                                        double shift) {
    if (n == 0 || nonzer == 0 || nonzer >= n) throw std::invalid_argument("make_cg_input: need 0 < nonzer < n");
    Lcg rng{314159265ull};
    rng.next();  // NPB: zeta = randlc(tran, amult) before makea
    std::uint32_t nn1 = 1;
    while (nn1 < n) nn1 *= 2;

    // sprnvc + vecset per outer index: nonzer distinct random positions
    // (values drawn before positions, out-of-range and repeated positions
    // rejected), then position i itself with value 0.5
    const std::uint32_t w = nonzer + 1;
    std::vector<std::uint32_t> cnt(n), col(static_cast<std::size_t>(n) * w);
    std::vector<double> val(static_cast<std::size_t>(n) * w);
    for (std::uint32_t i = 0; i < n; ++i) {
        std::uint32_t* c = &col[static_cast<std::size_t>(i) * w];
        double* v = &val[static_cast<std::size_t>(i) * w];
        std::uint32_t k = 0;
        while (k < nonzer) {
            const double vecelt = rng.next();
            const double vecloc = rng.next();
            const std::uint32_t pos = static_cast<std::uint32_t>(nn1 * vecloc);  // 0-based
            if (pos >= n || std::find(c, c + k, pos) != c + k) continue;
            c[k] = pos;
            v[k] = vecelt;
            ++k;
        }
        std::uint32_t* self = std::find(c, c + k, i);
        if (self != c + k) {
            v[self - c] = 0.5;
        } else {
            c[k] = i;
            v[k] = 0.5;
            ++k;
        }
        cnt[i] = k;
    }

    // contributions size_i * v_a * v_b at (c_a, c_b), bucketed by row in
    // increasing i; the diagonal of outer i gets rcond - shift on its own
    // entry (i, i)
    std::vector<std::uint64_t> start(n + 1, 0);
    for (std::uint32_t i = 0; i < n; ++i)
        for (std::uint32_t a = 0; a < cnt[i]; ++a) start[col[static_cast<std::size_t>(i) * w + a] + 1] += cnt[i];
    for (std::uint32_t j = 0; j < n; ++j) start[j + 1] += start[j];
    struct Entry {
        std::uint32_t col;
        double v;
    };
    std::vector<Entry> ent(start[n]);
    std::vector<std::uint64_t> fill(start.begin(), start.end() - 1);
    const double ratio = std::pow(kRcond, 1.0 / static_cast<double>(n));
    double size = 1.0;
    for (std::uint32_t i = 0; i < n; ++i) {
        const std::uint32_t* c = &col[static_cast<std::size_t>(i) * w];
        const double* v = &val[static_cast<std::size_t>(i) * w];
        for (std::uint32_t a = 0; a < cnt[i]; ++a) {
            const std::uint32_t row = c[a];
            const double scale = size * v[a];
            for (std::uint32_t b = 0; b < cnt[i]; ++b) {
                double va = v[b] * scale;
                if (c[b] == row && row == i) va = va + kRcond - shift;
                ent[fill[row]++] = {c[b], va};
            }
        }
        size *= ratio;
    }

    // per row: stable sort by column, sum each column's run in order
    std::vector<std::uint32_t> rowstr(n + 1, 0), colidx;
    std::vector<double> a;
    colidx.reserve(ent.size());
    a.reserve(ent.size());
    for (std::uint32_t j = 0; j < n; ++j) {
        auto b0 = ent.begin() + static_cast<std::ptrdiff_t>(start[j]);
        auto b1 = ent.begin() + static_cast<std::ptrdiff_t>(start[j + 1]);
        std::stable_sort(b0, b1, [](const Entry& x, const Entry& y) { return x.col < y.col; });
        for (auto it = b0; it != b1;) {
            double s = 0.0;
            const std::uint32_t cj = it->col;
            for (; it != b1 && it->col == cj; ++it) s += it->v;
            colidx.push_back(cj);
            a.push_back(s);
        }
        rowstr[j + 1] = static_cast<std::uint32_t>(colidx.size());
    }

    const std::uint32_t nnz = static_cast<std::uint32_t>(colidx.size());
    std::vector<std::uint8_t> out(vgpu_cg_input_bytes(n, nnz), 0);
    vgpu_cg_header h{};
    h.n = n;
    h.nnz = nnz;
    h.niter = niter;
    h.cgitmax = 25;
    h.shift = shift;
    std::uint8_t* p = out.data();
    std::memcpy(p, &h, sizeof h);
    std::memcpy(p + sizeof h, rowstr.data(), 4ull * (n + 1));
    const std::uint64_t off_col = sizeof h + 4ull * (n + 1);
    std::memcpy(p + off_col, colidx.data(), 4ull * nnz);
    const std::uint64_t off_a = (off_col + 4ull * nnz + 7u) & ~7ull;
    std::memcpy(p + off_a, a.data(), 8ull * nnz);
    return out;
}

}  // namespace vgpu::npb
