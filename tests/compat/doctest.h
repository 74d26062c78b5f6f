// doctest-compatible shim (doctest is not vendored in this image): maps the
// macros the reference's unit tests use onto tests/cpp/minitest.hpp, so the
// reference's own test sources compile unmodified against vgpu-b200.
#pragma once
#include <algorithm>
#include <cmath>
#include <limits>

#include "../cpp/minitest.hpp"

namespace doctest {
struct Approx {
    explicit Approx(double v) : value(v) {}
    Approx& epsilon(double e) {
        eps = e;
        return *this;
    }
    double value;
    double eps = std::numeric_limits<float>::epsilon() * 100;
};
inline bool operator==(double lhs, const Approx& a) {
    return std::fabs(lhs - a.value) < a.eps * (1.0 + std::max(std::fabs(lhs), std::fabs(a.value)));
}
inline bool operator==(const Approx& a, double rhs) { return rhs == a; }
inline bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
}  // namespace doctest
