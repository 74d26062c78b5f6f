// Minimal doctest-compatible test harness (doctest.h is not available in
// this image). Supports TEST_CASE / CHECK / CHECK_FALSE / REQUIRE /
// CHECK_THROWS_AS / FAIL / MESSAGE. Test names containing "[gpu]" need a
// CUDA device; the runner selects them with --only-gpu / --exclude-gpu.
#pragma once

#include <cstdio>
#include <cstring>
#include <functional>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

namespace minitest {

struct Case {
    const char* name;
    const char* file;
    int line;
    std::function<void()> fn;
};

inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}

struct Abort {};  // thrown by REQUIRE failures

struct State {
    int failures = 0;
    int checks = 0;
};
inline State& state() {
    static State s;
    return s;
}

inline void report(const char* file, int line, const std::string& what) {
    ++state().failures;
    std::fprintf(stderr, "  %s:%d: FAILED: %s\n", file, line, what.c_str());
}

struct Registrar {
    Registrar(const char* name, const char* file, int line, std::function<void()> fn) {
        registry().push_back({name, file, line, std::move(fn)});
    }
};

inline int run(int argc, char** argv) {
    bool only_gpu = false, exclude_gpu = false;
    std::vector<std::string> filters, files, skips;
    for (int i = 1; i < argc; ++i) {
        if (!std::strcmp(argv[i], "--only-gpu")) only_gpu = true;
        else if (!std::strcmp(argv[i], "--exclude-gpu")) exclude_gpu = true;
        else if (!std::strcmp(argv[i], "--file") && i + 1 < argc) files.emplace_back(argv[++i]);
        else if (!std::strcmp(argv[i], "--skip") && i + 1 < argc) skips.emplace_back(argv[++i]);
        else if (!std::strcmp(argv[i], "--list")) {
            for (auto& c : registry()) std::printf("%s\n", c.name);
            return 0;
        } else filters.emplace_back(argv[i]);
    }
    int ran = 0, failed = 0;
    for (auto& c : registry()) {
        const bool gpu = std::strstr(c.name, "[gpu]") != nullptr;
        if ((only_gpu && !gpu) || (exclude_gpu && gpu)) continue;
        if (!files.empty()) {
            bool hit = false;
            for (auto& f : files) hit |= std::strstr(c.file, f.c_str()) != nullptr;
            if (!hit) continue;
        }
        bool skipped = false;
        for (auto& s : skips) skipped |= std::strstr(c.name, s.c_str()) != nullptr;
        if (skipped) continue;
        if (!filters.empty()) {
            bool hit = false;
            for (auto& f : filters) hit |= std::strstr(c.name, f.c_str()) != nullptr;
            if (!hit) continue;
        }
        ++ran;
        const int before = state().failures;
        std::fprintf(stderr, "[ RUN  ] %s\n", c.name);
        try {
            c.fn();
        } catch (const Abort&) {
        } catch (const std::exception& e) {
            report(c.file, c.line, std::string("unexpected exception: ") + e.what());
        } catch (...) {
            report(c.file, c.line, "unexpected non-std exception");
        }
        const bool ok = state().failures == before;
        if (!ok) ++failed;
        std::fprintf(stderr, "[ %s ] %s\n", ok ? " OK " : "FAIL", c.name);
    }
    std::printf("minitest: %d test cases, %d failed, %d checks\n", ran, failed, state().checks);
    return failed == 0 ? 0 : 1;
}

}  // namespace minitest

#define MT_CAT2(a, b) a##b
#define MT_CAT(a, b) MT_CAT2(a, b)
#define TEST_CASE(name)                                                                   \
    static void MT_CAT(mt_case_, __LINE__)();                                             \
    static ::minitest::Registrar MT_CAT(mt_reg_, __LINE__)(name, __FILE__, __LINE__,      \
                                                           &MT_CAT(mt_case_, __LINE__)); \
    static void MT_CAT(mt_case_, __LINE__)()

#define CHECK(...)                                                                   \
    do {                                                                             \
        ++::minitest::state().checks;                                                \
        if (!(__VA_ARGS__)) ::minitest::report(__FILE__, __LINE__, #__VA_ARGS__);    \
    } while (0)
#define CHECK_FALSE(...) CHECK(!(__VA_ARGS__))
#define REQUIRE(...)                                                                 \
    do {                                                                             \
        ++::minitest::state().checks;                                                \
        if (!(__VA_ARGS__)) {                                                        \
            ::minitest::report(__FILE__, __LINE__, "REQUIRE " #__VA_ARGS__);         \
            throw ::minitest::Abort{};                                               \
        }                                                                            \
    } while (0)
#define CHECK_THROWS_AS(expr, type)                                                  \
    do {                                                                             \
        ++::minitest::state().checks;                                                \
        bool mt_ok = false;                                                          \
        try {                                                                        \
            (void)(expr);                                                            \
        } catch (const type&) {                                                      \
            mt_ok = true;                                                            \
        } catch (...) {                                                              \
        }                                                                            \
        if (!mt_ok) ::minitest::report(__FILE__, __LINE__, "throws " #type ": " #expr); \
    } while (0)
#define FAIL(msg)                                                  \
    do {                                                           \
        ::minitest::report(__FILE__, __LINE__, std::string(msg));  \
        throw ::minitest::Abort{};                                 \
    } while (0)
#define MESSAGE(msg) std::fprintf(stderr, "  note: %s\n", std::string(msg).c_str())
