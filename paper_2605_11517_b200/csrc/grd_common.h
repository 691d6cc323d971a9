// Shared helpers for the grinder_b200 C ABI: thread-local error reporting.
#pragma once

#include <cstdarg>
#include <cstdio>
#include <string>

namespace grd {

// Thread-local message returned by grd_last_error().
std::string& last_error_slot();

inline int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    std::vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    last_error_slot() = buf;
    return code;
}

inline void clear_error() { last_error_slot().clear(); }

constexpr int kErrArg = -1;
constexpr int kErrAlloc = -2;
constexpr int kErrState = -3;

inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

}  // namespace grd
