// Host-side plumbing shared by the C ABI implementation: status codes
// carried by C++ exceptions inside the library and converted exactly once at
// the extern "C" boundary (include/dimg.h).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>

#include "dimg.h"

namespace dimg {

// Thrown inside the library; caught by DIMG_API_GUARD at the C boundary.
struct Error : std::runtime_error {
    dimg_status code;
    int parse_kind;
    Error(dimg_status c, const std::string& what, int pk = -1)
        : std::runtime_error(what), code(c), parse_kind(pk) {}
};

[[noreturn]] inline void fail(dimg_status c, const std::string& what) { throw Error(c, what); }
[[noreturn]] inline void fail_parse(dimg_parse_kind k, const std::string& what) {
    throw Error(DIMG_EPARSE, what, int(k));
}

void set_last_error(dimg_status code, const char* msg, int parse_kind = -1);

constexpr int64_t kOne = int64_t(1) << 16;  // Q16 unit (proj/include/dim/q16.hpp:21)

}  // namespace dimg

#define DIMG_API_GUARD(...)                                              \
    try {                                                                \
        __VA_ARGS__;                                                     \
        ::dimg::set_last_error(DIMG_OK, "");                             \
        return DIMG_OK;                                                  \
    } catch (const ::dimg::Error& e) {                                   \
        ::dimg::set_last_error(e.code, e.what(), e.parse_kind);          \
        return e.code;                                                   \
    } catch (const std::bad_alloc&) {                                    \
        ::dimg::set_last_error(DIMG_ENOMEM, "host allocation failed");   \
        return DIMG_ENOMEM;                                              \
    } catch (const std::exception& e) {                                  \
        ::dimg::set_last_error(DIMG_EINVAL, e.what());                   \
        return DIMG_EINVAL;                                              \
    }
