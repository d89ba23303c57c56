// hybridsim/errors.hpp — the reference's exception types (errors.hpp:9-21)
// for C++ callers of libhybridcache_b200.so, plus the status -> exception
// bridge every wrapper in this header tree uses.
//
// Drop-in header tree: a reference caller built against
// /root/reference/proj/include compiles unchanged against this directory and
// links -lhybridcache_b200 instead of the reference library.
#pragma once
#include <stdexcept>
#include <string>

#include "hybridcache.h"

namespace hybridsim {

struct InputError : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct CapacityError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct ConfigError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

namespace b200 {
// C-ABI status (hybridcache.h: 1 InputError, 2 CapacityError, 3 ConfigError,
// 4 CUDA / runtime) -> the reference's exception, message from hc_last_error()
inline void check(int status) {
    if (status == 0) return;
    const std::string msg = hc_last_error();
    switch (status) {
        case 1: throw InputError(msg);
        case 2: throw CapacityError(msg);
        case 3: throw ConfigError(msg);
        default: throw std::runtime_error(msg);
    }
}
}  // namespace b200

}  // namespace hybridsim
