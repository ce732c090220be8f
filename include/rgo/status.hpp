// rgo/status.hpp -- maps C-ABI status codes back to the exception types the
// reference API throws (std::invalid_argument for validation,
// std::runtime_error for I/O and device failures).
#pragma once

#include <stdexcept>
#include <string>

#include "rgo/capi.h"

namespace rgo::detail {

inline void check(int rc) {
    if (rc == RGO_OK) return;
    const std::string msg = rgo_last_error();
    if (rc == RGO_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

}  // namespace rgo::detail
