// Internal umbrella header for the host-side implementation.
#pragma once

#include <stdexcept>

#include "../../include/pipesim/pipesim_b200.hpp"

namespace pb {
// Caller-provided output buffer is too small (C ABI: PB_ERR_CAPACITY).
struct capacity_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
}  // namespace pb
