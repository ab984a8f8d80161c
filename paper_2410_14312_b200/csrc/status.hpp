// Error plumbing shared by the C ABI: every entry point returns an int
// status and leaves a human-readable message in a thread-local slot.
// Status codes mirror the reference's exception taxonomy
// (proj/include/pipesim/errors.hpp:25-65) so the host mirror can re-raise
// the same exception types.
#pragma once

#include <cuda_runtime.h>

#include <stdexcept>
#include <string>

#include "../../include/pipesim_b200.h"

namespace pb {

void set_last_error(const std::string& msg);

struct cuda_failure : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void cuda_check(cudaError_t e, const char* what, const char* file,
                       int line) {
  if (e != cudaSuccess)
    throw cuda_failure(std::string(what) + ": " + cudaGetErrorString(e) +
                       " (" + file + ":" + std::to_string(line) + ")");
}

}  // namespace pb

#define PB_CUDA(x) ::pb::cuda_check((x), #x, __FILE__, __LINE__)
