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

#include <cstddef>
#include <cstdint>
#include <functional>
#include <string>
#include <vector>

namespace pb {

// A contiguous run of values to format (one stage's params, one version ...).
struct value_span {
  const double* data;
  int64_t n;
};

// Formats every value of `spans` (in order) as its shortest round-trip
// decimal followed by '\n' -- exactly the text the reference builds in
// params_digest / checkpoint_stage (proj/src/trainer.cpp:599-607,
// checkpoint.cpp:39-67) -- and hands the text to `sink` in order, chunk by
// chunk.  Formatting runs on host worker threads; the sink runs on the
// calling thread, overlapped with the formatting of later chunks.
void format_values_ordered(const std::vector<value_span>& spans,
                           const std::function<void(const char*, size_t)>& sink);

// Streaming FNV-1a 64 as the reference computes it (proj/src/text.cpp:39-51).
// Its offset basis is 1469598103934665603 -- the decimal of the standard FNV
// basis 14695981039346656037 with the last digit dropped -- so the digests
// differ from textbook FNV-1a; parity is with the reference's value.  The
// fold is a serial chain of one xor and one 64-bit multiply per byte
// (~4 cycles/byte): the floor of any digest of the reference's format.
struct fnv1a64 {
  uint64_t h = 1469598103934665603ull;
  void update(const char* p, size_t n) {
    uint64_t x = h;
    for (size_t i = 0; i < n; ++i) {
      x ^= static_cast<unsigned char>(p[i]);
      x *= 0x100000001b3ull;
    }
    h = x;
  }
  std::string hex() const;
};

// fnv1a64_hex of the formatted text of `spans`, without materialising it.
std::string digest_spans(const std::vector<value_span>& spans);

}  // namespace pb
