// The reference's parameter digest on the device (A14: params_digest,
// proj/src/trainer.cpp:599-607; fnv1a64_hex / format_double,
// proj/src/text.cpp:24-52).
//
// The reference formats every parameter as its shortest round-trip decimal,
// appends '\n', and folds the whole text with FNV-1a 64 -- for the
// 268M-parameter benchmark net a 5.6 GB string, 6 s of host time per digest
// even with the formatting spread over threads (the fold is a serial chain).
// Here the text is never materialised as one string and the fold is not
// serial:
//
//   FNV-1a step: h' = (h ^ c) * P  (mod 2^64), P = 0x100000001b3.
//   h ^ c = h + d with d = ((h & 0xFF) ^ c) - (h & 0xFF): the xor only
//   touches the low byte, so the low byte l evolves on its own,
//   l' = ((l ^ c) * 0xB3) mod 256 -- a permutation of 256 states per byte --
//   and given the low-byte trajectory the full state is affine in its start:
//   h_out = c + P^n * h_in.
//   The low nibble of l depends only on itself (l'_lo = 3 * (l ^ c)_lo mod
//   16), and the high nibble is affine in itself given the low nibble
//   (l'_hi = 3 * (l ^ c)_hi + 11 * x_lo + (3 * x_lo >> 4) mod 16).
//
// So each thread formats R values into 32-byte slots and runs its bytes three
// times: (A) the low-nibble map of all 16 starting nibbles at once (SWAR, one
// 64-bit word), (B) the high-nibble map given its now known low-nibble
// trajectory, (C) the exact fold from its known low byte, as an affine map.
// Maps compose in order per block, block maps are chained from the segment's
// known incoming state, and the affine maps reduce to the final hash.  The
// result is bit-identical to the serial fold (tests/test_digest.py).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

namespace pb {

// One run of the flat parameter stream: rows x cols row-major values with
// leading dimension ld, fp32 (f32) or split masters (hi bf16 + lo int16
// residual, bits = hi << 16 + lo).  `start` = index of its first value in the
// stream (spans are consecutive).
struct DigestSpan {
  const float* f32 = nullptr;
  const __nv_bfloat16* hi = nullptr;
  const uint16_t* lo = nullptr;
  int64_t rows = 0, cols = 0, ld = 0;
  int64_t start = 0;
};

constexpr uint64_t kFnvBasis = 1469598103934665603ull;  // the reference's basis (text.cpp:40)

// Scratch shared by every digest issued on one stream (digests on one
// DeviceDigest must be serialised on one stream).
class DeviceDigest {
 public:
  explicit DeviceDigest(int64_t seg_values = int64_t{1} << 22);
  ~DeviceDigest();
  DeviceDigest(const DeviceDigest&) = delete;
  DeviceDigest& operator=(const DeviceDigest&) = delete;

  // A digest plan: the span table in device memory (valid for graph replay).
  struct Plan {
    DigestSpan* d_spans = nullptr;
    int nspans = 0;
    int64_t total = 0;
  };
  Plan make_plan(const std::vector<DigestSpan>& spans);
  void free_plan(Plan& p);
  // Enqueues the digest of the plan's stream on `st`: *d_state = FNV-1a 64 of
  // the text (kernel launches only, graph-capturable).
  void enqueue(const Plan& p, uint64_t* d_state, cudaStream_t st);
  int launches_per(const Plan& p) const;

 private:
  void ensure();
  int64_t seg_;
  int blocks_ = 0;
  char* slots_ = nullptr;
  uint8_t* lens_ = nullptr;
  uint64_t* tmap_ = nullptr;   // per thread: low / high nibble maps
  uint8_t* tlo_ = nullptr;     // per thread: incoming low nibble
  uint64_t* bmap_ = nullptr;   // per block map
  uint8_t* bin_ = nullptr;     // per block incoming nibble
  uint64_t* baff_ = nullptr;   // per block affine map (c, m)
};

std::vector<DigestSpan> digest_spans_contiguous(const float* p, int64_t n);

}  // namespace pb
