// Shortest round-trip decimal text of a double, exactly as std::to_chars
// (no format / precision arguments) writes it -- the text the reference
// digests and checkpoints (proj/src/text.cpp:24-28, format_double).
//
// The same code is compiled for the host (tests pin it against
// std::to_chars) and for the device (the GPU digest, digest.cu).
//
// Algorithm: Steele & White / Burger & Dybvig free-format digit generation
// on exact 256-bit integers.  v = r / s with the rounding interval
// [(r - m-) / s, (r + m+) / s] (inclusive: every double here has an even
// significand); scaled by 10^-k so v < 1, digits are generated until the
// remainder falls inside the interval; the last digit is the closer of d and
// d + 1 (ties to even).  For v < 1 (every weight this ever formats) s is a
// power of two, so a digit is a shift and a mask -- no bignum division.
// Range: doubles that are exactly representable in fp32 (the masters), i.e.
// binary exponents -201..75; 256 bits then hold every intermediate.  The
// choice between fixed and scientific notation follows [charconv.to.chars]:
// the shorter string, fixed on a tie.
#pragma once

#include <cstdint>
#include <cstring>

#if defined(__CUDACC__)
#define PB_FMT_HD __host__ __device__ __forceinline__
#else
#define PB_FMT_HD inline
#endif

namespace pb {
namespace fmt {

// 10^k, k = 0..48, as four little-endian 64-bit limbs
#if defined(__CUDACC__)
// (global memory: lanes of a warp index different rows, which the constant
// cache would serialise)
__device__ const uint64_t kPow10Dev[49][4] = {
  {0x0000000000000001ull, 0x0000000000000000ull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x000000000000000aull, 0x0000000000000000ull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x0000000000000064ull, 0x0000000000000000ull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x00000000000003e8ull, 0x0000000000000000ull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x0000000000002710ull, 0x0000000000000000ull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x00000000000186a0ull, 0x0000000000000000ull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x00000000000f4240ull, 0x0000000000000000ull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x0000000000989680ull, 0x0000000000000000ull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x0000000005f5e100ull, 0x0000000000000000ull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x000000003b9aca00ull, 0x0000000000000000ull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x00000002540be400ull, 0x0000000000000000ull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x000000174876e800ull, 0x0000000000000000ull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x000000e8d4a51000ull, 0x0000000000000000ull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x000009184e72a000ull, 0x0000000000000000ull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x00005af3107a4000ull, 0x0000000000000000ull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x00038d7ea4c68000ull, 0x0000000000000000ull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x002386f26fc10000ull, 0x0000000000000000ull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x016345785d8a0000ull, 0x0000000000000000ull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x0de0b6b3a7640000ull, 0x0000000000000000ull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x8ac7230489e80000ull, 0x0000000000000000ull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x6bc75e2d63100000ull, 0x0000000000000005ull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x35c9adc5dea00000ull, 0x0000000000000036ull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x19e0c9bab2400000ull, 0x000000000000021eull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x02c7e14af6800000ull, 0x000000000000152dull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x1bcecceda1000000ull, 0x000000000000d3c2ull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x161401484a000000ull, 0x0000000000084595ull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0xdcc80cd2e4000000ull, 0x000000000052b7d2ull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x9fd0803ce8000000ull, 0x00000000033b2e3cull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x3e25026110000000ull, 0x00000000204fce5eull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x6d7217caa0000000ull, 0x00000001431e0faeull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x4674edea40000000ull, 0x0000000c9f2c9cd0ull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0xc0914b2680000000ull, 0x0000007e37be2022ull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x85acef8100000000ull, 0x000004ee2d6d415bull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x38c15b0a00000000ull, 0x0000314dc6448d93ull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x378d8e6400000000ull, 0x0001ed09bead87c0ull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x2b878fe800000000ull, 0x0013426172c74d82ull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0xb34b9f1000000000ull, 0x00c097ce7bc90715ull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x00f436a000000000ull, 0x0785ee10d5da46d9ull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x098a224000000000ull, 0x4b3b4ca85a86c47aull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x5f65568000000000ull, 0xf050fe938943acc4ull, 0x0000000000000002ull, 0x0000000000000000ull},
  {0xb9f5610000000000ull, 0x6329f1c35ca4bfabull, 0x000000000000001dull, 0x0000000000000000ull},
  {0x4395ca0000000000ull, 0xdfa371a19e6f7cb5ull, 0x0000000000000125ull, 0x0000000000000000ull},
  {0xa3d9e40000000000ull, 0xbc627050305adf14ull, 0x0000000000000b7aull, 0x0000000000000000ull},
  {0x6682e80000000000ull, 0x5bd86321e38cb6ceull, 0x00000000000072cbull, 0x0000000000000000ull},
  {0x011d100000000000ull, 0x9673df52e37f2410ull, 0x0000000000047bf1ull, 0x0000000000000000ull},
  {0x0b22a00000000000ull, 0xe086b93ce2f768a0ull, 0x00000000002cd76full, 0x0000000000000000ull},
  {0x6f5a400000000000ull, 0xc5433c60ddaa1640ull, 0x0000000001c06a5eull, 0x0000000000000000ull},
  {0x5986800000000000ull, 0xb4a05bc8a8a4de84ull, 0x00000000118427b3ull, 0x0000000000000000ull},
  {0x7f41000000000000ull, 0x0e4395d69670b12bull, 0x00000000af298d05ull, 0x0000000000000000ull},
};
#endif
static const uint64_t kPow10Host[49][4] = {
  {0x0000000000000001ull, 0x0000000000000000ull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x000000000000000aull, 0x0000000000000000ull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x0000000000000064ull, 0x0000000000000000ull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x00000000000003e8ull, 0x0000000000000000ull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x0000000000002710ull, 0x0000000000000000ull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x00000000000186a0ull, 0x0000000000000000ull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x00000000000f4240ull, 0x0000000000000000ull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x0000000000989680ull, 0x0000000000000000ull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x0000000005f5e100ull, 0x0000000000000000ull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x000000003b9aca00ull, 0x0000000000000000ull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x00000002540be400ull, 0x0000000000000000ull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x000000174876e800ull, 0x0000000000000000ull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x000000e8d4a51000ull, 0x0000000000000000ull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x000009184e72a000ull, 0x0000000000000000ull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x00005af3107a4000ull, 0x0000000000000000ull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x00038d7ea4c68000ull, 0x0000000000000000ull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x002386f26fc10000ull, 0x0000000000000000ull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x016345785d8a0000ull, 0x0000000000000000ull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x0de0b6b3a7640000ull, 0x0000000000000000ull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x8ac7230489e80000ull, 0x0000000000000000ull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x6bc75e2d63100000ull, 0x0000000000000005ull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x35c9adc5dea00000ull, 0x0000000000000036ull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x19e0c9bab2400000ull, 0x000000000000021eull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x02c7e14af6800000ull, 0x000000000000152dull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x1bcecceda1000000ull, 0x000000000000d3c2ull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x161401484a000000ull, 0x0000000000084595ull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0xdcc80cd2e4000000ull, 0x000000000052b7d2ull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x9fd0803ce8000000ull, 0x00000000033b2e3cull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x3e25026110000000ull, 0x00000000204fce5eull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x6d7217caa0000000ull, 0x00000001431e0faeull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x4674edea40000000ull, 0x0000000c9f2c9cd0ull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0xc0914b2680000000ull, 0x0000007e37be2022ull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x85acef8100000000ull, 0x000004ee2d6d415bull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x38c15b0a00000000ull, 0x0000314dc6448d93ull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x378d8e6400000000ull, 0x0001ed09bead87c0ull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x2b878fe800000000ull, 0x0013426172c74d82ull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0xb34b9f1000000000ull, 0x00c097ce7bc90715ull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x00f436a000000000ull, 0x0785ee10d5da46d9ull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x098a224000000000ull, 0x4b3b4ca85a86c47aull, 0x0000000000000000ull, 0x0000000000000000ull},
  {0x5f65568000000000ull, 0xf050fe938943acc4ull, 0x0000000000000002ull, 0x0000000000000000ull},
  {0xb9f5610000000000ull, 0x6329f1c35ca4bfabull, 0x000000000000001dull, 0x0000000000000000ull},
  {0x4395ca0000000000ull, 0xdfa371a19e6f7cb5ull, 0x0000000000000125ull, 0x0000000000000000ull},
  {0xa3d9e40000000000ull, 0xbc627050305adf14ull, 0x0000000000000b7aull, 0x0000000000000000ull},
  {0x6682e80000000000ull, 0x5bd86321e38cb6ceull, 0x00000000000072cbull, 0x0000000000000000ull},
  {0x011d100000000000ull, 0x9673df52e37f2410ull, 0x0000000000047bf1ull, 0x0000000000000000ull},
  {0x0b22a00000000000ull, 0xe086b93ce2f768a0ull, 0x00000000002cd76full, 0x0000000000000000ull},
  {0x6f5a400000000000ull, 0xc5433c60ddaa1640ull, 0x0000000001c06a5eull, 0x0000000000000000ull},
  {0x5986800000000000ull, 0xb4a05bc8a8a4de84ull, 0x00000000118427b3ull, 0x0000000000000000ull},
  {0x7f41000000000000ull, 0x0e4395d69670b12bull, 0x00000000af298d05ull, 0x0000000000000000ull},
};

PB_FMT_HD const uint64_t* pow10_limbs(int k) {
#if defined(__CUDA_ARCH__)
  return kPow10Dev[k];
#else
  return kPow10Host[k];
#endif
}

struct U256 {
  uint64_t w[4];
};

PB_FMT_HD void u_set(U256& a, uint64_t v) {
  a.w[0] = v;
  a.w[1] = a.w[2] = a.w[3] = 0;
}
PB_FMT_HD void u_load(U256& a, const uint64_t* p) {
  a.w[0] = p[0]; a.w[1] = p[1]; a.w[2] = p[2]; a.w[3] = p[3];
}
PB_FMT_HD uint64_t mulhi64(uint64_t a, uint64_t b) {
#if defined(__CUDA_ARCH__)
  return __umul64hi(a, b);
#else
  return static_cast<uint64_t>((static_cast<unsigned __int128>(a) * b) >> 64);
#endif
}
// a *= m (m < 2^64), truncated to 256 bits
PB_FMT_HD void u_mul_small(U256& a, uint64_t m) {
  uint64_t carry = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint64_t lo = a.w[i] * m;
    const uint64_t hi = mulhi64(a.w[i], m);
    const uint64_t t = lo + carry;
    carry = hi + (t < lo);
    a.w[i] = t;
  }
}
// a *= b where a < 2^64 on entry (a 64 x 256 product, truncated)
PB_FMT_HD void u_mul_u64_by(U256& a, const uint64_t* b) {
  const uint64_t x = a.w[0];
  uint64_t carry = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint64_t lo = x * b[i];
    const uint64_t hi = mulhi64(x, b[i]);
    const uint64_t t = lo + carry;
    carry = hi + (t < lo);
    a.w[i] = t;
  }
}
PB_FMT_HD void u_add(U256& a, const U256& b) {
  uint64_t c = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint64_t t = a.w[i] + b.w[i];
    const uint64_t c1 = t < a.w[i];
    a.w[i] = t + c;
    c = c1 | (a.w[i] < t);
  }
}
PB_FMT_HD void u_sub(U256& a, const U256& b) {  // a >= b
  uint64_t br = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint64_t t = a.w[i] - b.w[i];
    const uint64_t b1 = a.w[i] < b.w[i];
    a.w[i] = t - br;
    br = b1 | (t < br);
  }
}
PB_FMT_HD int u_cmp(const U256& a, const U256& b) {
#pragma unroll
  for (int i = 3; i >= 0; --i)
    if (a.w[i] != b.w[i]) return a.w[i] < b.w[i] ? -1 : 1;
  return 0;
}
PB_FMT_HD void u_pow2(U256& a, int s) {  // 2^s, 0 <= s < 256
  a.w[0] = a.w[1] = a.w[2] = a.w[3] = 0;
  a.w[s >> 6] = uint64_t{1} << (s & 63);
}
PB_FMT_HD void u_shl(U256& a, int s) {  // 0 <= s < 256
  const int q = s >> 6, b = s & 63;
#pragma unroll
  for (int i = 3; i >= 0; --i) {
    uint64_t v = i - q >= 0 ? a.w[i - q] << b : 0;
    if (b && i - q - 1 >= 0) v |= a.w[i - q - 1] >> (64 - b);
    a.w[i] = v;
  }
}
// (a >> s) for a result known to fit in 64 bits; a &= 2^s - 1
PB_FMT_HD uint64_t u_split(U256& a, int s) {
  const int q = s >> 6, b = s & 63;
  uint64_t hi = 0;
  if (q < 4) hi = a.w[q] >> b;
  if (b && q + 1 < 4) hi |= a.w[q + 1] << (64 - b);
  // mask
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if (i > q) a.w[i] = 0;
    else if (i == q) a.w[i] &= b ? ((uint64_t{1} << b) - 1) : 0;
  }
  return hi;
}

// Writes the text of v (fp32-exact double) to out; returns its length
// (at most 24 characters: "-1.2345678901234567e-45").
PB_FMT_HD int format_shortest(double v, char* out) {
  uint64_t bits;
  memcpy(&bits, &v, 8);
  int n = 0;
  if (bits >> 63) out[n++] = '-';
  const uint64_t frac = bits & ((uint64_t{1} << 52) - 1);
  const int eraw = static_cast<int>((bits >> 52) & 0x7FF);
  if (eraw == 0 && frac == 0) {
    out[n++] = '0';
    return n;
  }
  const uint64_t f = eraw ? (frac | (uint64_t{1} << 52)) : frac;
  const int e = eraw ? eraw - 1075 : -1074;
  const bool even = (f & 1) == 0;        // inclusive interval ends
  const bool lower_half = frac == 0 && eraw > 1;  // gap below is half the gap above
  // v = r / s; interval [(r - mm) / s, (r + mp) / s]
  U256 r, s, mp, mm;
  int sh = -1;  // s == 2^sh when >= 0
  if (e >= 0) {
    u_set(r, f);
    u_shl(r, e + (lower_half ? 2 : 1));
    u_set(s, lower_half ? 4 : 2);
    u_pow2(mp, e + (lower_half ? 1 : 0));
    u_pow2(mm, e);
  } else {
    u_set(r, f << (lower_half ? 2 : 1));
    sh = (lower_half ? 2 : 1) - e;
    u_pow2(s, sh);
    u_set(mp, lower_half ? 2 : 1);
    u_set(mm, 1);
  }
  // k: smallest with high bound <= 10^k (< when exclusive); estimate from
  // log10, never too large, fixed up by one step
  double lg = 0.0;
  {
    // log10(v) from the exponent and the leading bits (|error| < 1e-9)
    const double m = static_cast<double>(f) / 4503599627370496.0;  // f / 2^52
    lg = (e + 52) * 0.30102999566398119521 + log10(m);
  }
  int k = static_cast<int>(ceil(lg - 1e-9));
  U256 r0 = r, mp0 = mp, mm0 = mm, s0 = s;
  for (int pass = 0; pass < 3; ++pass) {
    r = r0; mp = mp0; mm = mm0; s = s0;
    if (k >= 0) {
      U256 p;
      u_load(p, pow10_limbs(k));
      // s * 10^k: s is a power of two or small
      if (sh >= 0) {
        U256 t = p;
        u_shl(t, sh);
        s = t;
      } else {
        const uint64_t sv = s.w[0];
        s = p;
        u_mul_small(s, sv);
      }
      if (k > 0) sh = -1;
    } else {
      const uint64_t* p = pow10_limbs(-k);
      // r, mp, mm are < 2^64 here (f << 2 < 2^55, mp/mm <= 2)
      u_mul_u64_by(r, p);
      u_mul_u64_by(mp, p);
      u_mul_u64_by(mm, p);
    }
    U256 hi = r;
    u_add(hi, mp);
    const int c = u_cmp(hi, s);
    if (even ? c >= 0 : c > 0) {
      ++k;
      if (e < 0) sh = (lower_half ? 2 : 1) - e;
      continue;
    }
    break;
  }
  char dig[20];
  int nd = 0;
  int X = k - 1;  // scientific exponent: v = d1.d2..dn x 10^X
  if (sh >= 0) {
    // Fast path (s = 2^sh, v < 1): the 18-digit truncations of v and of both
    // interval ends, exact, in one multiply-shift each (the interval is >= 16
    // units wide at 18 digits, so at least one digit is always dropped and
    // `last` is a real digit of v); then drop digits
    // while the ends still differ above them (Ryu's removal loop, with the
    // exactness flags from the shifted-out bits) and round the last kept
    // digit of v half to even.
    auto scaled = [&](const U256& x, bool* exact) {
      // floor(x * 10^18 / 2^sh) (< 10^18: x / s < 1), *exact = no remainder
      uint64_t p[5];
      uint64_t carry = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint64_t m = 1000000000000000000ull;
        const uint64_t lo = x.w[i] * m, hi = mulhi64(x.w[i], m);
        const uint64_t t = lo + carry;
        carry = hi + (t < lo);
        p[i] = t;
      }
      p[4] = carry;
      const int q = sh >> 6, bsh = sh & 63;
      uint64_t rem = 0;
      for (int i = 0; i < q; ++i) rem |= p[i];
      if (bsh) rem |= p[q] & ((uint64_t{1} << bsh) - 1);
      *exact = rem == 0;
      uint64_t v0 = p[q] >> bsh;
      if (bsh && q + 1 < 5) v0 |= p[q + 1] << (64 - bsh);
      return v0;
    };
    U256 up = r, dn = r;
    u_add(up, mp);
    u_sub(dn, mm);
    bool vr_ex, vp_ex, vm_ex;
    uint64_t vr = scaled(r, &vr_ex), vp = scaled(up, &vp_ex), vm = scaled(dn, &vm_ex);
    // inclusive ends (even significand): the upper end counts as it is;
    // the lower end only if exactly representable at the kept length
    bool vm_tz = vm_ex, vr_tz = vr_ex;
    int removed = 0;
    uint32_t last = 0;
    (void)vp_ex;
    for (;;) {
      const uint64_t vp10 = vp / 10, vm10 = vm / 10;
      if (vp10 <= vm10) break;
      const uint64_t vr10 = vr / 10;
      vm_tz &= (vm - 10 * vm10) == 0;
      vr_tz &= last == 0;
      last = static_cast<uint32_t>(vr - 10 * vr10);
      vr = vr10; vp = vp10; vm = vm10;
      ++removed;
    }
    if (vm_tz) {
      for (;;) {
        const uint64_t vm10 = vm / 10;
        if (vm - 10 * vm10 != 0) break;
        const uint64_t vr10 = vr / 10;
        vr_tz &= last == 0;
        last = static_cast<uint32_t>(vr - 10 * vr10);
        vr = vr10; vp /= 10; vm = vm10;
        ++removed;
      }
    }
    if (vr_tz && last == 5 && (vr & 1) == 0) last = 4;  // exactly ..50..0: to even
    const uint64_t out_digits = vr + ((vr == vm && !(even && vm_tz)) || last >= 5);
    // digits of out_digits, most significant first
    char tmp[20];
    int nt = 0;
    for (uint64_t q = out_digits; q; q /= 10) tmp[nt++] = static_cast<char>('0' + q % 10);
    if (nt == 0) tmp[nt++] = '0';
    while (nt) dig[nd++] = tmp[--nt];
    X = (k - 18) + removed + nd - 1;
  } else {
    for (;;) {
      u_mul_small(r, 10);
      u_mul_small(mp, 10);
      u_mul_small(mm, 10);
      int d;
      if (sh >= 0) {
        d = static_cast<int>(u_split(r, sh));
      } else {
        d = 0;
        while (u_cmp(r, s) >= 0) {
          u_sub(r, s);
          ++d;
        }
      }
      const int cl = u_cmp(r, mm);
      const bool tc1 = even ? cl <= 0 : cl < 0;
      U256 hi = r;
      u_add(hi, mp);
      const int ch = u_cmp(hi, s);
      const bool tc2 = even ? ch >= 0 : ch > 0;
      if (!tc1 && !tc2) {
        dig[nd++] = static_cast<char>('0' + d);
        if (nd >= 19) break;  // unreachable for doubles (<= 17 digits)
        continue;
      }
      if (tc1 && tc2) {
        U256 r2 = r;
        u_add(r2, r);
        const int c2 = u_cmp(r2, s);
        if (c2 > 0 || (c2 == 0 && (d & 1))) ++d;
      } else if (tc2) {
        ++d;
      }
      dig[nd++] = static_cast<char>('0' + d);
      break;
    }
  }
  // notation: v = d1.d2..dn x 10^X
  const int ax = X < 0 ? -X : X;
  const int sci_len = nd + (nd > 1 ? 1 : 0) + 2 + (ax >= 100 ? 3 : 2);
  int fix_len;
  if (X >= 0)
    fix_len = nd <= X + 1 ? X + 1 : nd + 1;
  else
    fix_len = nd + 1 - X;
  if (fix_len <= sci_len) {
    if (X >= 0) {
      if (nd < X + 1) {
        // the shortest digits would need trailing zeros: then v is an integer
        // (its rounding interval holds a representable integer, so it is
        // that double), and its exact digits (same length, zero difference)
        // are the representation [charconv.to.chars] selects
        U256 q;
        u_set(q, e >= 0 ? f : f >> -e);
        if (e > 0) u_shl(q, e);
        char tmp[48];
        int nt = 0;
        while (q.w[0] | q.w[1] | q.w[2] | q.w[3]) {
          // q /= 10 (limb-wise long division, remainder -> digit)
          uint64_t rem = 0;
          for (int i = 3; i >= 0; --i) {
            const unsigned __int128 cur = (static_cast<unsigned __int128>(rem) << 64) | q.w[i];
            q.w[i] = static_cast<uint64_t>(cur / 10);
            rem = static_cast<uint64_t>(cur % 10);
          }
          tmp[nt++] = static_cast<char>('0' + rem);
        }
        while (nt) out[n++] = tmp[--nt];
      } else if (nd == X + 1) {
        for (int i = 0; i < nd; ++i) out[n++] = dig[i];
      } else {
        for (int i = 0; i <= X; ++i) out[n++] = dig[i];
        out[n++] = '.';
        for (int i = X + 1; i < nd; ++i) out[n++] = dig[i];
      }
    } else {
      out[n++] = '0';
      out[n++] = '.';
      for (int i = 0; i < -X - 1; ++i) out[n++] = '0';
      for (int i = 0; i < nd; ++i) out[n++] = dig[i];
    }
  } else {
    out[n++] = dig[0];
    if (nd > 1) {
      out[n++] = '.';
      for (int i = 1; i < nd; ++i) out[n++] = dig[i];
    }
    out[n++] = 'e';
    out[n++] = X < 0 ? '-' : '+';
    if (ax >= 100) out[n++] = static_cast<char>('0' + ax / 100);
    out[n++] = static_cast<char>('0' + (ax / 10) % 10);
    out[n++] = static_cast<char>('0' + ax % 10);
  }
  return n;
}

}  // namespace fmt
}  // namespace pb
