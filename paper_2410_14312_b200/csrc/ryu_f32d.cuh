// Fast shortest round-trip text of a double that holds an fp32 value -- the
// same text as format_shortest (shortest.cuh) and std::to_chars, computed
// with Ryu's digit generation (Adams, PLDI 2018: the interval ends scaled by
// a 128-bit power of five, the removal loop over them) instead of 256-bit
// integer arithmetic, and with the text assembled in registers (no local
// memory).  The device digest formats every parameter with it; the rare
// fixed-notation integers with padded digits fall back to format_shortest.
// Pinned against format_shortest (itself exhaustively checked against
// std::to_chars) over every finite fp32 bit pattern: tools/shortest_fast_check.cu.
#pragma once

#include <cstdint>
#include <cstring>

#include "shortest.cuh"

namespace pb {
namespace fmt {

// Ryu's tables for the exponent range of fp32 values held in doubles:
// kRyuPow5InvSplit[q] = floor(2^(pow5bits(q) - 1 + 125) / 5^q) + 1,
// kRyuPow5Split[i] = 5^i scaled to 125 significant bits (128-bit, lo, hi).
#if defined(__CUDACC__)
__device__ const uint64_t kRyuPow5InvSplitDev[32][2] = {
  {0x0000000000000001ull, 0x2000000000000000ull},
  {0x999999999999999aull, 0x1999999999999999ull},
  {0x47ae147ae147ae15ull, 0x147ae147ae147ae1ull},
  {0x6c8b4395810624deull, 0x10624dd2f1a9fbe7ull},
  {0x7a786c226809d496ull, 0x1a36e2eb1c432ca5ull},
  {0x61f9f01b866e43abull, 0x14f8b588e368f084ull},
  {0xb4c7f34938583622ull, 0x10c6f7a0b5ed8d36ull},
  {0x87a6520ec08d236aull, 0x1ad7f29abcaf4857ull},
  {0x9fb841a566d74f88ull, 0x15798ee2308c39dfull},
  {0xe62d01511f12a607ull, 0x112e0be826d694b2ull},
  {0xd6ae6881cb5109a4ull, 0x1b7cdfd9d7bdbab7ull},
  {0xdef1ed34a2a73aeaull, 0x15fd7fe17964955full},
  {0x7f27f0f6e885c8bbull, 0x119799812dea1119ull},
  {0x650cb4be40d60df8ull, 0x1c25c268497681c2ull},
  {0xea70909833de7193ull, 0x16849b86a12b9b01ull},
  {0x21f3a6e0297ec143ull, 0x1203af9ee756159bull},
  {0x6985d7cd0f313537ull, 0x1cd2b297d889bc2bull},
  {0x2137dfd73f5a90f9ull, 0x170ef54646d49689ull},
  {0xe75fe645cc4873faull, 0x12725dd1d243aba0ull},
  {0xa5663d3c7a0d865dull, 0x1d83c94fb6d2ac34ull},
  {0x511e976394d79eb1ull, 0x179ca10c9242235dull},
  {0xda7edf82dd794bc1ull, 0x12e3b40a0e9b4f7dull},
  {0x2a6498d1625bac68ull, 0x1e392010175ee596ull},
  {0xeeb6e0a781e2f053ull, 0x182db34012b25144ull},
  {0x58924d52ce4f26a9ull, 0x1357c299a88ea76aull},
  {0x27507bb7b07ea441ull, 0x1ef2d0f5da7dd8aaull},
  {0x52a6c95fc0655034ull, 0x18c240c4aecb13bbull},
  {0x0eebd44c99eaa690ull, 0x13ce9a36f23c0fc9ull},
  {0xb17953adc3110a80ull, 0x1fb0f6be50601941ull},
  {0xc12ddc8b02740867ull, 0x195a5efea6b34767ull},
  {0x3424b06f3529a052ull, 0x14484bfeebc29f86ull},
  {0x901d59f290ee19dbull, 0x1039d66589687f9eull},
};
__device__ const uint64_t kRyuPow5SplitDev[80][2] = {
  {0x0000000000000000ull, 0x1000000000000000ull},
  {0x0000000000000000ull, 0x1400000000000000ull},
  {0x0000000000000000ull, 0x1900000000000000ull},
  {0x0000000000000000ull, 0x1f40000000000000ull},
  {0x0000000000000000ull, 0x1388000000000000ull},
  {0x0000000000000000ull, 0x186a000000000000ull},
  {0x0000000000000000ull, 0x1e84800000000000ull},
  {0x0000000000000000ull, 0x1312d00000000000ull},
  {0x0000000000000000ull, 0x17d7840000000000ull},
  {0x0000000000000000ull, 0x1dcd650000000000ull},
  {0x0000000000000000ull, 0x12a05f2000000000ull},
  {0x0000000000000000ull, 0x174876e800000000ull},
  {0x0000000000000000ull, 0x1d1a94a200000000ull},
  {0x0000000000000000ull, 0x12309ce540000000ull},
  {0x0000000000000000ull, 0x16bcc41e90000000ull},
  {0x0000000000000000ull, 0x1c6bf52634000000ull},
  {0x0000000000000000ull, 0x11c37937e0800000ull},
  {0x0000000000000000ull, 0x16345785d8a00000ull},
  {0x0000000000000000ull, 0x1bc16d674ec80000ull},
  {0x0000000000000000ull, 0x1158e460913d0000ull},
  {0x0000000000000000ull, 0x15af1d78b58c4000ull},
  {0x0000000000000000ull, 0x1b1ae4d6e2ef5000ull},
  {0x0000000000000000ull, 0x10f0cf064dd59200ull},
  {0x0000000000000000ull, 0x152d02c7e14af680ull},
  {0x0000000000000000ull, 0x1a784379d99db420ull},
  {0x0000000000000000ull, 0x108b2a2c28029094ull},
  {0x0000000000000000ull, 0x14adf4b7320334b9ull},
  {0x4000000000000000ull, 0x19d971e4fe8401e7ull},
  {0x8800000000000000ull, 0x1027e72f1f128130ull},
  {0xaa00000000000000ull, 0x1431e0fae6d7217cull},
  {0xd480000000000000ull, 0x193e5939a08ce9dbull},
  {0xc9a0000000000000ull, 0x1f8def8808b02452ull},
  {0xbe04000000000000ull, 0x13b8b5b5056e16b3ull},
  {0xad85000000000000ull, 0x18a6e32246c99c60ull},
  {0xd8e6400000000000ull, 0x1ed09bead87c0378ull},
  {0x878fe80000000000ull, 0x13426172c74d822bull},
  {0x6973e20000000000ull, 0x1812f9cf7920e2b6ull},
  {0x03d0da8000000000ull, 0x1e17b84357691b64ull},
  {0x8262889000000000ull, 0x12ced32a16a1b11eull},
  {0x22fb2ab400000000ull, 0x178287f49c4a1d66ull},
  {0xabb9f56100000000ull, 0x1d6329f1c35ca4bfull},
  {0xcb54395ca0000000ull, 0x125dfa371a19e6f7ull},
  {0xbe2947b3c8000000ull, 0x16f578c4e0a060b5ull},
  {0x2db399a0ba000000ull, 0x1cb2d6f618c878e3ull},
  {0xfc90400474400000ull, 0x11efc659cf7d4b8dull},
  {0x7bb4500591500000ull, 0x166bb7f0435c9e71ull},
  {0xdaa16406f5a40000ull, 0x1c06a5ec5433c60dull},
  {0xa8a4de8459868000ull, 0x118427b3b4a05bc8ull},
  {0xd2ce16256fe82000ull, 0x15e531a0a1c872baull},
  {0x87819baecbe22800ull, 0x1b5e7e08ca3a8f69ull},
  {0xf4b1014d3f6d5900ull, 0x111b0ec57e6499a1ull},
  {0x71dd41a08f48af40ull, 0x1561d276ddfdc00aull},
  {0x0e549208b31adb10ull, 0x1aba4714957d300dull},
  {0x28f4db456ff0c8eaull, 0x10b46c6cdd6e3e08ull},
  {0x33321216cbecfb24ull, 0x14e1878814c9cd8aull},
  {0xbffe969c7ee839edull, 0x1a19e96a19fc40ecull},
  {0xf7ff1e21cf512434ull, 0x105031e2503da893ull},
  {0xf5fee5aa43256d41ull, 0x14643e5ae44d12b8ull},
  {0x337e9f14d3eec892ull, 0x197d4df19d605767ull},
  {0x005e46da08ea7ab6ull, 0x1fdca16e04b86d41ull},
  {0xa03aec4845928cb2ull, 0x13e9e4e4c2f34448ull},
  {0xc849a75a56f72fdeull, 0x18e45e1df3b0155aull},
  {0x7a5c1130ecb4fbd6ull, 0x1f1d75a5709c1ab1ull},
  {0xec798abe93f11d65ull, 0x13726987666190aeull},
  {0xa797ed6e38ed64bfull, 0x184f03e93ff9f4daull},
  {0x517de8c9c728bdefull, 0x1e62c4e38ff87211ull},
  {0xd2eeb17e1c7976b5ull, 0x12fdbb0e39fb474aull},
  {0x87aa5ddda397d462ull, 0x17bd29d1c87a191dull},
  {0xe994f5550c7dc97bull, 0x1dac74463a989f64ull},
  {0x11fd195527ce9dedull, 0x128bc8abe49f639full},
  {0xd67c5faa71c24568ull, 0x172ebad6ddc73c86ull},
  {0x8c1b77950e32d6c2ull, 0x1cfa698c95390ba8ull},
  {0x57912abd28dfc639ull, 0x121c81f7dd43a749ull},
  {0xad75756c7317b7c8ull, 0x16a3a275d494911bull},
  {0x98d2d2c78fdda5baull, 0x1c4c8b1349b9b562ull},
  {0x9f83c3bcb9ea8794ull, 0x11afd6ec0e14115dull},
  {0x0764b4abe8652979ull, 0x161bcca7119915b5ull},
  {0x493de1d6e27e73d7ull, 0x1ba2bfd0d5ff5b22ull},
  {0x6dc6ad264d8f0866ull, 0x1145b7e285bf98f5ull},
  {0xc938586fe0f2ca80ull, 0x159725db272f7f32ull},
};
#endif
static const uint64_t kRyuPow5InvSplitHost[32][2] = {
  {0x0000000000000001ull, 0x2000000000000000ull},
  {0x999999999999999aull, 0x1999999999999999ull},
  {0x47ae147ae147ae15ull, 0x147ae147ae147ae1ull},
  {0x6c8b4395810624deull, 0x10624dd2f1a9fbe7ull},
  {0x7a786c226809d496ull, 0x1a36e2eb1c432ca5ull},
  {0x61f9f01b866e43abull, 0x14f8b588e368f084ull},
  {0xb4c7f34938583622ull, 0x10c6f7a0b5ed8d36ull},
  {0x87a6520ec08d236aull, 0x1ad7f29abcaf4857ull},
  {0x9fb841a566d74f88ull, 0x15798ee2308c39dfull},
  {0xe62d01511f12a607ull, 0x112e0be826d694b2ull},
  {0xd6ae6881cb5109a4ull, 0x1b7cdfd9d7bdbab7ull},
  {0xdef1ed34a2a73aeaull, 0x15fd7fe17964955full},
  {0x7f27f0f6e885c8bbull, 0x119799812dea1119ull},
  {0x650cb4be40d60df8ull, 0x1c25c268497681c2ull},
  {0xea70909833de7193ull, 0x16849b86a12b9b01ull},
  {0x21f3a6e0297ec143ull, 0x1203af9ee756159bull},
  {0x6985d7cd0f313537ull, 0x1cd2b297d889bc2bull},
  {0x2137dfd73f5a90f9ull, 0x170ef54646d49689ull},
  {0xe75fe645cc4873faull, 0x12725dd1d243aba0ull},
  {0xa5663d3c7a0d865dull, 0x1d83c94fb6d2ac34ull},
  {0x511e976394d79eb1ull, 0x179ca10c9242235dull},
  {0xda7edf82dd794bc1ull, 0x12e3b40a0e9b4f7dull},
  {0x2a6498d1625bac68ull, 0x1e392010175ee596ull},
  {0xeeb6e0a781e2f053ull, 0x182db34012b25144ull},
  {0x58924d52ce4f26a9ull, 0x1357c299a88ea76aull},
  {0x27507bb7b07ea441ull, 0x1ef2d0f5da7dd8aaull},
  {0x52a6c95fc0655034ull, 0x18c240c4aecb13bbull},
  {0x0eebd44c99eaa690ull, 0x13ce9a36f23c0fc9ull},
  {0xb17953adc3110a80ull, 0x1fb0f6be50601941ull},
  {0xc12ddc8b02740867ull, 0x195a5efea6b34767ull},
  {0x3424b06f3529a052ull, 0x14484bfeebc29f86ull},
  {0x901d59f290ee19dbull, 0x1039d66589687f9eull},
};
static const uint64_t kRyuPow5SplitHost[80][2] = {
  {0x0000000000000000ull, 0x1000000000000000ull},
  {0x0000000000000000ull, 0x1400000000000000ull},
  {0x0000000000000000ull, 0x1900000000000000ull},
  {0x0000000000000000ull, 0x1f40000000000000ull},
  {0x0000000000000000ull, 0x1388000000000000ull},
  {0x0000000000000000ull, 0x186a000000000000ull},
  {0x0000000000000000ull, 0x1e84800000000000ull},
  {0x0000000000000000ull, 0x1312d00000000000ull},
  {0x0000000000000000ull, 0x17d7840000000000ull},
  {0x0000000000000000ull, 0x1dcd650000000000ull},
  {0x0000000000000000ull, 0x12a05f2000000000ull},
  {0x0000000000000000ull, 0x174876e800000000ull},
  {0x0000000000000000ull, 0x1d1a94a200000000ull},
  {0x0000000000000000ull, 0x12309ce540000000ull},
  {0x0000000000000000ull, 0x16bcc41e90000000ull},
  {0x0000000000000000ull, 0x1c6bf52634000000ull},
  {0x0000000000000000ull, 0x11c37937e0800000ull},
  {0x0000000000000000ull, 0x16345785d8a00000ull},
  {0x0000000000000000ull, 0x1bc16d674ec80000ull},
  {0x0000000000000000ull, 0x1158e460913d0000ull},
  {0x0000000000000000ull, 0x15af1d78b58c4000ull},
  {0x0000000000000000ull, 0x1b1ae4d6e2ef5000ull},
  {0x0000000000000000ull, 0x10f0cf064dd59200ull},
  {0x0000000000000000ull, 0x152d02c7e14af680ull},
  {0x0000000000000000ull, 0x1a784379d99db420ull},
  {0x0000000000000000ull, 0x108b2a2c28029094ull},
  {0x0000000000000000ull, 0x14adf4b7320334b9ull},
  {0x4000000000000000ull, 0x19d971e4fe8401e7ull},
  {0x8800000000000000ull, 0x1027e72f1f128130ull},
  {0xaa00000000000000ull, 0x1431e0fae6d7217cull},
  {0xd480000000000000ull, 0x193e5939a08ce9dbull},
  {0xc9a0000000000000ull, 0x1f8def8808b02452ull},
  {0xbe04000000000000ull, 0x13b8b5b5056e16b3ull},
  {0xad85000000000000ull, 0x18a6e32246c99c60ull},
  {0xd8e6400000000000ull, 0x1ed09bead87c0378ull},
  {0x878fe80000000000ull, 0x13426172c74d822bull},
  {0x6973e20000000000ull, 0x1812f9cf7920e2b6ull},
  {0x03d0da8000000000ull, 0x1e17b84357691b64ull},
  {0x8262889000000000ull, 0x12ced32a16a1b11eull},
  {0x22fb2ab400000000ull, 0x178287f49c4a1d66ull},
  {0xabb9f56100000000ull, 0x1d6329f1c35ca4bfull},
  {0xcb54395ca0000000ull, 0x125dfa371a19e6f7ull},
  {0xbe2947b3c8000000ull, 0x16f578c4e0a060b5ull},
  {0x2db399a0ba000000ull, 0x1cb2d6f618c878e3ull},
  {0xfc90400474400000ull, 0x11efc659cf7d4b8dull},
  {0x7bb4500591500000ull, 0x166bb7f0435c9e71ull},
  {0xdaa16406f5a40000ull, 0x1c06a5ec5433c60dull},
  {0xa8a4de8459868000ull, 0x118427b3b4a05bc8ull},
  {0xd2ce16256fe82000ull, 0x15e531a0a1c872baull},
  {0x87819baecbe22800ull, 0x1b5e7e08ca3a8f69ull},
  {0xf4b1014d3f6d5900ull, 0x111b0ec57e6499a1ull},
  {0x71dd41a08f48af40ull, 0x1561d276ddfdc00aull},
  {0x0e549208b31adb10ull, 0x1aba4714957d300dull},
  {0x28f4db456ff0c8eaull, 0x10b46c6cdd6e3e08ull},
  {0x33321216cbecfb24ull, 0x14e1878814c9cd8aull},
  {0xbffe969c7ee839edull, 0x1a19e96a19fc40ecull},
  {0xf7ff1e21cf512434ull, 0x105031e2503da893ull},
  {0xf5fee5aa43256d41ull, 0x14643e5ae44d12b8ull},
  {0x337e9f14d3eec892ull, 0x197d4df19d605767ull},
  {0x005e46da08ea7ab6ull, 0x1fdca16e04b86d41ull},
  {0xa03aec4845928cb2ull, 0x13e9e4e4c2f34448ull},
  {0xc849a75a56f72fdeull, 0x18e45e1df3b0155aull},
  {0x7a5c1130ecb4fbd6ull, 0x1f1d75a5709c1ab1ull},
  {0xec798abe93f11d65ull, 0x13726987666190aeull},
  {0xa797ed6e38ed64bfull, 0x184f03e93ff9f4daull},
  {0x517de8c9c728bdefull, 0x1e62c4e38ff87211ull},
  {0xd2eeb17e1c7976b5ull, 0x12fdbb0e39fb474aull},
  {0x87aa5ddda397d462ull, 0x17bd29d1c87a191dull},
  {0xe994f5550c7dc97bull, 0x1dac74463a989f64ull},
  {0x11fd195527ce9dedull, 0x128bc8abe49f639full},
  {0xd67c5faa71c24568ull, 0x172ebad6ddc73c86ull},
  {0x8c1b77950e32d6c2ull, 0x1cfa698c95390ba8ull},
  {0x57912abd28dfc639ull, 0x121c81f7dd43a749ull},
  {0xad75756c7317b7c8ull, 0x16a3a275d494911bull},
  {0x98d2d2c78fdda5baull, 0x1c4c8b1349b9b562ull},
  {0x9f83c3bcb9ea8794ull, 0x11afd6ec0e14115dull},
  {0x0764b4abe8652979ull, 0x161bcca7119915b5ull},
  {0x493de1d6e27e73d7ull, 0x1ba2bfd0d5ff5b22ull},
  {0x6dc6ad264d8f0866ull, 0x1145b7e285bf98f5ull},
  {0xc938586fe0f2ca80ull, 0x159725db272f7f32ull},
};

PB_FMT_HD const uint64_t* ryu_inv(int q) {
#if defined(__CUDA_ARCH__)
  return kRyuPow5InvSplitDev[q];
#else
  return kRyuPow5InvSplitHost[q];
#endif
}
PB_FMT_HD const uint64_t* ryu_pow5(int i) {
#if defined(__CUDA_ARCH__)
  return kRyuPow5SplitDev[i];
#else
  return kRyuPow5SplitHost[i];
#endif
}

PB_FMT_HD int ryu_pow5bits(int e) { return static_cast<int>((static_cast<uint32_t>(e) * 1217359u) >> 19) + 1; }
PB_FMT_HD int ryu_log10pow2(int e) { return static_cast<int>((static_cast<uint32_t>(e) * 78913u) >> 18); }
PB_FMT_HD int ryu_log10pow5(int e) { return static_cast<int>((static_cast<uint32_t>(e) * 732923u) >> 20); }

// (m * mul) >> j for a 128-bit mul, 64 < j < 128
PB_FMT_HD uint64_t ryu_mulshift(uint64_t m, const uint64_t* mul, int j) {
  const unsigned __int128 b0 = static_cast<unsigned __int128>(m) * mul[0];
  const unsigned __int128 b2 = static_cast<unsigned __int128>(m) * mul[1];
  return static_cast<uint64_t>(((b0 >> 64) + b2) >> (j - 64));
}

PB_FMT_HD bool ryu_multiple_of_pow5(uint64_t v, int p) {
  int c = 0;
  while (v != 0 && v % 5 == 0) {
    v /= 5;
    ++c;
  }
  return c >= p;
}

// Shortest digits of a positive finite double (bits): value = *digits * 10^*e10.
PB_FMT_HD void ryu_d2d(uint64_t bits, uint64_t* digits, int* e10out) {
  const uint64_t ieee_m = bits & ((uint64_t{1} << 52) - 1);
  const int ieee_e = static_cast<int>((bits >> 52) & 0x7FF);
  int e2;
  uint64_t m2;
  if (ieee_e == 0) {
    e2 = 1 - 1023 - 52 - 2;
    m2 = ieee_m;
  } else {
    e2 = ieee_e - 1023 - 52 - 2;
    m2 = (uint64_t{1} << 52) | ieee_m;
  }
  const bool accept = (m2 & 1) == 0;
  const uint64_t mv = 4 * m2;
  const uint32_t mm_shift = (ieee_m != 0 || ieee_e <= 1) ? 1 : 0;
  uint64_t vr, vp, vm;
  int e10;
  bool vm_tz = false, vr_tz = false;
  if (e2 >= 0) {
    const int q = ryu_log10pow2(e2) - (e2 > 3 ? 1 : 0);
    e10 = q;
    const int k = 125 + ryu_pow5bits(q) - 1;
    const int i = -e2 + q + k;
    const uint64_t* mul = ryu_inv(q);
    vr = ryu_mulshift(4 * m2, mul, i);
    vp = ryu_mulshift(4 * m2 + 2, mul, i);
    vm = ryu_mulshift(4 * m2 - 1 - mm_shift, mul, i);
    if (q <= 21) {
      if (mv % 5 == 0)
        vr_tz = ryu_multiple_of_pow5(mv, q);
      else if (accept)
        vm_tz = ryu_multiple_of_pow5(mv - 1 - mm_shift, q);
      else
        vp -= ryu_multiple_of_pow5(mv + 2, q) ? 1 : 0;
    }
  } else {
    const int q = ryu_log10pow5(-e2) - (-e2 > 1 ? 1 : 0);
    e10 = q + e2;
    const int i = -e2 - q;
    const int k = ryu_pow5bits(i) - 125;
    const int j = q - k;
    const uint64_t* mul = ryu_pow5(i);
    vr = ryu_mulshift(4 * m2, mul, j);
    vp = ryu_mulshift(4 * m2 + 2, mul, j);
    vm = ryu_mulshift(4 * m2 - 1 - mm_shift, mul, j);
    if (q <= 1) {
      vr_tz = true;
      if (accept)
        vm_tz = mm_shift == 1;
      else
        --vp;
    } else if (q < 63) {
      vr_tz = (mv & ((uint64_t{1} << q) - 1)) == 0;
    }
  }
  int removed = 0;
  uint64_t out;
  if (vm_tz || vr_tz) {
    uint32_t last = 0;
    for (;;) {
      const uint64_t vp10 = vp / 10, vm10 = vm / 10;
      if (vp10 <= vm10) break;
      const uint64_t vr10 = vr / 10;
      vm_tz &= vm - 10 * vm10 == 0;
      vr_tz &= last == 0;
      last = static_cast<uint32_t>(vr - 10 * vr10);
      vr = vr10;
      vp = vp10;
      vm = vm10;
      ++removed;
    }
    if (vm_tz) {
      for (;;) {
        const uint64_t vm10 = vm / 10;
        if (vm - 10 * vm10 != 0) break;
        const uint64_t vp10 = vp / 10, vr10 = vr / 10;
        vr_tz &= last == 0;
        last = static_cast<uint32_t>(vr - 10 * vr10);
        vr = vr10;
        vp = vp10;
        vm = vm10;
        ++removed;
      }
    }
    if (vr_tz && last == 5 && vr % 2 == 0) last = 4;
    out = vr + (((vr == vm && (!accept || !vm_tz)) || last >= 5) ? 1 : 0);
  } else {
    bool round_up = false;
    const uint64_t vp100 = vp / 100, vm100 = vm / 100;
    if (vp100 > vm100) {
      const uint64_t vr100 = vr / 100;
      round_up = vr - 100 * vr100 >= 50;
      vr = vr100;
      vp = vp100;
      vm = vm100;
      removed += 2;
    }
    for (;;) {
      const uint64_t vp10 = vp / 10, vm10 = vm / 10;
      if (vp10 <= vm10) break;
      const uint64_t vr10 = vr / 10;
      round_up = vr - 10 * vr10 >= 5;
      vr = vr10;
      vp = vp10;
      vm = vm10;
      ++removed;
    }
    out = vr + ((vr == vm || round_up) ? 1 : 0);
  }
  *digits = out;
  *e10out = e10 + removed;
}

// the exact-integer path of format_shortest, kept out of line so that its
// 256-bit temporaries do not weigh on the fast path's registers
#if defined(__CUDACC__)
__host__ __device__ __noinline__ inline int format_shortest_slow(double v, char* out) {
  return format_shortest(v, out);
}
#else
inline int format_shortest_slow(double v, char* out) { return format_shortest(v, out); }
#endif

// byte c at position pos of a 32-byte text held in four registers
PB_FMT_HD void text_put(uint64_t (&w)[4], int pos, uint32_t c) {
  const uint64_t v = static_cast<uint64_t>(c & 0xFF) << (8 * (pos & 7));
  switch (pos >> 3) {
    case 0: w[0] |= v; break;
    case 1: w[1] |= v; break;
    case 2: w[2] |= v; break;
    default: w[3] |= v; break;
  }
}

// The text of v (an fp32 value as a double) into w (32 bytes, zero padded);
// returns its length.  Same text as format_shortest.
PB_FMT_HD int format_shortest_fast(double v, uint64_t (&w)[4]) {
  w[0] = w[1] = w[2] = w[3] = 0;
  uint64_t bits;
  memcpy(&bits, &v, 8);
  int n = 0;
  if (bits >> 63) text_put(w, n++, '-');
  bits &= ~(uint64_t{1} << 63);
  if (bits == 0) {
    text_put(w, n++, '0');
    return n;
  }
  uint64_t dg;
  int e10;
  ryu_d2d(bits, &dg, &e10);
  // digit count (dg < 10^17)
  int nd = 1;
  {
    // digit count: 32-bit compares on the high part when it is non-zero
    const uint64_t h = dg / 100000000u;
    uint32_t x = h ? static_cast<uint32_t>(h) : static_cast<uint32_t>(dg);
    nd = h ? 9 : 1;
    while (x >= 10) {
      x /= 10;
      ++nd;
    }
  }
  const int X = e10 + nd - 1;  // v = d1.d2..dn x 10^X
  const int ax = X < 0 ? -X : X;
  const int sci_len = nd + (nd > 1 ? 1 : 0) + 2 + (ax >= 100 ? 3 : 2);
  const int fix_len = X >= 0 ? (nd <= X + 1 ? X + 1 : nd + 1) : nd + 1 - X;
  const bool fixed = fix_len <= sci_len;
  if (fixed && X >= 0 && nd < X + 1) {
    // padded integer digits: the exact integer (rare; the reference path)
    char buf[48];
    const int m = format_shortest_slow(v, buf);
    w[0] = w[1] = w[2] = w[3] = 0;
    for (int i = 0; i < m && i < 32; ++i) text_put(w, i, static_cast<uint8_t>(buf[i]));
    return m;
  }
  // digit i (0-based from the left) goes straight to its final position;
  // the digits come off dg from the right
  auto digit_pos = [&](int i) {
    if (!fixed) return n + (i == 0 ? 0 : i + 1);          // d . ddd
    if (X < 0) return n + 1 - X + i;                      // 0.000ddd
    return n + (i <= X ? i : i + 1);                      // dd.ddd / ddd
  };
  // dg < 10^17: the low 8 digits and the rest as 32-bit numbers (32-bit
  // divisions by 10 are a multiply-high; 64-bit ones are emulated)
  const uint64_t hi64 = dg / 100000000u;
  uint32_t lo = static_cast<uint32_t>(dg - hi64 * 100000000u);
  uint32_t hi = static_cast<uint32_t>(hi64);
  for (int i = nd - 1; i >= 0; --i) {
    uint32_t d;
    if (i >= nd - 8) {
      const uint32_t l10 = lo / 10;
      d = lo - 10 * l10;
      lo = l10;
    } else {
      const uint32_t h10 = hi / 10;
      d = hi - 10 * h10;
      hi = h10;
    }
    text_put(w, digit_pos(i), '0' + d);
  }
  int len;
  if (!fixed) {
    if (nd > 1) text_put(w, n + 1, '.');
    int p = n + nd + (nd > 1 ? 1 : 0);
    text_put(w, p++, 'e');
    text_put(w, p++, X < 0 ? '-' : '+');
    if (ax >= 100) text_put(w, p++, static_cast<uint32_t>('0' + ax / 100));
    text_put(w, p++, static_cast<uint32_t>('0' + (ax / 10) % 10));
    text_put(w, p++, static_cast<uint32_t>('0' + ax % 10));
    len = p;
  } else if (X < 0) {
    text_put(w, n, '0');
    text_put(w, n + 1, '.');
    for (int i = 0; i < -X - 1; ++i) text_put(w, n + 2 + i, '0');
    len = n + 1 - X + nd;
  } else if (nd == X + 1) {
    len = n + nd;
  } else {
    text_put(w, n + X + 1, '.');
    len = n + nd + 1;
  }
  return len;
}

}  // namespace fmt
}  // namespace pb
