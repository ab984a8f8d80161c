// Exhaustive host check of format_shortest_fast (csrc/ryu_f32d.cuh, the code
// the device digest runs) against std::to_chars over every finite fp32 bit
// pattern widened to double, on all host threads (~3 min on 8 cores):
//   g++ -O2 -std=c++20 -pthread -Ipaper_2410_14312_b200/csrc tests/cpp/shortest_fast_exhaustive.cpp
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>
#include <atomic>
#include "ryu_f32d.cuh"
int main() {
  const int T = std::thread::hardware_concurrency();
  std::atomic<long> bad{0}, checked{0};
  std::vector<std::thread> th;
  for (int t = 0; t < T; ++t)
    th.emplace_back([&, t] {
      long lb = 0, lc = 0;
      for (uint64_t u = t; u < (uint64_t{1} << 32); u += T) {
        uint32_t b = static_cast<uint32_t>(u);
        float x;
        memcpy(&x, &b, 4);
        if (!std::isfinite(x)) continue;
        double v = x;
        char ref[64];
        auto r = std::to_chars(ref, ref + 64, v);
        int lr = r.ptr - ref;
        uint64_t w[4];
        int lf = pb::fmt::format_shortest_fast(v, w);
        ++lc;
        if (lf != lr || memcmp(w, ref, lf)) {
          if (lb++ < 5) printf("MISMATCH %08x %.17g: got '%.*s' want '%.*s'\n", b, v, lf, (const char*)w, lr, ref);
        }
      }
      bad += lb;
      checked += lc;
    });
  for (auto& x : th) x.join();
  printf("exhaustive fast formatter: %ld finite floats, %ld mismatches\n", checked.load(), bad.load());
  return bad != 0;
}
