// Host check of the shortest round-trip formatter the device digest uses
// (paper_2410_14312_b200/csrc/shortest.cuh) against std::to_chars, the
// reference's format_double (proj/src/text.cpp:24-28): random fp32 bit
// patterns, typical weights, every binade edge, integers and powers of ten.
// Usage: shortest_check [n]; exit status 0 iff no mismatch.
#include <charconv>
#include <cmath>
#include <cstdio>
#include <random>
#include <string>
#include "shortest.cuh"
#include "ryu_f32d.cuh"
int main(int argc, char** argv) {
  long n = argc > 1 ? atol(argv[1]) : 1000000;
  std::mt19937_64 g(1);
  long bad = 0;
  auto check = [&](float x) {
    if (!std::isfinite(x)) return;
    double v = x;
    char a[64], b[64];
    int la = pb::fmt::format_shortest(v, a);
    auto r = std::to_chars(b, b + 64, v);
    int lb = r.ptr - b;
    if (la != lb || memcmp(a, b, la)) {
      if (bad++ < 20) printf("MISMATCH %.17g: got '%.*s' want '%.*s'\n", v, la, a, lb, b);
    }
    uint64_t w[4];
    const int lf = pb::fmt::format_shortest_fast(v, w);
    if (lf != lb || memcmp(w, b, lf)) {
      if (bad++ < 20) printf("FAST MISMATCH %.17g: got '%.*s' want '%.*s'\n", v, lf,
                             reinterpret_cast<const char*>(w), lb, b);
    }
  };
  for (long i = 0; i < n; ++i) { uint32_t u = g(); float x; memcpy(&x, &u, 4); check(x); }
  // typical weights
  std::uniform_real_distribution<float> U(-0.05f, 0.05f);
  for (long i = 0; i < n; ++i) check(U(g));
  // all powers of two / edge exponents, and neighbours
  for (int e = -149; e <= 127; ++e) for (int d = -3; d <= 3; ++d) { float x = std::ldexp(1.0f, e); uint32_t u; memcpy(&u,&x,4); u += d; memcpy(&x,&u,4); check(x); check(-x);}
  for (int i = 0; i < 100000; ++i) { check((float)i); check(i * 0.1f); check(i * 1e-5f); check(std::pow(10.0f, (float)(i % 77 - 40))); }
  printf("checked, %ld mismatches\n", bad);
  return bad != 0;
}
