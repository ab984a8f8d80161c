// Parallel formatting of parameter text for the reference's digest and
// checkpoint formats (proj/src/trainer.cpp:599-607, proj/src/text.cpp:24-52,
// proj/src/checkpoint.cpp:39-67).
//
// The reference formats every double with shortest round-trip std::to_chars,
// appends '\n', and folds the whole text with FNV-1a.  Formatting is ~80% of
// that cost and is embarrassingly parallel; the FNV-1a fold is a serial
// dependency chain.  Worker threads format fixed-size chunks into a ring of
// buffers while the calling thread folds (or writes) finished chunks in
// order, so the digest costs max(format / threads, fold) instead of their sum.
#include <algorithm>
#include <atomic>
#include <charconv>
#include <thread>

#include "pipesim_core.hpp"

namespace pb {

std::string fnv1a64::hex() const {
  std::string out(16, '0');
  static const char kHex[] = "0123456789abcdef";
  uint64_t x = h;
  for (int i = 15; i >= 0; --i, x >>= 4) out[i] = kHex[x & 0xF];
  return out;
}

namespace {

constexpr int64_t kChunk = 1 << 15;   // values per chunk (~650 KB of text)
constexpr int64_t kSerialBelow = 1 << 18;

// Formats values [a, b) of the concatenated spans into out.
void format_range(const std::vector<value_span>& spans, const std::vector<int64_t>& starts,
                  int64_t a, int64_t b, std::string& out) {
  out.resize(static_cast<size_t>(b - a) * 26);
  char* p = out.data();
  size_t si = std::upper_bound(starts.begin(), starts.end(), a) - starts.begin() - 1;
  int64_t i = a;
  while (i < b) {
    while (i >= starts[si + 1]) ++si;
    const int64_t end = std::min(b, starts[si + 1]);
    const double* v = spans[si].data + (i - starts[si]);
    for (int64_t k = 0; k < end - i; ++k) {
      p = std::to_chars(p, p + 25, v[k]).ptr;
      *p++ = '\n';
    }
    i = end;
  }
  out.resize(static_cast<size_t>(p - out.data()));
}

}  // namespace

void format_values_ordered(const std::vector<value_span>& spans,
                           const std::function<void(const char*, size_t)>& sink) {
  std::vector<int64_t> starts(spans.size() + 1, 0);
  for (size_t i = 0; i < spans.size(); ++i) starts[i + 1] = starts[i] + spans[i].n;
  const int64_t total = starts.back();
  if (total == 0) return;
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const int workers = static_cast<int>(std::min<unsigned>(hw > 1 ? hw - 1 : 1, 64));
  if (total < kSerialBelow || workers < 2) {
    std::string buf;
    for (int64_t a = 0; a < total; a += kChunk) {
      format_range(spans, starts, a, std::min(total, a + kChunk), buf);
      sink(buf.data(), buf.size());
    }
    return;
  }
  const int64_t chunks = (total + kChunk - 1) / kChunk;
  const int ring = 4 * workers;
  std::vector<std::string> bufs(ring);
  std::vector<std::atomic<int64_t>> ready(ring);   // chunk index held by the slot, -1 none
  for (auto& r : ready) r.store(-1);
  std::atomic<int64_t> next{0};       // next chunk to claim
  std::atomic<int64_t> consumed{0};   // chunks handed to the sink
  auto work = [&] {
    for (;;) {
      const int64_t c = next.fetch_add(1);
      if (c >= chunks) return;
      while (c - consumed.load(std::memory_order_acquire) >= ring) std::this_thread::yield();
      const int slot = static_cast<int>(c % ring);
      const int64_t a = c * kChunk;
      format_range(spans, starts, a, std::min(total, a + kChunk), bufs[slot]);
      ready[slot].store(c, std::memory_order_release);
    }
  };
  std::vector<std::thread> pool;
  pool.reserve(workers);
  for (int i = 0; i < workers; ++i) pool.emplace_back(work);
  try {
    for (int64_t c = 0; c < chunks; ++c) {
      const int slot = static_cast<int>(c % ring);
      while (ready[slot].load(std::memory_order_acquire) != c) std::this_thread::yield();
      sink(bufs[slot].data(), bufs[slot].size());
      consumed.store(c + 1, std::memory_order_release);
    }
  } catch (...) {
    next.store(chunks);                  // stop claiming, release the waiters
    consumed.store(chunks + ring);
    for (auto& t : pool) t.join();
    throw;
  }
  for (auto& t : pool) t.join();
}

std::string digest_spans(const std::vector<value_span>& spans) {
  fnv1a64 f;
  format_values_ordered(spans, [&](const char* p, size_t n) { f.update(p, n); });
  return f.hex();
}

}  // namespace pb
