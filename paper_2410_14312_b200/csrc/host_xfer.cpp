#include "host_xfer.hpp"

#include <algorithm>
#include <cstring>
#include <thread>
#include <vector>

#include "status.hpp"

namespace pb {

void parallel_memcpy(void* dst, const void* src, size_t bytes, int threads) {
  constexpr size_t kMinPiece = size_t{4} << 20;
  if (threads <= 0)
    threads = static_cast<int>(std::min(16u, std::max(1u, std::thread::hardware_concurrency())));
  const size_t pieces = std::min<size_t>(threads, std::max<size_t>(1, bytes / kMinPiece));
  if (pieces <= 1) {
    std::memcpy(dst, src, bytes);
    return;
  }
  const size_t per = (bytes / pieces + 4095) & ~size_t{4095};
  std::vector<std::thread> pool;
  pool.reserve(pieces - 1);
  for (size_t i = 1; i < pieces; ++i) {
    const size_t a = std::min(bytes, i * per), b = std::min(bytes, a + per);
    if (a >= b) break;
    pool.emplace_back([=] {
      std::memcpy(static_cast<char*>(dst) + a, static_cast<const char*>(src) + a, b - a);
    });
  }
  std::memcpy(dst, src, std::min(bytes, per));
  for (auto& t : pool) t.join();
}

HostStager::HostStager(size_t chunk_bytes) : chunk_(chunk_bytes) {}

HostStager::~HostStager() {
  for (int b = 0; b < 2; ++b) {
    if (done_[b]) cudaEventSynchronize(done_[b]), cudaEventDestroy(done_[b]);
    if (pinned_[b]) cudaFreeHost(pinned_[b]);
  }
}

void HostStager::ensure() {
  if (pinned_[0]) return;
  for (int b = 0; b < 2; ++b) {
    PB_CUDA(cudaMallocHost(&pinned_[b], chunk_));
    PB_CUDA(cudaEventCreateWithFlags(&done_[b], cudaEventDisableTiming));
    PB_CUDA(cudaEventRecord(done_[b], 0));
  }
}

void HostStager::h2d(void* dev, const void* host, size_t bytes, cudaStream_t st) {
  if (bytes == 0) return;
  if (bytes < (size_t{1} << 20)) {  // small: the driver's own staging is fine
    PB_CUDA(cudaMemcpyAsync(dev, host, bytes, cudaMemcpyHostToDevice, st));
    PB_CUDA(cudaStreamSynchronize(st));
    return;
  }
  ensure();
  int b = 0;
  for (size_t off = 0; off < bytes; off += chunk_, b ^= 1) {
    const size_t n = std::min(chunk_, bytes - off);
    PB_CUDA(cudaEventSynchronize(done_[b]));  // the DMA that last read this buffer
    parallel_memcpy(pinned_[b], static_cast<const char*>(host) + off, n);
    PB_CUDA(cudaMemcpyAsync(static_cast<char*>(dev) + off, pinned_[b], n,
                            cudaMemcpyHostToDevice, st));
    PB_CUDA(cudaEventRecord(done_[b], st));
  }
}

void HostStager::d2h(void* host, const void* dev, size_t bytes, cudaStream_t st) {
  if (bytes == 0) return;
  if (bytes < (size_t{1} << 20)) {
    PB_CUDA(cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, st));
    PB_CUDA(cudaStreamSynchronize(st));
    return;
  }
  ensure();
  const size_t chunks = (bytes + chunk_ - 1) / chunk_;
  auto issue = [&](size_t c) {
    const int b = static_cast<int>(c & 1);
    const size_t off = c * chunk_, n = std::min(chunk_, bytes - off);
    PB_CUDA(cudaMemcpyAsync(pinned_[b], static_cast<const char*>(dev) + off, n,
                            cudaMemcpyDeviceToHost, st));
    PB_CUDA(cudaEventRecord(done_[b], st));
  };
  PB_CUDA(cudaEventSynchronize(done_[0]));
  PB_CUDA(cudaEventSynchronize(done_[1]));
  issue(0);
  for (size_t c = 0; c < chunks; ++c) {
    if (c + 1 < chunks) issue(c + 1);  // its buffer was drained two chunks ago
    const int b = static_cast<int>(c & 1);
    const size_t off = c * chunk_, n = std::min(chunk_, bytes - off);
    PB_CUDA(cudaEventSynchronize(done_[b]));
    parallel_memcpy(static_cast<char*>(host) + off, pinned_[b], n);
  }
}

}  // namespace pb
