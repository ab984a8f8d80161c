// Bulk host <-> HBM transfers for the drop-in boundary.
//
// The reference API hands parameters over as pageable std::vector<double>
// (trainer.hpp:81-83, :99-103).  A plain cudaMemcpy from pageable memory is
// staged by the driver through one small pinned buffer by one CPU thread; for
// the 2 GB of a 268M-parameter network that, plus a single-threaded fp64 <->
// fp32 conversion on the host, cost seconds per epoch.  Here the conversion
// runs on the device (the fp64 bytes cross PCIe once) and the pageable <->
// pinned copies are split over host threads, double-buffered against the DMA.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>

namespace pb {

// memcpy split over up to `threads` host threads (0 = hardware concurrency,
// capped at 16); small copies stay on the calling thread.
void parallel_memcpy(void* dst, const void* src, size_t bytes, int threads = 0);

class HostStager {
 public:
  explicit HostStager(size_t chunk_bytes = size_t{64} << 20);
  ~HostStager();
  HostStager(const HostStager&) = delete;
  HostStager& operator=(const HostStager&) = delete;

  // pageable host -> device, ordered on `st`.  Returns once the host bytes
  // have been consumed (the last DMA may still be in flight on `st`).
  void h2d(void* dev, const void* host, size_t bytes, cudaStream_t st);
  // device -> pageable host after the work already queued on `st`;
  // synchronous.
  void d2h(void* host, const void* dev, size_t bytes, cudaStream_t st);

 private:
  void ensure();
  size_t chunk_;
  int device_ = -1;
  char* pinned_[2] = {nullptr, nullptr};
  cudaEvent_t done_[2] = {nullptr, nullptr};
};

}  // namespace pb
