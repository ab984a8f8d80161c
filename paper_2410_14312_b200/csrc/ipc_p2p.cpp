// Peer-memory transport (see ipc_p2p.hpp).
#include "ipc_p2p.hpp"

#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstring>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <tuple>

#include "status.hpp"

namespace pb {

namespace {

struct StreamMemOps {
  PFN_cuStreamWaitValue32_v2 wait = nullptr;
  PFN_cuStreamWriteValue32_v2 write = nullptr;
};

const StreamMemOps& memops() {
  static StreamMemOps ops;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    PB_CUDA(cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !p) throw cuda_failure("cuStreamWaitValue32 unavailable");
    ops.wait = reinterpret_cast<PFN_cuStreamWaitValue32_v2>(p);
    PB_CUDA(cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !p) throw cuda_failure("cuStreamWriteValue32 unavailable");
    ops.write = reinterpret_cast<PFN_cuStreamWriteValue32_v2>(p);
  });
  return ops;
}

void cu_check(CUresult r, const char* what) {
  if (r != CUDA_SUCCESS) throw cuda_failure(std::string(what) + " failed (CUresult " +
                                            std::to_string(static_cast<int>(r)) + ")");
}

// blob layout: magic, rank, device, n, arena handle, flags handle, n entries
constexpr uint32_t kMagic = 0x50424950;  // "PBIP"

template <typename T>
void put(std::vector<uint8_t>& b, const T& v) {
  const auto* p = reinterpret_cast<const uint8_t*>(&v);
  b.insert(b.end(), p, p + sizeof(T));
}
template <typename T>
T get(const std::vector<uint8_t>& b, size_t& at) {
  if (at + sizeof(T) > b.size()) throw std::invalid_argument("truncated IPC blob");
  T v;
  std::memcpy(&v, b.data() + at, sizeof(T));
  at += sizeof(T);
  return v;
}

}  // namespace

IpcLink::IpcLink(int rank, int world, int device, void* arena, std::vector<Msg> msgs)
    : rank_(rank), world_(world), device_(device), arena_(arena), msgs_(std::move(msgs)) {
  std::map<std::tuple<int, int, int>, int> next;  // (boundary, dir, send) -> count
  entries_.reserve(msgs_.size());
  for (size_t i = 0; i < msgs_.size(); ++i) {
    const Msg& m = msgs_[i];
    if (std::abs(m.peer - rank) != 1) throw std::invalid_argument("IPC peer must be a neighbour");
    Entry e{};
    e.boundary = std::min(rank, m.peer);
    e.dir = m.dir;
    e.send = m.send ? 1 : 0;
    e.index = next[{e.boundary, e.dir, e.send}]++;
    e.bytes = static_cast<int64_t>(m.bytes);
    e.flag_off = static_cast<int64_t>(i * sizeof(uint32_t));
    e.dst_off = m.send ? -1
                       : static_cast<int64_t>(static_cast<const char*>(m.dst) -
                                              static_cast<const char*>(arena_));
    entries_.push_back(e);
  }
  const size_t n = std::max<size_t>(1, msgs_.size());
  PB_CUDA(cudaMalloc(&flags_, n * sizeof(uint32_t)));
  PB_CUDA(cudaMemset(flags_, 0, n * sizeof(uint32_t)));
  remote_flag_.assign(msgs_.size(), nullptr);
  remote_dst_.assign(msgs_.size(), nullptr);
}

IpcLink::~IpcLink() {
  for (void* p : opened_) cudaIpcCloseMemHandle(p);
  if (flags_) cudaFree(flags_);
}

std::vector<uint8_t> IpcLink::export_blob() const {
  std::vector<uint8_t> b;
  put(b, kMagic);
  put(b, static_cast<int32_t>(rank_));
  put(b, static_cast<int32_t>(device_));
  put(b, static_cast<int32_t>(entries_.size()));
  cudaIpcMemHandle_t ha{}, hf{};
  PB_CUDA(cudaIpcGetMemHandle(&ha, arena_));
  PB_CUDA(cudaIpcGetMemHandle(&hf, flags_));
  put(b, ha);
  put(b, hf);
  for (const Entry& e : entries_) put(b, e);
  return b;
}

void IpcLink::connect(const std::vector<std::vector<uint8_t>>& blobs) {
  if (static_cast<int>(blobs.size()) != world_) throw std::invalid_argument("need one blob per rank");
  PB_CUDA(cudaSetDevice(device_));
  for (int peer : {rank_ - 1, rank_ + 1}) {
    if (peer < 0 || peer >= world_) continue;
    const std::vector<uint8_t>& b = blobs[peer];
    size_t at = 0;
    if (get<uint32_t>(b, at) != kMagic) throw std::invalid_argument("bad IPC blob");
    if (get<int32_t>(b, at) != peer) throw std::invalid_argument("IPC blob of the wrong rank");
    const int pdev = get<int32_t>(b, at);
    const int n = get<int32_t>(b, at);
    const auto ha = get<cudaIpcMemHandle_t>(b, at);
    const auto hf = get<cudaIpcMemHandle_t>(b, at);
    std::map<std::tuple<int, int, int, int>, Entry> theirs;  // (boundary, dir, send, index)
    for (int i = 0; i < n; ++i) {
      const Entry e = get<Entry>(b, at);
      theirs[{e.boundary, e.dir, e.send, e.index}] = e;
    }
    if (pdev != device_) {
      int can = 0;
      PB_CUDA(cudaDeviceCanAccessPeer(&can, device_, pdev));
      if (!can) throw cuda_failure("GPU " + std::to_string(device_) + " cannot access peer GPU " +
                                   std::to_string(pdev));
    }
    void* parena = nullptr;
    void* pflags = nullptr;
    PB_CUDA(cudaIpcOpenMemHandle(&parena, ha, cudaIpcMemLazyEnablePeerAccess));
    opened_.push_back(parena);
    PB_CUDA(cudaIpcOpenMemHandle(&pflags, hf, cudaIpcMemLazyEnablePeerAccess));
    opened_.push_back(pflags);
    for (size_t i = 0; i < entries_.size(); ++i) {
      const Entry& e = entries_[i];
      if (msgs_[i].peer != peer) continue;
      auto it = theirs.find({e.boundary, e.dir, 1 - e.send, e.index});
      if (it == theirs.end())
        throw std::logic_error("IPC transfer without a matching peer transfer");
      if (it->second.bytes != e.bytes)
        throw std::logic_error("IPC transfer sizes differ between neighbouring ranks");
      remote_flag_[i] = reinterpret_cast<uint32_t*>(static_cast<char*>(pflags) + it->second.flag_off);
      if (e.send) remote_dst_[i] = static_cast<char*>(parena) + it->second.dst_off;
    }
  }
  connected_ = true;
}

// Binary flags, reset by the side that waits on them right after its wait:
// the value waited for is always 1, so the enqueued operations are identical
// every epoch and the epoch can be a CUDA graph replayed as is.  A flag's next
// set cannot overtake its reset: the receiver posts message i of the next
// epoch only after (its stream order) waiting for done[i] of this one, which
// the sender writes after resetting posted[i]; the sender signals done[i] of
// the next epoch only after that post, which the receiver issues after
// resetting done[i].  (Writes carry the default system-scope memory barrier.)
void IpcLink::send(int idx, cudaStream_t st) {
  if (!connected_) throw std::logic_error("IPC transport is not connected");
  const StreamMemOps& ops = memops();
  const CUstream cs = reinterpret_cast<CUstream>(st);
  const CUdeviceptr own = reinterpret_cast<CUdeviceptr>(flags_ + idx);
  cu_check(ops.wait(cs, own, 1, CU_STREAM_WAIT_VALUE_GEQ), "cuStreamWaitValue32 (posted)");
  cu_check(ops.write(cs, own, 0, CU_STREAM_WRITE_VALUE_DEFAULT), "cuStreamWriteValue32 (reset)");
  PB_CUDA(cudaMemcpyAsync(remote_dst_[idx], msgs_[idx].src, msgs_[idx].bytes,
                          cudaMemcpyDeviceToDevice, st));
  cu_check(ops.write(cs, reinterpret_cast<CUdeviceptr>(remote_flag_[idx]), 1,
                     CU_STREAM_WRITE_VALUE_DEFAULT),
           "cuStreamWriteValue32 (done)");
}

void IpcLink::recv(int idx, cudaStream_t st) {
  if (!connected_) throw std::logic_error("IPC transport is not connected");
  const StreamMemOps& ops = memops();
  const CUstream cs = reinterpret_cast<CUstream>(st);
  const CUdeviceptr own = reinterpret_cast<CUdeviceptr>(flags_ + idx);
  cu_check(ops.write(cs, reinterpret_cast<CUdeviceptr>(remote_flag_[idx]), 1,
                     CU_STREAM_WRITE_VALUE_DEFAULT),
           "cuStreamWriteValue32 (posted)");
  cu_check(ops.wait(cs, own, 1, CU_STREAM_WAIT_VALUE_GEQ), "cuStreamWaitValue32 (done)");
  cu_check(ops.write(cs, own, 0, CU_STREAM_WRITE_VALUE_DEFAULT), "cuStreamWriteValue32 (reset)");
}

}  // namespace pb
