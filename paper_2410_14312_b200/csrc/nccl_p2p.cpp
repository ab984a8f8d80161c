// NCCL point-to-point transport (see nccl_p2p.hpp).
#include "nccl_p2p.hpp"

#include <dlfcn.h>

#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>

#include "status.hpp"

namespace pb {

// Minimal NCCL ABI surface (matches nccl.h 2.x: opaque comm pointer,
// 128-byte unique id, int result/type enums).
struct NcclApi {
  using Comm = void*;
  struct UniqueId {
    char internal[kNcclIdBytes];
  };
  int (*GetUniqueId)(UniqueId*) = nullptr;
  int (*CommInitRank)(Comm*, int, UniqueId, int) = nullptr;
  int (*CommDestroy)(Comm) = nullptr;
  int (*Send)(const void*, size_t, int, int, Comm, cudaStream_t) = nullptr;
  int (*Recv)(void*, size_t, int, int, Comm, cudaStream_t) = nullptr;
  int (*GroupStart)() = nullptr;
  int (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
  bool ok = false;
};

namespace {

constexpr int kNcclUint8 = 1;  // ncclUint8 / ncclChar

NcclApi& api() {
  static NcclApi a;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    auto sym = [&](const char* n) { return dlsym(h, n); };
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(sym("ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(sym("ncclCommInitRank"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
    a.Send = reinterpret_cast<decltype(a.Send)>(sym("ncclSend"));
    a.Recv = reinterpret_cast<decltype(a.Recv)>(sym("ncclRecv"));
    a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(sym("ncclGroupStart"));
    a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(sym("ncclGroupEnd"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(sym("ncclGetErrorString"));
    a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.Send && a.Recv &&
           a.GroupStart && a.GroupEnd;
  });
  if (!a.ok) throw cuda_failure("NCCL (libnccl.so.2) is not available");
  return a;
}

void nccl_check(int r, const char* what) {
  if (r != 0) {
    const char* s = api().GetErrorString ? api().GetErrorString(r) : "?";
    throw cuda_failure(std::string(what) + ": NCCL error " + std::to_string(r) + " (" + s + ")");
  }
}

}  // namespace

bool P2P::available() {
  try {
    return api().ok;
  } catch (...) {
    return false;
  }
}

void P2P::unique_id(uint8_t* out) {
  NcclApi::UniqueId id;
  nccl_check(api().GetUniqueId(&id), "ncclGetUniqueId");
  std::memcpy(out, id.internal, kNcclIdBytes);
}

P2P::P2P(int rank, int world, const uint8_t* ids, size_t ids_bytes)
    : rank_(rank), world_(world), comms_(2 * std::max(0, world - 1), nullptr) {
  if (world < 2) return;
  if (ids_bytes < static_cast<size_t>(2 * (world - 1)) * kNcclIdBytes)
    throw std::invalid_argument("need 2*(world-1) NCCL unique ids");
  NcclApi& a = api();
  // Boundary b links ranks b and b+1 (2-rank communicators: b -> local 0,
  // b+1 -> local 1).  Grouped so the inits of neighbouring boundaries cannot
  // wait on each other.
  nccl_check(a.GroupStart(), "ncclGroupStart");
  for (int b = std::max(0, rank - 1); b <= std::min(world - 2, rank); ++b)
    for (int dir = 0; dir < 2; ++dir) {
      NcclApi::UniqueId id;
      std::memcpy(id.internal, ids + static_cast<size_t>(2 * b + dir) * kNcclIdBytes,
                  kNcclIdBytes);
      NcclApi::Comm c = nullptr;
      nccl_check(a.CommInitRank(&c, 2, id, rank == b ? 0 : 1), "ncclCommInitRank");
      comms_[2 * b + dir] = c;
    }
  nccl_check(a.GroupEnd(), "ncclGroupEnd");
}

P2P::~P2P() {
  for (void* c : comms_)
    if (c) api().CommDestroy(c);
}

void* P2P::comm(int peer_rank, int direction) {
  const int b = std::min(rank_, peer_rank);
  if (std::abs(peer_rank - rank_) != 1 || b < 0 || b >= world_ - 1)
    throw std::invalid_argument("P2P peer must be a neighbouring rank");
  void* c = comms_[2 * b + direction];
  if (!c) throw std::logic_error("no communicator for this boundary");
  return c;
}

void P2P::send(const void* buf, size_t bytes, int peer_rank, int direction, cudaStream_t st) {
  const int peer_local = peer_rank > rank_ ? 1 : 0;
  nccl_check(api().Send(buf, bytes, kNcclUint8, peer_local, comm(peer_rank, direction), st),
             "ncclSend");
}

void P2P::recv(void* buf, size_t bytes, int peer_rank, int direction, cudaStream_t st) {
  const int peer_local = peer_rank > rank_ ? 1 : 0;
  nccl_check(api().Recv(buf, bytes, kNcclUint8, peer_local, comm(peer_rank, direction), st),
             "ncclRecv");
}

}  // namespace pb
