// Point-to-point transport between pipeline stages on different GPUs.
//
// One process per GPU; each process owns a contiguous stage range.  The only
// cross-GPU traffic of the TiMePReSt step is point-to-point:
// activations s -> s+1 (per coalesced forward) and deltas s+1 -> s (per
// mini-batch).  Each boundary and direction gets its own 2-rank NCCL
// communicator, used from exactly one stream on each side, so sends and
// receives of the two directions never serialize behind each other.
//
// NCCL is resolved at run time (dlopen "libnccl.so.2"): inside a torch
// process this binds the NCCL torch already loaded; elsewhere the system one.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

namespace pb {

constexpr int kNcclIdBytes = 128;

struct NcclApi;

class P2P {
 public:
  // ids: 4 * (world-1) unique ids of kNcclIdBytes: [boundary][fwd, bwd] pairs
  // (boundary b links rank b and b+1); only the ones of this rank are used.
  P2P(int rank, int world, const uint8_t* ids, size_t ids_bytes);
  ~P2P();
  P2P(const P2P&) = delete;
  P2P& operator=(const P2P&) = delete;

  // direction 0 = forward (activations, rank -> rank+1), 1 = backward.
  void send(const void* buf, size_t bytes, int peer_rank, int direction, cudaStream_t st);
  void recv(void* buf, size_t bytes, int peer_rank, int direction, cudaStream_t st);

  static void unique_id(uint8_t* out);  // ncclGetUniqueId
  static bool available();

 private:
  void* comm(int peer_rank, int direction);
  int rank_, world_;
  std::vector<void*> comms_;  // [boundary * 2 + direction], nullptr if not ours
};

}  // namespace pb
