// Peer-memory point-to-point transport between pipeline stages owned by
// different processes (one process per GPU over NVLink, or several processes
// sharing one GPU).  The receiver's slot buffers are mapped into the sender
// with CUDA IPC; a transfer is one copy straight into the receiver's slot on
// the sender's transfer stream.  Flow control is a two-flag handshake per
// message, all on the device (stream memory operations, no host round trip):
//
//   receiver stream:  write posted[msg] = 1   (the slot is free: its previous
//                                               occupant's backward is done)
//                     wait  done[msg] == 1;  write done[msg] = 0
//   sender stream:    wait  posted[msg] == 1; write posted[msg] = 0
//                     copy  src -> receiver slot (peer / same-device copy)
//                     write done[msg] = 1
//
// Every flag is reset by its waiter right after the wait, so the operations
// are the same every epoch: an epoch is captured once as a CUDA graph
// (memory-operation nodes) and replayed (ordering argument at send()).
// Each flag lives in the memory of the side that waits on it; the other side
// writes it through its IPC mapping.  The i-th send of a channel (boundary,
// direction) pairs with the i-th receive of the same channel: the programs of
// neighbouring ranks issue them in the same order with the same sizes
// (tests/test_multigpu_plan.py).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <vector>

namespace pb {

class IpcLink {
 public:
  struct Msg {
    bool send;     // false: receive
    int dir;       // 0 activations (s -> s+1), 1 deltas (s+1 -> s)
    int peer;      // neighbouring rank
    size_t bytes;
    const void* src = nullptr;  // send: local source
    void* dst = nullptr;        // receive: local destination (inside the arena)
  };

  // msgs: this rank's transfers in program order.  arena: the cudaMalloc'd
  // allocation every receive destination lies in.
  IpcLink(int rank, int world, int device, void* arena, std::vector<Msg> msgs);
  ~IpcLink();
  IpcLink(const IpcLink&) = delete;
  IpcLink& operator=(const IpcLink&) = delete;

  // What the neighbours need: device, IPC handles of the arena and the flag
  // block, and per message its channel, index, flag offset and (receives)
  // destination offset.
  std::vector<uint8_t> export_blob() const;
  // blobs[r] = export_blob() of rank r (only the neighbours' are read).
  void connect(const std::vector<std::vector<uint8_t>>& blobs);
  bool connected() const { return connected_; }

  // Enqueue message `idx` (program order) on `st`.
  void send(int idx, cudaStream_t st);
  void recv(int idx, cudaStream_t st);

 private:
  struct Entry {
    int boundary, dir, send, index;  // index within the channel
    int64_t bytes;
    int64_t flag_off;  // own flag (waited on here)
    int64_t dst_off;   // receive: destination offset in the arena
  };
  int rank_, world_, device_;
  void* arena_;
  std::vector<Msg> msgs_;
  std::vector<Entry> entries_;
  uint32_t* flags_ = nullptr;  // one word per message
  bool connected_ = false;
  // per message, resolved by connect(): remote flag to write, remote destination
  std::vector<uint32_t*> remote_flag_;
  std::vector<void*> remote_dst_;
  std::vector<void*> opened_;  // IPC mappings to close
};

}  // namespace pb
