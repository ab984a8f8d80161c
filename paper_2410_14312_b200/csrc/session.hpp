// Session: the B200 executor of the pipeline-parallel training step
// (reference: proj/src/trainer.cpp:388-508 replay_grid, :510-553
// sequential_epoch).
//
// A session owns, for one network / train configuration, every device buffer
// of every pipeline stage and a static program derived from the schedule
// grid and version ledger (plan.cpp):
//   * per stage a forward stream, a backward stream (dgrad chain, loss), a
//     side stream (wgrad + SGD) and a bias stream; forwards and backwards each
//     run in slot order, and the hazards a single slot-ordered stream would
//     order (pinned version committed, activation slot free, pool colour
//     free) are explicit events (session.cu);
//   * cross-stage edges (activation s -> s+1, delta s+1 -> s) are CUDA events;
//   * weight versions live in a per-stage bf16 pool sized by the retention
//     timeline's peak (interval colouring), fp32 masters ping-pong by version
//     parity; a commit writes the next version in the wgrad+SGD epilogue;
//   * per-stage activation slots are interval-coloured over
//     [first forward of mini k, backward of mini k];
//   * the whole epoch is captured once as a CUDA graph and relaunched.
// Version accounting is observed on the device: every forward copies the tag
// of the pool slot it read, every backward the tag of the weights it
// propagated through, every commit stamps the new slot / current version.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "layer_ops.cuh"
#include "pipesim_core.hpp"

namespace pb {

enum class RunMode { timeprest = 0, pipedream = 1, sequential = 2 };
// bf16: x already rounded to bf16 on the host (the bf16 path's operand type;
// copied straight into the device layout, no conversion kernel)
enum class HostDType { f64 = 0, f32 = 1, labels_i32 = 2, bf16 = 3 };

// One layer of a convolutional network (VGG-style stages, BASELINE
// configs[3]; the reference has only Linear layers).
//  linear: in -> out features.
//  conv3x3: in -> out channels on h x w NHWC images, pad 1, stride 1, then
//  the activation, then (pool) 2x2 / stride-2 max pooling.  Weights are
//  [out][9 * in] with K = (3r + s) * in + c (tap-major), then b[out].
// A network is conv layers followed by linear layers; the first linear layer
// reads the last conv output flattened in NHWC order.  The first layer may be
// a narrow conv (in * 9 <= 72: the network input, im2col'd), every other conv
// has in, out % 64 == 0.
enum class LayerKind { linear = 0, conv3x3 = 1 };
struct LayerSpec {
  LayerKind kind = LayerKind::linear;
  int in = 0, out = 0;
  int h = 0, w = 0;  // conv: input image size
  bool pool = false;
  int act = 0;
  // per-sample element counts of the layer's input and (pooled) output
  int64_t in_elems() const {
    return kind == LayerKind::linear ? in : static_cast<int64_t>(h) * w * in;
  }
  int64_t out_elems() const {
    if (kind == LayerKind::linear) return out;
    return pool ? static_cast<int64_t>(h / 2) * (w / 2) * out : static_cast<int64_t>(h) * w * out;
  }
  // GEMM K of the weights (fan-in) and forward flops per sample
  int fan_in() const { return kind == LayerKind::linear ? in : 9 * in; }
  double flops() const {
    return 2.0 * out * fan_in() * (kind == LayerKind::linear ? 1.0 : static_cast<double>(h) * w);
  }
};

// Contiguous partition of a layer list into W stages minimising the largest
// stage's forward flops (the reference's partition_model balances parameter
// counts, trainer.cpp:104-135, which for a CNN would put every conv layer on
// one stage).  Returns n_layers per stage.
std::vector<int> partition_by_flops(const std::vector<LayerSpec>& layers, int W);
// Validates a conv network description (throws std::invalid_argument).
void check_layers(const std::vector<LayerSpec>& layers);

struct SessionConfig {
  std::vector<int> widths;
  std::vector<int> acts;
  // convolutional network (empty: the MLP given by widths / acts).  When set,
  // widths / acts are derived (widths[l] = per-sample input elements of
  // layer l, widths.back() = classes) and the stages are a flop-balanced
  // partition (stage_layers overrides it).
  std::vector<LayerSpec> layers;
  std::vector<int> stage_layers;
  int loss = 1;
  int W = 2, N = 2, B = 20, M = 10;
  double lr = 0.05;
  RunMode mode = RunMode::timeprest;
  int device = 0;
  bool use_graph = true;
  bool snapshots = false;  // per-commit fp32 host snapshots (per-mini digests)
  // stage range owned by this process (multi-GPU: one process per GPU);
  // [stage_lo, stage_hi] 1-based inclusive.  Default: all stages.
  int stage_lo = 1, stage_hi = 0;
  // multi-GPU: this process's rank among `world` (one process per GPU); the
  // stage range defaults to an even contiguous split.  nccl_ids holds the
  // 2*(world-1) NCCL unique ids (boundary x direction), identical on all ranks.
  int rank = 0, world = 1;
  std::vector<uint8_t> nccl_ids;
  // build the program only (no CUDA calls): used to check the cross-GPU
  // transfer schedule on machines without GPUs
  bool plan_only = false;
  // max micro-batches per coalesced forward launch (0 = N: a whole run)
  int fwd_merge = 0;
  // per-stage side stream for wgrad/bias (overlaps the dgrad chain)
  bool side_streams = true;
  // 0 none, 1 fwd, 2 dgrad, 3 wgrad: CUDA events around every launch of that
  // GEMM kind, recorded inside the graph (kernel_times_ms)
  int timed_kernel = 0;
  // multi-process stage split: 0 NCCL send/recv, 1 CUDA IPC peer memory
  // (ipc_p2p.hpp; also works for several processes sharing one GPU)
  int transport = 0;
  // fp32 verify precision: CUDA-core FFMA GEMMs on fp32 activations, deltas
  // and weight versions (verify_fp32.cu) instead of bf16 tensor cores
  bool verify_fp32 = false;
  // forwards and backwards of a stage on separate streams, with the slot
  // order's hazards as explicit events (PIPESIM_SPLIT_FB overrides)
  bool split_fb = true;
  // the reference's params_digest (trainer.cpp:492-501, :506) on the device,
  // inside the epoch: after every mini-batch's stage-1 commit over all stages'
  // then-current masters, and once over the final ones (digest_dev.hpp)
  bool digests = false;
};

// One point-to-point transfer of the program, in this process's issue order.
struct Transfer {
  bool send;      // false: receive
  int dir;        // 0 activations (s -> s+1), 1 deltas (s+1 -> s)
  int peer;       // rank
  int64_t bytes;
};

struct EpochResult {
  std::vector<double> mini_loss;  // [M]
  std::vector<int> pinned;        // [M * units] (ledger)
  std::vector<int> consumed;      // [M] update_source (ledger)
  std::vector<int> dev_fwd;       // [M * units * W] tags seen by forwards
  std::vector<int> dev_bwd;       // [M * W] tags propagated through by backwards
  std::vector<int> dev_current;   // [W] current version after the epoch
  float device_ms = 0.f;          // graph/stream time of the epoch
  std::vector<uint64_t> digests;  // [M + 1] per-mini-batch, then final (digests on)
};

// Per-node device timeline of one epoch (profile_epoch): a node is one
// backward task or one coalesced run of forward tasks of a stage.
struct NodeTiming {
  int stage;           // 1-based
  int fwd;             // 1 forward run, 0 backward
  int mini;            // k
  int micro_lo, micro_hi;  // forward micro-batch range (0-based), 0/0 for backward
  float start_ms, end_ms;  // from the epoch start, after the node's cross-stage waits
};

struct EpochProfile {
  float makespan_ms = 0.f;
  std::vector<float> busy_ms;  // [W]: sum of node spans per stage (-1: other GPU)
  std::vector<NodeTiming> nodes;
};

class Session {
 public:
  explicit Session(const SessionConfig& cfg);
  ~Session();
  Session(const Session&) = delete;
  Session& operator=(const Session&) = delete;

  const SessionConfig& config() const { return cfg_; }
  int units() const { return cfg_.mode == RunMode::timeprest ? cfg_.N : 1; }
  int64_t param_count() const { return total_params_; }
  int64_t stage_param_count(int s) const;  // 1-based
  int64_t stage_param_offset(int s) const;
  int stage_first_layer(int s) const;  // 1-based stage; 0-based layer
  int stage_layer_count(int s) const;

  // Installs a flat whole-network parameter vector as version 0.
  void load_params(const double* flat);
  // params_digest (trainer.cpp:599-607) of every stage's current version,
  // computed on the device; single-process sessions
  // (version: 0 after load_params, M after an epoch)
  uint64_t params_digest(int version);
  const EpochResult& last_result() const { return last_; }
  // version 0 of one stage (1-based) := p, W then b per layer (fp64)
  void load_stage_params(int stage, const double* p);
  // Copies the current version's fp32 masters out as doubles (flat layout).
  void read_params(double* flat);
  // fp32 snapshot of `version` of stage s (requires snapshots=true).
  const float* snapshot(int s, int version) const;
  bool has_snapshots() const { return cfg_.snapshots; }
  // fp32 master buffer `parity` (0/1) of stage s: holds the last committed
  // version with that parity (versions M and M-1 after an epoch).
  // fp32 master of `version` (M or M-1 after an epoch) of one stage
  void read_stage_master(int stage, int version, double* out);

  // Host -> device copy of the epoch's data (rows = M*B), then conversion.
  void upload(const void* x, HostDType xt, const void* y, HostDType yt,
              cudaStream_t st = nullptr);
  // Runs one epoch on the uploaded data.  `epoch` only tags the result.
  EpochResult run_epoch();
  // One epoch from host buffers with the upload streamed inside it: mini-batch
  // k's rows are copied and converted on their own stream while earlier
  // mini-batches compute; stage 1's forwards and the loss of mini k wait
  // only for mini k's rows (the graph is re-captured when the buffers change).
  EpochResult train_epoch_host(const void* x, HostDType xt, const void* y, HostDType yt);
  // Runs one epoch without the CUDA graph, with timing events around every
  // node on its stage stream: per-stage busy time, the epoch makespan and
  // the node timeline (pipeline bubble = 1 - sum(busy) / (W * makespan)).
  EpochResult profile_epoch(EpochProfile* prof);

  // Ledger / plan of the session (for logs and checks).
  const pipesim::version_ledger& ledger() const { return ledger_; }
  const pipesim::schedule_grid* grid() const { return grid_.get(); }
  int horizon() const { return horizon_; }
  std::vector<int> pool_sizes() const;
  std::vector<int> act_slot_counts() const;
  // per stage: {weight-version bytes, activation bytes} this process allocated
  std::vector<std::pair<int64_t, int64_t>> stage_bytes() const;
  int64_t device_bytes() const { return arena_bytes_; }
  int kernels_per_epoch() const { return kernels_per_epoch_; }
  // Schedule document (export.cpp schema) of the last epoch with the version
  // numbers the device observed: each pin from the tag its stage-1 forward
  // read, and (timeprest) each consumption from the tag its backward
  // propagated through.  Single-process sessions with a schedule grid.
  std::string trace_document() const;
  // durations of the timed GEMM kind's launches in the last epoch (ms)
  std::vector<float> kernel_times_ms();
  const std::vector<double>& kernel_flops() const;
  std::vector<Transfer> transfers() const;
  // IPC transport: this rank's connection blob, and the connect step with
  // every rank's blob (exchanged by the caller, e.g. over torch.distributed)
  std::vector<uint8_t> ipc_export();
  void ipc_connect(const std::vector<std::vector<uint8_t>>& blobs);

  struct Impl;  // public so the program-issue helpers can see it

 private:
  EpochResult collect_result();
  EpochResult last_;  // the last epoch's result (trace_document)
  SessionConfig cfg_;
  std::unique_ptr<Impl> impl_;
  std::unique_ptr<pipesim::schedule_grid> grid_;
  pipesim::version_ledger ledger_;
  int horizon_ = 0;
  int64_t total_params_ = 0;
  int64_t arena_bytes_ = 0;
  int kernels_per_epoch_ = 0;
};

}  // namespace pb
