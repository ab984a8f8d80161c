// Session implementation — see session.hpp for the design summary.
#include "session.hpp"
#include "conv_ops.cuh"
#include "digest_dev.hpp"
#include "host_xfer.hpp"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <numeric>
#include <stdexcept>
#include <string>
#include <tuple>

#include "ipc_p2p.hpp"
#include "nccl_p2p.hpp"
#include "status.hpp"

namespace pb {

namespace {

constexpr size_t kAlign = 256;

int ld8(int cols) { return (cols + 7) / 8 * 8; }

// Greedy interval colouring over [start, end] (inclusive ends): a colour is
// reusable by an interval starting strictly after the colour's last end.
// Intervals are given in the order colours should be assigned (by start).
std::vector<int> colour(const std::vector<std::pair<int, int>>& iv, int* n_colours,
                        bool half_open) {
  std::vector<int> order(iv.size());
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(),
                   [&](int a, int b) { return iv[a].first < iv[b].first; });
  std::vector<int> busy_until;  // per colour: last end
  std::vector<int> out(iv.size(), -1);
  for (int i : order) {
    int pick = -1;
    for (size_t c = 0; c < busy_until.size(); ++c) {
      const bool free = half_open ? busy_until[c] <= iv[i].first
                                  : busy_until[c] < iv[i].first;
      if (free) {
        pick = static_cast<int>(c);
        break;
      }
    }
    if (pick < 0) {
      pick = static_cast<int>(busy_until.size());
      busy_until.push_back(0);
    }
    busy_until[pick] = iv[i].second;
    out[i] = pick;
  }
  *n_colours = static_cast<int>(busy_until.size());
  return out;
}

}  // namespace

// ------------------------------------------------------------------ conv nets
void check_layers(const std::vector<LayerSpec>& layers) {
  bool seen_linear = false;
  int64_t prev_out = -1;
  for (size_t i = 0; i < layers.size(); ++i) {
    const LayerSpec& l = layers[i];
    const std::string at = "layer " + std::to_string(i) + ": ";
    if (l.in < 1 || l.out < 1) throw std::invalid_argument(at + "empty layer");
    if (l.act < 0 || l.act > 3) throw std::invalid_argument(at + "bad activation");
    if (l.kind == LayerKind::conv3x3) {
      if (seen_linear) throw std::invalid_argument(at + "conv layers must precede linear layers");
      if (l.h < 1 || l.w < 1) throw std::invalid_argument(at + "conv needs an image size");
      if (l.out % 64 != 0) throw std::invalid_argument(at + "conv output channels % 64");
      if (i == 0 ? (l.in % 64 != 0 && 9 * l.in > 72) : l.in % 64 != 0)
        throw std::invalid_argument(at + "conv input channels % 64 (first layer: <= 8)");
      if (l.pool && (l.h % 2 != 0 || l.w % 2 != 0))
        throw std::invalid_argument(at + "pooling needs an even image size");
      if (l.pool && l.act != 0 && l.act != 1)
        throw std::invalid_argument(at + "pooling follows a linear or ReLU activation");
    } else {
      seen_linear = true;
      if (l.pool) throw std::invalid_argument(at + "linear layers do not pool");
    }
    if (prev_out >= 0 && l.in_elems() != prev_out)
      throw std::invalid_argument(at + "input size " + std::to_string(l.in_elems()) +
                                  " != previous output " + std::to_string(prev_out));
    prev_out = l.out_elems();
  }
  if (layers.empty() || layers.back().kind != LayerKind::linear)
    throw std::invalid_argument("a conv network ends with a linear layer");
}

std::vector<int> partition_by_flops(const std::vector<LayerSpec>& layers, int W) {
  const int L = static_cast<int>(layers.size());
  if (W < 1 || W > L)
    throw pipesim::domain_error("workers", "cannot split " + std::to_string(L) +
                                               " layers into " + std::to_string(W) + " stages");
  std::vector<double> pre(L + 1, 0.0);
  for (int i = 0; i < L; ++i) pre[i + 1] = pre[i] + layers[i].flops();
  const double inf = 1e300;
  // best[k][i]: smallest max-stage cost of the first i layers in k stages
  std::vector<std::vector<double>> best(W + 1, std::vector<double>(L + 1, inf));
  std::vector<std::vector<int>> cut(W + 1, std::vector<int>(L + 1, 0));
  best[0][0] = 0.0;
  for (int k = 1; k <= W; ++k)
    for (int i = k; i <= L; ++i)
      for (int j = k - 1; j < i; ++j) {
        const double v = std::max(best[k - 1][j], pre[i] - pre[j]);
        if (v < best[k][i]) {
          best[k][i] = v;
          cut[k][i] = j;
        }
      }
  std::vector<int> n(W);
  for (int k = W, i = L; k >= 1; --k) {
    n[k - 1] = i - cut[k][i];
    i = cut[k][i];
  }
  return n;
}

// ------------------------------------------------------------------ Impl
struct Session::Impl {
  struct LayerDev {
    // weights: out x in (in = GEMM K, the fan-in), rows of ld_in elements
    int in = 0, out = 0, act = 0;
    int ld_in = 0, ld_out = 0;
    // conv layers (LayerSpec): channels, input image, pooling; the network's
    // first conv reads an im2col of the input (first_conv)
    bool conv = false, pool = false, first_conv = false;
    int cin = 0, h = 0, w = 0;
    // per-sample elements of the layer's input / (pooled) output: the
    // activation rows (= ld_in / ld_out for a Linear layer)
    int ain = 0, aout = 0;
    int64_t pre_elems = 0;  // pooled conv: per-sample conv output before pooling
    float* w32[2] = {nullptr, nullptr};  // fp32 masters by version parity
    uint16_t* lo[2] = {nullptr, nullptr};  // split masters: residuals by parity
    float* b32[2] = {nullptr, nullptr};
  };
  struct PoolSlot {
    std::vector<__nv_bfloat16*> w16;
    std::vector<float*> b32;
    int* tag = nullptr;
  };
  struct ActSlot {
    std::vector<__nv_bfloat16*> out16;  // per layer (null for the logits layer)
    std::vector<__nv_bfloat16*> pre16;  // per layer: pooled conv output before pooling
    __nv_bfloat16* cols16 = nullptr;     // first conv: im2col of the input rows
    float* out32 = nullptr;              // last stage: logits / final output
    __nv_bfloat16* dzin = nullptr;       // delta into this stage's top layer
    // cross-GPU boundary buffers (only on a rank's first stage when the
    // upstream stage lives on another GPU): received input activation and
    // the outgoing delta for the upstream stage.
    __nv_bfloat16* in16 = nullptr;
    __nv_bfloat16* dzsend = nullptr;
  };
  struct Stage {
    int id = 0, first_layer = 0, L = 0;
    std::vector<LayerDev> layers;
    std::vector<PoolSlot> pool;
    std::vector<ActSlot> acts;
    std::vector<__nv_bfloat16*> scratch_dz;  // per layer < L-1
    std::vector<__nv_bfloat16*> scratch_pre;  // per pooled conv layer: dZ before pooling
    float* wg_ws = nullptr;    // conv wgrad split-K partial slabs (side stream)
    float* bias_ws = nullptr;  // conv bias-gradient row-block partials (bias stream)
    size_t wg_floats = 0, bias_floats = 0;
    // split-K forwards (one stage per GPU): fixup partials + tile counters
    // of the forward stream (its launches run one at a time)
    float* fix_ws = nullptr;
    int* fix_cnt = nullptr;
    size_t fix_floats = 0;
    int fix_counters = 0;
    std::vector<int> version_colour;         // [M+1]
    std::vector<int> mini_act;               // [M+1]
    int* cur_version = nullptr;
    cudaStream_t stream = nullptr;
    cudaStream_t side = nullptr;  // wgrad/bias of a backward run beside the dgrad chain
    cudaStream_t bstream = nullptr;  // backwards (split mode; forwards keep `stream`)
    cudaStream_t biasstream = nullptr;  // bias gradient + SGD of a backward
    int64_t param_offset = 0, param_count = 0;
    // device bytes held for this stage: weight versions (pool + masters) and
    // activations (slots, scratch deltas, boundary buffers, logits)
    int64_t bytes_weights = 0, bytes_acts = 0;
  };

  struct Task {
    bool fwd = true;
    int k = 0, jj = 0, s = 0, slot = 0;
    int version = 0;  // fwd: pinned; bwd: propagation version
  };

  enum class OpKind { wait, record, fwd, dgrad, wgrad, bias, loss, copy, memset_i32, snapshot,
                      send, recv, mark, ktime, xwait, digest,
                      // conv stages
                      im2col, pool_fwd, pool_bwd, wgrad_partial, reduce_sgd, colsum,
                      dgrad_chain, fwd_chain };
  // streams beyond the stage streams (Op::stream values)
  static constexpr int kFwdSend = -2, kFwdRecv = -3, kBwdSend = -4, kBwdRecv = -5;
  static constexpr int kDigest = -6;  // in-epoch params digests
  static constexpr int kSideBase = -100;  // side stream of stage s: kSideBase - s
  static constexpr int kBwdBase = -1000;  // backward stream of stage s (split mode)
  static constexpr int kBiasBase = -2000;  // bias-gradient stream of stage s
  struct Op {
    OpKind kind;
    int stream = 0;  // stage index (0-based); -1 = origin stream
    cudaEvent_t ev = nullptr;
    GemmLaunch g{};
    ChainLaunch chain{};  // dgrad_chain
    FwdChainLaunch fchain{};  // fwd_chain
    // bias
    const __nv_bfloat16* dz = nullptr;
    int rows = 0, cols = 0, ld = 0;
    const float* b_cur = nullptr;
    float* b_new = nullptr;
    float* b_copy = nullptr;
    int* tag_slot = nullptr;
    int* cur_version = nullptr;
    const int* trace_src = nullptr;
    int* trace_dst = nullptr;
    int version = 0;
    // loss
    const float* y = nullptr;
    const float* t = nullptr;
    const int* lab = nullptr;
    int ld_t = 0, loss = 0, act_last = 0, ld_dz = 0;
    float lr = 0.f;
    float denom = 1.f;
    __nv_bfloat16* dz_out = nullptr;
    float* row_loss = nullptr;
    // copy / memset
    void* dst = nullptr;
    const void* src = nullptr;
    size_t bytes = 0;
    int value = 0;
    // send / recv
    int peer = 0, dir = 0;
    // conv stages: images / size / channels (im2col, pooling), partial slabs
    // (reduce_sgd: S slabs of `slab` floats, rows x cols, lds)
    int n = 0, h = 0, w = 0, ch = 0;
    const __nv_bfloat16* in16 = nullptr;
    const __nv_bfloat16* aux16 = nullptr;
    __nv_bfloat16* out16 = nullptr;
    float* f32 = nullptr;
    const float* w_cur = nullptr;
    float* w_new = nullptr;
    int ldw = 0, ld16 = 0, S = 0;
    long long slab = 0;
    bool f32dz = false;  // bias: dz holds fp32 partial sums
    // logits forward with the softmax-CE fused into its epilogue, and the
    // loss op it replaces (both only when the targets are class labels)
    bool loss_fused = false;
  };

  const SessionConfig& cfg;
  int W, N, B, M, U, Rm;
  // fp32 verify precision: activation / delta / weight-copy buffers hold fp32
  // in the same layout; sc = bf16 slots per stored element (1 or 2)
  bool v32 = false;
  int sc = 1;
  bool pdl = false;  // GEMMs with programmatic dependent launch
  // split fp32 masters (gemm_sm100.cuh): version v's master is its pool
  // slot's bf16 weights (hi) plus lo[v % 2]; no separate fp32 masters
  bool split = false;
  // forwards and backwards of a stage on separate streams (split mode)
  bool split_fb = false;
  // bias gradients on their own stream (else on the wgrad side stream)
  bool bias_stream = true;
  std::vector<Stage> stages;
  // data
  __nv_bfloat16* x16 = nullptr;
  int ld_x = 0;
  float* y32 = nullptr;
  int* ylab = nullptr;        // class labels [rows] (labels upload: one-hot never materialised)
  bool use_labels = false;    // the last upload's targets were labels
  int graph_labels = -1;      // use_labels the resident graph was captured with
  int n_out = 0;
  void* stage_buf = nullptr;  // upload staging (f64 or f32 or i32)
  size_t stage_bytes = 0;
  float* row_loss = nullptr;
  int* fwd_trace = nullptr;  // [M][U][W]
  int* bwd_trace = nullptr;  // [M][W]
  // arena
  char* arena = nullptr;
  size_t arena_used = 0, arena_cap = 0;
  // program
  std::vector<Task> tasks;  // issue order
  std::vector<Op> ops;
  std::vector<cudaEvent_t> events;
  cudaStream_t origin = nullptr;
  cudaEvent_t t0 = nullptr, t1 = nullptr;
  cudaEvent_t fork_ev = nullptr;
  std::vector<cudaEvent_t> join_ev;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  // snapshots: [W][M+1] host pinned fp32
  std::vector<std::vector<float*>> snaps;
  int kernels = 0;
  int W_lo = 1, W_hi = 0;  // local stage range (1-based, inclusive)
  int rank = 0, world = 1;
  std::vector<int> owner;  // [stage 0-based] -> rank
  // profiling: node metadata (issue order) and its begin/end timing events
  std::vector<NodeTiming> node_meta;
  std::vector<cudaEvent_t> mark_ev;  // [2 * nodes], created on first profile
  bool profiling = false;
  std::vector<cudaEvent_t> kt_ev;  // [2 * timed launches]
  // streamed input (train_epoch from host buffers): the H2D copy and
  // conversion of mini-batch k's rows run on their own stream inside the
  // epoch; stage 1's forwards and the loss of mini k wait for x_ready[k]
  struct HostInput {
    const void* x = nullptr;
    const void* y = nullptr;
    HostDType xt = HostDType::f32, yt = HostDType::f32;
    bool operator==(const HostInput& o) const {
      return x == o.x && y == o.y && xt == o.xt && yt == o.yt;
    }
  };
  bool streaming = false;          // the program being issued uploads its input
  HostInput host_in;               // of the streamed graph
  cudaStream_t h2d = nullptr;   // copies (back to back on the copy engine)
  cudaStream_t h2dc = nullptr;  // conversions (high priority)
  std::vector<cudaEvent_t> x_ready, copy_ev;  // [M + 1]
  cudaGraph_t sgraph = nullptr;
  cudaGraphExec_t sexec = nullptr;
  HostInput sgraph_key;  // host buffers the streamed graph was captured with
  std::vector<double> kt_flops;    // [timed launches] 2*M*N*K
  // parameter transfers at the boundary (load / read of fp64 masters):
  // pinned double-buffered staging and per-layer device scratch
  std::unique_ptr<HostStager> stager;
  // device digests: scratch, one plan per digest (M per-mini + final), the
  // results [M + 1], and their stream
  std::unique_ptr<DeviceDigest> digest;
  std::vector<DeviceDigest::Plan> dplans;
  uint64_t* d_digest = nullptr;
  cudaStream_t dstream = nullptr;
  // the span table of every local stage's masters of `version(s)`
  std::vector<DigestSpan> digest_spans(const std::vector<int>& version) const {
    std::vector<DigestSpan> v;
    for (size_t s = 0; s < stages.size(); ++s) {
      const Stage& st = stages[s];
      const int ver = version[s], p = ver & 1;
      for (size_t l = 0; l < st.layers.size(); ++l) {
        const LayerDev& d = st.layers[l];
        DigestSpan w;
        w.rows = d.out;
        w.cols = d.in;
        if (split) {
          w.hi = st.pool[st.version_colour[ver]].w16[l];
          w.lo = d.lo[p];
          w.ld = d.ld_in;
        } else {
          w.f32 = d.w32[p];
          w.ld = d.in;
        }
        v.push_back(w);
        DigestSpan b;
        b.f32 = d.b32[p];
        b.rows = 1;
        b.cols = d.out;
        b.ld = d.out;
        v.push_back(b);
      }
    }
    return v;
  }
  double* p64 = nullptr;  // one layer's W then b, fp64
  float* p32 = nullptr;   // one layer's W, fp32
  size_t p_cap = 0;       // elements of p64 / p32
  bool staged_upload = false;  // Session::upload: pageable copies via the stager
  void ensure_stager() {
    if (!stager) stager = std::make_unique<HostStager>();
  }
  void copy_h2d(void* dst, const void* src, size_t bytes, cudaStream_t st) {
    if (staged_upload) {
      ensure_stager();
      stager->h2d(dst, src, bytes, st);
    } else {
      PB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
    }
  }
  void param_scratch() {
    if (p64) return;
    size_t mx = 0;
    for (auto& st : stages)
      for (auto& d : st.layers) mx = std::max(mx, static_cast<size_t>(d.in) * d.out + d.out);
    PB_CUDA(cudaMalloc(&p64, mx * 8));
    PB_CUDA(cudaMalloc(&p32, mx * 4));
    p_cap = mx;
    ensure_stager();
  }
  std::unique_ptr<P2P> p2p;
  // IPC peer-memory transport (SessionConfig::transport == 1)
  std::unique_ptr<IpcLink> ipc;
  std::vector<IpcLink::Msg> msgs;  // this rank's transfers in program order
  int add_msg(bool send, int dir, int peer, size_t bytes, const void* src, void* dst) {
    msgs.push_back(IpcLink::Msg{send, dir, peer, bytes, src, dst});
    return static_cast<int>(msgs.size()) - 1;
  }
  cudaStream_t comm[4] = {nullptr, nullptr, nullptr, nullptr};  // fwd send/recv, bwd send/recv
  bool local(int s0) const { return s0 >= W_lo - 1 && s0 <= W_hi - 1; }
  cudaStream_t stream_of(int idx) const {
    if (idx >= 0) return stages[idx].stream;
    if (idx <= kBiasBase) return stages[kBiasBase - idx].biasstream;
    if (idx <= kBwdBase) return stages[kBwdBase - idx].bstream;
    if (idx <= kSideBase) return stages[kSideBase - idx].side;
    if (idx == -1) return origin;
    if (idx == kDigest) return dstream;
    return comm[-idx - 2];
  }

  explicit Impl(const SessionConfig& c) : cfg(c) {}

  // PIPESIM_GUARD=1 (debugging): a 4 KB canary after every carve, checked
  // after each epoch (check_guards) -- finds kernels writing past a buffer
  // inside the one arena allocation, where compute-sanitizer cannot see it
  static constexpr size_t kGuard = 4096;
  bool guard = false;
  struct Carve {
    size_t off, bytes;
    std::string label;
  };
  std::vector<Carve> carves;
  template <typename T>
  T* carve(size_t count, const char* label = "") {
    size_t bytes = (count * sizeof(T) + kAlign - 1) / kAlign * kAlign;
    if (bytes == 0) bytes = kAlign;
    if (arena_used + bytes + (guard ? kGuard : 0) > arena_cap)
      throw std::runtime_error("arena overflow");
    T* p = reinterpret_cast<T*>(arena + arena_used);
    if (guard) carves.push_back(Carve{arena_used, bytes, label});
    arena_used += bytes + (guard ? kGuard : 0);
    return p;
  }
  void fill_guards() {
    for (const Carve& c : carves)
      PB_CUDA(cudaMemset(arena + c.off + c.bytes, 0xA5, kGuard));
  }
  // returns the number of buffers written past (messages on stderr)
  int check_guards() {
    int hits = 0;
    std::vector<unsigned char> h(kGuard);
    for (const Carve& c : carves) {
      PB_CUDA(cudaMemcpy(h.data(), arena + c.off + c.bytes, kGuard, cudaMemcpyDeviceToHost));
      size_t bad = 0, first = kGuard;
      for (size_t i = 0; i < kGuard; ++i)
        if (h[i] != 0xA5) {
          ++bad;
          first = std::min(first, i);
        }
      if (bad) {
        ++hits;
        std::fprintf(stderr, "PIPESIM_GUARD: %zu bytes written past '%s' (offset %zu, %zu bytes), "
                             "first at +%zu\n", bad, c.label.c_str(), c.off, c.bytes, first);
      }
    }
    return hits;
  }

  ~Impl() {
    if (sexec) cudaGraphExecDestroy(sexec);
    if (sgraph) cudaGraphDestroy(sgraph);
    if (h2d) cudaStreamDestroy(h2d);
    if (h2dc) cudaStreamDestroy(h2dc);
    for (cudaEvent_t e : mark_ev)
      if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : kt_ev)
      if (e) cudaEventDestroy(e);
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    if (!plan_only)
      for (cudaEvent_t e : events) cudaEventDestroy(e);
    if (t0) cudaEventDestroy(t0);
    if (t1) cudaEventDestroy(t1);
    for (Stage& s : stages) {
      if (s.stream) cudaStreamDestroy(s.stream);
      if (s.side) cudaStreamDestroy(s.side);
      if (s.bstream) cudaStreamDestroy(s.bstream);
      if (s.biasstream) cudaStreamDestroy(s.biasstream);
    }
    if (origin) cudaStreamDestroy(origin);
    for (cudaStream_t c : comm)
      if (c) cudaStreamDestroy(c);
    for (auto& v : snaps)
      for (float* p : v)
        if (p) cudaFreeHost(p);
    if (arena && !plan_only) cudaFree(arena);
    stager.reset();
    if (digest)
      for (auto& p : dplans) digest->free_plan(p);
    digest.reset();
    if (dstream) cudaStreamDestroy(dstream);
    if (p64) cudaFree(p64);
    if (p32) cudaFree(p32);
  }

  bool plan_only = false;
  uintptr_t fake_events = 0x10;
  cudaEvent_t new_event() {
    cudaEvent_t e;
    if (plan_only) return reinterpret_cast<cudaEvent_t>(fake_events += 0x10);
    PB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    events.push_back(e);
    return e;
  }
};

// ------------------------------------------------------------------ ctor
Session::Session(const SessionConfig& cfg_in) : cfg_(cfg_in) {
  SessionConfig& c = cfg_;
  const bool convnet = !c.layers.empty();
  if (convnet) {  // widths / acts of a layer list (per-sample elements)
    check_layers(c.layers);
    if (c.verify_fp32) throw std::invalid_argument("conv networks: bf16 precision only");
    c.widths.clear();
    c.acts.clear();
    for (const LayerSpec& l : c.layers) {
      c.widths.push_back(static_cast<int>(l.in_elems()));
      c.acts.push_back(l.act);
    }
    c.widths.push_back(static_cast<int>(c.layers.back().out_elems()));
  }
  if (c.widths.size() < 2 || c.acts.size() + 1 != c.widths.size())
    throw std::invalid_argument("bad network description");
  if (c.stage_hi == 0) c.stage_hi = c.W;
  if (c.B % (c.mode == RunMode::timeprest ? c.N : 1) != 0)
    throw pipesim::domain_error("mini_batch_size",
                                "mini-batch size " + std::to_string(c.B) +
                                    " is not divisible by micro-batch count " +
                                    std::to_string(c.N));
  if (!c.plan_only) {
    PB_CUDA(cudaSetDevice(c.device));
    init_gemm_attributes();
  }
  impl_ = std::make_unique<Impl>(cfg_);
  Impl& I = *impl_;
  I.plan_only = c.plan_only;
  I.v32 = c.verify_fp32;
  I.split_fb = c.split_fb;
  if (const char* e = std::getenv("PIPESIM_BIAS_STREAM")) I.bias_stream = std::atoi(e) != 0;
  if (const char* e = std::getenv("PIPESIM_SPLIT_FB")) I.split_fb = std::atoi(e) != 0;
  I.sc = c.verify_fp32 ? 2 : 1;
  I.W = c.W;
  I.N = c.N;
  I.B = c.B;
  I.M = c.M;
  I.U = units();
  I.Rm = c.B / I.U;
  const int W = c.W, M = c.M, U = I.U;
  I.rank = c.rank;
  I.world = c.world;
  if (c.world < 1 || c.rank < 0 || c.rank >= c.world || c.world > W)
    throw std::invalid_argument("bad rank/world for the stage count");
  I.owner.assign(W, 0);
  for (int s = 0; s < W; ++s) I.owner[s] = static_cast<int>((static_cast<long>(s) * c.world) / W);
  if (c.world > 1) {  // even contiguous split of the W stages over the ranks
    c.stage_lo = W + 1;
    c.stage_hi = 0;
    for (int s = 0; s < W; ++s)
      if (I.owner[s] == c.rank) {
        c.stage_lo = std::min(c.stage_lo, s + 1);
        c.stage_hi = std::max(c.stage_hi, s + 1);
      }
  } else {
    c.stage_lo = 1;
    c.stage_hi = W;
  }
  I.W_lo = c.stage_lo;
  I.W_hi = c.stage_hi;

  // ---------------- network partition (trainer.cpp:104-135)
  pipesim::network_spec net;
  net.widths = c.widths;
  for (int a : c.acts) net.activations.push_back(static_cast<pipesim::activation_kind>(a));
  net.loss = c.loss == 0 ? pipesim::loss_kind::mse : pipesim::loss_kind::softmax_cross_entropy;
  // stage s: layers [part_first[s], part_first[s] + part_count[s])
  std::vector<int> part_first(W), part_count(W);
  if (convnet) {
    std::vector<int> cnt = c.stage_layers.empty() ? partition_by_flops(c.layers, W) : c.stage_layers;
    if (static_cast<int>(cnt.size()) != W)
      throw std::invalid_argument("stage_layers must have one entry per stage");
    int f = 0;
    for (int s = 0; s < W; ++s) {
      if (cnt[s] < 1) throw std::invalid_argument("every stage needs at least one layer");
      part_first[s] = f;
      part_count[s] = cnt[s];
      f += cnt[s];
    }
    if (f != static_cast<int>(c.layers.size()))
      throw std::invalid_argument("stage_layers must cover the layers");
    total_params_ = 0;
    for (const LayerSpec& l : c.layers)
      total_params_ += static_cast<int64_t>(l.out) * l.fan_in() + l.out;
  } else {
    const std::vector<pipesim::stage_model> part = pipesim::partition_model(net, W);
    for (int s = 0; s < W; ++s) {
      part_first[s] = part[s].first_layer;
      part_count[s] = static_cast<int>(part[s].layers.size());
    }
    total_params_ = net.param_count();
  }

  // ---------------- plan
  // Per stage: ordered tasks (slot numbers) and the pins / prop versions.
  std::vector<std::vector<std::pair<int, int>>> version_iv(W);  // [s][v] = [from, freed)
  std::vector<std::vector<std::pair<int, int>>> act_iv(W);      // [s][k-1] = [first fwd, bwd]
  for (int s = 0; s < W; ++s) {
    version_iv[s].assign(M + 1, {0, 0});
    act_iv[s].assign(M, {1 << 30, 0});
  }

  if (c.mode == RunMode::sequential) {
    // sequential_epoch (trainer.cpp:510-553): whole mini-batch forward through
    // all stages, then backward W..1.  Synthetic slots keep the same machinery.
    int slot = 0;
    for (int k = 1; k <= M; ++k) {
      for (int s = 1; s <= W; ++s) {
        Impl::Task t;
        t.fwd = true;
        t.k = k;
        t.jj = 0;
        t.s = s;
        t.slot = ++slot;
        t.version = k - 1;
        I.tasks.push_back(t);
        auto& a = act_iv[s - 1][k - 1];
        a.first = std::min(a.first, t.slot);
      }
      for (int s = W; s >= 1; --s) {
        Impl::Task t;
        t.fwd = false;
        t.k = k;
        t.s = s;
        t.slot = ++slot;
        t.version = k - 1;
        I.tasks.push_back(t);
        act_iv[s - 1][k - 1].second = t.slot;
        version_iv[s - 1][k].first = t.slot;
        if (k >= 1) version_iv[s - 1][k - 1].second = t.slot + 1;
      }
    }
    for (int s = 0; s < W; ++s) version_iv[s][M].second = slot + 1;
    horizon_ = slot;
    ledger_.cfg.workers = W;
    ledger_.cfg.micro_batches = c.N;
    ledger_.cfg.mini_batches = M;
    for (int k = 1; k <= M; ++k) {
      ledger_.pins.push_back({k, 0, 0, k - 1});
      ledger_.update_source.push_back(k - 1);
    }
  } else {
    pipesim::sim_config sc;
    sc.workers = W;
    sc.micro_batches = c.N;
    sc.mini_batches = M;
    sc.samples_per_mini_batch = c.B;
    const bool nf1b = c.mode == RunMode::timeprest;
    grid_ = std::make_unique<pipesim::schedule_grid>(
        nf1b ? pipesim::build_nf1b_schedule(sc) : pipesim::build_1f1b_schedule(sc));
    ledger_ = pipesim::assign_versions(*grid_, sc);
    const pipesim::retention_timeline rt =
        pipesim::build_retention_timeline(ledger_, *grid_);
    horizon_ = grid_->horizon();
    std::map<std::pair<int, int>, int> pin;
    for (const auto& p : ledger_.pins) pin[{p.mini, p.micro}] = p.version;
    for (int t = 1; t <= horizon_; ++t)
      for (int s = 1; s <= W; ++s) {
        const pipesim::task& cell = grid_->at(s, t);
        if (cell.is_idle()) continue;
        Impl::Task tk;
        tk.fwd = cell.is_forward();
        tk.k = cell.mini;
        tk.s = s;
        tk.slot = t;
        if (tk.fwd) {
          tk.jj = nf1b ? cell.micro - 1 : 0;
          tk.version = pin.at({cell.mini, cell.micro});
          auto& a = act_iv[s - 1][tk.k - 1];
          a.first = std::min(a.first, t);
        } else {
          // nF1B propagates through the latest stage weights (trainer.cpp:479-480);
          // 1F1B through the stashed pin.  Per-stage latest == k-1 (commits in order).
          tk.version = nf1b ? tk.k - 1 : pin.at({cell.mini, 0});
          act_iv[s - 1][tk.k - 1].second = t;
        }
        I.tasks.push_back(tk);
      }
    for (int s = 0; s < W; ++s)
      for (int v = 0; v <= M; ++v)
        version_iv[s][v] = {rt.per_stage[s][v].retained_from_slot,
                            rt.per_stage[s][v].freed_at_slot};
  }

  // A stage fed over the network receives its input while the upstream stage
  // produces it, so its activation slot is held from the upstream forward.
  for (int s0 = 1; s0 < W; ++s0)
    if (I.owner[s0 - 1] != I.owner[s0])
      for (int k = 0; k < M; ++k)
        act_iv[s0][k].first = std::min(act_iv[s0][k].first, act_iv[s0 - 1][k].first);

  // Latency-bound networks (every Linear layer at most 1024 wide, no conv):
  // GEMMs use programmatic dependent launch (GemmLaunch::pdl), and every
  // stage holds one spare activation slot -- a mini-batch's slot stays
  // reserved until the next one's first forward, so that forward does not
  // wait for the previous backward's weight gradient, which reads the slot
  // (hazard (b); C1 45.6 -> see DESIGN.md; PIPESIM_SPARE_ACT=0: off).
  bool latency = !convnet;
  for (size_t l = 0; l + 1 < c.widths.size() && latency; ++l)
    if (c.widths[l] > 1024 || c.widths[l + 1] > 1024) latency = false;
  {
    const char* e = std::getenv("PIPESIM_SPARE_ACT");
    if (latency && !(e && std::string(e) == "0"))
      for (int s0 = 0; s0 < W; ++s0)
        for (int k = 0; k + 1 < M; ++k)
          act_iv[s0][k].second = std::max(act_iv[s0][k].second, act_iv[s0][k + 1].first);
  }

  // ---------------- colouring: version pool and activation slots
  I.stages.resize(W);
  std::vector<int> pool_n(W), act_n(W);
  for (int s = 0; s < W; ++s) {
    Impl::Stage& st = I.stages[s];
    st.id = s + 1;
    st.first_layer = part_first[s];
    st.L = part_count[s];
    st.version_colour = colour(version_iv[s], &pool_n[s], /*half_open=*/true);
    std::vector<int> ac = colour(act_iv[s], &act_n[s], /*half_open=*/false);
    st.mini_act.assign(M + 1, 0);
    for (int k = 1; k <= M; ++k) st.mini_act[k] = ac[k - 1];
  }

  // ---------------- split masters: every local layer's wgrad+SGD must run the
  // pair kernel's TMA epilogue (the verify precision and per-slot snapshots
  // keep fp32 masters)
  I.split = !I.v32 && !c.snapshots && !convnet;
  for (int s = 0; s < W && I.split; ++s) {
    if (!I.local(s)) continue;
    for (int gl = part_first[s]; gl < part_first[s] + part_count[s]; ++gl)
      if (!split_master_eligible(c.widths[gl + 1], c.widths[gl], ld8(c.widths[gl])))
        I.split = false;
  }

  I.pdl = latency;
  // Skinny forwards split K (lower latency, more SM-time) when this process
  // keeps few stages in flight; PIPESIM_SESSION_SPLIT=0/1 overrides.
  bool split_fwd = I.W_hi - I.W_lo + 1 <= 2;
  if (const char* e = std::getenv("PIPESIM_SESSION_SPLIT")) split_fwd = std::atoi(e) != 0;
  if (I.v32) split_fwd = false;
  // softmax-CE fused into the logits forward (small class counts, linear
  // head; applied when the targets are class labels): the loss kernel leaves
  // the backward's critical path.  PIPESIM_LOSS_FUSE=0 disables.
  // backwards wait for the downstream delta, not the downstream updates
  // (PIPESIM_DELTA_EDGES=0: the whole downstream backward, as before)
  bool delta_edges = true;
  if (const char* e = std::getenv("PIPESIM_DELTA_EDGES")) delta_edges = std::atoi(e) != 0;
  // forwards wait for the commit of their pinned version only (not for the
  // dgrad chain of that backward); PIPESIM_COMMIT_EDGES=0: the whole backward
  bool commit_edges = !c.snapshots;
  if (const char* e = std::getenv("PIPESIM_COMMIT_EDGES")) commit_edges = commit_edges && std::atoi(e) != 0;
  bool loss_fuse = !I.v32 && c.loss == 1 && c.acts.back() == kLinear && c.widths.back() <= 16;
  if (const char* e = std::getenv("PIPESIM_LOSS_FUSE")) loss_fuse = loss_fuse && std::atoi(e) != 0;

  // ---------------- sizes
  I.n_out = c.widths.back();
  I.ld_x = ld8(c.widths.front());
  auto bytes_of = [](size_t n, size_t sz) { return (n * sz + kAlign - 1) / kAlign * kAlign + kAlign; };
  size_t need = 0;
  int64_t off = 0;
  for (int s = 0; s < W; ++s) {
    Impl::Stage& st = I.stages[s];
    st.param_offset = off;
    size_t wb = 0, ab = 0;
    for (int l = 0; l < st.L; ++l) {
      const int gl = st.first_layer + l;
      Impl::LayerDev d;
      d.in = c.widths[gl];
      d.out = c.widths[gl + 1];
      d.act = c.acts[gl];
      d.ld_in = ld8(d.in);
      d.ld_out = ld8(d.out);
      d.ain = d.ld_in;
      d.aout = d.ld_out;
      if (convnet) {
        const LayerSpec& ls = c.layers[gl];
        d.in = ls.fan_in();
        d.out = ls.out;
        d.ld_in = ld8(d.in);
        d.ld_out = ld8(d.out);
        // activation rows: exact NHWC elements for conv layers (channels are
        // multiples of 64), the 8-aligned leading dimensions for linear ones
        // (their kernels address rows with ld_in / ld_out)
        d.ain = ls.kind == LayerKind::linear ? d.ld_in : static_cast<int>(ls.in_elems());
        d.aout = ls.kind == LayerKind::linear ? d.ld_out : static_cast<int>(ls.out_elems());
        if (ls.kind == LayerKind::conv3x3) {
          d.conv = true;
          d.pool = ls.pool;
          d.cin = ls.in;
          d.h = ls.h;
          d.w = ls.w;
          d.first_conv = gl == 0 && ls.in % 64 != 0;
          d.pre_elems = d.pool ? static_cast<int64_t>(ls.h) * ls.w * ls.out : 0;
        }
      }
      st.layers.push_back(d);
      st.param_count += static_cast<int64_t>(d.in) * d.out + d.out;
      if (!I.local(s)) continue;
      wb += 2 * ((I.split ? bytes_of(static_cast<size_t>(d.out) * d.ld_in, 2)
                          : bytes_of(static_cast<size_t>(d.in) * d.out, 4)) +
                 bytes_of(d.out, 4));
      wb += pool_n[s] * (bytes_of(static_cast<size_t>(d.out) * d.ld_in, 2 * I.sc) + bytes_of(d.out, 4));
      ab += act_n[s] * bytes_of(static_cast<size_t>(c.B) * d.aout, 2 * I.sc);
      if (l + 1 < st.L) ab += bytes_of(static_cast<size_t>(c.B) * d.aout, 2 * I.sc);
      if (d.pool)  // conv output before pooling (slots) + its delta (scratch)
        ab += (act_n[s] + 1) * bytes_of(static_cast<size_t>(c.B) * d.pre_elems, 2);
      if (d.first_conv)
        ab += act_n[s] * bytes_of(static_cast<size_t>(c.B) * d.h * d.w * d.ld_in, 2);
      if (split_fwd && !d.conv) {
        for (int j = 1; j <= U; ++j)
          st.fix_floats = std::max(st.fix_floats, fwd_fix_floats(j * I.Rm, d.out, d.in));
        st.fix_counters = std::max(st.fix_counters, fwd_fix_counters(c.B, d.out));
      }
      if (d.conv) {
        int lds = 0;
        const size_t f = d.first_conv ? wgrad_partial_floats(d.out, d.ld_in, c.B * d.h * d.w, &lds)
                                      : conv_wgrad_floats(d.out, d.cin, c.B * d.h * d.w);
        st.wg_floats = std::max(st.wg_floats, f);
        st.bias_floats = std::max(st.bias_floats, static_cast<size_t>(kColsumChunks) * d.out);
      }
    }
    off += st.param_count;
    if (!I.local(s)) continue;
    wb += bytes_of(st.wg_floats, 4) + bytes_of(st.bias_floats, 4);
    if (st.fix_floats) ab += bytes_of(st.fix_floats, 4) + bytes_of(st.fix_counters, 4);
    if (s > 0 && !I.local(s - 1))  // boundary buffers: received input + outgoing delta
      ab += 2 * act_n[s] * bytes_of(static_cast<size_t>(c.B) * st.layers.front().ain, 2 * I.sc);
    wb += pool_n[s] * bytes_of(1, 4) + bytes_of(1, 4);
    ab += act_n[s] * bytes_of(static_cast<size_t>(c.B) * st.layers.back().aout, 2 * I.sc);
    if (s == W - 1) ab += act_n[s] * bytes_of(static_cast<size_t>(c.B) * I.n_out, 4);
    st.bytes_weights = static_cast<int64_t>(wb);
    st.bytes_acts = static_cast<int64_t>(ab);
    need += wb + ab;
  }
  const size_t rows = static_cast<size_t>(M) * c.B;
  need += bytes_of(rows * I.ld_x, 2 * I.sc) + bytes_of(rows * I.n_out, 4) + bytes_of(rows, 4) +
          bytes_of(rows, 4);
  // upload staging: x rows (f64 at most) then y rows (f64 at most)
  I.stage_bytes = rows * (static_cast<size_t>(c.widths.front()) + I.n_out) * 8;
  need += bytes_of(I.stage_bytes, 1);
  need += bytes_of(static_cast<size_t>(M) * U * W, 4) + bytes_of(static_cast<size_t>(M) * W, 4);
  need += bytes_of(static_cast<size_t>(M) + 1, 8);
  need += 64 * kAlign;

  if (const char* e = std::getenv("PIPESIM_GUARD")) I.guard = std::atoi(e) != 0 && !c.plan_only;
  if (I.guard) need += need + (size_t{1} << 26);  // canaries (debugging only)
  if (c.plan_only) {
    I.arena = reinterpret_cast<char*>(uintptr_t{1} << 40);  // addresses only, never touched
  } else {
    PB_CUDA(cudaMalloc(&I.arena, need));
    PB_CUDA(cudaMemset(I.arena, 0, need));
  }
  I.arena_cap = need;
  arena_bytes_ = static_cast<int64_t>(need);

  for (int s = 0; s < W; ++s) {
    Impl::Stage& st = I.stages[s];
    if (!I.local(s)) continue;
    for (auto& d : st.layers)
      for (int p = 0; p < 2; ++p) {
        if (I.split)
          d.lo[p] = I.carve<uint16_t>(static_cast<size_t>(d.out) * d.ld_in, "master lo");
        else
          d.w32[p] = I.carve<float>(static_cast<size_t>(d.in) * d.out, "master w32");
        d.b32[p] = I.carve<float>(d.out, "master b32");
      }
    st.pool.resize(pool_n[s]);
    for (auto& ps : st.pool) {
      for (auto& d : st.layers) {
        ps.w16.push_back(I.carve<__nv_bfloat16>(static_cast<size_t>(d.out) * d.ld_in * I.sc, "pool w16"));
        ps.b32.push_back(I.carve<float>(d.out, "pool b32"));
      }
      ps.tag = I.carve<int>(1, "pool tag");
    }
    st.cur_version = I.carve<int>(1);
    st.acts.resize(act_n[s]);
    for (auto& as : st.acts) {
      for (int l = 0; l < st.L; ++l) {
        const auto& d = st.layers[l];
        const bool logits = (s == W - 1) && (l == st.L - 1);
        as.out16.push_back(logits ? nullptr
                                  : I.carve<__nv_bfloat16>(static_cast<size_t>(c.B) * I.sc *
                                                           d.aout, "slot out16"));
        as.pre16.push_back(d.pool ? I.carve<__nv_bfloat16>(static_cast<size_t>(c.B) * d.pre_elems)
                                  : nullptr);
        if (d.first_conv)
          as.cols16 = I.carve<__nv_bfloat16>(static_cast<size_t>(c.B) * d.h * d.w * d.ld_in);
      }
      if (s == W - 1) as.out32 = I.carve<float>(static_cast<size_t>(c.B) * I.n_out, "slot out32");
      as.dzin = I.carve<__nv_bfloat16>(static_cast<size_t>(c.B) * st.layers.back().aout * I.sc, "slot dzin");
      if (s > 0 && !I.local(s - 1)) {
        as.in16 = I.carve<__nv_bfloat16>(static_cast<size_t>(c.B) * st.layers.front().ain * I.sc);
        as.dzsend = I.carve<__nv_bfloat16>(static_cast<size_t>(c.B) * st.layers.front().ain * I.sc);
      }
    }
    for (int l = 0; l + 1 < st.L; ++l)
      st.scratch_dz.push_back(
          I.carve<__nv_bfloat16>(static_cast<size_t>(c.B) * st.layers[l].aout * I.sc, "scratch dz"));
    for (int l = 0; l < st.L; ++l)
      st.scratch_pre.push_back(
          st.layers[l].pool
              ? I.carve<__nv_bfloat16>(static_cast<size_t>(c.B) * st.layers[l].pre_elems)
              : nullptr);
    if (st.wg_floats) st.wg_ws = I.carve<float>(st.wg_floats);
    if (st.fix_floats) {  // the arena is zeroed: counters start at 0
      st.fix_ws = I.carve<float>(st.fix_floats);
      st.fix_cnt = I.carve<int>(st.fix_counters);
    }
    if (st.bias_floats) st.bias_ws = I.carve<float>(st.bias_floats);
  }
  I.x16 = I.carve<__nv_bfloat16>(rows * I.ld_x * I.sc);
  I.y32 = I.carve<float>(rows * I.n_out);
  I.ylab = I.carve<int>(rows);
  I.row_loss = I.carve<float>(rows);
  I.stage_buf = I.carve<char>(I.stage_bytes);
  I.fwd_trace = I.carve<int>(static_cast<size_t>(M) * U * W);
  I.bwd_trace = I.carve<int>(static_cast<size_t>(M) * W);
  I.d_digest = I.carve<uint64_t>(static_cast<size_t>(M) + 1);
  if (I.guard) I.fill_guards();

  if (!c.plan_only) {
  PB_CUDA(cudaStreamCreateWithFlags(&I.origin, cudaStreamNonBlocking));
  if (c.digests) PB_CUDA(cudaStreamCreateWithFlags(&I.dstream, cudaStreamNonBlocking));
  // Stream priorities (PIPESIM_PRIO): 0 all equal; 1 stage streams (forwards,
  // loss, the dgrad chain) above the side streams (wgrad + SGD); 2 also
  // later stages above earlier ones (their backwards start the chain).
  int prio_mode = 0;
  if (const char* e = std::getenv("PIPESIM_PRIO")) prio_mode = std::atoi(e);
  int lo_prio = 0, hi_prio = 0;
  PB_CUDA(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));  // hi is numerically lower
  for (int s = 0; s < W; ++s)
    if (I.local(s)) {
      int ps = lo_prio, pside = lo_prio;
      if (prio_mode >= 1) ps = hi_prio;
      if (prio_mode == 2) ps = std::max(hi_prio, lo_prio - 1 - s * (lo_prio - hi_prio) / W);
      // PIPESIM_PRIO=3: backward (dgrad chain) streams above forwards above
      // the wgrad / bias streams
      int pb = ps;
      if (prio_mode == 3) {
        pb = hi_prio;
        ps = std::min(lo_prio, hi_prio + 1);
      }
      PB_CUDA(cudaStreamCreateWithPriority(&I.stages[s].stream, cudaStreamNonBlocking, ps));
      if (c.side_streams) {
        PB_CUDA(cudaStreamCreateWithPriority(&I.stages[s].side, cudaStreamNonBlocking, pside));
        PB_CUDA(cudaStreamCreateWithPriority(&I.stages[s].biasstream, cudaStreamNonBlocking, pside));
      }
      if (I.split_fb)
        PB_CUDA(cudaStreamCreateWithPriority(&I.stages[s].bstream, cudaStreamNonBlocking, pb));
    }
  if (c.world > 1) {
    for (cudaStream_t& cs : I.comm) PB_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    if (c.transport == 0)
      I.p2p = std::make_unique<P2P>(c.rank, c.world, c.nccl_ids.data(), c.nccl_ids.size());
  }
  PB_CUDA(cudaEventCreate(&I.t0));
  PB_CUDA(cudaEventCreate(&I.t1));
  }  // !plan_only

  if (c.snapshots && !c.plan_only) {
    I.snaps.assign(W, std::vector<float*>(M + 1, nullptr));
    for (int s = 0; s < W; ++s)
      for (int v = 0; v <= M && I.local(s); ++v)
        PB_CUDA(cudaMallocHost(&I.snaps[s][v], sizeof(float) * std::max<int64_t>(1, I.stages[s].param_count)));
  }

  // ---------------- compile the program into ops
  using OK = Impl::OpKind;
  auto push = [&](Impl::Op op) {
    op.g.pdl = I.pdl;
    op.chain.pdl = I.pdl;
    op.fchain.pdl = I.pdl;
    const int kind = op.kind == OK::fwd ? 1 : op.kind == OK::dgrad ? 2 : op.kind == OK::wgrad ? 3 : 0;
    const bool timed = kind != 0 && kind == c.timed_kernel && !c.plan_only;
    if (timed) {
      Impl::Op t{OK::ktime};
      t.stream = op.stream;
      t.value = static_cast<int>(I.kt_ev.size());
      cudaEvent_t e0, e1;
      PB_CUDA(cudaEventCreate(&e0));
      PB_CUDA(cudaEventCreate(&e1));
      I.kt_ev.push_back(e0);
      I.kt_ev.push_back(e1);
      I.kt_flops.push_back(2.0 * op.g.sh.M * op.g.sh.N * op.g.sh.K);
      I.ops.push_back(t);
      I.ops.push_back(op);
      t.value += 1;
      I.ops.push_back(t);
      return;
    }
    I.ops.push_back(op);
  };
  const int last_s = W - 1;

  // Rebase (trainer.cpp:372-379): version 0 of this epoch = the previous
  // epoch's final version.  Masters ping-pong by parity, pool colours are
  // fixed by the plan, so copy when they differ.
  for (int s = 0; s < W; ++s) {
    if (!I.local(s)) continue;
    Impl::Stage& st = I.stages[s];
    const int cM = st.version_colour[M], c0 = st.version_colour[0];
    for (int l = 0; l < st.L; ++l) {
      auto& d = st.layers[l];
      if (M % 2 == 1) {
        Impl::Op o{OK::copy};
        o.stream = s;
        if (I.split) {
          o.dst = d.lo[0];
          o.src = d.lo[1];
          o.bytes = sizeof(uint16_t) * d.out * static_cast<size_t>(d.ld_in);
        } else {
          o.dst = d.w32[0];
          o.src = d.w32[1];
          o.bytes = sizeof(float) * d.in * static_cast<size_t>(d.out);
        }
        push(o);
        o.dst = d.b32[0];
        o.src = d.b32[1];
        o.bytes = sizeof(float) * d.out;
        push(o);
      }
      if (cM != c0) {
        Impl::Op o{OK::copy};
        o.stream = s;
        o.dst = st.pool[c0].w16[l];
        o.src = st.pool[cM].w16[l];
        o.bytes = sizeof(__nv_bfloat16) * I.sc * d.out * static_cast<size_t>(d.ld_in);
        push(o);
        o.dst = st.pool[c0].b32[l];
        o.src = st.pool[cM].b32[l];
        o.bytes = sizeof(float) * d.out;
        push(o);
      }
    }
    Impl::Op z{OK::memset_i32};
    z.stream = s;
    z.dst = st.pool[c0].tag;
    z.value = 0;
    push(z);
    z.dst = st.cur_version;
    push(z);
    if (c.digests && !c.plan_only) {  // the digest stream starts after the rebase
      Impl::Op r{OK::record};
      r.stream = s;
      r.ev = I.new_event();
      push(r);
      Impl::Op w{OK::wait};
      w.stream = Impl::kDigest;
      w.ev = r.ev;
      push(w);
    }
  }


  // per stage: pool colour of every version; previous occupant of each
  // mini-batch's activation slot (0: none)
  std::vector<std::vector<int>> stage_version_colour(W), act_prev_occupant(W);
  for (int s0 = 0; s0 < W; ++s0) {
    stage_version_colour[s0] = I.stages[s0].version_colour;
    act_prev_occupant[s0].assign(M + 1, 0);
    std::map<int, int> last;
    for (int k = 1; k <= M; ++k) {
      auto it = last.find(I.stages[s0].mini_act[k]);
      act_prev_occupant[s0][k] = it == last.end() ? 0 : it->second;
      last[I.stages[s0].mini_act[k]] = k;
    }
  }

  // ---------------- program: coalesce forwards, order the task DAG
  // A node is one backward task, or a run of consecutive forward tasks of one
  // stage with the same mini-batch and the same pinned version (coalesced
  // into one taller GEMM per layer: GEMM rows are independent, so the result
  // is bit-identical to per-micro-batch launches; each micro-batch's version
  // tag is still written to the device trace).
  struct Node {
    bool fwd;
    int s, k, version, jj0, jj1;  // s 0-based; forward micro range [jj0, jj1]
    int order;                     // position of the first member in issue order
    std::vector<int> deps;         // node ids (same-stage predecessor + cross-stage)
    // forward: hazard-(a) deps (the commit of its pinned version: only the
    // backward's wgrad / bias streams, not its dgrad chain), and the
    // hazard-(b) dep (slot reuse: the whole backward)
    std::vector<int> commit_deps;
    int slot_dep = -1;
    // backward: events on its wgrad and bias streams after the commit
    cudaEvent_t commit_side = nullptr, commit_bias = nullptr;
    cudaEvent_t done = nullptr;
    // backward of a stage s > 0: the delta for stage s-1 is written (its
    // wgrad / bias work on the side streams may still run)
    cudaEvent_t delta_done = nullptr;
    int digest = -1;               // >= 0: in-epoch digest node (index into dplans)
  };
  std::vector<Node> nodes;
  std::vector<std::vector<int>> digest_version;  // [digest][stage] version read
  const int merge = c.fwd_merge > 0 ? c.fwd_merge : U;
  {
    // last_on_stage: stream-order predecessor (split mode: per kind)
    std::vector<int> open(W, -1), last_on_stage(W, -1), last_fwd(W, -1), last_bwd(W, -1);
    std::map<std::tuple<int, int, int>, int> fwd_node;  // (k, jj, s) -> node
    std::map<std::pair<int, int>, int> bwd_node;         // (k, s) -> node
    int order = 0;
    for (const Impl::Task& tk : I.tasks) {
      const int s = tk.s - 1;
      ++order;
      if (tk.fwd) {
        const int o = open[s];
        if (o >= 0 && nodes[o].k == tk.k && nodes[o].version == tk.version &&
            nodes[o].jj1 + 1 == tk.jj && nodes[o].jj1 - nodes[o].jj0 + 1 < merge) {
          nodes[o].jj1 = tk.jj;
          fwd_node[{tk.k, tk.jj, s}] = o;
          continue;
        }
        Node n{true, s, tk.k, tk.version, tk.jj, tk.jj, order, {}};
        const int pred = I.split_fb ? last_fwd[s] : last_on_stage[s];
        if (pred >= 0) n.deps.push_back(pred);
        nodes.push_back(n);
        const int id = static_cast<int>(nodes.size()) - 1;
        open[s] = last_on_stage[s] = last_fwd[s] = id;
        fwd_node[{tk.k, tk.jj, s}] = id;
      } else {
        // a backward ends a coalescing run unless forwards have their own
        // stream (then a run may span it: same mini, same pinned version)
        if (!I.split_fb) open[s] = -1;
        Node n{false, s, tk.k, tk.version, 0, 0, order, {}};
        const int pred = I.split_fb ? last_bwd[s] : last_on_stage[s];
        if (pred >= 0) n.deps.push_back(pred);
        nodes.push_back(n);
        const int id = static_cast<int>(nodes.size()) - 1;
        last_on_stage[s] = last_bwd[s] = id;
        bwd_node[{tk.k, s}] = id;
      }
    }
    if (I.split_fb) {
      // Split mode: the hazards the single stage stream ordered by slot are
      // explicit edges (all point forward in slot order, so the DAG stays
      // acyclic):
      //  (a) a forward reads its pinned version v: after the commit of v on
      //      this stage (the backward of mini v);
      //  (b) the first forward of mini k writes activation slot colour(k):
      //      after the backward of the slot's previous occupant;
      //  (c) the backward of mini k reads mini k's activations: after the
      //      last forward of mini k on this stage;
      //  (d) the commit of version k overwrites pool colour(k): after the
      //      last forward that read the colour's previous version.
      std::map<std::pair<int, int>, int> last_fwd_of_mini, last_reader, first_fwd;
      for (int i = 0; i < static_cast<int>(nodes.size()); ++i) {
        const Node& n = nodes[i];
        if (!n.fwd) continue;
        last_fwd_of_mini[{n.k, n.s}] = i;
        last_reader[{n.version, n.s}] = i;
        if (!first_fwd.count({n.k, n.s})) first_fwd[{n.k, n.s}] = i;
      }
      for (int i = 0; i < static_cast<int>(nodes.size()); ++i) {
        Node& n = nodes[i];
        const auto& colour = stage_version_colour[n.s];
        if (n.fwd) {
          if (n.version >= 1) {                                                 // (a)
            n.deps.push_back(bwd_node.at({n.version, n.s}));
            n.commit_deps.push_back(n.deps.back());
          }
          if (first_fwd.at({n.k, n.s}) == i) {                                  // (b)
            const int pk = act_prev_occupant[n.s][n.k];
            if (pk > 0) {
              n.deps.push_back(bwd_node.at({pk, n.s}));
              n.slot_dep = n.deps.back();
            }
          }
        } else {
          n.deps.push_back(last_fwd_of_mini.at({n.k, n.s}));  // (c)
          int prev_v = -1;                                     // (d)
          for (int v = n.k - 1; v >= 0; --v)
            if (colour[v] == colour[n.k]) {
              prev_v = v;
              break;
            }
          if (prev_v >= 0) {
            auto it = last_reader.find({prev_v, n.s});
            if (it != last_reader.end()) n.deps.push_back(it->second);
          }
        }
      }
    }
    // The backward of mini k on stage s waits only for the delta of stage
    // s+1's backward (delta_done), not for stage s+1's weight / bias updates
    // still running on its side streams -- they read stage s's activation
    // slot of mini k (the wgrad operand x), so stage s's reuse of that slot
    // (its first forward of the slot's next occupant) waits for stage s+1's
    // whole backward of the previous occupant instead: edge (b').
    std::map<std::pair<int, int>, int> first_fwd_node;
    for (int i = 0; i < static_cast<int>(nodes.size()); ++i)
      if (nodes[i].fwd && !first_fwd_node.count({nodes[i].k, nodes[i].s}))
        first_fwd_node[{nodes[i].k, nodes[i].s}] = i;
    for (int i = 0; i < static_cast<int>(nodes.size()); ++i) {
      Node& n = nodes[i];
      if (!n.fwd || n.s + 1 >= W || first_fwd_node.at({n.k, n.s}) != i) continue;
      const int pk = act_prev_occupant[n.s][n.k];
      if (pk > 0) n.deps.push_back(bwd_node.at({pk, n.s + 1}));  // (b')
    }
    for (Node& n : nodes) {
      if (n.fwd && n.s > 0)
        for (int jj = n.jj0; jj <= n.jj1; ++jj) n.deps.push_back(fwd_node.at({n.k, jj, n.s - 1}));
      if (!n.fwd && n.s < last_s) n.deps.push_back(bwd_node.at({n.k, n.s + 1}));
      std::sort(n.deps.begin(), n.deps.end());
      n.deps.erase(std::unique(n.deps.begin(), n.deps.end()), n.deps.end());
    }
    // In-epoch digests (trainer.cpp:492-501): digest k reads, on every stage,
    // the version current when stage 1 commits mini k (stage s > 1: its latest
    // commit in an earlier slot); it runs after those commits and before each
    // stage's commit two versions later, which overwrites that version's
    // master residual / pool slot.  Both edges point forward in slot order,
    // so the DAG stays acyclic.  Digest M+1 is the final one (:506).
    if (c.digests && !c.plan_only) {
      if (c.world > 1)
        throw std::invalid_argument("in-epoch digests need every stage in one process");
      int max_order = 0;
      for (const Node& n : nodes) max_order = std::max(max_order, n.order);
      for (int k = 1; k <= M + 1; ++k) {
        std::vector<int> vs(W, std::min(k, M));
        if (grid_ && k <= M) {
          const int t1 = grid_->backward_slot(k, 1);
          for (int s0 = 1; s0 < W; ++s0) {
            int v = 0;
            for (int u = 1; u <= M; ++u)
              if (grid_->backward_slot(u, s0 + 1) < t1) v = u;
            vs[s0] = v;
          }
        }
        digest_version.push_back(vs);
        Node n{false, -1, std::min(k, M), 0, 0, 0,
               k <= M ? nodes[bwd_node.at({k, 0})].order : max_order + 1, {}};
        n.digest = k - 1;
        for (int s0 = 0; s0 < W; ++s0)
          if (vs[s0] >= 1) n.deps.push_back(bwd_node.at({vs[s0], s0}));
        nodes.push_back(n);
        const int id = static_cast<int>(nodes.size()) - 1;
        for (int s0 = 0; s0 < W; ++s0)
          if (vs[s0] + 2 <= M) nodes[bwd_node.at({vs[s0] + 2, s0})].deps.push_back(id);
      }
    }
  }
  // Kahn's algorithm, earliest original position first.
  std::vector<int> topo;
  {
    const int n = static_cast<int>(nodes.size());
    std::vector<int> indeg(n, 0);
    std::vector<std::vector<int>> succ(n);
    for (int i = 0; i < n; ++i)
      for (int d : nodes[i].deps) {
        ++indeg[i];
        succ[d].push_back(i);
      }
    std::vector<int> ready;
    for (int i = 0; i < n; ++i)
      if (indeg[i] == 0) ready.push_back(i);
    auto later = [&](int x, int y) { return nodes[x].order > nodes[y].order; };
    std::make_heap(ready.begin(), ready.end(), later);
    while (!ready.empty()) {
      std::pop_heap(ready.begin(), ready.end(), later);
      const int i = ready.back();
      ready.pop_back();
      topo.push_back(i);
      for (int j : succ[i])
        if (--indeg[j] == 0) {
          ready.push_back(j);
          std::push_heap(ready.begin(), ready.end(), later);
        }
    }
    if (static_cast<int>(topo.size()) != n)
      throw std::logic_error("coalesced task graph has a cycle");
  }

  auto stage_input = [&](int s, int k, int* row_off) -> Mat16 {
    // Activation entering stage s (0-based) for mini k: data rows or the
    // previous stage's output slot.
    if (s == 0) {
      *row_off = (k - 1) * c.B;
      return Mat16{I.x16, M * c.B, c.widths.front(), I.ld_x};
    }
    *row_off = 0;
    if (!I.local(s - 1)) {  // received over the network into this stage's slot
      const Impl::Stage& me = I.stages[s];
      const auto& fl = me.layers.front();
      return Mat16{me.acts[me.mini_act[k]].in16, c.B, fl.conv ? fl.ain : fl.in, fl.ain};
    }
    const Impl::Stage& pv = I.stages[s - 1];
    const auto& pl = pv.layers.back();
    return Mat16{pv.acts[pv.mini_act[k]].out16.back(), c.B, pl.conv ? pl.aout : pl.out,
                 pl.aout};
  };

  // Cross-GPU plumbing.  Previous occupant of each activation slot (slot reuse
  // guard for receives), first local forward node of each (k, s), and the
  // receive events (posted lazily, in the sender's order).
  std::vector<std::vector<int>> prev_occ(W, std::vector<int>(M + 1, 0));
  for (int s0 = 0; s0 < W; ++s0) {
    std::map<int, int> last;
    for (int k = 1; k <= M; ++k) {
      auto it = last.find(I.stages[s0].mini_act[k]);
      prev_occ[s0][k] = it == last.end() ? 0 : it->second;
      last[I.stages[s0].mini_act[k]] = k;
    }
  }
  std::map<std::pair<int, int>, int> bwd_id, first_fwd_id;  // (k, s0) -> node
  for (int i = 0; i < static_cast<int>(nodes.size()); ++i) {
    if (nodes[i].digest >= 0) continue;
    if (!nodes[i].fwd) bwd_id[{nodes[i].k, nodes[i].s}] = i;
    else if (!first_fwd_id.count({nodes[i].k, nodes[i].s})) first_fwd_id[{nodes[i].k, nodes[i].s}] = i;
  }
  std::map<int, cudaEvent_t> fwd_recv_done;  // upstream node id -> event

  // Transitive pruning of cross-stream waits: done[i] = the nodes whose
  // completion node i's start already implies (through full-completion
  // waits and stream order; a wait on a partial event -- delta, commit --
  // implies only that node's own predecessors).  A wait on d is dropped when
  // another dependency of the same node implies d.  Fewer graph edges, and a
  // GEMM left with a single upstream kernel gets a programmatic (PDL) edge
  // instead of a full one (PIPESIM_PRUNE_EDGES=0: off).
  const bool prune_edges = [] {
    const char* e = std::getenv("PIPESIM_PRUNE_EDGES");
    return !(e && std::string(e) == "0");
  }();
  const size_t words = (nodes.size() + 63) / 64;
  std::vector<std::vector<uint64_t>> done_set(nodes.size());
  auto implies = [&](int i, int d) {
    return !done_set[i].empty() && ((done_set[i][d >> 6] >> (d & 63)) & 1);
  };
  auto absorb = [&](int i, int d, bool with_d) {
    if (done_set[i].empty()) done_set[i].assign(words, 0);
    if (!done_set[d].empty())
      for (size_t w = 0; w < words; ++w) done_set[i][w] |= done_set[d][w];
    if (with_d) done_set[i][d >> 6] |= uint64_t{1} << (d & 63);
  };

  for (int id : topo) {
    Node& node = nodes[id];
    const int s = node.s;
    if (node.digest >= 0) {
      for (int d : node.deps) absorb(id, d, true);
      for (int d : node.deps) {
        Impl::Op w{OK::wait};
        w.stream = Impl::kDigest;
        w.ev = nodes[d].done;
        push(w);
      }
      Impl::Op o{OK::digest};
      o.stream = Impl::kDigest;
      o.value = node.digest;
      push(o);
      Impl::Op r{OK::record};
      r.stream = Impl::kDigest;
      r.ev = I.new_event();
      node.done = r.ev;
      push(r);
      continue;
    }
    if (!I.local(s)) continue;  // another GPU's stage
    Impl::Stage& st = I.stages[s];
    Impl::Task tk;
    tk.fwd = node.fwd;
    tk.k = node.k;
    tk.s = s + 1;
    tk.version = node.version;
    const int a = st.mini_act[tk.k];
    Impl::ActSlot& as = st.acts[a];
    // the node's stream: the stage stream, or (split mode) the stage's
    // backward stream for a backward
    const int ns = (!node.fwd && I.split_fb) ? Impl::kBwdBase - s : s;
    auto wait_on = [&](int stream, cudaEvent_t ev) {
      Impl::Op w{OK::wait};
      w.stream = stream;
      w.ev = ev;
      push(w);
    };
    auto record_on = [&](int stream) {
      Impl::Op r{OK::record};
      r.stream = stream;
      r.ev = I.new_event();
      push(r);
      return r.ev;
    };
    // classify every dependency: 0 stream order, 1 skipped (remote (b')),
    // 2 full wait, 3 delta wait, 4 commit wait, 5 remote
    std::vector<int> dep_kind(node.deps.size());
    for (size_t i = 0; i < node.deps.size(); ++i) {
      const int d = node.deps[i];
      int kind;
      if (nodes[d].s == s && (nodes[d].fwd == node.fwd || !I.split_fb)) {
        kind = 0;
      } else if (node.fwd && !nodes[d].fwd && nodes[d].digest < 0 && nodes[d].s == s + 1 &&
                 !I.local(nodes[d].s)) {
        kind = 1;
      } else if (nodes[d].digest >= 0 || I.local(nodes[d].s)) {
        // a backward waits for the downstream stage's delta only
        const bool delta_edge = !node.fwd && !nodes[d].fwd && nodes[d].digest < 0 &&
                                nodes[d].s == s + 1 && nodes[d].k == node.k &&
                                nodes[d].delta_done && delta_edges;
        // a forward waits for the commit of its pinned version only (the
        // wgrad + bias streams of that backward), unless the same backward
        // also frees the activation slot it writes
        const bool commit_edge =
            node.fwd && !nodes[d].fwd && nodes[d].digest < 0 && nodes[d].s == s &&
            d != node.slot_dep && nodes[d].commit_side && commit_edges &&
            std::find(node.commit_deps.begin(), node.commit_deps.end(), d) !=
                node.commit_deps.end();
        kind = commit_edge ? 4 : delta_edge ? 3 : 2;
      } else {
        kind = 5;
      }
      dep_kind[i] = kind;
      if (kind == 0 || kind == 2) absorb(id, d, true);
      else if (kind == 3 || kind == 4) absorb(id, d, false);
    }
    for (size_t i = 0; i < node.deps.size(); ++i) {
      const int d = node.deps[i];
      const int kind = dep_kind[i];
      if (kind <= 1) continue;
      if (kind <= 4) {
        if (prune_edges) {
          bool implied = false;
          for (size_t j = 0; j < node.deps.size() && !implied; ++j)
            implied = j != i && dep_kind[j] != 1 && dep_kind[j] != 5 &&
                      node.deps[j] != d && implies(node.deps[j], d);
          if (implied) continue;
        }
        const bool commit_edge = kind == 4, delta_edge = kind == 3;
        if (commit_edge) {
          wait_on(ns, nodes[d].commit_side);
          if (nodes[d].commit_bias) wait_on(ns, nodes[d].commit_bias);
          continue;
        }
        wait_on(ns, delta_edge ? nodes[d].delta_done : nodes[d].done);
        continue;
      }
      const Node& up = nodes[d];
      if (node.fwd) {
        // activation rows of the remote upstream group -> this stage's slot
        auto it = fwd_recv_done.find(d);
        if (it == fwd_recv_done.end()) {
          const int pk = prev_occ[s][tk.k];
          if (pk > 0) wait_on(Impl::kFwdRecv, nodes[bwd_id.at({pk, s})].done);
          const auto& fl = st.layers.front();
          Impl::Op rv{OK::recv};
          rv.stream = Impl::kFwdRecv;
          rv.dst = as.in16 + static_cast<size_t>(up.jj0) * I.Rm * fl.ain * I.sc;
          rv.bytes = static_cast<size_t>(up.jj1 - up.jj0 + 1) * I.Rm * fl.ain * 2 * I.sc;
          rv.peer = I.owner[up.s];
          rv.dir = 0;
          rv.value = I.add_msg(false, rv.dir, rv.peer, rv.bytes, nullptr, rv.dst);
          push(rv);
          it = fwd_recv_done.emplace(d, record_on(Impl::kFwdRecv)).first;
        }
        wait_on(ns, it->second);
      } else {
        // delta of the remote downstream stage -> this slot's dzin; the slot
        // belongs to mini k since its first forward here
        wait_on(Impl::kBwdRecv, nodes[first_fwd_id.at({tk.k, s})].done);
        Impl::Op rv{OK::recv};
        rv.stream = Impl::kBwdRecv;
        rv.dst = as.dzin;
        rv.bytes = static_cast<size_t>(c.B) * st.layers.back().aout * 2 * I.sc;
        rv.peer = I.owner[up.s];
        rv.dir = 1;
        rv.value = I.add_msg(false, rv.dir, rv.peer, rv.bytes, nullptr, rv.dst);
        push(rv);
        wait_on(ns, record_on(Impl::kBwdRecv));
      }
    }
    // streamed input: stage 1's first forward of mini k and the loss of mini
    // k wait for mini k's rows (no-ops when the input is resident)
    if ((node.fwd && s == 0 && first_fwd_id.at({tk.k, 0}) == id) || (!node.fwd && s == last_s)) {
      Impl::Op xw{OK::xwait};
      xw.stream = ns;
      xw.value = tk.k;
      xw.dir = node.fwd ? 1 : 0;  // the forward converts the rows, the loss reads labels
      push(xw);
    }
    const int node_idx = static_cast<int>(I.node_meta.size());
    I.node_meta.push_back(NodeTiming{s + 1, node.fwd ? 1 : 0, node.k, node.fwd ? node.jj0 : 0,
                                     node.fwd ? node.jj1 : 0, 0.f, 0.f});
    {
      Impl::Op mk{OK::mark};
      mk.stream = ns;
      mk.value = 2 * node_idx;
      push(mk);
    }
    if (node.fwd) {
      const Impl::PoolSlot& ps = st.pool[st.version_colour[tk.version]];
      const int r0 = node.jj0 * I.Rm;
      const int rows = (node.jj1 - node.jj0 + 1) * I.Rm;
      // the last two layers in one kernel (fwd_chain.cuh) on latency-bound
      // networks: layer L-2 at most 256 wide (a multiple of 64), layer L-1
      // at most 64
      int fchain = -1;
      if (st.L >= 2 && I.pdl && !I.v32) {
        const auto& la = st.layers[st.L - 2];
        const auto& lb = st.layers[st.L - 1];
        if (!la.conv && !lb.conv && !la.pool && fwd_chain_eligible(la.out, lb.out))
          fchain = st.L - 2;
      }
      for (int l = 0; l < st.L; ++l) {
        if (fchain >= 0 && l == fchain + 1) continue;  // computed by the chain
        const auto& d = st.layers[l];
        int in_off = 0;
        Mat16 x;
        if (l == 0) {
          x = stage_input(s, tk.k, &in_off);
        } else {
          x = Mat16{as.out16[l - 1], c.B, d.conv ? d.ain : d.in, d.ain};
        }
        const bool logits = (s == last_s) && (l == st.L - 1);
        Mat16 w{ps.w16[l], d.out, d.in, d.ld_in};
        if (l == fchain) {
          const auto& d2 = st.layers[l + 1];
          const bool logits2 = (s == last_s) && (l + 1 == st.L - 1);
          const Mat16 w2{ps.w16[l + 1], d2.out, d2.in, d2.ld_in};
          Impl::Op o{OK::fwd_chain};
          o.stream = ns;
          if (!c.plan_only) {
            const GemmLaunch g2 =
                plan_fwd(Mat16{as.out16[l], c.B, d2.in, d2.ain}, r0, rows, w2, ps.b32[l + 1],
                         d2.act, logits2 ? nullptr : as.out16[l + 1], d2.ld_out,
                         logits2 ? as.out32 : nullptr, I.n_out, r0, /*allow_split=*/false);
            o.fchain = plan_fwd_chain(x, in_off + r0, rows, w, ps.b32[l], d.act, as.out16[l],
                                      d.ld_out, r0, w2, g2);
          }
          if (logits2 && loss_fuse) {
            o.loss_fused = true;
            o.lab = I.ylab + static_cast<size_t>(tk.k - 1) * c.B;
            o.row_loss = I.row_loss + static_cast<size_t>(tk.k - 1) * c.B;
            o.dz_out = as.dzin;
            o.ld_dz = d2.ld_out;
            o.denom = static_cast<float>(c.B);
          }
          if (l == 0) {
            o.fchain.ep2.tag_src = ps.tag;
            o.fchain.ep2.tag_dst =
                I.fwd_trace + (static_cast<size_t>(tk.k - 1) * U + node.jj0) * W + s;
            o.fchain.ep2.tag_count = node.jj1 - node.jj0 + 1;
            o.fchain.ep2.tag_stride = W;
          }
          push(o);
          ++kernels_per_epoch_;
          continue;
        }
        Impl::Op o{OK::fwd};
        o.stream = ns;
        // a pooled conv writes its pre-pooling output, then pools it
        __nv_bfloat16* y16 = d.pool ? as.pre16[l] : as.out16[l];
        const int hw = d.h * d.w;
        if (d.first_conv) {
          // the network input's im2col (3-channel images: too narrow for an
          // im2col TMA box), then a plain GEMM over it
          Impl::Op ic{OK::im2col};
          ic.stream = ns;
          ic.in16 = x.ptr + static_cast<size_t>(in_off + r0) * x.ld;
          ic.ld = x.ld;
          ic.n = rows;
          ic.h = d.h;
          ic.w = d.w;
          ic.ch = d.cin;
          ic.out16 = as.cols16 + static_cast<size_t>(r0) * hw * d.ld_in;
          ic.ld16 = d.ld_in;
          push(ic);
          ++kernels_per_epoch_;
          if (!c.plan_only)
            o.g = plan_fwd(Mat16{as.cols16, c.B * hw, d.ld_in, d.ld_in}, r0 * hw, rows * hw, w,
                           ps.b32[l], d.act, y16, d.out, nullptr, 0, r0 * hw,
                           /*allow_split=*/false);
        } else if (d.conv) {
          if (!c.plan_only)
            o.g = plan_conv_fwd(Nhwc{x.ptr, x.rows, d.h, d.w, d.cin}, in_off + r0, rows, w,
                                ps.b32[l], d.act, y16, r0 * hw);
        } else if (!c.plan_only) {
          o.g = plan_fwd(x, in_off + r0, rows, w, ps.b32[l], d.act,
                         logits ? nullptr : as.out16[l], d.ld_out,
                         logits ? as.out32 : nullptr, I.n_out, r0,
                         /*allow_split=*/split_fwd, /*verify=*/I.v32, st.fix_ws, st.fix_cnt);
        }
        if (logits && loss_fuse && !o.g.simt && o.g.sh.splits <= 1) {
          o.loss_fused = true;
          o.lab = I.ylab + static_cast<size_t>(tk.k - 1) * c.B;
          o.row_loss = I.row_loss + static_cast<size_t>(tk.k - 1) * c.B;
          o.dz_out = as.dzin;
          o.ld_dz = d.ld_out;
          o.denom = static_cast<float>(c.B);
        }
        if (l == 0) {
          o.g.ep.tag_src = ps.tag;
          o.g.ep.tag_dst = I.fwd_trace + (static_cast<size_t>(tk.k - 1) * U + node.jj0) * W + s;
          o.g.ep.tag_count = node.jj1 - node.jj0 + 1;
          o.g.ep.tag_stride = W;
        }
        push(o);
        ++kernels_per_epoch_;
        if (d.pool) {
          Impl::Op pf{OK::pool_fwd};
          pf.stream = ns;
          pf.in16 = as.pre16[l] + static_cast<size_t>(r0) * d.pre_elems;
          pf.out16 = as.out16[l] + static_cast<size_t>(r0) * d.aout;
          pf.n = rows;
          pf.h = d.h;
          pf.w = d.w;
          pf.ch = d.out;
          push(pf);
          ++kernels_per_epoch_;
        }
      }
    } else {
      // ---------------- backward of mini k on stage s
      if (s == last_s) {
        // fused loss + gradient over the stacked mini-batch (trainer.cpp:461-473)
        Impl::Op o{OK::loss};
        o.stream = ns;
        o.y = as.out32;
        o.rows = c.B;
        o.cols = I.n_out;
        o.ld = I.n_out;
        o.t = I.y32 + static_cast<size_t>(tk.k - 1) * c.B * I.n_out;
        o.lab = I.ylab + static_cast<size_t>(tk.k - 1) * c.B;
        o.ld_t = I.n_out;
        o.loss = c.loss;
        o.act_last = st.layers.back().act;
        o.denom = static_cast<float>(c.B);
        o.dz_out = as.dzin;
        o.row_loss = I.row_loss + static_cast<size_t>(tk.k - 1) * c.B;
        o.ld_dz = st.layers.back().ld_out;
        o.loss_fused = loss_fuse;
        push(o);
        if (!loss_fuse) ++kernels_per_epoch_;
      }
      const Impl::PoolSlot& prop = st.pool[st.version_colour[tk.version]];
      Impl::PoolSlot& next = st.pool[st.version_colour[tk.k]];
      const int cur = (tk.k - 1) % 2, nxt = tk.k % 2;
      // wgrad+SGD of layer l runs on the side stream and its bias gradient +
      // SGD on the bias stream as soon as dZ_l exists, overlapping the dgrad
      // chain of the layers below (which only needs dZ) and each other;
      // both are joined back before the task completes.
      const int side = c.side_streams ? Impl::kSideBase - s : s;
      const int bstr = !c.side_streams ? s : (I.bias_stream ? Impl::kBiasBase - s : side);
      if (c.side_streams) {
        cudaEvent_t ev = record_on(ns);
        wait_on(side, ev);
        if (bstr != side) wait_on(bstr, ev);
      }
      // the input x of layer li (row offset *off inside its buffer)
      auto layer_x = [&](int li, int* off) {
        *off = 0;
        if (li == 0) return stage_input(s, tk.k, off);
        const auto& dl = st.layers[li];
        return Mat16{as.out16[li - 1], c.B, dl.conv ? dl.ain : dl.in, dl.ain};
      };
      // where layer li's dgrad writes (the layer below's dZ, or the delta of
      // the previous stage) and the activation whose act' gates it
      auto dgrad_dst = [&](int li, __nv_bfloat16** dst, int* act_prev) {
        if (li > 0) {
          *dst = st.scratch_dz[li - 1];
          *act_prev = st.layers[li - 1].act;
        } else if (!I.local(s - 1)) {
          *dst = as.dzsend;  // sent to the upstream GPU after this task
          *act_prev = I.stages[s - 1].layers.back().act;
        } else {
          const Impl::Stage& pv = I.stages[s - 1];
          *dst = pv.acts[pv.mini_act[tk.k]].dzin;
          *act_prev = pv.layers.back().act;
        }
      };
      // top two dgrads fused into one kernel (dgrad_chain.cuh): a narrow top
      // layer (out <= 64) over an input of <= 256 columns, both linear, the
      // lower one the stage's first (its dgrad is the delta of the previous
      // stage).  When the lower dgrad feeds another layer of the same stage,
      // two launches win: that layer's wgrad then starts after the first
      // (tiny) dgrad instead of after both (C2 sequential 50.5 vs 46.6 us
      // per mini-batch, tools/gpu/r2_c2seq.sh).
      int chain_top = -1;
      {
        const int lt = st.L - 1;
        if (lt == 1 && s > 0 && !I.v32 && !st.layers[lt].conv && !st.layers[lt - 1].conv &&
            dgrad_chain_eligible(st.layers[lt].out, st.layers[lt].in))
          chain_top = lt;
      }
      for (int l = st.L - 1; l >= 0; --l) {
        const auto& d = st.layers[l];
        __nv_bfloat16* dz = (l == st.L - 1) ? as.dzin : st.scratch_dz[l];
        int x_off = 0;
        Mat16 x;
        if (l == 0)
          x = stage_input(s, tk.k, &x_off);
        else
          x = Mat16{as.out16[l - 1], c.B, d.conv ? d.ain : d.in, d.ain};
        const int hw = d.h * d.w;
        // a pooled conv's delta arrives pooled (already gated by act' of the
        // pooled activation, which equals act' at each window's maximum);
        // route it to the first maximum of every window
        if (d.pool) {
          Impl::Op pb{OK::pool_bwd};
          pb.stream = ns;
          pb.in16 = dz;
          pb.aux16 = as.pre16[l];
          pb.dz = as.out16[l];
          pb.out16 = st.scratch_pre[l];
          pb.n = c.B;
          pb.h = d.h;
          pb.w = d.w;
          pb.ch = d.out;
          push(pb);
          ++kernels_per_epoch_;
          dz = st.scratch_pre[l];
          if (c.side_streams) {
            cudaEvent_t ev = record_on(ns);
            wait_on(side, ev);
            if (bstr != side) wait_on(bstr, ev);
          }
        }
        // conv: dz has one row per output pixel
        Mat16 mdz = d.conv ? Mat16{dz, c.B * hw, d.out, d.out} : Mat16{dz, c.B, d.out, d.ld_out};
        // dgrad: delta for the layer below (or the previous stage)
        if ((l > 0 || s > 0) && !d.first_conv && l == chain_top - 1) {
          // computed by the chain kernel of layer l + 1
          if (l == 0) node.delta_done = record_on(ns);  // stage s-1's delta is written
        } else if ((l > 0 || s > 0) && !d.first_conv && l == chain_top) {
          __nv_bfloat16 *dst, *dst2;
          int act_prev, act_prev2, x2_off = 0;
          dgrad_dst(l, &dst, &act_prev);
          dgrad_dst(l - 1, &dst2, &act_prev2);
          const auto& d2 = st.layers[l - 1];
          const Mat16 x2 = layer_x(l - 1, &x2_off);
          Impl::Op o{OK::dgrad_chain};
          o.stream = ns;
          if (!c.plan_only) {
            const __nv_bfloat16* xin = x.ptr + static_cast<size_t>(x_off) * x.ld * I.sc;
            const __nv_bfloat16* xin2 = x2.ptr + static_cast<size_t>(x2_off) * x2.ld * I.sc;
            const Mat16 mid{dst, c.B, d2.out, d.ld_in};
            const GemmLaunch g1 = plan_dgrad(mdz, Mat16{prop.w16[l], d.out, d.in, d.ld_in}, xin,
                                             x.ld, act_prev, dst, d.ld_in);
            const GemmLaunch g2 = plan_dgrad(mid, Mat16{prop.w16[l - 1], d2.out, d2.in, d2.ld_in},
                                             xin2, x2.ld, act_prev2, dst2, d2.ld_in);
            o.chain = plan_dgrad_chain(g1, g2, mid);
          }
          push(o);
          ++kernels_per_epoch_;
        } else if ((l > 0 || s > 0) && !d.first_conv) {
          __nv_bfloat16* dst;
          int act_prev;
          dgrad_dst(l, &dst, &act_prev);
          // act' of the layer below, recovered from the activation it produced
          // (= this layer's input x).
          const __nv_bfloat16* xin = x.ptr + static_cast<size_t>(x_off) * x.ld * I.sc;
          Impl::Op o{OK::dgrad};
          o.stream = ns;
          if (!c.plan_only) {
            if (d.conv)
              o.g = plan_conv_dgrad(Nhwc{dz, c.B, d.h, d.w, d.out}, prop.w16[l], d.cin, d.ld_in,
                                    xin, act_prev, dst);
            else
              o.g = plan_dgrad(mdz, Mat16{prop.w16[l], d.out, d.in, d.ld_in}, xin, x.ld,
                               act_prev, dst, d.ld_in, I.v32);
          }
          push(o);
          ++kernels_per_epoch_;
          if (l == 0) node.delta_done = record_on(ns);  // stage s-1's delta is written
        }
        // the side stream's work on layer l only reads dZ_l (and x); it was
        // made ready before this iteration (dZ_{L-1}: task start; dZ_l: the
        // previous iteration's dgrad, signalled below)
        // wgrad + SGD into the new version (trainer.cpp:244-249, :484-488)
        if (d.conv) {
          // conv: split-K fp32 partial slabs over the pixels, then their
          // in-order reduction fused with the SGD update and the bf16 copy
          Impl::Op o{OK::wgrad_partial};
          o.stream = side;
          ConvWgradInfo wi;
          wi.lds = d.ld_in;
          wi.slab = static_cast<long long>(d.out) * d.ld_in;
          if (!c.plan_only) {
            if (d.first_conv)
              o.g = plan_wgrad_partial(mdz, Mat16{as.cols16, c.B * hw, d.ld_in, d.ld_in},
                                       st.wg_ws, d.ld_in, &wi.splits);
            else
              o.g = plan_conv_wgrad_partial(mdz, Nhwc{x.ptr, x.rows, d.h, d.w, d.cin}, x_off,
                                            st.wg_ws, &wi);
          }
          push(o);
          ++kernels_per_epoch_;
          Impl::Op r{OK::reduce_sgd};
          r.stream = side;
          r.f32 = st.wg_ws;
          r.S = wi.splits;
          r.slab = wi.slab;
          r.value = wi.transposed ? 1 : 0;
          r.rows = d.out;
          r.cols = d.in;
          r.ld = wi.lds;
          r.w_cur = d.w32[cur];
          r.w_new = d.w32[nxt];
          r.ldw = d.in;
          r.out16 = next.w16[l];
          r.ld16 = d.ld_in;
          r.lr = static_cast<float>(c.lr);
          push(r);
          ++kernels_per_epoch_;
        } else {
          Impl::Op o{OK::wgrad};
          o.stream = side;
          if (!c.plan_only) {
            if (I.split)  // master(k-1) = hi in version k-1's pool slot + lo[cur]
              o.g = plan_wgrad_sgd_split(mdz, x, x_off,
                                         st.pool[st.version_colour[tk.k - 1]].w16[l], d.lo[cur],
                                         next.w16[l], d.lo[nxt], d.ld_in,
                                         static_cast<float>(c.lr));
            else
              o.g = plan_wgrad_sgd(mdz, x, x_off, d.w32[cur], d.w32[nxt], d.in, next.w16[l],
                                   d.ld_in, static_cast<float>(c.lr), I.v32,
                                   I.pdl ? latency_wgrad_bn(d.out, d.in) : 0);
          }
          push(o);
          ++kernels_per_epoch_;
        }
        // bias gradient + SGD; the last one stamps the commit.  Conv: column
        // sums of row blocks of dZ first (one pass over all its pixel rows
        // on the whole GPU), then the same kernel over the fp32 partials.
        {
          Impl::Op o{OK::bias};
          o.stream = bstr;
          o.dz = dz;
          o.rows = c.B;
          o.cols = d.out;
          o.ld = d.ld_out;
          if (d.conv) {
            Impl::Op cs{OK::colsum};
            cs.stream = bstr;
            cs.dz = dz;
            cs.rows = c.B * hw;
            cs.cols = d.out;
            cs.ld = d.out;
            cs.f32 = st.bias_ws;
            push(cs);
            ++kernels_per_epoch_;
            o.dz = reinterpret_cast<const __nv_bfloat16*>(st.bias_ws);
            o.rows = colsum_chunks(c.B * hw);
            o.ld = d.out;
            o.f32dz = true;
          }
          o.b_cur = d.b32[cur];
          o.b_new = d.b32[nxt];
          o.b_copy = next.b32[l];
          o.lr = static_cast<float>(c.lr);
          if (l == 0) {
            o.trace_src = prop.tag;
            o.trace_dst = I.bwd_trace + static_cast<size_t>(tk.k - 1) * W + s;
            o.tag_slot = next.tag;
            o.cur_version = st.cur_version;
            o.version = tk.k;
          }
          push(o);
          ++kernels_per_epoch_;
        }
        // dZ_{l-1} (written by this iteration's dgrad on the main stream) is
        // what the side stream needs next
        if (c.side_streams && l > 0) {
          cudaEvent_t ev = record_on(ns);
          wait_on(side, ev);
          if (bstr != side) wait_on(bstr, ev);
        }
      }
      if (c.side_streams) {  // join (the two events also mark the commit)
        node.commit_side = record_on(side);
        wait_on(ns, node.commit_side);
        if (bstr != side) {
          node.commit_bias = record_on(bstr);
          wait_on(ns, node.commit_bias);
        }
      }
      if (c.snapshots && !c.plan_only) {
        for (int l = 0, po = 0; l < st.L; ++l) {
          const auto& d = st.layers[l];
          Impl::Op o{OK::snapshot};
          o.stream = ns;
          o.dst = I.snaps[s][tk.k] + po;
          o.src = d.w32[nxt];
          o.bytes = sizeof(float) * d.in * static_cast<size_t>(d.out);
          push(o);
          o.dst = I.snaps[s][tk.k] + po + static_cast<size_t>(d.in) * d.out;
          o.src = d.b32[nxt];
          o.bytes = sizeof(float) * d.out;
          push(o);
          po += d.in * d.out + d.out;
        }
      }
    }
    Impl::Op r{OK::record};
    r.stream = ns;
    r.ev = I.new_event();
    node.done = r.ev;
    push(r);
    {
      Impl::Op mk{OK::mark};
      mk.stream = ns;
      mk.value = 2 * node_idx + 1;
      push(mk);
    }
    // outgoing cross-GPU edges of this node
    if (node.fwd && s + 1 < W && !I.local(s + 1)) {
      const auto& ll = st.layers.back();
      wait_on(Impl::kFwdSend, node.done);
      Impl::Op sd{OK::send};
      sd.stream = Impl::kFwdSend;
      sd.src = as.out16.back() + static_cast<size_t>(node.jj0) * I.Rm * ll.aout * I.sc;
      sd.bytes = static_cast<size_t>(node.jj1 - node.jj0 + 1) * I.Rm * ll.aout * 2 * I.sc;
      sd.peer = I.owner[s + 1];
      sd.dir = 0;
      sd.value = I.add_msg(true, sd.dir, sd.peer, sd.bytes, sd.src, nullptr);
      push(sd);
    }
    if (!node.fwd && s > 0 && !I.local(s - 1)) {
      wait_on(Impl::kBwdSend, node.delta_done && delta_edges ? node.delta_done : node.done);
      Impl::Op sd{OK::send};
      sd.stream = Impl::kBwdSend;
      sd.src = as.dzsend;
      sd.bytes = static_cast<size_t>(c.B) * st.layers.front().ain * 2 * I.sc;
      sd.peer = I.owner[s - 1];
      sd.dir = 1;
      sd.value = I.add_msg(true, sd.dir, sd.peer, sd.bytes, sd.src, nullptr);
      push(sd);
    }
  }
  if (c.world > 1 && c.transport == 1 && !c.plan_only)
    I.ipc = std::make_unique<IpcLink>(c.rank, c.world, c.device, I.arena, I.msgs);
  if (!digest_version.empty()) {
    I.digest = std::make_unique<DeviceDigest>(int64_t{1} << 24);
    for (const auto& vs : digest_version) {
      I.dplans.push_back(I.digest->make_plan(I.digest_spans(vs)));
      kernels_per_epoch_ += I.digest->launches_per(I.dplans.back());
    }
  }
  // PIPESIM_DUMP_OPS=file: the epoch's op program (stream, kind, event) for
  // reading the dependency chains (works with plan_only, no GPU)
  if (const char* path = std::getenv("PIPESIM_DUMP_OPS")) {
    static const char* kNames[] = {"wait", "record", "fwd", "dgrad", "wgrad", "bias", "loss",
                                   "copy", "memset", "snapshot", "send", "recv", "mark",
                                   "ktime", "xwait", "digest", "im2col", "pool_fwd",
                                   "pool_bwd", "wgrad_partial", "reduce_sgd", "colsum",
                                   "dgrad_chain", "fwd_chain"};
    if (FILE* f = std::fopen(path, "w")) {
      std::map<cudaEvent_t, int> ev_id;
      for (size_t i = 0; i < I.ops.size(); ++i) {
        const Impl::Op& o = I.ops[i];
        int e = -1;
        if (o.ev) e = ev_id.emplace(o.ev, static_cast<int>(ev_id.size())).first->second;
        std::fprintf(f, "%zu %d %s %d %d\n", i, o.stream, kNames[static_cast<int>(o.kind)], e,
                     o.g.sh.M);
      }
      std::fclose(f);
    }
  }
}

Session::~Session() = default;

std::vector<uint8_t> Session::ipc_export() {
  Impl& I = *impl_;
  if (!I.ipc) throw std::logic_error("session does not use the IPC transport");
  PB_CUDA(cudaSetDevice(cfg_.device));
  return I.ipc->export_blob();
}

void Session::ipc_connect(const std::vector<std::vector<uint8_t>>& blobs) {
  Impl& I = *impl_;
  if (!I.ipc) throw std::logic_error("session does not use the IPC transport");
  I.ipc->connect(blobs);
}

std::vector<Transfer> Session::transfers() const {
  std::vector<Transfer> out;
  using OK = Impl::OpKind;
  for (const auto& o : impl_->ops)
    if (o.kind == OK::send || o.kind == OK::recv)
      out.push_back(Transfer{o.kind == OK::send, o.dir, o.peer, static_cast<int64_t>(o.bytes)});
  return out;
}

int64_t Session::stage_param_count(int s) const { return impl_->stages.at(s - 1).param_count; }
int Session::stage_first_layer(int s) const { return impl_->stages.at(s - 1).first_layer; }
int Session::stage_layer_count(int s) const { return impl_->stages.at(s - 1).L; }
int64_t Session::stage_param_offset(int s) const {
  return impl_->stages.at(s - 1).param_offset;
}

std::vector<int> Session::pool_sizes() const {
  std::vector<int> v;
  for (const auto& s : impl_->stages) v.push_back(static_cast<int>(s.pool.size()));
  return v;
}

std::vector<std::pair<int64_t, int64_t>> Session::stage_bytes() const {
  std::vector<std::pair<int64_t, int64_t>> v;
  for (const auto& s : impl_->stages) v.push_back({s.bytes_weights, s.bytes_acts});
  return v;
}

std::vector<int> Session::act_slot_counts() const {
  std::vector<int> v;
  for (const auto& s : impl_->stages) v.push_back(static_cast<int>(s.acts.size()));
  return v;
}

const float* Session::snapshot(int s, int version) const {
  if (impl_->snaps.empty()) throw std::invalid_argument("session has no snapshots");
  return impl_->snaps.at(s - 1).at(version);
}

// ------------------------------------------------------------------ params
void Session::load_params(const double* flat) {
  for (auto& st : impl_->stages)
    if (impl_->local(st.id - 1)) load_stage_params(st.id, flat + st.param_offset);
}

// Version 0 of one stage := p (fp64, per layer W then b).  The fp64 values
// cross PCIe once (pinned, double-buffered, host copies split over threads);
// rounding to fp32 and the split into hi / lo (or the fp32 master and its
// bf16 copy) run on the device.
void Session::load_stage_params(int stage, const double* p) {
  Impl& I = *impl_;
  PB_CUDA(cudaSetDevice(cfg_.device));
  Impl::Stage& st = I.stages.at(stage - 1);
  if (!I.local(stage - 1)) throw std::invalid_argument("stage is not held by this process");
  I.param_scratch();
  const int c0 = st.version_colour[0];
  size_t po = 0;
  for (int l = 0; l < st.L; ++l) {
    auto& d = st.layers[l];
    const size_t nw = static_cast<size_t>(d.in) * d.out;
    // every step is ordered on the origin stream (its kernels read the
    // destination)
    I.stager->h2d(I.p64, p + po, (nw + d.out) * 8, I.origin);
    launch_convert_f64_f32(I.origin, I.p64 + nw, d.b32[0], d.out);
    PB_CUDA(cudaMemcpyAsync(st.pool[c0].b32[l], d.b32[0], d.out * 4, cudaMemcpyDeviceToDevice,
                            I.origin));
    PB_CUDA(cudaMemcpyAsync(d.b32[1], d.b32[0], d.out * 4, cudaMemcpyDeviceToDevice, I.origin));
    if (I.split) {  // version 0 = hi in pool colour(0) + lo[0] (lo[1] kept equal)
      launch_convert_f64_f32(I.origin, I.p64, I.p32, nw);
      launch_split_master(I.origin, I.p32, d.out, d.in, d.in, st.pool[c0].w16[l], d.lo[0],
                          d.ld_in);
      PB_CUDA(cudaMemcpyAsync(d.lo[1], d.lo[0], sizeof(uint16_t) * d.out * d.ld_in,
                              cudaMemcpyDeviceToDevice, I.origin));
    } else {
      launch_convert_f64_f32(I.origin, I.p64, d.w32[0], nw);
      if (I.v32)
        launch_rows_to_f32(I.origin, d.w32[0], false, d.out, d.in, d.in,
                           reinterpret_cast<float*>(st.pool[c0].w16[l]), d.ld_in);
      else
        launch_f32_to_bf16_rows(I.origin, d.w32[0], d.out, d.in, d.in, st.pool[c0].w16[l],
                                d.ld_in);
      // keep the odd master in sync so an M-odd rebase copy is always valid
      PB_CUDA(cudaMemcpyAsync(d.w32[1], d.w32[0], nw * 4, cudaMemcpyDeviceToDevice, I.origin));
    }
    po += nw + d.out;
  }
  // the rebase copies pool[colour(M)] -> pool[colour(0)]: make it a no-op
  const int cM = st.version_colour[cfg_.M];
  if (cM != c0)
    for (int l = 0; l < st.L; ++l) {
      auto& d = st.layers[l];
      PB_CUDA(cudaMemcpyAsync(st.pool[cM].w16[l], st.pool[c0].w16[l],
                              sizeof(__nv_bfloat16) * I.sc * d.out * static_cast<size_t>(d.ld_in),
                              cudaMemcpyDeviceToDevice, I.origin));
      PB_CUDA(cudaMemcpyAsync(st.pool[cM].b32[l], st.pool[c0].b32[l], 4 * d.out,
                              cudaMemcpyDeviceToDevice, I.origin));
    }
  PB_CUDA(cudaStreamSynchronize(I.origin));
  if (!I.snaps.empty()) {
    float* dst = I.snaps[stage - 1][0];
    for (int64_t i = 0; i < st.param_count; ++i) dst[i] = static_cast<float>(p[i]);
  }
}

uint64_t Session::params_digest(int version) {
  Impl& I = *impl_;
  if (cfg_.world > 1) throw std::logic_error("params_digest: multi-process session");
  if (version < 0 || version > cfg_.M) throw std::invalid_argument("version out of range");
  PB_CUDA(cudaSetDevice(cfg_.device));
  if (!I.digest) I.digest = std::make_unique<DeviceDigest>(int64_t{1} << 24);
  if (I.d_digest == nullptr) throw std::logic_error("session has no digest slot");
  DeviceDigest::Plan p =
      I.digest->make_plan(I.digest_spans(std::vector<int>(cfg_.W, version)));
  // after everything queued so far (the last epoch); the result goes to the
  // final slot and is read back here
  PB_CUDA(cudaStreamSynchronize(I.origin));
  uint64_t* out = I.d_digest + cfg_.M;
  I.digest->enqueue(p, out, I.origin);
  uint64_t h = 0;
  PB_CUDA(cudaMemcpyAsync(&h, out, 8, cudaMemcpyDeviceToHost, I.origin));
  PB_CUDA(cudaStreamSynchronize(I.origin));
  I.digest->free_plan(p);
  return h;
}

namespace {
// fp32 master of `version` of one stage's layers -> out (flat, W then b per
// layer, widened to fp64 on the device); split masters are joined first
void read_master(Session::Impl& I, Session::Impl::Stage& st, int version, double* out) {
  const int p = version & 1;
  I.param_scratch();
  size_t po = 0;
  for (size_t l = 0; l < st.layers.size(); ++l) {
    auto& d = st.layers[l];
    const size_t nw = static_cast<size_t>(d.in) * d.out;
    const float* w = d.w32[p];
    if (I.split) {
      launch_join_master(I.origin, st.pool[st.version_colour[version]].w16[l], d.lo[p], d.out,
                         d.in, d.ld_in, I.p32, d.in);
      w = I.p32;
    }
    launch_convert_f32_f64(I.origin, w, I.p64, nw);
    launch_convert_f32_f64(I.origin, d.b32[p], I.p64 + nw, d.out);
    I.stager->d2h(out + po, I.p64, (nw + d.out) * 8, I.origin);
    po += nw + d.out;
  }
}
}  // namespace

void Session::read_params(double* flat) {
  Impl& I = *impl_;
  PB_CUDA(cudaSetDevice(cfg_.device));
  PB_CUDA(cudaDeviceSynchronize());
  for (auto& st : I.stages) {
    if (!I.local(st.id - 1)) continue;  // other GPUs' stages stay untouched
    read_master(I, st, cfg_.M, flat + st.param_offset);  // current version M
  }
}

void Session::read_stage_master(int stage, int version, double* out) {
  Impl& I = *impl_;
  PB_CUDA(cudaSetDevice(cfg_.device));
  PB_CUDA(cudaDeviceSynchronize());
  read_master(I, I.stages.at(stage - 1), version, out);
}

// ------------------------------------------------------------------ data
namespace {
void upload_rows(Session::Impl& I, size_t r0, size_t n, const void* x, HostDType xt,
                 const void* y, HostDType yt, cudaStream_t st, cudaStream_t conv = nullptr,
                 cudaEvent_t copied = nullptr, bool skip_convert = false);
void convert_rows(Session::Impl& I, size_t r0, size_t n, HostDType xt, HostDType yt,
                  cudaStream_t cs, bool do_x = true, bool do_y = true);
}  // namespace

void Session::upload(const void* x, HostDType xt, const void* y, HostDType yt,
                     cudaStream_t st) {
  Impl& I = *impl_;
  PB_CUDA(cudaSetDevice(cfg_.device));
  if (!st) st = I.origin;
  // pageable host buffers: pinned staging with threaded host copies
  cudaPointerAttributes a{};
  const bool pinned = cudaPointerGetAttributes(&a, x) == cudaSuccess &&
                      a.type == cudaMemoryTypeHost;
  cudaGetLastError();
  I.staged_upload = !pinned;
  try {
    upload_rows(I, 0, static_cast<size_t>(cfg_.M) * cfg_.B, x, xt, y, yt, st);
  } catch (...) {
    I.staged_upload = false;
    throw;
  }
  I.staged_upload = false;
  if (st != I.origin) {
    cudaEvent_t e = I.new_event();
    PB_CUDA(cudaEventRecord(e, st));
    PB_CUDA(cudaStreamWaitEvent(I.origin, e, 0));
  }
}

// ------------------------------------------------------------------ run
namespace {
// Rows [r0, r0 + n) of the epoch's data: H2D into the staging buffer (x
// region, then y region) on `st`, then conversion into the device layout on
// `conv` (st if null; with a separate conversion stream the copies run back
// to back on the copy engine and never wait for SMs).
void upload_rows(Session::Impl& I, size_t r0, size_t n, const void* x, HostDType xt,
                 const void* y, HostDType yt, cudaStream_t st, cudaStream_t conv,
                 cudaEvent_t copied, bool skip_convert) {
  const int in = I.cfg.widths.front();
  const size_t rows = static_cast<size_t>(I.M) * I.B;
  char* xs = static_cast<char*>(I.stage_buf);
  char* ys = xs + rows * in * 8;  // y region after the largest x region
  __nv_bfloat16* xdst = I.x16 + r0 * I.ld_x * I.sc;
  float* ydst = I.y32 + r0 * I.n_out;
  const size_t xes = xt == HostDType::f64 ? 8 : xt == HostDType::f32 ? 4 : 2;
  char* xb = xs + r0 * in * xes;
  char* yb = ys + r0 * I.n_out * 8;
  // ---- copies
  if (xt == HostDType::bf16) {  // already the device operand type: one 2-D copy
    if (I.v32) throw std::invalid_argument("bf16 input needs a bf16-precision session");
    PB_CUDA(cudaMemcpy2DAsync(xdst, static_cast<size_t>(I.ld_x) * 2,
                              static_cast<const __nv_bfloat16*>(x) + r0 * in,
                              static_cast<size_t>(in) * 2, static_cast<size_t>(in) * 2, n,
                              cudaMemcpyHostToDevice, st));
  } else if (xt == HostDType::f64 || xt == HostDType::f32) {
    I.copy_h2d(xb, static_cast<const char*>(x) + r0 * in * xes, n * in * xes, st);
  } else {
    throw std::invalid_argument("x must be f64, f32 or bf16");
  }
  if (yt == HostDType::f64) {
    I.copy_h2d(yb, static_cast<const char*>(y) + r0 * I.n_out * 8, n * I.n_out * 8, st);
  } else if (yt == HostDType::f32) {
    I.copy_h2d(ydst, static_cast<const float*>(y) + r0 * I.n_out, n * I.n_out * 4, st);
  } else if (yt == HostDType::labels_i32) {  // the loss kernel reads labels directly
    PB_CUDA(cudaMemcpyAsync(I.ylab + r0, static_cast<const int*>(y) + r0, n * 4,
                            cudaMemcpyHostToDevice, st));
  } else {
    throw std::invalid_argument("y must be f64, f32 or int32 labels");
  }
  I.use_labels = yt == HostDType::labels_i32;
  if (copied) PB_CUDA(cudaEventRecord(copied, st));
  if (skip_convert) return;
  // ---- conversions
  cudaStream_t cs = st;
  if (conv && conv != st) {
    PB_CUDA(cudaStreamWaitEvent(conv, copied, 0));
    cs = conv;
  }
  convert_rows(I, r0, n, xt, yt, cs);
}

// Conversion of rows [r0, r0 + n) from the staging buffer into the device
// layout (f64 / f32 x -> the bf16 operand or fp32 verify rows; f64 y -> fp32).
void convert_rows(Session::Impl& I, size_t r0, size_t n, HostDType xt, HostDType yt,
                  cudaStream_t cs, bool do_x, bool do_y) {
  const int in = I.cfg.widths.front();
  const size_t rows = static_cast<size_t>(I.M) * I.B;
  char* xs = static_cast<char*>(I.stage_buf);
  char* ys = xs + rows * in * 8;
  __nv_bfloat16* xdst = I.x16 + r0 * I.ld_x * I.sc;
  float* ydst = I.y32 + r0 * I.n_out;
  const size_t xes = xt == HostDType::f64 ? 8 : xt == HostDType::f32 ? 4 : 2;
  char* xb = xs + r0 * in * xes;
  char* yb = ys + r0 * I.n_out * 8;
  if (do_x && (xt == HostDType::f64 || xt == HostDType::f32)) {
    if (I.v32)
      launch_rows_to_f32(cs, xb, xt == HostDType::f64, static_cast<int>(n), in, in,
                         reinterpret_cast<float*>(xdst), I.ld_x);
    else if (xt == HostDType::f64)
      launch_convert_f64_bf16(cs, reinterpret_cast<const double*>(xb), static_cast<int>(n), in,
                              in, xdst, I.ld_x);
    else if (!std::getenv("PIPESIM_H2D_DBG"))  // timing experiment: skip (wrong numerics)
      launch_convert_f32_bf16(cs, reinterpret_cast<const float*>(xb), static_cast<int>(n), in,
                              in, xdst, I.ld_x);
  }
  if (do_y && yt == HostDType::f64)
    launch_convert_f64_f32(cs, reinterpret_cast<const double*>(yb), ydst, n * I.n_out);
}

void issue(Session::Impl& I, cudaStream_t origin) {
  using OK = Session::Impl::OpKind;
  // every stream this process drives: local stage streams + P2P streams
  std::vector<cudaStream_t> streams;
  for (size_t i = 0; i < I.stages.size(); ++i)
    if (I.local(static_cast<int>(i))) {
      streams.push_back(I.stages[i].stream);
      if (I.stages[i].side) streams.push_back(I.stages[i].side);
      if (I.stages[i].bstream) streams.push_back(I.stages[i].bstream);
      if (I.stages[i].biasstream) streams.push_back(I.stages[i].biasstream);
    }
  for (cudaStream_t c : I.comm)
    if (c) streams.push_back(c);
  if (I.h2d) streams.push_back(I.h2d);
  if (I.h2dc) streams.push_back(I.h2dc);
  if (I.dstream) streams.push_back(I.dstream);
  if (!I.fork_ev) I.fork_ev = I.new_event();
  while (I.join_ev.size() < streams.size()) I.join_ev.push_back(I.new_event());
  cudaStreamCaptureStatus cap_status = cudaStreamCaptureStatusNone;
  PB_CUDA(cudaStreamIsCapturing(origin, &cap_status));
  const bool capturing = cap_status != cudaStreamCaptureStatusNone;
  cudaEvent_t fork = I.fork_ev;
  PB_CUDA(cudaEventRecord(fork, origin));
  for (cudaStream_t st : streams) PB_CUDA(cudaStreamWaitEvent(st, fork, 0));
  // mini-batch k's rows: the H2D copies run back to back on the copy engine
  // (copy_ev[k]); the conversion of x (f32 / f64 hosts) runs on stage 1's
  // forward stream right before its first forward of mini k (xwait), where
  // the rows are needed -- a conversion kernel on a side stream cost ~7 ms
  // per 16 x 4096 step (measured), against ~0.25 ms of conversion work.
  // PIPESIM_H2D_SIDE=1 restores the side-stream conversion (x_ready[k]).
  const bool side_conv = std::getenv("PIPESIM_H2D_SIDE") != nullptr;
  if (I.streaming)
    for (int k = 1; k <= I.M; ++k) {
      upload_rows(I, static_cast<size_t>(k - 1) * I.B, I.B, I.host_in.x, I.host_in.xt,
                  I.host_in.y, I.host_in.yt, I.h2d, I.h2dc, I.copy_ev[k], !side_conv);
      if (side_conv) PB_CUDA(cudaEventRecord(I.x_ready[k], I.h2dc));
    }
  for (const auto& o : I.ops) {
    cudaStream_t s = I.stream_of(o.stream);
    switch (o.kind) {
      case OK::wait: PB_CUDA(cudaStreamWaitEvent(s, o.ev, 0)); break;
      case OK::record: PB_CUDA(cudaEventRecord(o.ev, s)); break;
      case OK::fwd:
        if (o.loss_fused && I.use_labels) {
          GemmLaunch g = o.g;
          g.ep.loss_labels = o.lab;
          g.ep.loss_dz = o.dz_out;
          g.ep.loss_ld_dz = o.ld_dz;
          g.ep.loss_row = o.row_loss;
          g.ep.loss_denom = o.denom;
          g.ep.rowwise = 1;  // the row-per-thread epilogue holds whole rows
          launch_fwd(g, s);
        } else {
          launch_fwd(o.g, s);
        }
        break;
      case OK::dgrad: launch_dgrad(o.g, s); break;
      case OK::dgrad_chain: launch_dgrad_chain(o.chain, s); break;
      case OK::fwd_chain:
        if (o.loss_fused && I.use_labels) {
          EpiParams ep = o.fchain.ep2;
          ep.loss_labels = o.lab;
          ep.loss_dz = o.dz_out;
          ep.loss_ld_dz = o.ld_dz;
          ep.loss_row = o.row_loss;
          ep.loss_denom = o.denom;
          ep.rowwise = 1;  // the row-per-thread epilogue holds whole rows
          launch_fwd_chain(o.fchain, s, ep);
        } else {
          launch_fwd_chain(o.fchain, s);
        }
        break;
      case OK::wgrad: launch_wgrad(o.g, s); break;
      case OK::bias:
        launch_bias_sgd(s, o.dz, o.rows, o.cols, o.ld, o.b_cur, o.b_new, o.b_copy, o.lr,
                        o.tag_slot, o.cur_version, o.version, o.trace_src, o.trace_dst,
                        I.v32 || o.f32dz);
        break;
      case OK::im2col:
        launch_im2col_first(s, o.in16, o.ld, o.n, o.h, o.w, o.ch, o.out16, o.ld16);
        break;
      case OK::pool_fwd:
        launch_maxpool2_fwd(s, o.in16, o.n, o.h, o.w, o.ch, o.out16);
        break;
      case OK::pool_bwd:  // in16 = d_out (pooled), aux16 = conv output, dz = pooled output
        launch_maxpool2_bwd(s, o.in16, o.aux16, o.dz, o.n, o.h, o.w, o.ch, o.out16);
        break;
      case OK::wgrad_partial: launch_wgrad_partial(o.g, s); break;
      case OK::reduce_sgd:
        launch_reduce_sgd(s, o.f32, o.S, o.slab, o.rows, o.cols, o.ld, o.w_cur, o.w_new, o.ldw,
                          o.out16, o.ld16, o.lr, o.value != 0);
        break;
      case OK::colsum:
        launch_colsum_partial(s, o.dz, o.rows, o.cols, o.ld, o.f32);
        break;
      case OK::loss:
        if (o.loss_fused && I.use_labels) break;  // done by the logits forward
        launch_loss(s, o.y, o.rows, o.cols, o.ld, o.t, o.ld_t, o.loss, o.act_last, o.denom,
                    o.dz_out, o.ld_dz, o.row_loss, I.v32, I.use_labels ? o.lab : nullptr);
        break;
      case OK::copy:
        PB_CUDA(cudaMemcpyAsync(o.dst, o.src, o.bytes, cudaMemcpyDeviceToDevice, s));
        break;
      case OK::snapshot:
        PB_CUDA(cudaMemcpyAsync(o.dst, o.src, o.bytes, cudaMemcpyDeviceToHost, s));
        break;
      case OK::memset_i32:
        PB_CUDA(cudaMemsetAsync(o.dst, 0, sizeof(int), s));
        break;
      case OK::send:
        if (I.ipc)
          I.ipc->send(o.value, s);
        else
          I.p2p->send(o.src, o.bytes, o.peer, o.dir, s);
        break;
      case OK::recv:
        if (I.ipc)
          I.ipc->recv(o.value, s);
        else
          I.p2p->recv(o.dst, o.bytes, o.peer, o.dir, s);
        break;
      case OK::mark:
        if (I.profiling) PB_CUDA(cudaEventRecord(I.mark_ev[o.value], s));
        break;
      case OK::xwait:
        if (I.streaming) {
          if (std::getenv("PIPESIM_H2D_SIDE")) {
            PB_CUDA(cudaStreamWaitEvent(s, I.x_ready[o.value], 0));
          } else {
            PB_CUDA(cudaStreamWaitEvent(s, I.copy_ev[o.value], 0));
            // stage 1's first forward of mini k converts its x rows, the loss
            // its (f64) targets
            convert_rows(I, static_cast<size_t>(o.value - 1) * I.B, I.B, I.host_in.xt,
                         I.host_in.yt, s, o.dir == 1, o.dir == 0);
          }
        }
        break;
      case OK::digest:
        I.digest->enqueue(I.dplans[o.value], I.d_digest + o.value, s);
        break;
      case OK::ktime:  // an event record node when captured
        PB_CUDA(cudaEventRecordWithFlags(I.kt_ev[o.value], s,
                                         capturing ? cudaEventRecordExternal : 0));
        break;
    }
  }
  for (size_t i = 0; i < streams.size(); ++i) {
    PB_CUDA(cudaEventRecord(I.join_ev[i], streams[i]));
    PB_CUDA(cudaStreamWaitEvent(origin, I.join_ev[i], 0));
  }
}
}  // namespace

EpochResult Session::run_epoch() {
  Impl& I = *impl_;
  PB_CUDA(cudaSetDevice(cfg_.device));
  if (I.ipc && !I.ipc->connected())
    throw std::logic_error("IPC transport: call ipc_connect first");
  PB_CUDA(cudaEventRecord(I.t0, I.origin));
  if (cfg_.use_graph) {
    if (I.exec && I.graph_labels != static_cast<int>(I.use_labels)) {
      cudaGraphExecDestroy(I.exec);
      cudaGraphDestroy(I.graph);
      I.exec = nullptr;
      I.graph = nullptr;
    }
    if (!I.exec) {
      I.graph_labels = static_cast<int>(I.use_labels);
      PB_CUDA(cudaStreamBeginCapture(I.origin, cudaStreamCaptureModeThreadLocal));
      try {
        issue(I, I.origin);
      } catch (...) {
        cudaGraph_t g;
        cudaStreamEndCapture(I.origin, &g);
        if (g) cudaGraphDestroy(g);
        throw;
      }
      PB_CUDA(cudaStreamEndCapture(I.origin, &I.graph));
      // PIPESIM_GRAPH_DOT=file: the captured graph (nodes, edges, edge types)
      if (const char* dot = std::getenv("PIPESIM_GRAPH_DOT"))
        cudaGraphDebugDotPrint(I.graph, dot, cudaGraphDebugDotFlagsVerbose);
      PB_CUDA(cudaGraphInstantiate(&I.exec, I.graph, 0));
    }
    PB_CUDA(cudaGraphLaunch(I.exec, I.origin));
  } else {
    issue(I, I.origin);
  }
  PB_CUDA(cudaEventRecord(I.t1, I.origin));
  PB_CUDA(cudaEventSynchronize(I.t1));
  if (I.guard && I.check_guards() > 0)
    throw std::logic_error("PIPESIM_GUARD: a kernel wrote past a session buffer (see stderr)");
  return collect_result();
}

const std::vector<double>& Session::kernel_flops() const { return impl_->kt_flops; }

std::vector<float> Session::kernel_times_ms() {
  Impl& I = *impl_;
  std::vector<float> out;
  for (size_t i = 0; i + 1 < I.kt_ev.size(); i += 2) {
    float ms = 0.f;
    PB_CUDA(cudaEventElapsedTime(&ms, I.kt_ev[i], I.kt_ev[i + 1]));
    out.push_back(ms);
  }
  return out;
}

EpochResult Session::train_epoch_host(const void* x, HostDType xt, const void* y,
                                      HostDType yt) {
  Impl& I = *impl_;
  PB_CUDA(cudaSetDevice(cfg_.device));
  auto pinned = [](const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    return a.type == cudaMemoryTypeHost;  // page-locked (cudaHostAlloc / registered)
  };
  // pageable buffers (not capturable): upload, then the epoch
  if (!pinned(x) || !pinned(y)) {
    upload(x, xt, y, yt);
    return run_epoch();
  }
  if (!I.h2d) {
    int lo = 0, hi = 0;
    PB_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    PB_CUDA(cudaStreamCreateWithFlags(&I.h2d, cudaStreamNonBlocking));
    const char* pe = std::getenv("PIPESIM_H2D_PRIO");
    PB_CUDA(cudaStreamCreateWithPriority(&I.h2dc, cudaStreamNonBlocking,
                                         pe && std::atoi(pe) == 0 ? lo : hi));
    I.x_ready.assign(cfg_.M + 1, nullptr);
    I.copy_ev.assign(cfg_.M + 1, nullptr);
    for (int k = 1; k <= cfg_.M; ++k) {
      I.x_ready[k] = I.new_event();
      I.copy_ev[k] = I.new_event();
    }
  }
  const Impl::HostInput in{x, y, xt, yt};
  PB_CUDA(cudaEventRecord(I.t0, I.origin));
  I.streaming = true;
  I.host_in = in;
  try {
    if (cfg_.use_graph) {
      if (!I.sexec || !(I.sgraph_key == in)) {
        if (I.sexec) cudaGraphExecDestroy(I.sexec);
        if (I.sgraph) cudaGraphDestroy(I.sgraph);
        I.sexec = nullptr;
        I.sgraph = nullptr;
        PB_CUDA(cudaStreamBeginCapture(I.origin, cudaStreamCaptureModeThreadLocal));
        try {
          issue(I, I.origin);
        } catch (...) {
          cudaGraph_t g;
          cudaStreamEndCapture(I.origin, &g);
          if (g) cudaGraphDestroy(g);
          throw;
        }
        PB_CUDA(cudaStreamEndCapture(I.origin, &I.sgraph));
        PB_CUDA(cudaGraphInstantiate(&I.sexec, I.sgraph, 0));
        I.sgraph_key = in;
      }
      PB_CUDA(cudaGraphLaunch(I.sexec, I.origin));
    } else {
      issue(I, I.origin);
    }
  } catch (...) {
    I.streaming = false;
    throw;
  }
  I.streaming = false;
  PB_CUDA(cudaEventRecord(I.t1, I.origin));
  PB_CUDA(cudaEventSynchronize(I.t1));
  if (I.guard && I.check_guards() > 0)
    throw std::logic_error("PIPESIM_GUARD: a kernel wrote past a session buffer (see stderr)");
  return collect_result();
}

EpochResult Session::profile_epoch(EpochProfile* prof) {
  Impl& I = *impl_;
  PB_CUDA(cudaSetDevice(cfg_.device));
  if (I.mark_ev.empty()) {
    I.mark_ev.assign(2 * I.node_meta.size(), nullptr);
    for (cudaEvent_t& e : I.mark_ev) PB_CUDA(cudaEventCreate(&e));
  }
  if (I.ipc && !I.ipc->connected())
    throw std::logic_error("IPC transport: call ipc_connect first");
  PB_CUDA(cudaEventRecord(I.t0, I.origin));
  I.profiling = true;
  try {
    issue(I, I.origin);
  } catch (...) {
    I.profiling = false;
    throw;
  }
  I.profiling = false;
  PB_CUDA(cudaEventRecord(I.t1, I.origin));
  PB_CUDA(cudaEventSynchronize(I.t1));
  EpochResult r = collect_result();
  if (prof) {
    prof->makespan_ms = r.device_ms;
    prof->busy_ms.assign(cfg_.W, -1.f);
    for (int s = 0; s < cfg_.W; ++s)
      if (I.local(s)) prof->busy_ms[s] = 0.f;
    prof->nodes = I.node_meta;
    for (size_t i = 0; i < prof->nodes.size(); ++i) {
      NodeTiming& n = prof->nodes[i];
      PB_CUDA(cudaEventElapsedTime(&n.start_ms, I.t0, I.mark_ev[2 * i]));
      PB_CUDA(cudaEventElapsedTime(&n.end_ms, I.t0, I.mark_ev[2 * i + 1]));
      prof->busy_ms[n.stage - 1] += n.end_ms - n.start_ms;
    }
  }
  return r;
}

EpochResult Session::collect_result() {
  Impl& I = *impl_;
  EpochResult r;
  PB_CUDA(cudaEventElapsedTime(&r.device_ms, I.t0, I.t1));
  const int M = cfg_.M, U = I.U, W = cfg_.W, B = cfg_.B;
  std::vector<float> rl(static_cast<size_t>(M) * B);
  PB_CUDA(cudaMemcpy(rl.data(), I.row_loss, rl.size() * 4, cudaMemcpyDeviceToHost));
  r.dev_fwd.resize(static_cast<size_t>(M) * U * W);
  r.dev_bwd.resize(static_cast<size_t>(M) * W);
  PB_CUDA(cudaMemcpy(r.dev_fwd.data(), I.fwd_trace, r.dev_fwd.size() * 4, cudaMemcpyDeviceToHost));
  PB_CUDA(cudaMemcpy(r.dev_bwd.data(), I.bwd_trace, r.dev_bwd.size() * 4, cudaMemcpyDeviceToHost));
  for (auto& st : I.stages) {
    int v = -1;  // -1: stage owned by another GPU
    if (I.local(st.id - 1)) PB_CUDA(cudaMemcpy(&v, st.cur_version, 4, cudaMemcpyDeviceToHost));
    r.dev_current.push_back(v);
  }
  // mini loss: mean over micro-batches of the micro mean (trainer.cpp:462-469)
  const int Rm = I.Rm;
  for (int k = 0; k < M; ++k) {
    double tot = 0.0;
    for (int j = 0; j < U; ++j) {
      double part = 0.0;
      for (int q = 0; q < Rm; ++q) part += rl[static_cast<size_t>(k) * B + j * Rm + q];
      tot += part / Rm;
    }
    r.mini_loss.push_back(tot / U);
  }
  for (const auto& p : ledger_.pins) r.pinned.push_back(p.version);
  r.consumed = ledger_.update_source;
  if (!I.dplans.empty()) {
    r.digests.resize(static_cast<size_t>(M) + 1);
    PB_CUDA(cudaMemcpy(r.digests.data(), I.d_digest, r.digests.size() * 8,
                       cudaMemcpyDeviceToHost));
  }
  last_ = r;
  return r;
}

std::string Session::trace_document() const {
  if (!grid_) throw std::logic_error("trace_document: the sequential mode has no schedule grid");
  if (cfg_.world > 1) throw std::logic_error("trace_document: multi-process session");
  if (last_.dev_fwd.empty()) throw std::logic_error("trace_document: run an epoch first");
  const int W = cfg_.W, U = units();
  pipesim::version_ledger L = ledger_;
  for (auto& p : L.pins) {
    const int j = U > 1 ? p.micro - 1 : 0;
    p.version = last_.dev_fwd[(static_cast<size_t>(p.mini - 1) * U + j) * W + 0];
  }
  if (cfg_.mode == RunMode::timeprest)
    for (auto& c : L.consumptions)
      c.version = last_.dev_bwd[static_cast<size_t>(c.mini - 1) * W + (c.stage - 1)];
  return pipesim::schedule_document_json(*grid_, L);
}

}  // namespace pb
