// C ABI over the pipeline session (include/pipesim_b200.h, "pipeline session").
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "nccl_p2p.hpp"
#include "session.hpp"
#include "status.hpp"

namespace pb {
int translate_exception();
}

struct pb_session {
  std::unique_ptr<pb::Session> impl;
};

#define PB_GUARD_BEGIN try {
#define PB_GUARD_END \
  return PB_OK;      \
  }                  \
  catch (...) {      \
    return pb::translate_exception(); \
  }

namespace {

pb::Session& S(pb_session* s) {
  if (!s || !s->impl) throw std::invalid_argument("null session");
  return *s->impl;
}

pb::HostDType dtype(int d) {
  switch (d) {
    case PB_DTYPE_F64: return pb::HostDType::f64;
    case PB_DTYPE_F32: return pb::HostDType::f32;
    case PB_DTYPE_LABELS_I32: return pb::HostDType::labels_i32;
    case PB_DTYPE_BF16: return pb::HostDType::bf16;
    default: throw std::invalid_argument("bad dtype " + std::to_string(d));
  }
}

void fill(const pb::EpochResult& r, const pb::Session& s, pb_epoch_out* out) {
  if (!out) return;
  const int M = s.config().M, W = s.config().W, U = s.units();
  auto put = [](auto* dst, const auto& v, size_t n) {
    if (dst)
      for (size_t i = 0; i < n && i < v.size(); ++i) dst[i] = v[i];
  };
  put(out->mini_loss, r.mini_loss, M);
  put(out->pinned, r.pinned, static_cast<size_t>(M) * U);
  put(out->consumed, r.consumed, M);
  put(out->dev_fwd, r.dev_fwd, static_cast<size_t>(M) * U * W);
  put(out->dev_bwd, r.dev_bwd, static_cast<size_t>(M) * W);
  put(out->dev_current, r.dev_current, W);
  out->device_ms = r.device_ms;
}

}  // namespace

extern "C" {

namespace {
pb::SessionConfig make_config(const pb_net_spec* net, const pb_train_config* cfg) {
  if (!net || !cfg) throw std::invalid_argument("null argument");
  if (cfg->micro_batches < 1)
    throw pipesim::domain_error("micro_batches", "micro-batch count must be >= 1");
  if (cfg->mini_batch_size < 1 || cfg->mini_batches < 1)
    throw pipesim::domain_error("mini_batches", "mini-batch count/size must be >= 1");
  pb::SessionConfig c;
  c.widths.assign(net->widths, net->widths + net->n_layers + 1);
  c.acts.assign(net->activations, net->activations + net->n_layers);
  c.loss = net->loss;
  c.W = cfg->workers;
  c.N = cfg->micro_batches;
  c.B = cfg->mini_batch_size;
  c.M = cfg->mini_batches;
  c.lr = cfg->learning_rate;
  c.mode = static_cast<pb::RunMode>(cfg->mode);
  c.device = cfg->device;
  c.use_graph = cfg->use_graph != 0;
  c.snapshots = cfg->snapshots != 0;
  c.fwd_merge = cfg->fwd_merge;
  c.timed_kernel = cfg->timed_kernel;
  c.transport = cfg->transport;
  c.verify_fp32 = cfg->precision == 1;
  c.digests = cfg->digests != 0;
  if (const char* e = std::getenv("PIPESIM_FWD_MERGE")) c.fwd_merge = std::atoi(e);
  if (const char* e = std::getenv("PIPESIM_SIDE")) c.side_streams = std::atoi(e) != 0;
  return c;
}
}  // namespace

int pb_session_create(const pb_net_spec* net, const pb_train_config* cfg,
                      pb_session** out) {
  return pb_session_create_dist(net, cfg, 0, 1, nullptr, 0, out);
}

int pb_session_create_dist(const pb_net_spec* net, const pb_train_config* cfg, int rank,
                           int world, const uint8_t* nccl_ids, size_t ids_bytes,
                           pb_session** out) {
  PB_GUARD_BEGIN
  if (!out) throw std::invalid_argument("null argument");
  pb::SessionConfig c = make_config(net, cfg);
  c.rank = rank;
  c.world = world;
  if (nccl_ids && ids_bytes) c.nccl_ids.assign(nccl_ids, nccl_ids + ids_bytes);
  auto* s = new pb_session;
  try {
    s->impl = std::make_unique<pb::Session>(c);
  } catch (...) {
    delete s;
    throw;
  }
  *out = s;
  PB_GUARD_END
}

namespace {
std::vector<pb::LayerSpec> layer_list(const pb_layer_net* net) {
  if (!net || net->n_layers < 1 || !net->layers) throw std::invalid_argument("empty layer list");
  std::vector<pb::LayerSpec> v;
  for (int i = 0; i < net->n_layers; ++i) {
    const pb_layer_spec& a = net->layers[i];
    if (a.kind != PB_LAYER_LINEAR && a.kind != PB_LAYER_CONV3X3)
      throw std::invalid_argument("bad layer kind " + std::to_string(a.kind));
    pb::LayerSpec l;
    l.kind = a.kind == PB_LAYER_CONV3X3 ? pb::LayerKind::conv3x3 : pb::LayerKind::linear;
    l.in = a.in;
    l.out = a.out;
    l.h = a.height;
    l.w = a.width;
    l.pool = a.pool != 0;
    l.act = a.act;
    v.push_back(l);
  }
  pb::check_layers(v);
  return v;
}
}  // namespace

int pb_partition_layers(const pb_layer_net* net, int workers, int* first_layer, int* n_layers) {
  PB_GUARD_BEGIN
  const std::vector<int> n = pb::partition_by_flops(layer_list(net), workers);
  for (int s = 0, f = 0; s < workers; ++s) {
    if (first_layer) first_layer[s] = f;
    if (n_layers) n_layers[s] = n[s];
    f += n[s];
  }
  PB_GUARD_END
}

int pb_session_create_layers(const pb_layer_net* net, const pb_train_config* cfg, int rank,
                             int world, const uint8_t* nccl_ids, size_t ids_bytes,
                             pb_session** out) {
  PB_GUARD_BEGIN
  if (!out || !net || !cfg) throw std::invalid_argument("null argument");
  pb::SessionConfig c;
  {
    // the train-config fields (make_config needs a net spec: a 1-layer stub)
    const int w[2] = {1, 1}, a[1] = {0};
    const pb_net_spec stub{1, w, a, net->loss};
    c = make_config(&stub, cfg);
  }
  c.layers = layer_list(net);
  c.widths.clear();
  c.acts.clear();
  c.loss = net->loss;
  if (net->stage_layers) c.stage_layers.assign(net->stage_layers, net->stage_layers + cfg->workers);
  c.rank = rank;
  c.world = world;
  if (nccl_ids && ids_bytes) c.nccl_ids.assign(nccl_ids, nccl_ids + ids_bytes);
  auto* s = new pb_session;
  try {
    s->impl = std::make_unique<pb::Session>(c);
  } catch (...) {
    delete s;
    throw;
  }
  *out = s;
  PB_GUARD_END
}

int pb_session_ipc_export(pb_session* s, uint8_t* buf, int64_t cap, int64_t* len) {
  PB_GUARD_BEGIN
  const std::vector<uint8_t> b = S(s).ipc_export();
  if (len) *len = static_cast<int64_t>(b.size());
  if (buf) std::memcpy(buf, b.data(), std::min<size_t>(b.size(), static_cast<size_t>(cap)));
  PB_GUARD_END
}

int pb_session_ipc_connect(pb_session* s, const uint8_t* blobs, const int64_t* lens, int world) {
  PB_GUARD_BEGIN
  std::vector<std::vector<uint8_t>> v;
  size_t at = 0;
  for (int r = 0; r < world; ++r) {
    v.emplace_back(blobs + at, blobs + at + lens[r]);
    at += static_cast<size_t>(lens[r]);
  }
  S(s).ipc_connect(v);
  PB_GUARD_END
}

int pb_nccl_unique_id(uint8_t* out128) {
  PB_GUARD_BEGIN
  pb::P2P::unique_id(out128);
  PB_GUARD_END
}

int pb_plan_transfers(const pb_net_spec* net, const pb_train_config* cfg, int rank, int world,
                      int* n, int* kinds, int* dirs, int* peers, int64_t* bytes, int cap) {
  PB_GUARD_BEGIN
  pb::SessionConfig c = make_config(net, cfg);
  c.rank = rank;
  c.world = world;
  c.plan_only = true;
  c.use_graph = false;
  c.snapshots = false;
  pb::Session sess(c);
  const std::vector<pb::Transfer> t = sess.transfers();
  *n = static_cast<int>(t.size());
  for (int i = 0; i < *n && i < cap; ++i) {
    if (kinds) kinds[i] = t[i].send ? 1 : 0;
    if (dirs) dirs[i] = t[i].dir;
    if (peers) peers[i] = t[i].peer;
    if (bytes) bytes[i] = t[i].bytes;
  }
  PB_GUARD_END
}

int pb_plan_memory(const pb_net_spec* net, const pb_train_config* cfg, int rank, int world,
                   int64_t* weight_bytes, int64_t* act_bytes, int* pool, int* act_slots) {
  PB_GUARD_BEGIN
  pb::SessionConfig c = make_config(net, cfg);
  c.rank = rank;
  c.world = world;
  c.plan_only = true;
  c.use_graph = false;
  pb::Session sess(c);
  const auto b = sess.stage_bytes();
  const auto ps = sess.pool_sizes();
  const auto as = sess.act_slot_counts();
  for (size_t i = 0; i < b.size(); ++i) {
    if (weight_bytes) weight_bytes[i] = b[i].first;
    if (act_bytes) act_bytes[i] = b[i].second;
    if (pool) pool[i] = ps[i];
    if (act_slots) act_slots[i] = as[i];
  }
  PB_GUARD_END
}

namespace {
void hex16(uint64_t h, char* out) {
  static const char kHex[] = "0123456789abcdef";
  for (int i = 15; i >= 0; --i, h >>= 4) out[i] = kHex[h & 15];
  out[16] = 0;
}
}  // namespace

int pb_session_digests(pb_session* s, char* hex, int64_t cap) {
  PB_GUARD_BEGIN
  pb::Session& x = S(s);
  const auto& d = x.last_result().digests;
  if (d.empty()) throw std::logic_error("no digests: create the session with digests = 1 and run an epoch");
  if (cap < static_cast<int64_t>(d.size())) throw pb::capacity_error("digest buffer too small");
  for (size_t i = 0; i < d.size(); ++i) hex16(d[i], hex + 17 * i);
  PB_GUARD_END
}

int pb_session_params_digest(pb_session* s, int version, char* out17) {
  PB_GUARD_BEGIN
  hex16(S(s).params_digest(version), out17);
  PB_GUARD_END
}

int pb_session_destroy(pb_session* s) {
  PB_GUARD_BEGIN
  delete s;
  PB_GUARD_END
}

int pb_session_info_get(pb_session* s, pb_session_info* info) {
  PB_GUARD_BEGIN
  pb::Session& x = S(s);
  info->horizon = x.horizon();
  info->units = x.units();
  info->kernels_per_epoch = x.kernels_per_epoch();
  info->device_bytes = x.device_bytes();
  info->param_count = x.param_count();
  const auto ps = x.pool_sizes();
  const auto as = x.act_slot_counts();
  for (size_t i = 0; i < ps.size(); ++i) {
    if (info->pool_sizes) info->pool_sizes[i] = ps[i];
    if (info->act_slots) info->act_slots[i] = as[i];
  }
  for (int i = 0; i < x.config().W; ++i) {
    if (info->stage_first_layer) info->stage_first_layer[i] = x.stage_first_layer(i + 1);
    if (info->stage_layers) info->stage_layers[i] = x.stage_layer_count(i + 1);
  }
  PB_GUARD_END
}

int pb_session_load_params(pb_session* s, const double* flat, int64_t n) {
  PB_GUARD_BEGIN
  pb::Session& x = S(s);
  if (n != x.param_count())
    throw pipesim::structural_error(n < x.param_count()
                                        ? "parameter vector shorter than the network"
                                        : "parameter vector longer than the network");
  x.load_params(flat);
  PB_GUARD_END
}

int pb_session_load_stage_params(pb_session* s, int stage, const double* p, int64_t n) {
  PB_GUARD_BEGIN
  pb::Session& x = S(s);
  if (stage < 1 || stage > x.config().W) throw std::invalid_argument("stage out of range");
  if (n != x.stage_param_count(stage))
    throw pipesim::structural_error(n < x.stage_param_count(stage)
                                        ? "parameter vector shorter than the stage"
                                        : "parameter vector longer than the stage");
  x.load_stage_params(stage, p);
  PB_GUARD_END
}

int pb_session_read_params(pb_session* s, double* flat, int64_t n) {
  PB_GUARD_BEGIN
  pb::Session& x = S(s);
  if (n != x.param_count()) throw pb::capacity_error("parameter count mismatch");
  x.read_params(flat);
  PB_GUARD_END
}

int pb_session_upload(pb_session* s, const void* x, int x_dtype, const void* y,
                      int y_dtype) {
  PB_GUARD_BEGIN
  S(s).upload(x, dtype(x_dtype), y, dtype(y_dtype));
  PB_GUARD_END
}

int pb_session_run_epoch(pb_session* s, pb_epoch_out* out) {
  PB_GUARD_BEGIN
  pb::Session& x = S(s);
  const pb::EpochResult r = x.run_epoch();
  fill(r, x, out);
  PB_GUARD_END
}

int pb_session_train_epoch(pb_session* s, const void* x, int x_dtype,
                           const void* y, int y_dtype, pb_epoch_out* out) {
  PB_GUARD_BEGIN
  pb::Session& ss = S(s);
  const pb::EpochResult r = ss.train_epoch_host(x, dtype(x_dtype), y, dtype(y_dtype));
  fill(r, ss, out);
  PB_GUARD_END
}

int pb_session_trace_document(pb_session* s, char* buf, int64_t cap, int64_t* len) {
  PB_GUARD_BEGIN
  const std::string d = S(s).trace_document();
  if (len) *len = static_cast<int64_t>(d.size());
  if (buf && cap > 0) {
    const size_t n = std::min<size_t>(d.size(), static_cast<size_t>(cap - 1));
    std::memcpy(buf, d.data(), n);
    buf[n] = '\0';
  }
  PB_GUARD_END
}

int pb_session_kernel_times(pb_session* s, float* ms, double* flops, int max, int* n) {
  PB_GUARD_BEGIN
  const std::vector<float> t = S(s).kernel_times_ms();
  const std::vector<double>& f = S(s).kernel_flops();
  if (n) *n = static_cast<int>(t.size());
  for (int i = 0; i < max && i < static_cast<int>(t.size()); ++i) {
    if (ms) ms[i] = t[i];
    if (flops) flops[i] = f[i];
  }
  PB_GUARD_END
}

int pb_session_profile_epoch(pb_session* s, pb_epoch_out* out, pb_epoch_profile* prof) {
  PB_GUARD_BEGIN
  pb::Session& x = S(s);
  pb::EpochProfile p;
  const pb::EpochResult r = x.profile_epoch(&p);
  fill(r, x, out);
  if (prof) {
    prof->makespan_ms = p.makespan_ms;
    if (prof->stage_busy_ms)
      for (size_t i = 0; i < p.busy_ms.size(); ++i) prof->stage_busy_ms[i] = p.busy_ms[i];
    prof->n_nodes = static_cast<int>(p.nodes.size());
    const int n = std::min(prof->n_nodes, prof->max_nodes);
    for (int i = 0; i < n; ++i) {
      const pb::NodeTiming& t = p.nodes[i];
      if (prof->node_stage) prof->node_stage[i] = t.stage;
      if (prof->node_fwd) prof->node_fwd[i] = t.fwd;
      if (prof->node_mini) prof->node_mini[i] = t.mini;
      if (prof->node_micro_lo) prof->node_micro_lo[i] = t.micro_lo;
      if (prof->node_micro_hi) prof->node_micro_hi[i] = t.micro_hi;
      if (prof->node_start_ms) prof->node_start_ms[i] = t.start_ms;
      if (prof->node_end_ms) prof->node_end_ms[i] = t.end_ms;
    }
  }
  PB_GUARD_END
}

int pb_session_snapshot(pb_session* s, int stage, int version, double* out, int64_t n) {
  PB_GUARD_BEGIN
  pb::Session& x = S(s);
  if (n != x.stage_param_count(stage)) throw pb::capacity_error("stage parameter count mismatch");
  const float* p = x.snapshot(stage, version);
  for (int64_t i = 0; i < n; ++i) out[i] = p[i];
  PB_GUARD_END
}

int pb_session_read_version(pb_session* s, int stage, int version, double* out,
                            int64_t n) {
  PB_GUARD_BEGIN
  pb::Session& x = S(s);
  if (n != x.stage_param_count(stage)) throw pb::capacity_error("stage parameter count mismatch");
  const int M = x.config().M;
  if (x.has_snapshots()) {
    const float* p = x.snapshot(stage, version);
    for (int64_t i = 0; i < n; ++i) out[i] = p[i];
  } else if (version == M || version == M - 1) {
    x.read_stage_master(stage, version, out);
  } else {
    throw pipesim::structural_error("stage " + std::to_string(stage) + " does not hold version " +
                                    std::to_string(version) + " (no snapshots)");
  }
  PB_GUARD_END
}

int pb_make_classification_task(int rows, int features, int classes, uint64_t seed,
                                double* x64, float* x32, int* labels) {
  PB_GUARD_BEGIN
  if (rows < 0 || features < 1 || classes < 1) throw std::invalid_argument("bad shape");
  std::mt19937_64 g(seed);
  const size_t n = static_cast<size_t>(rows) * features;
  for (size_t i = 0; i < n; ++i) {
    const double v = static_cast<double>(g() >> 11) * 0x1.0p-53;
    if (x64) x64[i] = v;
    if (x32) x32[i] = static_cast<float>(v);
  }
  for (int r = 0; r < rows; ++r) {
    const int c = static_cast<int>(g() % static_cast<uint64_t>(classes));
    if (labels) labels[r] = c;
  }
  PB_GUARD_END
}

}  // extern "C"
