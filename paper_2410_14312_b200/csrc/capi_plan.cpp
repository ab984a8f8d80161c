// C ABI over the host plan layer and model helpers (include/pipesim_b200.h).
// Marshals flat arrays to / from the pipesim:: value types.
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "pipesim_core.hpp"
#include "status.hpp"

namespace pb {
int translate_exception();
}

#define PB_GUARD_BEGIN try {
#define PB_GUARD_END \
  return PB_OK;      \
  }                  \
  catch (...) {      \
    return pb::translate_exception(); \
  }

namespace {

using namespace pipesim;

sim_config to_cfg(const pb_sim_config* c) {
  if (!c) throw std::invalid_argument("null sim_config");
  sim_config s;
  s.workers = c->workers;
  s.micro_batches = c->micro_batches;
  s.mini_batches = c->mini_batches;
  s.backward_cost_factor = c->backward_cost_factor;
  s.samples_per_mini_batch = c->samples_per_mini_batch;
  s.seed = c->seed;
  return s;
}

schedule_mode to_mode(int m) {
  if (m == PB_MODE_TIMEPREST) return schedule_mode::timeprest;
  if (m == PB_MODE_PIPEDREAM) return schedule_mode::pipedream;
  throw std::invalid_argument("unknown schedule mode " + std::to_string(m));
}

task_kind to_kind(int k) {
  switch (k) {
    case PB_TASK_FORWARD: return task_kind::forward_micro;
    case PB_TASK_BACKWARD: return task_kind::backward_mini;
    default: return task_kind::idle;
  }
}

int from_kind(task_kind k) {
  switch (k) {
    case task_kind::forward_micro: return PB_TASK_FORWARD;
    case task_kind::backward_mini: return PB_TASK_BACKWARD;
    default: return PB_TASK_IDLE;
  }
}

schedule_grid grid_from(const sim_config& cfg, int mode, const pb_task* cells,
                        int horizon) {
  schedule_grid g(cfg, to_mode(mode));
  if (horizon < 0) throw std::invalid_argument("negative horizon");
  for (int w = 1; w <= cfg.workers; ++w)
    for (int t = 1; t <= horizon; ++t) {
      const pb_task& c = cells[static_cast<size_t>(w - 1) * horizon + (t - 1)];
      // put() on every cell fixes the horizon even for trailing idle slots
      g.put(w, t, task{to_kind(c.kind), c.mini, c.micro});
    }
  return g;
}

network_spec net_from(const pb_net_spec* n) {
  if (!n || n->n_layers < 0) throw std::invalid_argument("bad network spec");
  network_spec s;
  s.widths.assign(n->widths, n->widths + n->n_layers + 1);
  for (int l = 0; l < n->n_layers; ++l) {
    const int a = n->activations[l];
    if (a < 0 || a > 3) throw std::invalid_argument("bad activation id");
    s.activations.push_back(static_cast<activation_kind>(a));
  }
  if (n->loss != PB_LOSS_MSE && n->loss != PB_LOSS_SOFTMAX_CE)
    throw std::invalid_argument("bad loss id");
  s.loss = n->loss == PB_LOSS_MSE ? loss_kind::mse : loss_kind::softmax_cross_entropy;
  return s;
}

}  // namespace

extern "C" {

int pb_validate_config(const pb_sim_config* cfg) {
  PB_GUARD_BEGIN
  validate(to_cfg(cfg));
  PB_GUARD_END
}

int pb_schedule_build(const pb_sim_config* cfg, int mode, int* horizon,
                      pb_task* cells, int cap_slots) {
  PB_GUARD_BEGIN
  const sim_config c = to_cfg(cfg);
  const schedule_grid g = to_mode(mode) == schedule_mode::timeprest
                              ? build_nf1b_schedule(c)
                              : build_1f1b_schedule(c);
  *horizon = g.horizon();
  if (!cells || cap_slots < g.horizon())
    throw pb::capacity_error("schedule needs " + std::to_string(g.horizon()) +
                             " slots");
  for (int w = 1; w <= c.workers; ++w)
    for (int t = 1; t <= g.horizon(); ++t) {
      const task& k = g.at(w, t);
      cells[static_cast<size_t>(w - 1) * cap_slots + (t - 1)] =
          pb_task{from_kind(k.kind), k.mini, k.micro};
    }
  PB_GUARD_END
}

int pb_schedule_document(const pb_sim_config* cfg, int mode, char* buf, int64_t cap,
                         int64_t* len) {
  PB_GUARD_BEGIN
  const sim_config c = to_cfg(cfg);
  const schedule_grid g = to_mode(mode) == schedule_mode::timeprest ? build_nf1b_schedule(c)
                                                                     : build_1f1b_schedule(c);
  const std::string d = schedule_document_json(g, assign_versions(g, c));
  if (len) *len = static_cast<int64_t>(d.size());
  if (buf && cap > 0) {
    const size_t n = std::min<size_t>(d.size(), static_cast<size_t>(cap - 1));
    std::memcpy(buf, d.data(), n);
    buf[n] = '\0';
  }
  PB_GUARD_END
}

int pb_schedule_validate(const pb_sim_config* cfg, int mode, const pb_task* cells,
                         int horizon, int* n_violations, int* kinds, int cap_kinds,
                         char* messages, int cap_messages) {
  PB_GUARD_BEGIN
  const sim_config c = to_cfg(cfg);
  const validation_report r = validate_schedule(grid_from(c, mode, cells, horizon), c);
  *n_violations = static_cast<int>(r.violations.size());
  std::string text;
  for (size_t i = 0; i < r.violations.size(); ++i) {
    if (kinds && static_cast<int>(i) < cap_kinds)
      kinds[i] = static_cast<int>(r.violations[i].kind);
    text += r.violations[i].message;
    text.push_back('\n');
  }
  if (messages && cap_messages > 0) {
    const size_t n = std::min(text.size(), static_cast<size_t>(cap_messages - 1));
    std::memcpy(messages, text.data(), n);
    messages[n] = '\0';
  }
  PB_GUARD_END
}

int pb_assign_versions(const pb_sim_config* cfg, int mode, const pb_task* cells,
                       int horizon, pb_commit* commits, pb_pin* pins,
                       pb_consume* consumptions, int* update_source,
                       int* full_commit_slot) {
  PB_GUARD_BEGIN
  const sim_config c = to_cfg(cfg);
  const version_ledger L = assign_versions(grid_from(c, mode, cells, horizon), c);
  for (size_t i = 0; i < L.commits.size(); ++i)
    commits[i] = {L.commits[i].version, L.commits[i].mini, L.commits[i].stage,
                  L.commits[i].slot};
  for (size_t i = 0; i < L.pins.size(); ++i)
    pins[i] = {L.pins[i].mini, L.pins[i].micro, L.pins[i].slot, L.pins[i].version};
  for (size_t i = 0; i < L.consumptions.size(); ++i)
    consumptions[i] = {L.consumptions[i].mini, L.consumptions[i].stage,
                       L.consumptions[i].slot, L.consumptions[i].version};
  for (size_t i = 0; i < L.update_source.size(); ++i) update_source[i] = L.update_source[i];
  for (size_t i = 0; i < L.full_commit_slot.size(); ++i)
    full_commit_slot[i] = L.full_commit_slot[i];
  PB_GUARD_END
}

int pb_measure_version_difference(const pb_sim_config* cfg,
                                  const int* update_source, int strict, int* v) {
  PB_GUARD_BEGIN
  version_ledger L;
  L.cfg = to_cfg(cfg);
  L.update_source.assign(update_source, update_source + L.cfg.mini_batches);
  *v = measure_version_difference(L, strict != 0);
  PB_GUARD_END
}

int pb_closed_form_v(int workers, int micro_batches, int* v) {
  PB_GUARD_BEGIN
  *v = closed_form_v(workers, micro_batches);
  PB_GUARD_END
}

int pb_forward_span(int workers, int micro_batches, int mini_ordinal, int* span) {
  PB_GUARD_BEGIN
  *span = forward_span(workers, micro_batches, mini_ordinal);
  PB_GUARD_END
}

int pb_backward_span(int workers, int* span) {
  PB_GUARD_BEGIN
  *span = backward_span(workers);
  PB_GUARD_END
}

int pb_overlap_condition(int workers, int micro_batches, int* out) {
  PB_GUARD_BEGIN
  *out = overlap_condition(workers, micro_batches) ? 1 : 0;
  PB_GUARD_END
}

int pb_decompose_sequences(const pb_sim_config* cfg, const int* update_source,
                           int mini_batches, int* n_sequences, int* seq_len,
                           int* seq_mini, int* v_measured) {
  PB_GUARD_BEGIN
  version_ledger L;
  L.cfg = to_cfg(cfg);
  L.update_source.assign(update_source, update_source + L.cfg.mini_batches);
  const sequence_decomposition d = decompose_sequences(L, mini_batches);
  *n_sequences = static_cast<int>(d.sequences.size());
  size_t pos = 0;
  for (size_t i = 0; i < d.sequences.size(); ++i) {
    seq_len[i] = static_cast<int>(d.sequences[i].size());
    for (int m : d.sequences[i]) seq_mini[pos++] = m;
  }
  *v_measured = d.version_difference_measured;
  PB_GUARD_END
}

int pb_retention_timeline(const pb_sim_config* cfg, int mode, const pb_task* cells,
                          int horizon, const pb_pin* pins, pb_interval* intervals,
                          int* peak) {
  PB_GUARD_BEGIN
  const sim_config c = to_cfg(cfg);
  const schedule_grid g = grid_from(c, mode, cells, horizon);
  version_ledger L;
  L.cfg = c;
  L.mode = to_mode(mode);
  const int units = L.mode == schedule_mode::timeprest ? c.micro_batches : 1;
  for (int i = 0; i < c.mini_batches * units; ++i)
    L.pins.push_back({pins[i].mini, pins[i].micro, pins[i].slot, pins[i].version});
  const retention_timeline T = build_retention_timeline(L, g);
  for (int s = 0; s < c.workers; ++s) {
    peak[s] = T.peak_concurrent[s];
    for (int v = 0; v <= c.mini_batches; ++v) {
      const retention_interval& iv = T.per_stage[s][v];
      intervals[static_cast<size_t>(s) * (c.mini_batches + 1) + v] = {
          iv.version, iv.retained_from_slot, iv.freed_at_slot};
    }
  }
  PB_GUARD_END
}

int pb_staleness(const pb_sim_config* cfg, const pb_commit* commits,
                 const pb_consume* consumptions, int* staleness) {
  PB_GUARD_BEGIN
  version_ledger L;
  L.cfg = to_cfg(cfg);
  const int n = L.cfg.mini_batches * L.cfg.workers;
  for (int i = 0; i < n; ++i) {
    L.commits.push_back({commits[i].version, commits[i].mini, commits[i].stage,
                         commits[i].slot});
    L.consumptions.push_back({consumptions[i].mini, consumptions[i].stage,
                              consumptions[i].slot, consumptions[i].version});
  }
  const staleness_report_t r = staleness_report(L);
  for (size_t i = 0; i < r.entries.size(); ++i) staleness[i] = r.entries[i].staleness;
  PB_GUARD_END
}

int pb_partition_model(const pb_net_spec* net, int workers, int* first_layer,
                       int* n_layers) {
  PB_GUARD_BEGIN
  const std::vector<stage_model> st = partition_model(net_from(net), workers);
  for (size_t s = 0; s < st.size(); ++s) {
    first_layer[s] = st[s].first_layer;
    n_layers[s] = static_cast<int>(st[s].layers.size());
  }
  PB_GUARD_END
}

int64_t pb_param_count(const pb_net_spec* net) {
  try {
    return net_from(net).param_count();
  } catch (...) {
    pb::translate_exception();
    return -1;
  }
}

int pb_init_network_params(const pb_net_spec* net, uint64_t seed, double* out,
                           int64_t n) {
  PB_GUARD_BEGIN
  const std::vector<double> p = init_network_params(net_from(net), seed);
  if (static_cast<int64_t>(p.size()) != n)
    throw pb::capacity_error("parameter count is " + std::to_string(p.size()));
  std::memcpy(out, p.data(), p.size() * sizeof(double));
  PB_GUARD_END
}

int pb_make_synthetic_task(int samples, uint64_t seed, double* x, double* y) {
  PB_GUARD_BEGIN
  const dataset d = make_synthetic_task(samples, seed);
  std::memcpy(x, d.x.data.data(), d.x.data.size() * sizeof(double));
  std::memcpy(y, d.y.data.data(), d.y.data.size() * sizeof(double));
  PB_GUARD_END
}

int pb_params_digest(const double* values, int64_t n, char* out17) {
  PB_GUARD_BEGIN
  const std::string h = pb::digest_spans({{values, n}});
  std::memcpy(out17, h.c_str(), 17);
  PB_GUARD_END
}

int pb_checkpoint_stage(int stage_id, int first_layer, int n_layers, const int* layers,
                        int version, const double* params, int64_t n, int loss, int epoch,
                        const char* path) {
  PB_GUARD_BEGIN
  if (!path || (n > 0 && !params) || n_layers < 1 || !layers)
    throw std::invalid_argument("pb_checkpoint_stage: null argument");
  stage_model st;
  st.stage_id = stage_id;
  st.first_layer = first_layer;
  for (int i = 0; i < n_layers; ++i)
    st.layers.push_back({layers[3 * i], layers[3 * i + 1],
                         static_cast<activation_kind>(layers[3 * i + 2])});
  if (st.param_count() != n)
    throw pipesim::structural_error("stage holds " + std::to_string(st.param_count()) +
                                    " params, got " + std::to_string(n));
  st.version_store[version].assign(params, params + n);
  st.current_version = version;
  checkpoint_stage(st, loss == PB_LOSS_MSE ? loss_kind::mse : loss_kind::softmax_cross_entropy,
                   epoch, path);
  PB_GUARD_END
}

int pb_restore_stage(const char* path, int expected_stage, int expected_epoch,
                     pb_restored_stage* info, int* layers, int layers_cap, double* params,
                     int64_t cap) {
  PB_GUARD_BEGIN
  if (!path || !info) throw std::invalid_argument("pb_restore_stage: null argument");
  const restored_stage r = restore_stage(path, expected_stage, expected_epoch);
  const std::vector<double>& p = r.stage.current_params();
  info->stage_id = r.stage.stage_id;
  info->first_layer = r.stage.first_layer;
  info->n_layers = static_cast<int>(r.stage.layers.size());
  info->version = r.stage.current_version;
  info->loss = r.loss == loss_kind::mse ? PB_LOSS_MSE : PB_LOSS_SOFTMAX_CE;
  info->epoch = r.epoch;
  info->n_values = static_cast<int64_t>(p.size());
  if (info->n_layers > layers_cap || info->n_values > cap)
    throw pb::capacity_error("checkpoint holds " + std::to_string(info->n_layers) +
                             " layers / " + std::to_string(info->n_values) + " values");
  for (int i = 0; i < info->n_layers; ++i) {
    layers[3 * i] = r.stage.layers[i].in;
    layers[3 * i + 1] = r.stage.layers[i].out;
    layers[3 * i + 2] = static_cast<int>(r.stage.layers[i].act);
  }
  std::memcpy(params, p.data(), p.size() * sizeof(double));
  PB_GUARD_END
}

}  // extern "C"
