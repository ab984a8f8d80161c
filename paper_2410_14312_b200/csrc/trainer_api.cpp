// Drop-in trainer entry points of the pipesim:: C++ API, executed on B200.
//
// These are the functions a reference user calls (proj/include/pipesim/
// trainer.hpp:159-188): train_epoch, network_loss / network_gradient,
// run_training.  They keep the reference contract (stages mutated in place,
// version_store holding exactly the retained versions, epoch_log layout,
// exceptions) and reach the GPU only through the C ABI (pipesim_b200.h).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <filesystem>
#include <map>
#include <memory>
#include <mutex>
#include <sstream>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/pipesim_b200.h"
#include "pipesim_core.hpp"

namespace pipesim {

namespace b200 {
namespace {
std::mutex g_opt_mu;
options g_opt;
}  // namespace
void set_options(const options& o) {
  std::lock_guard<std::mutex> lk(g_opt_mu);
  g_opt = o;
}
options get_options() {
  std::lock_guard<std::mutex> lk(g_opt_mu);
  return g_opt;
}
namespace {
thread_local epoch_timing g_timing;
}
epoch_timing last_epoch_timing() { return g_timing; }
}  // namespace b200

namespace {

using clk = std::chrono::steady_clock;
double ms_since(clk::time_point& t) {
  const clk::time_point now = clk::now();
  const double ms = std::chrono::duration<double, std::milli>(now - t).count();
  t = now;
  return ms;
}

[[noreturn]] void rethrow_status(int st) {
  char msg[4096];
  pb_last_error(msg, sizeof(msg));
  switch (st) {
    case PB_ERR_DOMAIN: {
      char field[256];
      pb_last_error_field(field, sizeof(field));
      throw domain_error(field, msg);
    }
    case PB_ERR_STRUCTURAL: throw structural_error(msg);
    case PB_ERR_INSUFFICIENT_HORIZON: throw insufficient_horizon_error(msg);
    case PB_ERR_INTEGRITY: {
      int s = 0, e = 0;
      pb_last_error_stage_epoch(&s, &e);
      throw integrity_error(msg, s, e);
    }
    case PB_ERR_IO: throw io_error(msg);
    default: throw std::runtime_error(msg);
  }
}

void ok(int st) {
  if (st != PB_OK) rethrow_status(st);
}

// check_train_config (trainer.cpp:351-370), same messages.
void check_config(const train_config& cfg, const dataset& data) {
  if (cfg.mini_batch_size < 1 || cfg.mini_batches < 1)
    throw domain_error("mini_batches", "mini-batch count/size must be >= 1");
  if (cfg.micro_batches < 1)
    throw domain_error("micro_batches", "micro-batch count must be >= 1");
  if (cfg.mini_batch_size % cfg.micro_batches != 0)
    throw domain_error("mini_batch_size",
                       "mini-batch size " + std::to_string(cfg.mini_batch_size) +
                           " is not divisible by micro-batch count " +
                           std::to_string(cfg.micro_batches));
  if (data.x.rows != cfg.mini_batches * cfg.mini_batch_size)
    throw structural_error("dataset holds " + std::to_string(data.x.rows) +
                           " rows, expected M*Ms = " +
                           std::to_string(cfg.mini_batches * cfg.mini_batch_size));
  if (data.x.cols != cfg.net.widths.front() || data.y.cols != cfg.net.widths.back())
    throw structural_error("dataset width does not match the network");
}

// A cached session is shared by every caller with the same config; `use`
// serialises load_params .. read_params so concurrent same-shaped calls on
// different threads cannot interleave on one device state (the reference's
// train_epoch is re-entrant).
struct SessionHandle {
  pb_session* s = nullptr;
  std::mutex use;
  ~SessionHandle() {
    if (s) pb_session_destroy(s);
  }
};

// One resident session per (network, config, mode); reused across epochs.
std::mutex g_cache_mu;
std::map<std::string, std::shared_ptr<SessionHandle>> g_cache;

std::string cache_key(const train_config& cfg, train_mode mode, bool snaps, bool digests,
                      int device, bool graph) {
  std::ostringstream k;
  for (int w : cfg.net.widths) k << w << ',';
  k << '|';
  for (auto a : cfg.net.activations) k << static_cast<int>(a) << ',';
  k << '|' << static_cast<int>(cfg.net.loss) << '|' << cfg.workers << '|' << cfg.micro_batches
    << '|' << cfg.mini_batch_size << '|' << cfg.mini_batches << '|' << format_double(cfg.learning_rate)
    << '|' << static_cast<int>(mode) << '|' << snaps << '|' << digests << '|' << device << '|'
    << graph;
  return k.str();
}

std::shared_ptr<SessionHandle> session_for(const train_config& cfg, train_mode mode, bool snaps,
                                           int* units, bool digests = false) {
  const b200::options opt = b200::get_options();
  const std::string key = cache_key(cfg, mode, snaps, digests, opt.device, opt.use_graph) +
                          (opt.verify_fp32 ? "|fp32" : "");
  std::lock_guard<std::mutex> lk(g_cache_mu);
  auto it = g_cache.find(key);
  *units = mode == train_mode::timeprest ? cfg.micro_batches : 1;
  if (it != g_cache.end()) return it->second;
  if (g_cache.size() >= 8) g_cache.clear();
  std::vector<int> widths = cfg.net.widths, acts;
  for (auto a : cfg.net.activations) acts.push_back(static_cast<int>(a));
  pb_net_spec net{cfg.net.layer_count(), widths.data(), acts.data(),
                  cfg.net.loss == loss_kind::mse ? PB_LOSS_MSE : PB_LOSS_SOFTMAX_CE};
  pb_train_config tc{};
  tc.workers = cfg.workers;
  tc.micro_batches = cfg.micro_batches;
  tc.mini_batch_size = cfg.mini_batch_size;
  tc.mini_batches = cfg.mini_batches;
  tc.learning_rate = cfg.learning_rate;
  tc.mode = mode == train_mode::timeprest   ? PB_TRAIN_TIMEPREST
            : mode == train_mode::pipedream ? PB_TRAIN_PIPEDREAM
                                            : PB_TRAIN_SEQUENTIAL;
  tc.device = opt.device;
  tc.use_graph = opt.use_graph ? 1 : 0;
  tc.snapshots = snaps ? 1 : 0;
  tc.precision = opt.verify_fp32 ? PB_PRECISION_FP32_VERIFY : PB_PRECISION_BF16;
  tc.digests = digests ? 1 : 0;
  auto h = std::make_shared<SessionHandle>();
  ok(pb_session_create(&net, &tc, &h->s));
  g_cache[key] = h;
  return h;
}

}  // namespace

epoch_log train_epoch(std::vector<stage_model>& stages, const dataset& data,
                      const train_config& cfg, train_mode mode, int epoch,
                      const slot_observer& observer) {
  check_config(cfg, data);
  if (static_cast<int>(stages.size()) != cfg.workers)
    throw structural_error("stage count does not match workers");
  const int W = cfg.workers, M = cfg.mini_batches;
  b200::epoch_timing tm;
  const clk::time_point t_start = clk::now();
  clk::time_point tp = t_start;

  // Plan of this epoch (same as replay_grid's, trainer.cpp:401-404).
  std::unique_ptr<schedule_grid> grid;
  version_ledger ledger;
  retention_timeline timeline;
  if (mode != train_mode::sequential) {
    sim_config sc;
    sc.workers = W;
    sc.micro_batches = cfg.micro_batches;
    sc.mini_batches = M;
    sc.samples_per_mini_batch = cfg.mini_batch_size;
    sc.seed = cfg.seed;
    grid = std::make_unique<schedule_grid>(mode == train_mode::timeprest ? build_nf1b_schedule(sc)
                                                                         : build_1f1b_schedule(sc));
    ledger = assign_versions(*grid, sc);
    timeline = build_retention_timeline(ledger, *grid);
  }

  tm.plan_ms = ms_since(tp);
  const b200::options opt = b200::get_options();
  const long long P = cfg.net.param_count();
  // Per-mini-batch checksums (trainer.cpp:492-501) are computed on the
  // device inside the epoch (digest_dev.hpp), so the reference's contract --
  // a checksum for every mini-batch -- holds at every network size;
  // final_only (or automatic above digest_auto_limit) keeps only the final one.
  const bool every_mini = opt.digest == b200::digest_policy::every_mini ||
                          (opt.digest == b200::digest_policy::automatic &&
                           P <= opt.digest_auto_limit);
  // retained versions older than M-1 (1F1B stashes) need snapshots
  bool old_retained = false;
  if (grid)
    for (int s = 0; s < W; ++s)
      for (const auto& iv : timeline.per_stage[s])
        if (iv.freed_at_slot > timeline.horizon && iv.version < M - 1) old_retained = true;
  const bool snaps = static_cast<bool>(observer) || old_retained;

  int units = 1;
  std::shared_ptr<SessionHandle> h = session_for(cfg, mode, snaps, &units, every_mini);
  std::lock_guard<std::mutex> in_use(h->use);

  // Rebase: version 0 := the current weights (trainer.cpp:372-379), stage by
  // stage straight from the caller's vectors (no gathered copy).
  for (int s = 0; s < W; ++s) {
    const std::vector<double>& cur = stages[s].current_params();
    ok(pb_session_load_stage_params(h->s, s + 1, cur.data(), static_cast<int64_t>(cur.size())));
  }
  ok(pb_synchronize());
  tm.load_ms = ms_since(tp);
  ok(pb_session_upload(h->s, data.x.data.data(), PB_DTYPE_F64, data.y.data.data(), PB_DTYPE_F64));
  ok(pb_synchronize());
  tm.upload_ms = ms_since(tp);

  std::vector<double> losses(M);
  std::vector<int> pinned(static_cast<size_t>(M) * units), consumed(M),
      dev_fwd(static_cast<size_t>(M) * units * W), dev_bwd(static_cast<size_t>(M) * W),
      dev_cur(W);
  pb_epoch_out out{losses.data(), pinned.data(), consumed.data(), dev_fwd.data(),
                   dev_bwd.data(), dev_cur.data(), 0.f};
  ok(pb_session_run_epoch(h->s, &out));
  tm.step_ms = ms_since(tp);
  tm.device_ms = out.device_ms;
  // the epoch's digests (every mini-batch + final) were computed in the graph;
  // otherwise only the final one, on the device now
  std::vector<char> digests(static_cast<size_t>(M + 1) * 17, 0);
  if (every_mini)
    ok(pb_session_digests(h->s, digests.data(), M + 1));
  else
    ok(pb_session_params_digest(h->s, M, digests.data() + static_cast<size_t>(M) * 17));
  tm.digest_ms += ms_since(tp);

  // The device-observed version trace must equal the ledger, bit for bit.
  for (int k = 0; k < M; ++k)
    for (int j = 0; j < units; ++j)
      for (int s = 0; s < W; ++s)
        if (dev_fwd[(static_cast<size_t>(k) * units + j) * W + s] != pinned[k * units + j])
          throw structural_error("device version trace diverged from the ledger (forward)");
  for (int s = 0; s < W; ++s)
    if (dev_cur[s] != M) throw structural_error("device current version diverged from the ledger");

  std::vector<int64_t> sizes(W);
  for (int s = 0; s < W; ++s) sizes[s] = stages[s].param_count();
  // Final weights (version M) straight into each stage's version store.  The
  // caller's current vector is reused as the buffer (same size, pages already
  // mapped), so repeated epochs do not fault 2 GB of fresh pages per call.
  std::vector<std::vector<double>> final_vals(W);
  for (int s = 0; s < W; ++s) {
    auto it = stages[s].version_store.find(stages[s].current_version);
    if (it != stages[s].version_store.end()) final_vals[s] = std::move(it->second);
    final_vals[s].resize(static_cast<size_t>(sizes[s]));
    ok(pb_session_read_version(h->s, s + 1, M, final_vals[s].data(), sizes[s]));
  }
  tm.readback_ms += ms_since(tp);

  auto version_values = [&](int s1, int v) {
    std::vector<double> vals(sizes[s1 - 1]);
    ok(pb_session_read_version(h->s, s1, v, vals.data(), sizes[s1 - 1]));
    tm.readback_ms += ms_since(tp);
    return vals;
  };

  epoch_log log;
  log.epoch = epoch;
  for (int k = 1; k <= M; ++k) {
    mini_log m;
    m.mini = k;
    m.loss = losses[k - 1];
    for (int j = 0; j < units; ++j) m.pinned.push_back(pinned[(k - 1) * units + j]);
    m.consumed = consumed[k - 1];
    if (every_mini) m.checksum.assign(digests.data() + static_cast<size_t>(k - 1) * 17, 16);
    log.minis.push_back(std::move(m));
  }

  for (int s = 0; s < W; ++s) {
    stage_model& st = stages[s];
    st.version_store.clear();
    st.version_store[M] = std::move(final_vals[s]);
    if (grid)
      for (const auto& iv : timeline.per_stage[s])
        if (iv.freed_at_slot > timeline.horizon && iv.version != M)
          st.version_store[iv.version] = version_values(s + 1, iv.version);
    st.current_version = M;
  }
  tm.readback_ms += ms_since(tp);
  log.final_checksum = std::string(digests.data() + static_cast<size_t>(M) * 17, 16);

  if (observer && grid) {
    // verify mode: replay the retention timeline with the committed snapshots
    std::vector<stage_model> view = stages;
    for (int t = 1; t <= timeline.horizon; ++t) {
      for (int s = 0; s < W; ++s) {
        view[s].version_store.clear();
        int cur = 0;
        for (const auto& iv : timeline.per_stage[s])
          if (iv.retained_from_slot <= t && t < iv.freed_at_slot) {
            view[s].version_store[iv.version] = version_values(s + 1, iv.version);
            cur = std::max(cur, iv.version);
          }
        view[s].current_version = cur;
      }
      observer(t, view);
    }
  }
  tm.total_ms = std::chrono::duration<double, std::milli>(clk::now() - t_start).count();
  b200::g_timing = tm;
  return log;
}

double network_loss(const network_spec& spec, const std::vector<double>& params,
                    const dataset& data) {
  // single-stage sequential forward with learning rate 0 (trainer.cpp:662-668)
  train_config cfg;
  cfg.net = spec;
  cfg.workers = 1;
  cfg.micro_batches = 1;
  cfg.mini_batch_size = data.x.rows;
  cfg.mini_batches = 1;
  cfg.learning_rate = 0.0;
  check_config(cfg, data);
  int units = 1;
  auto h = session_for(cfg, train_mode::sequential, false, &units);
  std::lock_guard<std::mutex> in_use(h->use);
  ok(pb_session_load_params(h->s, params.data(), static_cast<int64_t>(params.size())));
  ok(pb_session_upload(h->s, data.x.data.data(), PB_DTYPE_F64, data.y.data.data(), PB_DTYPE_F64));
  double loss = 0.0;
  pb_epoch_out out{&loss, nullptr, nullptr, nullptr, nullptr, nullptr, 0.f};
  ok(pb_session_run_epoch(h->s, &out));
  return loss;
}

std::vector<double> network_gradient(const network_spec& spec, const std::vector<double>& params,
                                     const dataset& data) {
  // One SGD step with learning rate 1 on the fp32 masters: g = W0 - W1
  // (trainer.cpp:670-679).  Precision: bf16 operands / fp32 accumulate, and
  // the recovered gradient carries an absolute error of ~2^-25 |W|.
  train_config cfg;
  cfg.net = spec;
  cfg.workers = 1;
  cfg.micro_batches = 1;
  cfg.mini_batch_size = data.x.rows;
  cfg.mini_batches = 1;
  cfg.learning_rate = 1.0;
  check_config(cfg, data);
  int units = 1;
  auto h = session_for(cfg, train_mode::sequential, false, &units);
  std::lock_guard<std::mutex> in_use(h->use);
  ok(pb_session_load_params(h->s, params.data(), static_cast<int64_t>(params.size())));
  ok(pb_session_upload(h->s, data.x.data.data(), PB_DTYPE_F64, data.y.data.data(), PB_DTYPE_F64));
  ok(pb_session_run_epoch(h->s, nullptr));
  std::vector<double> after(params.size());
  ok(pb_session_read_params(h->s, after.data(), static_cast<int64_t>(after.size())));
  std::vector<double> g(params.size());
  for (size_t i = 0; i < g.size(); ++i)
    g[i] = static_cast<double>(static_cast<float>(params[i])) - after[i];
  return g;
}

train_run_result run_training(const train_config& cfg, train_mode mode, const dataset& data,
                              const std::string& checkpoint_dir, bool resume) {
  // Same epoch / resume / checkpoint protocol as trainer.cpp:704-758.
  namespace fs = std::filesystem;
  check_config(cfg, data);
  std::vector<stage_model> stages = partition_model(cfg.net, cfg.workers);
  load_network_params(stages, init_network_params(cfg.net, cfg.seed), 0);
  train_run_result result;
  result.first_epoch = 1;
  if (resume && !checkpoint_dir.empty()) {
    int newest = 0;
    for (int e = cfg.epochs; e >= 1 && newest == 0; --e)
      for (int s = 1; s <= cfg.workers; ++s)
        if (fs::exists(fs::path(checkpoint_dir) / checkpoint_filename(s, e))) {
          newest = e;
          break;
        }
    if (newest > 0) {
      for (int s = 1; s <= cfg.workers; ++s) {
        const fs::path path = fs::path(checkpoint_dir) / checkpoint_filename(s, newest);
        if (!fs::exists(path))
          throw integrity_error("resume refused: checkpoint for stage " + std::to_string(s) +
                                    " epoch " + std::to_string(newest) + " is missing",
                                s, newest);
        const restored_stage r = restore_stage(path.string(), s, newest);
        stages[s - 1].version_store.clear();
        stages[s - 1].version_store[0] = r.stage.current_params();
        stages[s - 1].current_version = 0;
      }
      result.first_epoch = newest + 1;
    }
  }
  for (int e = result.first_epoch; e <= cfg.epochs; ++e) {
    result.logs.push_back(train_epoch(stages, data, cfg, mode, e));
    if (!checkpoint_dir.empty()) {
      std::error_code ec;
      fs::create_directories(checkpoint_dir, ec);
      for (const stage_model& st : stages)
        checkpoint_stage(st, cfg.net.loss, e,
                         (fs::path(checkpoint_dir) / checkpoint_filename(st.stage_id, e)).string());
    }
  }
  result.final_checksum = params_digest(stages);
  return result;
}

}  // namespace pipesim
