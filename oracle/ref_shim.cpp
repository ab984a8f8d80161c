// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" shim over the UNMODIFIED reference library (pipesim, compiled
// from /root/reference/proj/src by oracle/Makefile into oracle/_ref/) so the
// Python tests, golden-fixture generators and bench.py's cpu_baseline leg can
// call the reference itself.  Only the reference's public API
// (proj/include/pipesim/*.hpp) is used.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <set>
#include <string>
#include <vector>

#include "pipesim/checkpoint.hpp"
#include "pipesim/errors.hpp"
#include "pipesim/export.hpp"
#include "pipesim/ledger.hpp"
#include "pipesim/metrics.hpp"
#include "pipesim/render.hpp"
#include "pipesim/schedule.hpp"
#include "pipesim/trainer.hpp"

using namespace pipesim;

namespace {
thread_local std::string g_err;

int fail() {
  try {
    throw;
  } catch (const domain_error& e) {
    g_err = std::string(e.field()) + "|" + e.what();
    return 1;
  } catch (const structural_error& e) {
    g_err = e.what();
    return 2;
  } catch (const insufficient_horizon_error& e) {
    g_err = e.what();
    return 3;
  } catch (const integrity_error& e) {
    g_err = e.what();
    return 4;
  } catch (const io_error& e) {
    g_err = e.what();
    return 5;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 9;
  }
}

sim_config mk(int w, int n, int m) {
  sim_config c;
  c.workers = w;
  c.micro_batches = n;
  c.mini_batches = m;
  return c;
}

schedule_grid build(int w, int n, int m, int mode) {
  const sim_config c = mk(w, n, m);
  return mode == 0 ? build_nf1b_schedule(c) : build_1f1b_schedule(c);
}

network_spec net_of(int n_layers, const int* widths, const int* acts, int loss) {
  network_spec s;
  s.widths.assign(widths, widths + n_layers + 1);
  for (int l = 0; l < n_layers; ++l)
    s.activations.push_back(static_cast<activation_kind>(acts[l]));
  s.loss = loss == 0 ? loss_kind::mse : loss_kind::softmax_cross_entropy;
  return s;
}

void put_str(const std::string& s, char* buf, int cap) {
  if (!buf || cap <= 0) return;
  size_t n = s.size() < static_cast<size_t>(cap - 1) ? s.size() : cap - 1;
  std::memcpy(buf, s.data(), n);
  buf[n] = 0;
}
}  // namespace

extern "C" {

int ref_last_error(char* buf, int cap) {
  put_str(g_err, buf, cap);
  return static_cast<int>(g_err.size());
}

// cells: [W][cap] of (kind, mini, micro)
int ref_schedule(int w, int n, int m, int mode, int* horizon, int* cells, int cap) {
  try {
    const schedule_grid g = build(w, n, m, mode);
    *horizon = g.horizon();
    if (!cells || cap < g.horizon()) return 7;
    for (int s = 1; s <= w; ++s)
      for (int t = 1; t <= g.horizon(); ++t) {
        const task& k = g.at(s, t);
        int* c = cells + 3 * (static_cast<size_t>(s - 1) * cap + (t - 1));
        c[0] = static_cast<int>(k.kind);
        c[1] = k.mini;
        c[2] = k.micro;
      }
    return 0;
  } catch (...) {
    return fail();
  }
}

// validate_schedule on an arbitrary (possibly hand-mutated) grid given as
// [W][H][3] cells; kinds[i] / '\n'-joined messages.
int ref_validate(int w, int n, int m, int mode, const int* cells, int h, int* n_viol,
                 int* kinds, int cap, char* msgs, int msg_cap) {
  try {
    const sim_config c = mk(w, n, m);
    schedule_grid g(c, mode == 0 ? schedule_mode::timeprest : schedule_mode::pipedream);
    for (int s = 1; s <= w; ++s)
      for (int t = 1; t <= h; ++t) {
        const int* x = cells + 3 * (static_cast<size_t>(s - 1) * h + (t - 1));
        g.put(s, t, task{static_cast<task_kind>(x[0]), x[1], x[2]});
      }
    const validation_report r = validate_schedule(g, c);
    *n_viol = static_cast<int>(r.violations.size());
    std::string text;
    for (size_t i = 0; i < r.violations.size(); ++i) {
      if (static_cast<int>(i) < cap) kinds[i] = static_cast<int>(r.violations[i].kind);
      text += r.violations[i].message + "\n";
    }
    put_str(text, msgs, msg_cap);
    return 0;
  } catch (...) {
    return fail();
  }
}

int ref_render_ascii(int w, int n, int m, int mode, char* buf, int cap) {
  try {
    put_str(render_ascii(build(w, n, m, mode)), buf, cap);
    return 0;
  } catch (...) {
    return fail();
  }
}

// schedule document JSON (export.cpp:78-139) of a (w, n, m, mode) config
int ref_schedule_document(int w, int n, int m, int mode, char* buf, int cap) {
  try {
    const sim_config c = mk(w, n, m);
    const schedule_grid g = build(w, n, m, mode);
    put_str(schedule_document_json(g, assign_versions(g, c)), buf, cap);
    return 0;
  } catch (...) {
    return fail();
  }
}

// commits [M*W][4], pins [M*units][4], cons [M*W][4], us [M], fcs [M+1]
int ref_ledger(int w, int n, int m, int mode, int* commits, int* pins, int* cons,
               int* us, int* fcs) {
  try {
    const schedule_grid g = build(w, n, m, mode);
    const version_ledger L = assign_versions(g, mk(w, n, m));
    for (size_t i = 0; i < L.commits.size(); ++i) {
      const auto& c = L.commits[i];
      int* o = commits + 4 * i;
      o[0] = c.version; o[1] = c.mini; o[2] = c.stage; o[3] = c.slot;
    }
    for (size_t i = 0; i < L.pins.size(); ++i) {
      const auto& p = L.pins[i];
      int* o = pins + 4 * i;
      o[0] = p.mini; o[1] = p.micro; o[2] = p.slot; o[3] = p.version;
    }
    for (size_t i = 0; i < L.consumptions.size(); ++i) {
      const auto& c = L.consumptions[i];
      int* o = cons + 4 * i;
      o[0] = c.mini; o[1] = c.stage; o[2] = c.slot; o[3] = c.version;
    }
    for (size_t i = 0; i < L.update_source.size(); ++i) us[i] = L.update_source[i];
    for (size_t i = 0; i < L.full_commit_slot.size(); ++i) fcs[i] = L.full_commit_slot[i];
    return 0;
  } catch (...) {
    return fail();
  }
}

// intervals [W][M+1][3], peak [W]
int ref_retention(int w, int n, int m, int mode, int* intervals, int* peak) {
  try {
    const schedule_grid g = build(w, n, m, mode);
    const retention_timeline T = build_retention_timeline(assign_versions(g, mk(w, n, m)), g);
    for (int s = 0; s < w; ++s) {
      peak[s] = T.peak_concurrent[s];
      for (int v = 0; v <= m; ++v) {
        int* o = intervals + 3 * (static_cast<size_t>(s) * (m + 1) + v);
        o[0] = T.per_stage[s][v].version;
        o[1] = T.per_stage[s][v].retained_from_slot;
        o[2] = T.per_stage[s][v].freed_at_slot;
      }
    }
    return 0;
  } catch (...) {
    return fail();
  }
}

int ref_measure_v(int w, int n, int m, int mode, int strict, int* v) {
  try {
    *v = measure_version_difference(assign_versions(build(w, n, m, mode), mk(w, n, m)),
                                    strict != 0);
    return 0;
  } catch (...) {
    return fail();
  }
}

int ref_closed_form_v(int w, int n, int* v) {
  try {
    *v = closed_form_v(w, n);
    return 0;
  } catch (...) {
    return fail();
  }
}

int ref_init_params(int n_layers, const int* widths, const int* acts, int loss,
                    uint64_t seed, double* out) {
  try {
    const auto p = init_network_params(net_of(n_layers, widths, acts, loss), seed);
    std::memcpy(out, p.data(), p.size() * sizeof(double));
    return 0;
  } catch (...) {
    return fail();
  }
}

int ref_partition(int n_layers, const int* widths, const int* acts, int loss, int w,
                  int* first_layer, int* n_stage_layers) {
  try {
    const auto st = partition_model(net_of(n_layers, widths, acts, loss), w);
    for (size_t s = 0; s < st.size(); ++s) {
      first_layer[s] = st[s].first_layer;
      n_stage_layers[s] = static_cast<int>(st[s].layers.size());
    }
    return 0;
  } catch (...) {
    return fail();
  }
}

int ref_synthetic(int samples, uint64_t seed, double* x, double* y) {
  try {
    const dataset d = make_synthetic_task(samples, seed);
    std::memcpy(x, d.x.data.data(), d.x.data.size() * sizeof(double));
    std::memcpy(y, d.y.data.data(), d.y.data.size() * sizeof(double));
    return 0;
  } catch (...) {
    return fail();
  }
}

// Runs `epochs` epochs of train_epoch from `params_in` (flat) on the given
// data.  Outputs: params_out (flat, current versions), loss/consumed per
// mini per epoch, pinned [epochs][M][units], log text of all epochs,
// held (optional): [horizon][W][M+1] 0/1 version-store membership after each
// slot of the LAST epoch (slot_observer), seconds: wall time of train_epoch.
int ref_train(int n_layers, const int* widths, const int* acts, int loss, int w,
              int n, int b, int m, double lr, uint64_t seed, int mode, int epochs,
              const double* x, const double* y, const double* params_in,
              double* params_out, double* losses, int* pinned, int* consumed,
              char* log_text, int log_cap, int* held, int held_cap_slots,
              double* seconds) {
  try {
    train_config cfg;
    cfg.net = net_of(n_layers, widths, acts, loss);
    cfg.workers = w;
    cfg.micro_batches = n;
    cfg.mini_batch_size = b;
    cfg.mini_batches = m;
    cfg.learning_rate = lr;
    cfg.seed = seed;
    dataset data;
    data.x = matrix(m * b, widths[0]);
    data.y = matrix(m * b, widths[n_layers]);
    std::memcpy(data.x.data.data(), x, data.x.data.size() * sizeof(double));
    std::memcpy(data.y.data.data(), y, data.y.data.size() * sizeof(double));
    std::vector<stage_model> stages = partition_model(cfg.net, w);
    const int total = cfg.net.param_count();
    load_network_params(stages, std::vector<double>(params_in, params_in + total), 0);
    const train_mode tm = mode == 0   ? train_mode::timeprest
                          : mode == 1 ? train_mode::pipedream
                                      : train_mode::sequential;
    std::string text;
    double secs = 0.0;
    for (int e = 1; e <= epochs; ++e) {
      slot_observer obs;
      if (held && e == epochs)
        obs = [&](int slot, const std::vector<stage_model>& st) {
          if (slot > held_cap_slots) return;
          for (const auto& s : st)
            for (const auto& kv : s.version_store)
              if (kv.first >= 0 && kv.first <= m)
                held[(static_cast<size_t>(slot - 1) * w + (s.stage_id - 1)) * (m + 1) +
                     kv.first] = 1;
        };
      const auto t0 = std::chrono::steady_clock::now();
      const epoch_log log = train_epoch(stages, data, cfg, tm, e, obs);
      secs += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      text += log.to_text();
      const int units = mode == 0 ? n : 1;
      for (int k = 0; k < m; ++k) {
        losses[(e - 1) * m + k] = log.minis[k].loss;
        consumed[(e - 1) * m + k] = log.minis[k].consumed;
        for (int j = 0; j < units && j < static_cast<int>(log.minis[k].pinned.size()); ++j)
          pinned[((e - 1) * m + k) * units + j] = log.minis[k].pinned[j];
      }
    }
    const auto flat = gather_network_params(stages);
    std::memcpy(params_out, flat.data(), flat.size() * sizeof(double));
    put_str(text, log_text, log_cap);
    if (seconds) *seconds = secs;
    return 0;
  } catch (...) {
    return fail();
  }
}

int ref_network_loss(int n_layers, const int* widths, const int* acts, int loss,
                     const double* params, int rows, const double* x, const double* y,
                     double* out) {
  try {
    const network_spec net = net_of(n_layers, widths, acts, loss);
    dataset d;
    d.x = matrix(rows, widths[0]);
    d.y = matrix(rows, widths[n_layers]);
    std::memcpy(d.x.data.data(), x, d.x.data.size() * sizeof(double));
    std::memcpy(d.y.data.data(), y, d.y.data.size() * sizeof(double));
    *out = network_loss(net, std::vector<double>(params, params + net.param_count()), d);
    return 0;
  } catch (...) {
    return fail();
  }
}

int ref_network_gradient(int n_layers, const int* widths, const int* acts, int loss,
                         const double* params, int rows, const double* x,
                         const double* y, double* out) {
  try {
    const network_spec net = net_of(n_layers, widths, acts, loss);
    dataset d;
    d.x = matrix(rows, widths[0]);
    d.y = matrix(rows, widths[n_layers]);
    std::memcpy(d.x.data.data(), x, d.x.data.size() * sizeof(double));
    std::memcpy(d.y.data.data(), y, d.y.data.size() * sizeof(double));
    const auto g =
        network_gradient(net, std::vector<double>(params, params + net.param_count()), d);
    std::memcpy(out, g.data(), g.size() * sizeof(double));
    return 0;
  } catch (...) {
    return fail();
  }
}

// checkpoint_stage of the reference (checkpoint.cpp:39-67) for one stage
// given as (stage_id, first_layer, layers as in/out/act triples, version,
// params); used to byte-compare checkpoint files and cross-restore them.
int ref_checkpoint_stage(int stage_id, int first_layer, int n_layers, const int* layers,
                         int version, const double* params, int n, int loss, int epoch,
                         const char* path) {
  try {
    stage_model st;
    st.stage_id = stage_id;
    st.first_layer = first_layer;
    for (int i = 0; i < n_layers; ++i) {
      layer_spec l;
      l.in = layers[3 * i];
      l.out = layers[3 * i + 1];
      l.act = static_cast<activation_kind>(layers[3 * i + 2]);
      st.layers.push_back(l);
    }
    st.version_store[version] = std::vector<double>(params, params + n);
    st.current_version = version;
    checkpoint_stage(st, loss == 0 ? loss_kind::mse : loss_kind::softmax_cross_entropy, epoch,
                     path);
    return 0;
  } catch (...) {
    return fail();
  }
}

// restore_stage of the reference; writes the current params (n = count).
int ref_restore_stage(const char* path, int expected_stage, int expected_epoch, double* params,
                      int cap, int* n, int* version, int* epoch) {
  try {
    const restored_stage r = restore_stage(path, expected_stage, expected_epoch);
    const auto& p = r.stage.current_params();
    if (static_cast<int>(p.size()) > cap) return 9;
    std::memcpy(params, p.data(), p.size() * sizeof(double));
    *n = static_cast<int>(p.size());
    *version = r.stage.current_version;
    *epoch = r.epoch;
    return 0;
  } catch (...) {
    return fail();
  }
}

// Seconds the reference's params_digest (trainer.cpp:599-607) takes over the
// given values (one stage holding them): the per-mini-batch fixed cost of
// replay_grid, reported beside the reference arm's throughput.
int ref_digest_seconds(const double* values, int64_t n, double* seconds, char* out17) {
  try {
    std::vector<stage_model> st(1);
    st[0].stage_id = 1;
    st[0].version_store[0] = std::vector<double>(values, values + n);
    const auto t0 = std::chrono::steady_clock::now();
    const std::string d = params_digest(st);
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    put_str(d, out17, 17);
    return 0;
  } catch (...) {
    return fail();
  }
}

}  // extern "C"
