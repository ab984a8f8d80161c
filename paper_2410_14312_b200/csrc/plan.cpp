// Plan layer: nF1B / 1F1B slot schedules, structural validation, the weight
// version ledger, retention timelines and staleness — host C++.
//
// Semantics follow the reference exactly (bit-exact traces are a parity
// requirement): proj/src/schedule.cpp:95-346 and proj/src/ledger.cpp:24-293.
// The data structures differ: the grid is a flat slot-major array, the
// generator keeps reservations in per-stage slot vectors, and the ledger
// derives every slot lookup from one O(W*H) index instead of repeated grid
// scans.
#include <algorithm>
#include <deque>
#include <string>
#include <utility>
#include <vector>

#include "pipesim_core.hpp"

namespace pipesim {

// ----------------------------------------------------------------- config
void validate(const sim_config& c) {
  auto bad = [](const char* field, const std::string& msg) {
    throw domain_error(field, msg);
  };
  if (c.workers < 2)
    bad("workers", "workers: W must satisfy W >= 2 (got " +
                       std::to_string(c.workers) + ")");
  if (c.micro_batches < 2)
    bad("micro_batches", "micro_batches: N must satisfy N >= 2 (got " +
                             std::to_string(c.micro_batches) + ")");
  if (c.mini_batches < 1)
    bad("mini_batches", "mini_batches: M must satisfy M >= 1 (got " +
                            std::to_string(c.mini_batches) + ")");
  if (c.backward_cost_factor < 1.0)
    bad("backward_cost_factor", "backward_cost_factor must be >= 1");
  if (c.samples_per_mini_batch < 1)
    bad("samples_per_mini_batch", "samples_per_mini_batch must be >= 1");
}

const char* to_string(schedule_mode mode) {
  return mode == schedule_mode::pipedream ? "pipedream" : "timeprest";
}

// ----------------------------------------------------------------- grid
namespace {
const task kIdleTask{};

std::string label_of(const task& t) {
  if (t.is_backward()) return "B" + std::to_string(t.mini);
  std::string s = std::to_string(t.mini);
  if (t.micro > 0) s.push_back(static_cast<char>('A' + (t.micro - 1) % 26));
  return s;
}
}  // namespace

const task& schedule_grid::at(int worker, int slot) const {
  const int w = workers();
  if (worker < 1 || worker > w || slot < 1 || slot > horizon_) return kIdleTask;
  return cells_[static_cast<size_t>(slot - 1) * w + (worker - 1)];
}

void schedule_grid::put(int worker, int slot, task t) {
  const int w = workers();
  if (slot > horizon_) {
    cells_.resize(static_cast<size_t>(slot) * w);
    horizon_ = slot;
  }
  cells_[static_cast<size_t>(slot - 1) * w + (worker - 1)] = t;
}

void schedule_grid::clear(int worker, int slot) {
  if (worker < 1 || worker > workers() || slot < 1 || slot > horizon_) return;
  cells_[static_cast<size_t>(slot - 1) * workers() + (worker - 1)] = kIdleTask;
}

int schedule_grid::forward_slot(int mini, int micro, int stage) const {
  for (int t = 1; t <= horizon_; ++t) {
    const task& c = at(stage, t);
    if (c.is_forward() && c.mini == mini && c.micro == micro) return t;
  }
  return 0;
}

int schedule_grid::backward_slot(int mini, int stage) const {
  for (int t = 1; t <= horizon_; ++t) {
    const task& c = at(stage, t);
    if (c.is_backward() && c.mini == mini) return t;
  }
  return 0;
}

bool operator==(const schedule_grid& a, const schedule_grid& b) {
  if (a.workers() != b.workers() || a.horizon() != b.horizon()) return false;
  for (int t = 1; t <= a.horizon(); ++t)
    for (int w = 1; w <= a.workers(); ++w)
      if (!(a.at(w, t) == b.at(w, t))) return false;
  return true;
}

// ----------------------------------------------------------------- generator
namespace {

// Slot-stepping generator shared by both disciplines.  Units are micro-batches
// (nF1B) or whole mini-batches (1F1B, micro id 0).  Backward chains are
// reserved in full when released, which is how they win contended slots.
struct slot_stepper {
  struct unit {
    int mini, micro;
  };
  struct waiting {
    unit u;
    int left_at;  // slot in which u finished on the previous stage
  };

  const sim_config cfg;
  const int units;
  const int cap;  // admission cap on concurrently started minis (0 = none)
  schedule_grid grid;

  std::vector<unit> inject;  // stage-1 injection order (strict FIFO)
  size_t next_inject = 0;
  std::vector<std::deque<waiting>> fifo;       // per stage
  std::vector<std::vector<int>> reserved;      // [stage][slot] -> mini (0 none)
  std::vector<int> exited;                     // per mini: units past stage W
  int started = 0, finished = 0;

  slot_stepper(const sim_config& c, schedule_mode mode, int units_per_mini,
               int admission_cap)
      : cfg(c), units(units_per_mini), cap(admission_cap), grid(c, mode),
        fifo(c.workers + 1), reserved(c.workers + 1),
        exited(c.mini_batches + 1, 0) {
    const bool micro_ids = mode == schedule_mode::timeprest;
    inject.reserve(static_cast<size_t>(c.mini_batches) * units);
    for (int k = 1; k <= c.mini_batches; ++k)
      for (int j = 1; j <= units; ++j) inject.push_back({k, micro_ids ? j : 0});
  }

  int reservation(int s, int t) const {
    const auto& row = reserved[s];
    return t < static_cast<int>(row.size()) ? row[t] : 0;
  }
  void reserve(int s, int t, int mini) {
    auto& row = reserved[s];
    if (static_cast<int>(row.size()) <= t) row.resize(t + 1, 0);
    row[t] = mini;
  }

  bool admissible() const {
    if (cap <= 0) return true;
    if (inject[next_inject].micro > 1) return true;  // continues a started mini
    return started - finished < cap;
  }

  void place_forward(int s, int t, unit u) {
    grid.put(s, t, task{task_kind::forward_micro, u.mini, u.micro});
    if (s == 1 && u.micro <= 1) ++started;
    const int W = cfg.workers;
    if (s < W) {
      fifo[s + 1].push_back({u, t});
    } else if (++exited[u.mini] == units) {
      // Average-loss barrier passed: backward occupies W..1 at t+1..t+W.
      for (int d = 0; d < W; ++d) reserve(W - d, t + 1 + d, u.mini);
    }
  }

  schedule_grid run() {
    const int W = cfg.workers;
    long todo = static_cast<long>(cfg.mini_batches) * W * (units + 1);
    for (int t = 1; todo > 0; ++t) {
      for (int s = 1; s <= W; ++s) {
        if (const int k = reservation(s, t)) {
          grid.put(s, t, task{task_kind::backward_mini, k, 0});
          if (s == 1) ++finished;
          --todo;
          continue;
        }
        if (s == 1) {
          if (next_inject < inject.size() && admissible()) {
            place_forward(1, t, inject[next_inject++]);
            --todo;
          }
          continue;
        }
        auto& q = fifo[s];
        if (!q.empty() && q.front().left_at < t) {
          const unit u = q.front().u;
          q.pop_front();
          place_forward(s, t, u);
          --todo;
        }
      }
    }
    return grid;
  }
};

}  // namespace

schedule_grid build_nf1b_schedule(const sim_config& cfg) {
  validate(cfg);
  return slot_stepper(cfg, schedule_mode::timeprest, cfg.micro_batches, 0).run();
}

schedule_grid build_1f1b_schedule(const sim_config& cfg) {
  validate(cfg);
  return slot_stepper(cfg, schedule_mode::pipedream, 1, cfg.workers).run();
}

// ----------------------------------------------------------------- validator
namespace {

void forward_chain_check(const schedule_grid& g, int mini, int micro,
                         validation_report& rep) {
  const int W = g.workers();
  const task want{task_kind::forward_micro, mini, micro};
  std::vector<int> at_stage(W + 1, 0);
  for (int s = 1; s <= W; ++s) {
    int hits = 0;
    for (int t = 1; t <= g.horizon(); ++t)
      if (g.at(s, t) == want) {
        at_stage[s] = t;
        ++hits;
      }
    if (hits != 1) {
      rep.violations.push_back(
          {violation_kind::completeness,
           "completeness violation: forward " + label_of(want) + " appears " +
               std::to_string(hits) + " times on stage " + std::to_string(s)});
      return;
    }
  }
  for (int s = 1; s < W; ++s) {
    const int from = at_stage[s], to = at_stage[s + 1];
    if (to <= from) {
      rep.violations.push_back(
          {violation_kind::task_invariant,
           "task invariant violation: forward " + label_of(want) +
               " does not advance from stage " + std::to_string(s)});
      return;
    }
    for (int u = from + 1; u < to; ++u)
      if (g.at(s + 1, u).is_idle()) {
        rep.violations.push_back(
            {violation_kind::stage_continuity,
             "stage-continuity violation: forward " + label_of(want) +
                 " idles before stage " + std::to_string(s + 1) + " at slot " +
                 std::to_string(u) + " (stage " + std::to_string(s) + " slot " +
                 std::to_string(from) + ", stage " + std::to_string(s + 1) +
                 " slot " + std::to_string(to) + ")"});
        return;
      }
  }
}

void backward_chain_check(const schedule_grid& g, int mini, int exit_slot,
                          validation_report& rep) {
  const int W = g.workers();
  const task want{task_kind::backward_mini, mini, 0};
  std::vector<int> at_stage(W + 1, 0);
  for (int s = 1; s <= W; ++s) {
    int hits = 0;
    for (int t = 1; t <= g.horizon(); ++t)
      if (g.at(s, t) == want) {
        at_stage[s] = t;
        ++hits;
      }
    if (hits != 1) {
      rep.violations.push_back(
          {violation_kind::completeness,
           "completeness violation: backward B" + std::to_string(mini) +
               " appears " + std::to_string(hits) + " times on stage " +
               std::to_string(s)});
      return;
    }
  }
  for (int s = W; s > 1; --s)
    if (at_stage[s - 1] != at_stage[s] + 1) {
      rep.violations.push_back(
          {violation_kind::task_invariant,
           "task invariant violation: backward B" + std::to_string(mini) +
               " is not contiguous between stages " + std::to_string(s) +
               " and " + std::to_string(s - 1)});
      return;
    }
  if (exit_slot > 0 && at_stage[W] != exit_slot + 1)
    rep.violations.push_back(
        {violation_kind::backward_priority,
         "backward-priority violation: B" + std::to_string(mini) +
             " starts at slot " + std::to_string(at_stage[W]) +
             " but was ready at slot " + std::to_string(exit_slot + 1)});
}

}  // namespace

validation_report validate_schedule(const schedule_grid& g, const sim_config& cfg) {
  validation_report rep;
  const int W = cfg.workers;
  const bool nf1b = g.mode() == schedule_mode::timeprest;
  const int units = nf1b ? cfg.micro_batches : 1;
  auto micro_id = [&](int j) { return nf1b ? j : 0; };

  for (int k = 1; k <= cfg.mini_batches; ++k)
    for (int j = 1; j <= units; ++j) forward_chain_check(g, k, micro_id(j), rep);

  for (int k = 1; k <= cfg.mini_batches; ++k) {
    int last_exit = 0;
    bool complete = true;
    for (int j = 1; j <= units; ++j) {
      const int t = g.forward_slot(k, micro_id(j), W);
      complete = complete && t != 0;
      last_exit = std::max(last_exit, t);
    }
    backward_chain_check(g, k, complete ? last_exit : 0, rep);
  }

  for (int k = 1; k <= cfg.mini_batches; ++k) {
    int last_exit = 0;
    for (int j = 1; j <= units; ++j)
      last_exit = std::max(last_exit, g.forward_slot(k, micro_id(j), W));
    for (int s = W; s >= 1; --s) {
      const int b = g.backward_slot(k, s);
      if (b == 0) continue;
      int ready;
      if (s == W)
        ready = last_exit > 0 ? last_exit + 1 : b;
      else
        ready = g.backward_slot(k, s + 1) + 1;
      for (int u = ready; u < b; ++u)
        if (g.at(s, u).is_forward())
          rep.violations.push_back(
              {violation_kind::backward_priority,
               "backward-priority violation: stage " + std::to_string(s) +
                   " ran forward " + label_of(g.at(s, u)) + " at slot " +
                   std::to_string(u) + " while B" + std::to_string(k) +
                   " was ready"});
    }
  }
  return rep;
}

// ----------------------------------------------------------------- ledger
namespace {

void require_pair(int workers, int micro_batches) {
  if (workers < 2) throw domain_error("workers", "workers: W must satisfy W >= 2");
  if (micro_batches < 2)
    throw domain_error("micro_batches", "micro_batches: N must satisfy N >= 2");
}

// One pass over the grid: first forward slot per (mini, micro, stage) and
// first backward slot per (mini, stage).
struct slot_index {
  int W, M, U;  // U = micro ids 0..N
  std::vector<int> fwd, bwd;
  slot_index(const schedule_grid& g, int micro_max)
      : W(g.workers()), M(g.config().mini_batches), U(micro_max + 1),
        fwd(static_cast<size_t>(M + 1) * U * (W + 1), 0),
        bwd(static_cast<size_t>(M + 1) * (W + 1), 0) {
    for (int t = 1; t <= g.horizon(); ++t)
      for (int s = 1; s <= W; ++s) {
        const task& c = g.at(s, t);
        if (c.mini < 1 || c.mini > M) continue;
        if (c.is_forward() && c.micro >= 0 && c.micro < U) {
          int& f = fwd[(static_cast<size_t>(c.mini) * U + c.micro) * (W + 1) + s];
          if (f == 0) f = t;
        } else if (c.is_backward()) {
          int& b = bwd[static_cast<size_t>(c.mini) * (W + 1) + s];
          if (b == 0) b = t;
        }
      }
  }
  int f(int mini, int micro, int s) const {
    return fwd[(static_cast<size_t>(mini) * U + micro) * (W + 1) + s];
  }
  int b(int mini, int s) const { return bwd[static_cast<size_t>(mini) * (W + 1) + s]; }
};

// Newest version v >= 1 whose stage-1 commit slot is strictly before `slot`.
int newest_full_commit_before(const std::vector<int>& full_commit, int slot) {
  int v = 0;
  for (int k = 1; k < static_cast<int>(full_commit.size()); ++k)
    if (full_commit[k] < slot) v = k;
  return v;
}

}  // namespace

int version_ledger::pinned_version(int mini, int micro) const {
  for (const pin_record& p : pins)
    if (p.mini == mini && p.micro == micro) return p.version;
  throw structural_error("no pin recorded for mini " + std::to_string(mini) +
                         " micro " + std::to_string(micro));
}

version_ledger assign_versions(const schedule_grid& g, const sim_config& cfg) {
  validate(cfg);
  if (g.workers() != cfg.workers || g.config().mini_batches != cfg.mini_batches)
    throw structural_error("grid does not match config");
  {
    const validation_report rep = validate_schedule(g, cfg);
    if (!rep.valid())
      throw structural_error("invalid grid: " + rep.violations.front().message);
  }
  const int W = cfg.workers, M = cfg.mini_batches;
  const bool nf1b = g.mode() == schedule_mode::timeprest;
  const int units = nf1b ? cfg.micro_batches : 1;
  const slot_index idx(g, nf1b ? cfg.micro_batches : 0);

  version_ledger L;
  L.cfg = cfg;
  L.mode = g.mode();
  L.full_commit_slot.assign(M + 1, 0);
  L.update_source.assign(M, 0);

  for (int k = 1; k <= M; ++k) {
    for (int s = W; s >= 1; --s) L.commits.push_back({k, k, s, idx.b(k, s)});
    L.full_commit_slot[k] = idx.b(k, 1);
  }
  std::stable_sort(L.commits.begin(), L.commits.end(),
                   [](const commit_event& x, const commit_event& y) {
                     return x.slot < y.slot;
                   });

  for (int k = 1; k <= M; ++k)
    for (int j = 1; j <= units; ++j) {
      const int micro = nf1b ? j : 0;
      const int inj = idx.f(k, micro, 1);
      L.pins.push_back(
          {k, micro, inj, newest_full_commit_before(L.full_commit_slot, inj)});
    }

  for (int k = 1; k <= M; ++k) {
    if (nf1b) {
      L.update_source[k - 1] =
          newest_full_commit_before(L.full_commit_slot, idx.b(k, W));
      for (int s = W; s >= 1; --s) {
        const int arrival = idx.b(k, s);
        int used = 0;
        for (int v = 1; v < k; ++v)
          if (idx.b(v, s) < arrival) used = v;
        L.consumptions.push_back({k, s, arrival, used});
      }
    } else {
      const int stashed = L.pinned_version(k, 0);
      L.update_source[k - 1] = stashed;
      for (int s = W; s >= 1; --s)
        L.consumptions.push_back({k, s, idx.b(k, s), stashed});
    }
  }
  return L;
}

int measure_version_difference(const version_ledger& L, bool strict) {
  const int M = L.cfg.mini_batches;
  const int floor_m = 2 * (L.cfg.workers + L.cfg.micro_batches);
  if (strict && M < floor_m)
    throw insufficient_horizon_error(
        "M = " + std::to_string(M) + " is below the steady-state horizon " +
        std::to_string(floor_m) + " = 2(W+N)");
  if (M < 2) throw insufficient_horizon_error("at least two mini-batches required");
  int v = 0;
  for (int k = M / 2 + 1; k <= M; ++k) {
    const int gap = k - L.update_source[k - 1];
    if (v == 0) v = gap;
    if (gap != v)
      throw insufficient_horizon_error(
          "version-difference not steady: gap " + std::to_string(gap) +
          " at mini-batch " + std::to_string(k) + " vs " + std::to_string(v));
  }
  return v;
}

int closed_form_v(int workers, int micro_batches) {
  require_pair(workers, micro_batches);
  return (workers + micro_batches - 2) / micro_batches;
}

int forward_span(int workers, int micro_batches, int mini_ordinal) {
  require_pair(workers, micro_batches);
  if (mini_ordinal < 1)
    throw domain_error("mini_ordinal", "mini-batch ordinal must be >= 1");
  return workers + micro_batches - 2 + mini_ordinal;
}

int backward_span(int workers) {
  if (workers < 2) throw domain_error("workers", "workers: W must satisfy W >= 2");
  return workers;
}

bool overlap_condition(int workers, int micro_batches) {
  require_pair(workers, micro_batches);
  return workers > micro_batches + 1;
}

sequence_decomposition decompose_sequences(const version_ledger& L,
                                           int mini_batches) {
  const int M = mini_batches;
  if (M > L.cfg.mini_batches)
    throw structural_error("ledger covers fewer mini-batches than requested");
  // next_of[i]: the mini-batch whose backward consumed version i (0: none).
  std::vector<int> next_of(M + 1, 0);
  for (int k = 1; k <= M; ++k) {
    const int src = L.update_source[k - 1];
    if (src == 0) continue;
    if (src <= M && next_of[src] != 0)
      throw structural_error("version " + std::to_string(src) +
                             " consumed by two backwards");
    if (src <= M) next_of[src] = k;
  }
  sequence_decomposition out;
  std::vector<char> used(M + 1, 0);
  auto walk = [&](int head, bool stop_on_used) {
    std::vector<int> chain;
    for (int cur = head; cur != 0 && cur <= M; cur = next_of[cur]) {
      if (stop_on_used && used[cur]) break;
      chain.push_back(cur);
      used[cur] = 1;
    }
    out.sequences.push_back(std::move(chain));
  };
  for (int k = 1; k <= M; ++k)
    if (!used[k] && L.update_source[k - 1] == 0) walk(k, false);
  for (int k = 1; k <= M; ++k)
    if (!used[k]) walk(k, true);
  std::sort(out.sequences.begin(), out.sequences.end(),
            [](const std::vector<int>& a, const std::vector<int>& b) {
              return a.front() < b.front();
            });
  out.version_difference_measured = measure_version_difference(L, false);
  return out;
}

int retention_timeline::retained_count(int stage, int slot) const {
  int n = 0;
  for (const retention_interval& iv : per_stage[stage - 1])
    n += (iv.retained_from_slot <= slot && slot < iv.freed_at_slot) ? 1 : 0;
  return n;
}

retention_timeline build_retention_timeline(const version_ledger& L,
                                            const schedule_grid& g) {
  if (g.mode() != L.mode || g.config().mini_batches != L.cfg.mini_batches)
    throw structural_error("ledger does not match grid");
  const int W = L.cfg.workers, M = L.cfg.mini_batches;
  const bool nf1b = L.mode == schedule_mode::timeprest;
  const slot_index idx(g, nf1b ? L.cfg.micro_batches : 0);

  retention_timeline T;
  T.horizon = g.horizon();
  T.per_stage.assign(W, {});
  T.peak_concurrent.assign(W, 0);

  std::vector<std::vector<std::pair<int, int>>> riders(M + 1);  // by version
  for (const pin_record& p : L.pins)
    if (p.version >= 0 && p.version <= M) riders[p.version].push_back({p.mini, p.micro});

  for (int s = 1; s <= W; ++s) {
    auto commit_at = [&](int v) { return v == 0 ? 0 : idx.b(v, s); };
    auto& ivs = T.per_stage[s - 1];
    for (int v = 0; v <= M; ++v) {
      int last = v < M ? commit_at(v + 1) : g.horizon();
      for (const auto& [mini, micro] : riders[v]) {
        last = std::max(last, idx.f(mini, micro, s));
        if (!nf1b) last = std::max(last, idx.b(mini, s));
      }
      ivs.push_back({v, commit_at(v), last + 1});
    }
    // Peak live count: sweep over the interval endpoints.
    int peak = 0;
    for (int t = 1; t <= g.horizon(); ++t) peak = std::max(peak, T.retained_count(s, t));
    T.peak_concurrent[s - 1] = peak;
  }
  return T;
}

bool staleness_report_t::all_zero() const {
  for (const staleness_entry& e : entries)
    if (e.staleness != 0) return false;
  return true;
}

int staleness_report_t::steady_state_staleness(int first_steady_mini) const {
  int worst = 0;
  for (const staleness_entry& e : entries)
    if (e.mini >= first_steady_mini) worst = std::max(worst, e.staleness);
  return worst;
}

staleness_report_t staleness_report(const version_ledger& L) {
  const int W = L.cfg.workers, M = L.cfg.mini_batches;
  // commit slot per (version, stage); 0 = no commit recorded.
  std::vector<int> at(static_cast<size_t>(M + 1) * (W + 1), 0);
  std::vector<char> has(at.size(), 0);
  for (const commit_event& c : L.commits)
    if (c.version >= 0 && c.version <= M && c.stage >= 1 && c.stage <= W) {
      at[static_cast<size_t>(c.version) * (W + 1) + c.stage] = c.slot;
      has[static_cast<size_t>(c.version) * (W + 1) + c.stage] = 1;
    }
  staleness_report_t r;
  for (const consume_record& use : L.consumptions) {
    int newest = 0;
    for (int v = 1; v <= M; ++v) {
      const size_t i = static_cast<size_t>(v) * (W + 1) + use.stage;
      if (use.stage >= 1 && use.stage <= W && has[i] && at[i] < use.slot) newest = v;
    }
    r.entries.push_back({use.mini, use.stage, newest - use.version});
  }
  return r;
}

}  // namespace pipesim
