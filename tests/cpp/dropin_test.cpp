// Drop-in check: code written against the reference's C++ API
// (#include "pipesim/trainer.hpp" ...) compiled and linked against the B200
// build.  Mirrors proj/tests/test_trainer.cpp cases that exercise the step.
// Exit code 0 = all checks passed.  Needs a GPU for the train_epoch checks;
// `--plan-only` runs the host plan-layer checks (CPU).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <set>
#include <string>
#include <vector>

#include "pipesim/checkpoint.hpp"
#include "pipesim/ledger.hpp"
#include "pipesim/schedule.hpp"
#include "pipesim/trainer.hpp"

using namespace pipesim;

static int failures = 0;
#define CHECK(c)                                                    \
  do {                                                              \
    if (!(c)) {                                                     \
      std::fprintf(stderr, "CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #c); \
      ++failures;                                                   \
    }                                                               \
  } while (0)

static network_spec demo_net() {
  network_spec net;
  net.widths = {2, 8, 2};
  net.activations = {activation_kind::tanh, activation_kind::linear};
  net.loss = loss_kind::softmax_cross_entropy;
  return net;
}

static void plan_checks() {
  sim_config c;
  c.workers = 4;
  c.micro_batches = 2;
  c.mini_batches = 7;
  const schedule_grid g = build_nf1b_schedule(c);
  CHECK(validate_schedule(g, c).valid());
  const version_ledger L = assign_versions(g, c);
  CHECK(L.update_source.size() == 7);
  CHECK(L.update_source[2] == 1);
  CHECK(closed_form_v(8, 2) == 4);
  sim_config s = c;
  s.mini_batches = 20;
  s.workers = 8;
  CHECK(measure_version_difference(assign_versions(build_nf1b_schedule(s), s)) == 3);
  bool threw = false;
  try {
    sim_config bad = c;
    bad.micro_batches = 1;
    build_nf1b_schedule(bad);
  } catch (const domain_error& e) {
    threw = std::string(e.field()) == "micro_batches";
  }
  CHECK(threw);
}

static void train_checks() {
  train_config cfg;
  cfg.net.widths = {2, 6, 6, 6, 2};
  cfg.net.activations = {activation_kind::tanh, activation_kind::tanh, activation_kind::tanh,
                         activation_kind::linear};
  cfg.net.loss = loss_kind::softmax_cross_entropy;
  cfg.workers = 4;
  cfg.micro_batches = 2;
  cfg.mini_batch_size = 4;
  cfg.mini_batches = 7;
  cfg.learning_rate = 0.05;
  cfg.seed = 2;
  dataset data = make_synthetic_task(28, 2);
  std::vector<stage_model> stages = partition_model(cfg.net, cfg.workers);
  load_network_params(stages, init_network_params(cfg.net, cfg.seed), 0);
  epoch_log log = train_epoch(stages, data, cfg, train_mode::timeprest, 1);
  CHECK(log.minis.size() == 7);
  CHECK(log.minis[2].consumed == 1);
  CHECK(log.minis[4].consumed == 3);
  for (const auto& m : log.minis) CHECK(std::isfinite(m.loss));
  CHECK(log.final_checksum == log.minis.back().checksum);
  std::printf("%s", log.to_text().c_str());

  // observer sees exactly the retention timeline (test_trainer.cpp:387-433)
  sim_config sc;
  sc.workers = 4;
  sc.micro_batches = 2;
  sc.mini_batches = 7;
  const schedule_grid g = build_nf1b_schedule(sc);
  const retention_timeline T = build_retention_timeline(assign_versions(g, sc), g);
  int observed = 0;
  train_epoch(stages, data, cfg, train_mode::timeprest, 2,
              [&](int slot, const std::vector<stage_model>& st) {
                ++observed;
                for (const auto& s : st) {
                  std::set<int> live, held;
                  for (const auto& iv : T.per_stage[s.stage_id - 1])
                    if (iv.retained_from_slot <= slot && slot < iv.freed_at_slot) live.insert(iv.version);
                  for (const auto& kv : s.version_store) held.insert(kv.first);
                  CHECK(live == held);
                }
              });
  CHECK(observed == g.horizon());

  // zero learning rate keeps the (fp32-rounded) weights (test_trainer.cpp:261-279)
  train_config z;
  z.net = demo_net();
  z.workers = 2;
  z.micro_batches = 2;
  z.mini_batch_size = 10;
  z.mini_batches = 4;
  z.learning_rate = 0.0;
  z.seed = 5;
  dataset d2 = make_synthetic_task(40, 23);
  std::vector<double> init = init_network_params(z.net, z.seed);
  for (train_mode m : {train_mode::timeprest, train_mode::sequential, train_mode::pipedream}) {
    std::vector<stage_model> st = partition_model(z.net, 2);
    load_network_params(st, init, 0);
    train_epoch(st, d2, z, m, 1);
    const std::vector<double> got = gather_network_params(st);
    for (size_t i = 0; i < got.size(); ++i)
      CHECK(got[i] == static_cast<double>(static_cast<float>(init[i])));
  }

  // run_training with per-stage checkpoints + resume (checkpoint format is
  // the reference's, so either build can resume the other's files)
  namespace fs = std::filesystem;
  const std::string dir = (fs::temp_directory_path() / "pipesim_b200_ckpt").string();
  fs::remove_all(dir);
  train_config rc = z;
  rc.learning_rate = 0.05;
  rc.epochs = 2;
  const train_run_result a = run_training(rc, train_mode::timeprest, d2, dir, false);
  CHECK(a.logs.size() == 2);
  rc.epochs = 3;
  const train_run_result b = run_training(rc, train_mode::timeprest, d2, dir, true);
  CHECK(b.first_epoch == 3);
  const restored_stage r = restore_stage((fs::path(dir) / checkpoint_filename(1, 3)).string(), 1, 3);
  CHECK(r.epoch == 3);
  bool threw = false;
  try {
    restore_stage((fs::path(dir) / checkpoint_filename(2, 9)).string(), 2, 9);
  } catch (const integrity_error& e) {
    threw = e.stage_id() == 2 && e.epoch() == 9;
  }
  CHECK(threw);
}

int main(int argc, char** argv) {
  plan_checks();
  if (!(argc > 1 && std::strcmp(argv[1], "--plan-only") == 0)) train_checks();
  if (failures) {
    std::fprintf(stderr, "%d check(s) failed\n", failures);
    return 1;
  }
  std::printf("dropin_test: all checks passed\n");
  return 0;
}
