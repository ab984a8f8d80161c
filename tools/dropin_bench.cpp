// End-to-end timing of the reference-facing C++ call (measurement harness).
//
// A program written against the reference's API (pipesim/trainer.hpp) calls
// pipesim::train_epoch exactly as a reference user does: fp64 stages and an
// fp64 dataset (x plus one-hot y) in host memory, the log returned by value,
// version_store refilled, digests computed.  Prints one JSON line with
// samples/s over the timed epochs and the per-phase breakdown
// (pipesim::b200::last_epoch_timing).
//
//   dropin_bench c1|c3 [epochs=3] [digest=auto|every|final]
//
// c1: 784-512-256-10 (ReLU, ReLU, linear; softmax-CE), W=2, N=4, B=256, M=32
// c3: 16 x Linear(4096->4096) (ReLU x15, linear; softmax-CE over 4096),
//     W=8, N=8, B=1024, M=32 (BASELINE configs[2])
// The first epoch is a warm-up (session creation, graph capture).
#include <chrono>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "pipesim/trainer.hpp"
#include "pipesim_b200.h"

using namespace pipesim;

int main(int argc, char** argv) {
  const std::string which = argc > 1 ? argv[1] : "c1";
  const int epochs = argc > 2 ? std::atoi(argv[2]) : 3;
  const std::string digest = argc > 3 ? argv[3] : "auto";
  train_config cfg;
  if (which == "c3") {
    cfg.net.widths.assign(17, 4096);
    cfg.net.activations.assign(16, activation_kind::relu);
    cfg.net.activations.back() = activation_kind::linear;
    cfg.workers = 8;
    cfg.micro_batches = 8;
    cfg.mini_batch_size = 1024;
  } else {
    cfg.net.widths = {784, 512, 256, 10};
    cfg.net.activations = {activation_kind::relu, activation_kind::relu, activation_kind::linear};
    cfg.workers = 2;
    cfg.micro_batches = 4;
    cfg.mini_batch_size = 256;
  }
  cfg.net.loss = loss_kind::softmax_cross_entropy;
  cfg.mini_batches = 32;
  cfg.learning_rate = 0.05;
  cfg.seed = 1;
  b200::options opt = b200::get_options();
  if (digest == "every") opt.digest = b200::digest_policy::every_mini;
  if (digest == "final") opt.digest = b200::digest_policy::final_only;
  b200::set_options(opt);

  const int rows = cfg.mini_batches * cfg.mini_batch_size;
  const int in = cfg.net.widths.front(), classes = cfg.net.widths.back();
  dataset data;
  data.x = matrix(rows, in);
  data.y = matrix(rows, classes);
  std::vector<int> labels(rows);
  if (pb_make_classification_task(rows, in, classes, 7, data.x.data.data(), nullptr,
                                  labels.data()) != PB_OK) {
    std::fprintf(stderr, "data generation failed\n");
    return 1;
  }
  for (int r = 0; r < rows; ++r) data.y.at(r, labels[r]) = 1.0;

  std::vector<stage_model> stages = partition_model(cfg.net, cfg.workers);
  load_network_params(stages, init_network_params(cfg.net, cfg.seed), 0);

  b200::epoch_timing sum;
  double wall_ms = 0;
  int timed = 0;
  std::string checksum;
  for (int e = 1; e <= epochs; ++e) {
    const auto t0 = std::chrono::steady_clock::now();
    const epoch_log log = train_epoch(stages, data, cfg, train_mode::timeprest, e);
    const double ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    checksum = log.final_checksum;
    if (e == 1 && epochs > 1) continue;
    const b200::epoch_timing t = b200::last_epoch_timing();
    sum.plan_ms += t.plan_ms;
    sum.load_ms += t.load_ms;
    sum.upload_ms += t.upload_ms;
    sum.step_ms += t.step_ms;
    sum.device_ms += t.device_ms;
    sum.readback_ms += t.readback_ms;
    sum.digest_ms += t.digest_ms;
    sum.total_ms += t.total_ms;
    wall_ms += ms;
    ++timed;
  }
  const double n = timed;
  const double per = wall_ms / n;
  std::printf(
      "{\"config\": \"%s\", \"samples_per_epoch\": %d, \"epochs_timed\": %d, "
      "\"ms_per_epoch\": %.3f, \"samples_per_s\": %.3f, \"params\": %d, "
      "\"digest\": \"%s\", \"final_checksum\": \"%s\", \"breakdown_ms\": {\"plan\": %.3f, "
      "\"load_params\": %.3f, \"upload_data\": %.3f, \"step\": %.3f, \"step_device\": %.3f, "
      "\"readback\": %.3f, \"digest\": %.3f, \"other\": %.3f}}\n",
      which.c_str(), rows, timed, per, rows / (per / 1000.0), cfg.net.param_count(),
      digest.c_str(), checksum.c_str(), sum.plan_ms / n, sum.load_ms / n, sum.upload_ms / n,
      sum.step_ms / n, sum.device_ms / n, sum.readback_ms / n, sum.digest_ms / n,
      (sum.total_ms - sum.plan_ms - sum.load_ms - sum.upload_ms - sum.step_ms -
       sum.readback_ms - sum.digest_ms) / n);
  return 0;
}
