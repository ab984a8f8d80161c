// pipesim_b200.hpp — drop-in C++ API of the B200-native TiMePReSt step.
//
// Declares the same `pipesim::` names, value types and signatures as the
// reference headers (proj/include/pipesim/{errors,config,schedule,ledger,
// trainer,text,checkpoint}.hpp) so code written against the reference
// compiles and links against libpipesim_b200 unchanged.  The plan layer
// (schedule / ledger / retention) is native host C++; the trainer entry
// points execute on B200 through the C ABI in pipesim_b200.h.
//
// The per-file headers next to this one (pipesim/trainer.hpp, ...) only
// forward here.
#ifndef PIPESIM_B200_HPP_
#define PIPESIM_B200_HPP_

#include <cstdint>
#include <functional>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

namespace pipesim {

// ===================================================================== errors
// errors.hpp:25-65 — same five exception types, same accessors.
class domain_error : public std::runtime_error {
 public:
  domain_error(std::string field, const std::string& message)
      : std::runtime_error(message), field_(std::move(field)) {}
  const std::string& field() const { return field_; }

 private:
  std::string field_;
};

class structural_error : public std::runtime_error {
  using std::runtime_error::runtime_error;
};
class insufficient_horizon_error : public std::runtime_error {
  using std::runtime_error::runtime_error;
};
class io_error : public std::runtime_error {
  using std::runtime_error::runtime_error;
};

class integrity_error : public std::runtime_error {
 public:
  integrity_error(const std::string& message, int stage_id, int epoch)
      : std::runtime_error(message), stage_id_(stage_id), epoch_(epoch) {}
  int stage_id() const { return stage_id_; }
  int epoch() const { return epoch_; }

 private:
  int stage_id_;
  int epoch_;
};

// ===================================================================== config
// config.hpp:25-66
enum class schedule_mode { timeprest, pipedream };

struct sim_config {
  int workers = 2;
  int micro_batches = 2;
  int mini_batches = 1;
  double backward_cost_factor = 2.0;
  int samples_per_mini_batch = 64;
  std::uint64_t seed = 0;
};

// Domain contract: W >= 2, N >= 2, M >= 1, cost factor >= 1, samples >= 1.
// Throws domain_error naming the field.
void validate(const sim_config& cfg);
const char* to_string(schedule_mode mode);

// =================================================================== schedule
// schedule.hpp:25-113
enum class task_kind { idle, forward_micro, backward_mini };

struct task {
  task_kind kind = task_kind::idle;
  int mini = 0;
  int micro = 0;
  bool is_idle() const { return kind == task_kind::idle; }
  bool is_forward() const { return kind == task_kind::forward_micro; }
  bool is_backward() const { return kind == task_kind::backward_mini; }
  friend bool operator==(const task&, const task&) = default;
};

class schedule_grid {
 public:
  schedule_grid(sim_config cfg, schedule_mode mode) : cfg_(cfg), mode_(mode) {}

  const sim_config& config() const { return cfg_; }
  schedule_mode mode() const { return mode_; }
  int workers() const { return cfg_.workers; }
  int horizon() const { return horizon_; }

  const task& at(int worker, int slot) const;
  void put(int worker, int slot, task t);
  void clear(int worker, int slot);
  int forward_slot(int mini, int micro, int stage) const;
  int backward_slot(int mini, int stage) const;

  friend bool operator==(const schedule_grid& a, const schedule_grid& b);

 private:
  sim_config cfg_;
  schedule_mode mode_;
  int horizon_ = 0;
  std::vector<task> cells_;  // slot-major: cells_[(slot-1)*W + (worker-1)]
};

schedule_grid build_nf1b_schedule(const sim_config& cfg);
schedule_grid build_1f1b_schedule(const sim_config& cfg);

enum class violation_kind {
  task_invariant,
  stage_continuity,
  completeness,
  backward_priority,
};
struct violation {
  violation_kind kind;
  std::string message;
};
struct validation_report {
  std::vector<violation> violations;
  bool valid() const { return violations.empty(); }
};
validation_report validate_schedule(const schedule_grid& grid,
                                    const sim_config& cfg);

// ===================================================================== ledger
// ledger.hpp:29-139
struct commit_event {
  int version;
  int mini;
  int stage;
  int slot;
};
struct pin_record {
  int mini;
  int micro;
  int slot;
  int version;
};
struct consume_record {
  int mini;
  int stage;
  int slot;
  int version;
};

struct version_ledger {
  sim_config cfg;
  schedule_mode mode = schedule_mode::timeprest;
  std::vector<commit_event> commits;
  std::vector<pin_record> pins;
  std::vector<consume_record> consumptions;
  std::vector<int> update_source;
  std::vector<int> full_commit_slot;
  int pinned_version(int mini, int micro) const;
};

version_ledger assign_versions(const schedule_grid& grid, const sim_config& cfg);
int measure_version_difference(const version_ledger& ledger, bool strict = true);
int closed_form_v(int workers, int micro_batches);
int forward_span(int workers, int micro_batches, int mini_ordinal);
int backward_span(int workers);
bool overlap_condition(int workers, int micro_batches);

struct sequence_decomposition {
  std::vector<std::vector<int>> sequences;
  int version_difference_measured = 0;
};
sequence_decomposition decompose_sequences(const version_ledger& ledger,
                                           int mini_batches);

// Schedule document JSON (export.hpp; export.cpp:78-139): config, non-idle
// cells, ledger and v analysis, schema version 1.
std::string schedule_document_json(const schedule_grid& grid, const version_ledger& ledger);

struct retention_interval {
  int version;
  int retained_from_slot;
  int freed_at_slot;
};
struct retention_timeline {
  std::vector<std::vector<retention_interval>> per_stage;
  std::vector<int> peak_concurrent;
  int horizon = 0;
  int retained_count(int stage, int slot) const;
};
retention_timeline build_retention_timeline(const version_ledger& ledger,
                                            const schedule_grid& grid);

struct staleness_entry {
  int mini;
  int stage;
  int staleness;
};
struct staleness_report_t {
  std::vector<staleness_entry> entries;
  bool all_zero() const;
  int steady_state_staleness(int first_steady_mini) const;
};
staleness_report_t staleness_report(const version_ledger& ledger);

// ======================================================================= text
// text.hpp:23-30
std::string format_double(double value);
double parse_double(const std::string& text);
std::string fnv1a64_hex(const std::string& data);

// ==================================================================== trainer
// trainer.hpp:28-188
enum class activation_kind { linear, relu, tanh, sigmoid };
enum class loss_kind { mse, softmax_cross_entropy };

const char* to_string(activation_kind a);
const char* to_string(loss_kind l);
activation_kind activation_from_string(const std::string& s);
loss_kind loss_from_string(const std::string& s);

struct matrix {
  int rows = 0;
  int cols = 0;
  std::vector<double> data;
  matrix() = default;
  matrix(int r, int c) : rows(r), cols(c), data(static_cast<size_t>(r) * c) {}
  double& at(int r, int c) { return data[static_cast<size_t>(r) * cols + c]; }
  double at(int r, int c) const { return data[static_cast<size_t>(r) * cols + c]; }
};

struct layer_spec {
  int in = 0;
  int out = 0;
  activation_kind act = activation_kind::linear;
  int param_count() const { return out * in + out; }
};

struct network_spec {
  std::vector<int> widths;
  std::vector<activation_kind> activations;
  loss_kind loss = loss_kind::mse;
  int layer_count() const { return static_cast<int>(widths.size()) - 1; }
  layer_spec layer(int index) const;
  int param_count() const;
};

struct stage_model {
  int stage_id = 0;
  int first_layer = 0;
  std::vector<layer_spec> layers;
  std::map<int, std::vector<double>> version_store;
  int current_version = 0;
  int param_count() const;
  const std::vector<double>& params(int version) const;
  const std::vector<double>& current_params() const {
    return params(current_version);
  }
};

std::vector<stage_model> partition_model(const network_spec& spec, int workers);
std::vector<double> init_network_params(const network_spec& spec,
                                        std::uint64_t seed);
void load_network_params(std::vector<stage_model>& stages,
                         const std::vector<double>& flat, int version);
std::vector<double> gather_network_params(const std::vector<stage_model>& stages);
std::string params_digest(const std::vector<stage_model>& stages);

struct dataset {
  matrix x;
  matrix y;
};
dataset make_synthetic_task(int samples, std::uint64_t seed);

struct train_config {
  network_spec net;
  int workers = 2;
  int micro_batches = 2;
  int mini_batch_size = 20;
  int mini_batches = 10;
  int epochs = 1;
  double learning_rate = 0.05;
  std::uint64_t seed = 1;
};

enum class train_mode { timeprest, sequential, pipedream };
const char* to_string(train_mode m);
train_mode train_mode_from_string(const std::string& s);

struct mini_log {
  int mini = 0;
  double loss = 0.0;
  std::vector<int> pinned;
  int consumed = 0;
  std::string checksum;
};

struct epoch_log {
  int epoch = 0;
  std::vector<mini_log> minis;
  std::string final_checksum;
  std::string to_text() const;
};

using slot_observer =
    std::function<void(int slot, const std::vector<stage_model>&)>;

// The pipeline step, executed on B200.  Same contract as
// trainer.hpp:159-161: stages are mutated in place, the log is returned.
epoch_log train_epoch(std::vector<stage_model>& stages, const dataset& data,
                      const train_config& cfg, train_mode mode, int epoch,
                      const slot_observer& observer = {});

double network_loss(const network_spec& spec, const std::vector<double>& params,
                    const dataset& data);
std::vector<double> network_gradient(const network_spec& spec,
                                     const std::vector<double>& params,
                                     const dataset& data);

struct train_run_result {
  std::vector<epoch_log> logs;
  int first_epoch = 1;
  std::string final_checksum;
};
train_run_result run_training(const train_config& cfg, train_mode mode,
                              const dataset& data,
                              const std::string& checkpoint_dir, bool resume);

// ================================================================ checkpoint
// checkpoint.hpp:29-44
void checkpoint_stage(const stage_model& stage, loss_kind loss, int epoch,
                      const std::string& path);
struct restored_stage {
  stage_model stage;
  loss_kind loss = loss_kind::mse;
  int epoch = 0;
};
restored_stage restore_stage(const std::string& path, int expected_stage = 0,
                             int expected_epoch = 0);
std::string checkpoint_filename(int stage_id, int epoch);

// ============================================================ B200 controls
// Not part of the reference API: execution knobs of the GPU build.  Defaults
// keep the reference semantics; they never change the schedule or versions.
namespace b200 {
enum class digest_policy { automatic, every_mini, final_only };
struct options {
  int device = 0;
  bool use_graph = true;                 // capture the epoch as a CUDA graph
  // mini_log::checksum of every mini-batch (trainer.cpp:492-501) is computed
  // on the device inside the epoch (digest_dev.hpp); automatic = every
  // mini-batch for networks up to digest_auto_limit params, final only above
  digest_policy digest = digest_policy::automatic;
  long long digest_auto_limit = 1LL << 40;
  bool verify_fp32 = false;              // fp32 FFMA verify precision (no bf16 rounding)
};
void set_options(const options& o);
options get_options();

// Host wall-clock breakdown of the calling thread's last train_epoch (ms):
// plan (grid / ledger / retention), load (fp64 params -> device masters and
// version 0), upload (the epoch's fp64 x / y), step (the epoch on the device,
// launch to completion; device_ms = its CUDA-event time), readback (final
// masters + retained versions -> fp64 version_store), digest (fetching the
// device digests; the per-mini-batch ones run inside the epoch, in step), total.
struct epoch_timing {
  double plan_ms = 0, load_ms = 0, upload_ms = 0, step_ms = 0, device_ms = 0,
         readback_ms = 0, digest_ms = 0, total_ms = 0;
};
epoch_timing last_epoch_timing();
}  // namespace b200

}  // namespace pipesim

#endif  // PIPESIM_B200_HPP_
