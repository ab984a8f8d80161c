// Model-side host helpers of the drop-in API: enum tags, network / stage
// value types, the parameter-count partition, seeded init, the synthetic
// task, digests and the epoch-log text.  Semantics follow
// proj/src/trainer.cpp:35-135, :557-640 and proj/src/text.cpp:24-52.
#include <charconv>
#include <cmath>
#include <random>
#include <string>
#include <vector>

#include "pipesim_core.hpp"

namespace pipesim {

// ----------------------------------------------------------------- text
std::string format_double(double value) {
  char buf[64];
  const auto res = std::to_chars(buf, buf + sizeof(buf), value);
  return std::string(buf, res.ptr);
}

double parse_double(const std::string& text) {
  double v = 0.0;
  const char* b = text.data();
  const char* e = b + text.size();
  const auto res = std::from_chars(b, e, v);
  if (res.ec != std::errc{} || res.ptr != e)
    throw io_error("malformed decimal value: '" + text + "'");
  return v;
}

std::string fnv1a64_hex(const std::string& data) {
  pb::fnv1a64 f;
  f.update(data.data(), data.size());
  return f.hex();
}

// ----------------------------------------------------------------- tags
const char* to_string(activation_kind a) {
  switch (a) {
    case activation_kind::relu: return "relu";
    case activation_kind::tanh: return "tanh";
    case activation_kind::sigmoid: return "sigmoid";
    case activation_kind::linear: break;
  }
  return "linear";
}

const char* to_string(loss_kind l) {
  return l == loss_kind::softmax_cross_entropy ? "softmax_cross_entropy" : "mse";
}

activation_kind activation_from_string(const std::string& s) {
  for (activation_kind a : {activation_kind::linear, activation_kind::relu,
                            activation_kind::tanh, activation_kind::sigmoid})
    if (s == to_string(a)) return a;
  throw domain_error("activation", "unknown activation tag: " + s);
}

loss_kind loss_from_string(const std::string& s) {
  if (s == "mse") return loss_kind::mse;
  if (s == "softmax_cross_entropy") return loss_kind::softmax_cross_entropy;
  throw domain_error("loss", "unknown loss tag: " + s);
}

const char* to_string(train_mode m) {
  switch (m) {
    case train_mode::timeprest: return "timeprest";
    case train_mode::pipedream: return "pipedream";
    case train_mode::sequential: break;
  }
  return "sequential";
}

train_mode train_mode_from_string(const std::string& s) {
  for (train_mode m :
       {train_mode::timeprest, train_mode::sequential, train_mode::pipedream})
    if (s == to_string(m)) return m;
  throw domain_error("mode", "unknown training mode: " + s);
}

// ----------------------------------------------------------------- network
layer_spec network_spec::layer(int index) const {
  return layer_spec{widths[index], widths[index + 1], activations[index]};
}

int network_spec::param_count() const {
  int n = 0;
  for (int l = 0; l < layer_count(); ++l) n += layer(l).param_count();
  return n;
}

int stage_model::param_count() const {
  int n = 0;
  for (const layer_spec& l : layers) n += l.param_count();
  return n;
}

const std::vector<double>& stage_model::params(int version) const {
  const auto it = version_store.find(version);
  if (it == version_store.end())
    throw structural_error("stage " + std::to_string(stage_id) +
                           " does not hold version " + std::to_string(version));
  return it->second;
}

// Greedy contiguous split by parameter count (trainer.cpp:104-135): a stage
// takes layers until it reaches total/W, always leaving one layer for each
// stage still to come.
std::vector<stage_model> partition_model(const network_spec& spec, int workers) {
  const int L = spec.layer_count();
  if (workers < 1) throw domain_error("workers", "workers must be >= 1");
  if (L < workers)
    throw domain_error("layers", "cannot split " + std::to_string(L) +
                                     " layers across " + std::to_string(workers) +
                                     " stages");
  if (static_cast<int>(spec.activations.size()) != L)
    throw structural_error("one activation tag per layer required");

  const double share = static_cast<double>(spec.param_count()) / workers;
  std::vector<stage_model> out(workers);
  int next = 0;
  for (int s = 0; s < workers; ++s) {
    stage_model& st = out[s];
    st.stage_id = s + 1;
    st.first_layer = next;
    const bool last = s + 1 == workers;
    const int limit = L - (workers - 1 - s);  // leave one layer per later stage
    double taken = 0.0;
    while (next < limit) {
      if (!last && taken >= share) break;
      st.layers.push_back(spec.layer(next));
      taken += spec.layer(next).param_count();
      ++next;
      if (!last && taken >= share) break;
    }
  }
  return out;
}

namespace {
double unit_uniform(std::mt19937_64& g) {
  return static_cast<double>(g() >> 11) * 0x1.0p-53;
}
}  // namespace

std::vector<double> init_network_params(const network_spec& spec,
                                        std::uint64_t seed) {
  std::mt19937_64 g(seed);
  std::vector<double> p;
  p.reserve(spec.param_count());
  for (int l = 0; l < spec.layer_count(); ++l) {
    const layer_spec ls = spec.layer(l);
    const double bound = 1.0 / std::sqrt(static_cast<double>(ls.in));
    for (int i = 0, n = ls.param_count(); i < n; ++i)
      p.push_back((2.0 * unit_uniform(g) - 1.0) * bound);
  }
  return p;
}

void load_network_params(std::vector<stage_model>& stages,
                         const std::vector<double>& flat, int version) {
  size_t off = 0;
  for (stage_model& st : stages) {
    const size_t n = st.param_count();
    if (off + n > flat.size())
      throw structural_error("parameter vector shorter than the network");
    st.version_store.clear();
    st.version_store[version].assign(flat.begin() + off, flat.begin() + off + n);
    st.current_version = version;
    off += n;
  }
  if (off != flat.size())
    throw structural_error("parameter vector longer than the network");
}

std::vector<double> gather_network_params(const std::vector<stage_model>& stages) {
  std::vector<double> flat;
  for (const stage_model& st : stages) {
    const std::vector<double>& p = st.current_params();
    flat.insert(flat.end(), p.begin(), p.end());
  }
  return flat;
}

std::string params_digest(const std::vector<stage_model>& stages) {
  // same text and hash as trainer.cpp:599-607, formatted on host threads
  std::vector<pb::value_span> spans;
  for (const stage_model& st : stages) {
    const std::vector<double>& p = st.current_params();
    spans.push_back({p.data(), static_cast<int64_t>(p.size())});
  }
  return pb::digest_spans(spans);
}

dataset make_synthetic_task(int samples, std::uint64_t seed) {
  std::mt19937_64 g(seed);
  dataset d;
  d.x = matrix(samples, 2);
  d.y = matrix(samples, 2);
  for (int i = 0; i < samples; ++i) {
    double a, b, margin;
    do {
      a = 2.0 * unit_uniform(g) - 1.0;
      b = 2.0 * unit_uniform(g) - 1.0;
      margin = 0.8 * a - 0.6 * b;
    } while (std::abs(margin) < 0.1);
    d.x.at(i, 0) = a;
    d.x.at(i, 1) = b;
    d.y.at(i, margin > 0.0 ? 0 : 1) = 1.0;
  }
  return d;
}

std::string epoch_log::to_text() const {
  std::string s;
  const std::string ep = "epoch " + std::to_string(epoch);
  for (const mini_log& m : minis) {
    s += ep + " mini " + std::to_string(m.mini) + " loss " + format_double(m.loss) +
         " pinned";
    for (int p : m.pinned) s += " " + std::to_string(p);
    s += " consumed " + std::to_string(m.consumed) + " checksum " + m.checksum + "\n";
  }
  s += ep + " final checksum " + final_checksum + "\n";
  return s;
}

}  // namespace pipesim
