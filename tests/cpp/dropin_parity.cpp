// Numeric parity driver for the reference-facing C++ API (test infrastructure).
//
// Written against the reference's headers only (pipesim/trainer.hpp, ...),
// linked against libpipesim_b200.  tests/test_cpp_dropin.py writes the
// network, config and data, runs one command, and compares the outputs with
// the CPU oracle:
//
//   dropin_parity train    IN OUT   epochs of pipesim::train_epoch
//   dropin_parity gradient IN OUT   pipesim::network_gradient (fp32 verify)
//   dropin_parity resume   IN OUT   run_training: continuous vs resumed
//
// IN (text): "widths w0 w1 ..", "acts a0 ..", "loss L", "cfg W N B M epochs lr
// seed mode", "x rows cols v..", "y rows cols v..", "params v..".
// OUT (text): one "key v1 v2 .." line per array, shortest round-trip decimals.
#include <charconv>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "pipesim/checkpoint.hpp"
#include "pipesim/trainer.hpp"

using namespace pipesim;

namespace {

struct input {
  train_config cfg;
  train_mode mode = train_mode::timeprest;
  dataset data;
  std::vector<double> params;
};

std::vector<double> doubles(std::istringstream& is) {
  std::vector<double> v;
  std::string tok;
  while (is >> tok) {
    double d = 0.0;
    std::from_chars(tok.data(), tok.data() + tok.size(), d);
    v.push_back(d);
  }
  return v;
}

matrix read_matrix(std::istringstream& is) {
  int r = 0, c = 0;
  is >> r >> c;
  matrix m(r, c);
  m.data = doubles(is);
  return m;
}

input read_input(const char* path) {
  std::ifstream f(path);
  input in;
  std::string line;
  while (std::getline(f, line)) {
    std::istringstream is(line);
    std::string key;
    is >> key;
    if (key == "widths") {
      int w;
      while (is >> w) in.cfg.net.widths.push_back(w);
    } else if (key == "acts") {
      int a;
      while (is >> a) in.cfg.net.activations.push_back(static_cast<activation_kind>(a));
    } else if (key == "loss") {
      int l;
      is >> l;
      in.cfg.net.loss = l == 0 ? loss_kind::mse : loss_kind::softmax_cross_entropy;
    } else if (key == "cfg") {
      std::string mode;
      is >> in.cfg.workers >> in.cfg.micro_batches >> in.cfg.mini_batch_size >>
          in.cfg.mini_batches >> in.cfg.epochs >> in.cfg.learning_rate >> in.cfg.seed >> mode;
      in.mode = train_mode_from_string(mode);
    } else if (key == "x") {
      in.data.x = read_matrix(is);
    } else if (key == "y") {
      in.data.y = read_matrix(is);
    } else if (key == "params") {
      in.params = doubles(is);
    }
  }
  return in;
}

struct writer {
  std::ofstream f;
  explicit writer(const char* path) : f(path) {}
  template <class T>
  void put(const std::string& key, const std::vector<T>& v) {
    f << key;
    for (const T& x : v) {
      if constexpr (std::is_floating_point_v<T>) {
        char buf[64];
        f << ' ' << std::string(buf, std::to_chars(buf, buf + 64, x).ptr);
      } else {
        f << ' ' << x;
      }
    }
    f << '\n';
  }
  void text(const std::string& key, const std::string& t) {
    std::istringstream is(t);
    std::string line;
    while (std::getline(is, line)) f << key << ' ' << line << '\n';
  }
};

void dump_log(writer& w, const epoch_log& log, const std::string& tag) {
  std::vector<double> losses;
  std::vector<int> pinned, consumed;
  for (const mini_log& m : log.minis) {
    losses.push_back(m.loss);
    consumed.push_back(m.consumed);
    pinned.insert(pinned.end(), m.pinned.begin(), m.pinned.end());
  }
  w.put(tag + ".losses", losses);
  w.put(tag + ".pinned", pinned);
  w.put(tag + ".consumed", consumed);
  w.text(tag + ".log", log.to_text());
}

void dump_stages(writer& w, const std::vector<stage_model>& stages, const std::string& tag) {
  w.put(tag + ".params", gather_network_params(stages));
  for (const stage_model& st : stages) {
    std::vector<int> keys;
    for (const auto& kv : st.version_store) keys.push_back(kv.first);
    keys.push_back(-1);
    keys.push_back(st.current_version);
    w.put(tag + ".stage" + std::to_string(st.stage_id) + ".versions", keys);
    for (const auto& kv : st.version_store)
      w.put(tag + ".stage" + std::to_string(st.stage_id) + ".v" + std::to_string(kv.first),
            kv.second);
  }
}

}  // namespace

int main(int argc, char** argv) {
  if (argc != 4) {
    std::fprintf(stderr, "usage: dropin_parity train|gradient|resume IN OUT\n");
    return 2;
  }
  const std::string cmd = argv[1];
  input in = read_input(argv[2]);
  writer w(argv[3]);
  try {
    if (cmd == "train") {
      std::vector<stage_model> stages = partition_model(in.cfg.net, in.cfg.workers);
      load_network_params(stages, in.params, 0);
      for (int e = 1; e <= in.cfg.epochs; ++e) {
        const epoch_log log = train_epoch(stages, in.data, in.cfg, in.mode, e);
        dump_log(w, log, "e" + std::to_string(e));
      }
      dump_stages(w, stages, "final");
    } else if (cmd == "gradient") {
      b200::options o = b200::get_options();
      o.verify_fp32 = true;
      b200::set_options(o);
      w.put("gradient", network_gradient(in.cfg.net, in.params, in.data));
      w.put("loss", std::vector<double>{network_loss(in.cfg.net, in.params, in.data)});
    } else if (cmd == "resume") {
      namespace fs = std::filesystem;
      const fs::path root = fs::path(argv[3]).parent_path() / "ckpt";
      fs::remove_all(root);
      train_config c = in.cfg;
      const train_run_result full = run_training(c, in.mode, in.data, (root / "a").string(), false);
      c.epochs = in.cfg.epochs - 1;
      const train_run_result part = run_training(c, in.mode, in.data, (root / "b").string(), false);
      c.epochs = in.cfg.epochs;
      const train_run_result resumed =
          run_training(c, in.mode, in.data, (root / "b").string(), true);
      w.put("first_epoch", std::vector<int>{full.first_epoch, part.first_epoch,
                                            resumed.first_epoch});
      w.text("full.checksum", full.final_checksum);
      w.text("resumed.checksum", resumed.final_checksum);
      dump_log(w, full.logs.back(), "full.last");
      dump_log(w, resumed.logs.back(), "resumed.last");
      for (int s = 1; s <= c.workers; ++s) {
        const std::string f = checkpoint_filename(s, c.epochs);
        std::ifstream a(root / "a" / f, std::ios::binary), b(root / "b" / f, std::ios::binary);
        std::stringstream sa, sb;
        sa << a.rdbuf();
        sb << b.rdbuf();
        w.put("ckpt_equal", std::vector<int>{s, sa.str() == sb.str() ? 1 : 0});
      }
    } else {
      std::fprintf(stderr, "unknown command %s\n", cmd.c_str());
      return 2;
    }
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
  return 0;
}
