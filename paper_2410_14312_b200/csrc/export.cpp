// Schedule document (reference: proj/src/export.cpp:78-139, schema version 1):
// config, the grid's non-idle cells, the version ledger (commits,
// consumptions, pins) and the v analysis, as 2-space-indented JSON in the
// reference's key order.  The same writer serialises the device-observed
// trace of a session epoch (Session::trace_document), so a GPU run's version
// trace can be byte-diffed against the reference's `pipesim simulate` output.
#include <string>
#include <utility>
#include <vector>

#include "pipesim_core.hpp"

namespace pipesim {

namespace {

constexpr int kDocumentSchemaVersion = 1;

// A minimal ordered JSON value with the reference's pretty-printer layout.
struct J {
  enum Kind { kNull, kInt, kDouble, kString, kArray, kObject } kind = kNull;
  long long i = 0;
  double d = 0.0;
  std::string s;
  std::vector<J> a;
  std::vector<std::pair<std::string, J>> o;

  static J null() { return J{}; }
  static J integer(long long v) {
    J j;
    j.kind = kInt;
    j.i = v;
    return j;
  }
  static J real(double v) {
    J j;
    j.kind = kDouble;
    j.d = v;
    return j;
  }
  static J str(std::string v) {
    J j;
    j.kind = kString;
    j.s = std::move(v);
    return j;
  }
  static J array() {
    J j;
    j.kind = kArray;
    return j;
  }
  static J object() {
    J j;
    j.kind = kObject;
    return j;
  }
  J& set(const std::string& k, J v) {
    o.emplace_back(k, std::move(v));
    return *this;
  }
  J& push(J v) {
    a.push_back(std::move(v));
    return *this;
  }
};

void dump(const J& v, int depth, std::string& out) {
  const std::string ind(2 * (depth + 1), ' ');
  const std::string close(2 * depth, ' ');
  switch (v.kind) {
    case J::kNull: out += "null"; break;
    case J::kInt: out += std::to_string(v.i); break;
    case J::kDouble: {
      std::string t = format_double(v.d);  // shortest round trip
      if (t.find_first_of(".eEn") == std::string::npos) t += ".0";
      out += t;
      break;
    }
    case J::kString: out += "\"" + v.s + "\""; break;
    case J::kArray:
      if (v.a.empty()) {
        out += "[]";
        break;
      }
      out += "[\n";
      for (size_t k = 0; k < v.a.size(); ++k) {
        out += ind;
        dump(v.a[k], depth + 1, out);
        out += k + 1 < v.a.size() ? ",\n" : "\n";
      }
      out += close + "]";
      break;
    case J::kObject:
      if (v.o.empty()) {
        out += "{}";
        break;
      }
      out += "{\n";
      for (size_t k = 0; k < v.o.size(); ++k) {
        out += ind + "\"" + v.o[k].first + "\": ";
        dump(v.o[k].second, depth + 1, out);
        out += k + 1 < v.o.size() ? ",\n" : "\n";
      }
      out += close + "}";
      break;
  }
}

J opt_micro(int micro) { return micro > 0 ? J::integer(micro) : J::null(); }

}  // namespace

std::string schedule_document_json(const schedule_grid& grid, const version_ledger& ledger) {
  const sim_config& cfg = grid.config();
  const bool nf1b = grid.mode() == schedule_mode::timeprest;
  J doc = J::object();
  doc.set("schema_version", J::integer(kDocumentSchemaVersion));
  J c = J::object();
  c.set("workers", J::integer(cfg.workers))
      .set("micro_batches", J::integer(cfg.micro_batches))
      .set("mini_batches", J::integer(cfg.mini_batches))
      .set("mode", J::str(to_string(grid.mode())))
      .set("backward_cost_factor", J::real(cfg.backward_cost_factor))
      .set("samples_per_mini_batch", J::integer(cfg.samples_per_mini_batch))
      .set("seed", J::integer(static_cast<long long>(cfg.seed)));
  doc.set("config", std::move(c));

  J cells = J::array();
  for (int w = 1; w <= grid.workers(); ++w)
    for (int t = 1; t <= grid.horizon(); ++t) {
      const task& cell = grid.at(w, t);
      if (cell.is_idle()) continue;
      J e = J::object();
      e.set("worker", J::integer(w))
          .set("slot", J::integer(t))
          .set("kind", J::str(cell.is_forward() ? "forward" : "backward"))
          .set("mini", J::integer(cell.mini))
          .set("micro", cell.is_forward() ? opt_micro(cell.micro) : J::null());
      cells.push(std::move(e));
    }
  doc.set("cells", std::move(cells));

  J commits = J::array(), cons = J::array(), pins = J::array();
  for (const auto& e : ledger.commits)
    commits.push(J::object()
                     .set("version", J::integer(e.version))
                     .set("mini", J::integer(e.mini))
                     .set("stage", J::integer(e.stage))
                     .set("slot", J::integer(e.slot)));
  for (const auto& e : ledger.consumptions)
    cons.push(J::object()
                  .set("mini", J::integer(e.mini))
                  .set("stage", J::integer(e.stage))
                  .set("slot", J::integer(e.slot))
                  .set("version", J::integer(e.version)));
  for (const auto& e : ledger.pins)
    pins.push(J::object()
                  .set("mini", J::integer(e.mini))
                  .set("micro", opt_micro(e.micro))
                  .set("slot", J::integer(e.slot))
                  .set("version", J::integer(e.version)));
  J led = J::object();
  led.set("commits", std::move(commits)).set("consumptions", std::move(cons)).set("pins", std::move(pins));
  doc.set("ledger", std::move(led));

  // analysis (export.cpp:43-72): mini-batch 1's forward span, backward span,
  // v laws and the sequence decomposition (nF1B only)
  J an = J::object();
  an.set("f1", J::integer(nf1b ? cfg.workers + cfg.micro_batches - 1 : cfg.workers));
  an.set("b", J::integer(cfg.workers));
  if (nf1b) {
    an.set("v_closed_form", J::integer(closed_form_v(cfg.workers, cfg.micro_batches)));
    try {
      an.set("v_measured", J::integer(measure_version_difference(ledger, /*strict=*/false)));
    } catch (const insufficient_horizon_error&) {
      an.set("v_measured", J::null());
    }
    J seqs = J::array();
    try {
      for (const auto& seq : decompose_sequences(ledger, cfg.mini_batches).sequences) {
        J one = J::array();
        for (int k : seq) one.push(J::integer(k));
        seqs.push(std::move(one));
      }
    } catch (const insufficient_horizon_error&) {
      seqs = J::array();
    }
    an.set("sequences", std::move(seqs));
  } else {
    an.set("v_closed_form", J::null()).set("v_measured", J::null()).set("sequences", J::array());
  }
  doc.set("analysis", std::move(an));

  std::string out;
  dump(doc, 0, out);
  return out + "\n";
}

}  // namespace pipesim
