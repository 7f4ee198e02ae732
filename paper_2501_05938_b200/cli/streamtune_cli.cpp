// streamtune_cli.cpp -- the `streamtune` command-line front end
// (module "cli").
//
//   streamtune fit --stage-csv F --runs-csv F [--seed 42] [--size-threshold 1000000]
//                  [--overhead-fit ols|anchored] --out M
//   streamtune predict --model M|paper|b200 --sizes N[,N...] [--precision fp64|fp32]
//   streamtune baseline --stage-csv F --tau T [--model M]
//   streamtune simulate --h2d1 . --comp1 . --d2h1 . --cpu . --h2d3 . --comp3 . --d2h3 .
//                       --streams n [--tau T] [--hw-queues 32] [--trace out.csv]
//   streamtune report --model M|paper|b200 --reference table1|table2|table4|table5
//   streamtune dump-reference --reference table1|table2|table4|table5|tau
// Every command takes --json (machine-readable output: the same numbers at
// full precision).  Exit codes (errors.hpp:9-21): 0 success,
// 1 ValidationError (bad flags, malformed CSV/bundle, invalid stream count),
// 2 ComputationError (too few observations, rank deficiency, tau <= 0, FAIL
// cells in a report).  Human output prints milliseconds with 6 decimals.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "streamtune/bundle_io.hpp"
#include "streamtune/dataset.hpp"
#include "streamtune/predictor.hpp"
#include "streamtune/simulator.hpp"
#include "streamtune/timing_model.hpp"

using namespace streamtune;

namespace {

struct Flags {
  std::map<std::string, std::string> kv;
  bool json = false;

  bool has(const std::string& k) const { return kv.count(k) != 0; }
  const std::string& need(const std::string& k) const {
    auto it = kv.find(k);
    if (it == kv.end()) throw ValidationError("missing required flag --" + k);
    return it->second;
  }
  std::string get(const std::string& k, const std::string& def) const {
    auto it = kv.find(k);
    return it == kv.end() ? def : it->second;
  }
  double num(const std::string& k, double def, bool required = false) const {
    if (!has(k)) {
      if (required) need(k);
      return def;
    }
    const std::string& s = kv.at(k);
    char* end = nullptr;
    const double v = std::strtod(s.c_str(), &end);
    if (end == s.c_str() || *end != '\0')
      throw ValidationError("flag --" + k + " is not a number: '" + s + "'");
    return v;
  }
  std::uint64_t u64(const std::string& k, std::uint64_t def) const {
    if (!has(k)) return def;
    const double v = num(k, 0.0);
    if (!(v >= 0.0) || v != std::floor(v)) throw ValidationError("flag --" + k + " must be a non-negative integer");
    return static_cast<std::uint64_t>(v);
  }
};

Flags parse(int argc, char** argv, int first) {
  Flags f;
  for (int i = first; i < argc; ++i) {
    std::string a = argv[i];
    if (a.rfind("--", 0) != 0) throw ValidationError("unexpected argument '" + a + "'");
    a = a.substr(2);
    if (a == "json") {
      f.json = true;
      continue;
    }
    const size_t eq = a.find('=');
    if (eq != std::string::npos) {
      f.kv[a.substr(0, eq)] = a.substr(eq + 1);
    } else {
      if (i + 1 >= argc) throw ValidationError("flag --" + a + " needs a value");
      f.kv[a] = argv[++i];
    }
  }
  return f;
}

std::string read_file(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw ValidationError("cannot read file '" + path + "'");
  std::ostringstream s;
  s << in.rdbuf();
  return s.str();
}

ModelBundle load_model(const std::string& spec) {
  if (spec == "paper") return ModelBundle::paper();
  if (spec == "b200") return ModelBundle::b200();
  return bundle_from_document(read_file(spec));
}

std::string f6(double v) {
  char b[64];
  std::snprintf(b, sizeof(b), "%.6f", v);
  return b;
}
std::string g17(double v) {
  char b[64];
  std::snprintf(b, sizeof(b), "%.17g", v);
  return b;
}

std::vector<std::uint64_t> parse_sizes(const std::string& s) {
  std::vector<std::uint64_t> out;
  std::stringstream ss(s);
  std::string tok;
  while (std::getline(ss, tok, ',')) {
    if (tok.empty()) continue;
    char* end = nullptr;
    const double v = std::strtod(tok.c_str(), &end);
    if (end == tok.c_str() || *end != '\0' || !(v >= 1.0) || v != std::floor(v))
      throw ValidationError("bad SLAE size '" + tok + "'");
    out.push_back(static_cast<std::uint64_t>(v));
  }
  if (out.empty()) throw ValidationError("--sizes is empty");
  return out;
}

int cmd_fit(const Flags& f) {
  std::istringstream s1(read_file(f.need("stage-csv"))), s2(read_file(f.need("runs-csv")));
  const StageTimingsTable st = load_stage_timings(s1);
  const StreamedRunTable rt = load_streamed_runs(s2);
  const std::string mode = f.get("overhead-fit", "ols");
  if (mode != "ols" && mode != "anchored") throw ValidationError("--overhead-fit must be ols or anchored");
  BundleFit fit = fit_bundle(st, rt, f.u64("size-threshold", 1000000), f.u64("seed", 42), mode == "anchored");
  fit.bundle.fitted_on = f.get("fitted-on", f.need("stage-csv"));
  const FitMetricsDoc met = fit.metrics();
  const std::string doc = bundle_to_document(fit.bundle, &met);
  if (f.has("out")) {
    std::ofstream o(f.need("out"));
    if (!o) throw ValidationError("cannot write '" + f.need("out") + "'");
    o << doc;
  }
  if (f.json) {
    std::cout << doc;
    return 0;
  }
  const std::pair<const char*, const FitReport*> reps[3] = {
      {"sum (Eq. 4)", &fit.sum}, {"overhead small (Eq. 7)", &fit.small}, {"overhead big (Eq. 7)", &fit.big}};
  for (const auto& r : reps) {
    std::cout << r.first << ": coefficients";
    for (double c : r.second->coefficients) std::cout << ' ' << g17(c);
    std::cout << "\n  train R2 " << r.second->train.r_squared << " RMSE " << r.second->train.rmse
              << " (n=" << r.second->n_train << ")  test R2 " << r.second->test.r_squared << " RMSE "
              << r.second->test.rmse << " (n=" << r.second->n_test << ")\n";
  }
  if (f.has("out")) std::cout << "wrote " << f.need("out") << "\n";
  return 0;
}

int cmd_predict(const Flags& f) {
  const ModelBundle b = load_model(f.get("model", "paper"));
  const std::string prec = f.get("precision", "fp64");
  if (prec != "fp64" && prec != "fp32") throw ValidationError("--precision must be fp64 or fp32");
  const auto sizes = parse_sizes(f.need("sizes"));
  std::ostringstream js;
  js << "{\"precision\": \"" << prec << "\", \"predictions\": [";
  for (size_t i = 0; i < sizes.size(); ++i) {
    const Recommendation r = recommend(b, sizes[i]);
    const int chosen = prec == "fp32" ? recommend_fp32(b, sizes[i]).value() : r.chosen.value();
    if (f.json) {
      js << (i ? ", " : "") << "{\"slae_size\": " << sizes[i] << ", \"chosen\": " << chosen
         << ", \"model_used\": \"" << (r.model_used == OverheadModel::small ? "small" : "big")
         << "\", \"rows\": [";
      for (size_t k = 0; k < r.rows.size(); ++k)
        js << (k ? ", " : "") << "{\"n\": " << r.rows[k].n.value() << ", \"predicted_sum\": "
           << g17(r.rows[k].predicted_sum) << ", \"predicted_overhead\": "
           << g17(r.rows[k].predicted_overhead) << ", \"benefit\": " << g17(r.rows[k].benefit) << "}";
      js << "]}";
    } else {
      std::cout << "N = " << sizes[i] << "  (" << (r.model_used == OverheadModel::small ? "small" : "big")
                << " overhead model)\n";
      std::cout << "  n   predicted_sum   overhead        benefit\n";
      for (const BenefitRow& row : r.rows)
        std::cout << "  " << row.n.value() << (row.n.value() < 10 ? "   " : "  ") << f6(row.predicted_sum)
                  << "        " << f6(row.predicted_overhead) << "        " << f6(row.benefit) << "\n";
      std::cout << "  chosen streams (" << prec << "): " << chosen << "\n";
    }
  }
  if (f.json) std::cout << js.str() << "]}\n";
  return 0;
}

int cmd_baseline(const Flags& f) {
  const double tau = f.num("tau", ReferenceData::tau_ms, true);
  std::istringstream s1(read_file(f.need("stage-csv")));
  const StageTimingsTable st = load_stage_timings(s1);
  const ModelBundle b = load_model(f.get("model", "paper"));
  std::ostringstream js;
  js << "{\"tau_ms\": " << g17(tau) << ", \"rows\": [";
  if (!f.json) std::cout << "slae_size      sum             gomez_luna   recommend\n";
  for (size_t i = 0; i < st.rows.size(); ++i) {
    const StageTimings& t = st.rows[i];
    const double s = overlap_sum(t);
    const double gl = gomez_luna_optimum(s, tau);  // throws NonpositiveTauError
    const int rec = recommend(b, t.slae_size).chosen.value();
    if (f.json)
      js << (i ? ", " : "") << "{\"slae_size\": " << t.slae_size << ", \"sum\": " << g17(s)
         << ", \"gomez_luna\": " << g17(gl) << ", \"recommend\": " << rec << "}";
    else
      std::cout << t.slae_size << "\t" << f6(s) << "\t" << f6(gl) << "\t" << rec << "\n";
  }
  if (st.rows.empty() && tau <= 0.0) gomez_luna_optimum(0.0, tau);
  if (f.json) std::cout << js.str() << "]}\n";
  return 0;
}

int cmd_simulate(const Flags& f) {
  PipelineSpec p;
  p.stage1 = StageSpec{f.num("h2d1", 0), f.num("comp1", 0), f.num("d2h1", 0)};
  p.cpu_ms = f.num("cpu", 0);
  p.stage3 = StageSpec{f.num("h2d3", 0), f.num("comp3", 0), f.num("d2h3", 0)};
  const double n = f.num("streams", 1);
  if (n != std::floor(n)) throw InvalidStreamCountError(static_cast<int>(n));
  p.num_streams = StreamCount(static_cast<int>(n));
  p.tau_ms = f.num("tau", 0);
  p.hw_queues = static_cast<int>(f.num("hw-queues", 32));
  const SimResult r = simulate(p);
  const double bound = streamed_lower_bound(p.timings(), p.num_streams, p.num_streams.value() * p.tau_ms);
  const double eq1 = total_unstreamed(p.timings());
  if (f.has("trace")) {
    std::ofstream o(f.need("trace"));
    if (!o) throw ValidationError("cannot write '" + f.need("trace") + "'");
    write_trace_csv(o, r);
  }
  if (f.json) {
    std::cout << "{\"total_ms\": " << g17(r.total_ms) << ", \"stage1_makespan_ms\": "
              << g17(r.stage1_makespan_ms) << ", \"stage3_makespan_ms\": " << g17(r.stage3_makespan_ms)
              << ", \"eq1_total_unstreamed_ms\": " << g17(eq1) << ", \"eq2_lower_bound_ms\": " << g17(bound)
              << ", \"lower_bound_holds\": " << (verify_lower_bound(p) ? "true" : "false")
              << ", \"dominance\": " << (dominance_holds(p) ? "true" : "false") << "}\n";
  } else {
    std::cout << "total            " << f6(r.total_ms) << " ms\n"
              << "stage 1 makespan " << f6(r.stage1_makespan_ms) << " ms\n"
              << "stage 3 makespan " << f6(r.stage3_makespan_ms) << " ms\n"
              << "Eq. 1 (unstreamed) " << f6(eq1) << " ms\n"
              << "Eq. 2 lower bound  " << f6(bound) << " ms ("
              << (dominance_holds(p) ? "exact: dominance regime" : "strict unless dominant copies") << ")\n";
  }
  return 0;
}

int cmd_report(const Flags& f) {
  const ModelBundle b = load_model(f.get("model", "paper"));
  const TableReport r = report_table(b, f.need("reference"));
  static const char* st[3] = {"PASS", "FAIL", "KNOWN"};
  if (f.json) {
    std::cout << "{\"table\": \"" << r.table << "\", \"passed\": " << r.passed << ", \"failed\": " << r.failed
              << ", \"known\": " << r.known << ", \"cells\": [";
    for (size_t i = 0; i < r.cells.size(); ++i) {
      const ReportCell& c = r.cells[i];
      std::cout << (i ? ", " : "") << "{\"row\": \"" << c.row << "\", \"column\": \"" << c.column
                << "\", \"expected\": " << g17(c.expected) << ", \"got\": " << g17(c.got)
                << ", \"tolerance\": " << g17(c.tolerance) << ", \"status\": \""
                << st[static_cast<int>(c.status)] << "\"}";
    }
    std::cout << "]}\n";
  } else {
    for (const ReportCell& c : r.cells) {
      std::cout << st[static_cast<int>(c.status)] << "  " << c.row << "  " << c.column << "  expected "
                << f6(c.expected) << "  got " << f6(c.got) << "  (tol " << c.tolerance << ")";
      if (!c.note.empty()) std::cout << "  -- " << c.note;
      std::cout << "\n";
    }
    std::cout << r.table << ": " << r.passed << " PASS, " << r.failed << " FAIL, " << r.known
              << " KNOWN\n";
  }
  return r.failed ? 2 : 0;
}

int cmd_dump(const Flags& f) {
  std::cout << dump_reference(f.need("reference"));
  return 0;
}

void usage() {
  std::cerr << "usage: streamtune {fit|predict|baseline|simulate|report|dump-reference} [--flags] [--json]\n";
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    usage();
    return 1;
  }
  const std::string cmd = argv[1];
  try {
    const Flags f = parse(argc, argv, 2);
    if (cmd == "fit") return cmd_fit(f);
    if (cmd == "predict") return cmd_predict(f);
    if (cmd == "baseline") return cmd_baseline(f);
    if (cmd == "simulate") return cmd_simulate(f);
    if (cmd == "report") return cmd_report(f);
    if (cmd == "dump-reference") return cmd_dump(f);
    usage();
    return 1;
  } catch (const ComputationError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 2;
  } catch (const ValidationError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  }
}
