// st_capi.cpp -- extern "C" wrappers of the streamtune C++ API (include/streamtune_c.h).
#include "streamtune_c.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <sstream>
#include <string>
#include <vector>

#include "streamtune/bundle_io.hpp"
#include "streamtune/dataset.hpp"
#include "streamtune/predictor.hpp"
#include "streamtune/regression.hpp"
#include "streamtune/simulator.hpp"
#include "streamtune/timing_model.hpp"

namespace {

using namespace streamtune;

void put(char* err, int errlen, const std::string& s) {
  if (!err || errlen <= 0) return;
  std::strncpy(err, s.c_str(), (size_t)errlen - 1);
  err[errlen - 1] = '\0';
}

// Runs f, mapping the exception taxonomy (errors.hpp) to status codes and
// "<Class>: <message>" strings.
template <class F>
int guarded(char* err, int errlen, F&& f) {
  try {
    f();
    return ST_OK;
  } catch (const MalformedRowError& e) {
    put(err, errlen, std::string("MalformedRowError: ") + e.what());
  } catch (const NegativeDurationError& e) {
    put(err, errlen, std::string("NegativeDurationError: ") + e.what());
  } catch (const DuplicateSizeError& e) {
    put(err, errlen, std::string("DuplicateSizeError: ") + e.what());
  } catch (const InvalidStreamCountError& e) {
    put(err, errlen, std::string("InvalidStreamCountError: ") + e.what());
  } catch (const MissingStageTimingsError& e) {
    put(err, errlen, std::string("MissingStageTimingsError: ") + e.what());
  } catch (const ValidationError& e) {
    put(err, errlen, std::string("ValidationError: ") + e.what());
    return ST_VALIDATION;
  } catch (const TooFewObservationsError& e) {
    put(err, errlen, std::string("TooFewObservationsError: ") + e.what());
    return ST_COMPUTATION;
  } catch (const RankDeficiencyError& e) {
    put(err, errlen, std::string("RankDeficiencyError: ") + e.what());
    return ST_COMPUTATION;
  } catch (const ZeroVarianceError& e) {
    put(err, errlen, std::string("ZeroVarianceError: ") + e.what());
    return ST_COMPUTATION;
  } catch (const NonpositiveTauError& e) {
    put(err, errlen, std::string("NonpositiveTauError: ") + e.what());
    return ST_COMPUTATION;
  } catch (const ComputationError& e) {
    put(err, errlen, std::string("ComputationError: ") + e.what());
    return ST_COMPUTATION;
  } catch (const std::exception& e) {
    put(err, errlen, std::string("ValidationError: ") + e.what());
    return ST_VALIDATION;
  }
  return ST_VALIDATION;  // the ValidationError subclasses above
}

StageTimings from_c(const pm_stage_timings& c) {
  StageTimings t;
  t.slae_size = c.slae_size;
  t.t1_h2d = c.t1_h2d; t.t1_comp = c.t1_comp; t.t1_d2h = c.t1_d2h; t.t2_comp = c.t2_comp;
  t.t3_h2d = c.t3_h2d; t.t3_comp = c.t3_comp; t.t3_d2h = c.t3_d2h;
  return t;
}

ModelBundle bundle_from_c(const pm_model_bundle* c) {
  if (!c) return ModelBundle::paper();
  ModelBundle b;
  b.sum_a = c->sum_a; b.sum_b = c->sum_b;
  b.small_a = c->small_a; b.small_b = c->small_b; b.small_c = c->small_c;
  b.big_a = c->big_a; b.big_b = c->big_b; b.big_c = c->big_c;
  b.size_threshold = c->size_threshold;
  b.candidates.clear();
  if (c->num_candidates < 0 || c->num_candidates > 5) throw ValidationError("bad candidate count");
  for (int k = 0; k < c->num_candidates; ++k) b.candidates.emplace_back(c->candidates[k]);
  b.validate();
  return b;
}

}  // namespace

extern "C" {

int st_stream_count_is_valid(int n) { return StreamCount::is_valid(n) ? 1 : 0; }

int st_validate_stage_timings(const pm_stage_timings* t, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    if (!t) throw ValidationError("null StageTimings");
    from_c(*t).validate();
  });
}

double st_total_unstreamed(const pm_stage_timings* t) { return total_unstreamed(from_c(*t)); }
double st_overlap_sum(const pm_stage_timings* t) { return overlap_sum(from_c(*t)); }

int st_streamed_lower_bound(const pm_stage_timings* t, int n, double overhead_ms, double* out,
                            char* err, int errlen) {
  return guarded(err, errlen, [&] { *out = streamed_lower_bound(from_c(*t), StreamCount(n), overhead_ms); });
}

int st_overhead_from_measurement(double t_str, double t_non_str, int n, double sum, double* out,
                                 char* err, int errlen) {
  return guarded(err, errlen,
                 [&] { *out = overhead_from_measurement(t_str, t_non_str, StreamCount(n), sum); });
}

int st_overlap_benefit(int n, double sum, double overhead_ms, double* out, char* err, int errlen) {
  return guarded(err, errlen, [&] { *out = overlap_benefit(StreamCount(n), sum, overhead_ms); });
}

int st_predict_sum(const pm_model_bundle* b, uint64_t n, double* out, char* err, int errlen) {
  return guarded(err, errlen, [&] { *out = predict_sum(bundle_from_c(b), n); });
}

int st_predict_overhead(const pm_model_bundle* b, uint64_t n, int streams, double* out, char* err,
                        int errlen) {
  return guarded(err, errlen,
                 [&] { *out = predict_overhead(bundle_from_c(b), n, StreamCount(streams)); });
}

int st_recommend(const pm_model_bundle* b, uint64_t n, int* chosen, double* benefits,
                 double* overheads, double* predicted_sum, int* model_used, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    if (n < 1) throw ValidationError("SLAE size must be at least 1");
    Recommendation r = recommend(bundle_from_c(b), n);
    if (chosen) *chosen = r.chosen.value();
    for (size_t k = 0; k < r.rows.size(); ++k) {
      if (benefits) benefits[k] = r.rows[k].benefit;
      if (overheads) overheads[k] = r.rows[k].predicted_overhead;
    }
    if (predicted_sum && !r.rows.empty()) *predicted_sum = r.rows[0].predicted_sum;
    if (model_used) *model_used = r.model_used == OverheadModel::small ? 0 : 1;
  });
}

int st_recommend_fp32(const pm_model_bundle* b, uint64_t n, int* chosen, char* err, int errlen) {
  return guarded(err, errlen, [&] { *chosen = recommend_fp32(bundle_from_c(b), n).value(); });
}

int st_gomez_luna_optimum(double sum, double tau, double* out, char* err, int errlen) {
  return guarded(err, errlen, [&] { *out = gomez_luna_optimum(sum, tau); });
}

int st_train_test_split(int n, double train_fraction, int shuffle, uint64_t seed, int* order,
                        int* n_train, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    std::vector<Observation> data(n < 0 ? 0 : n);
    for (int k = 0; k < n; ++k) data[k].target = k;  // carry the index
    SplitConfig cfg{train_fraction, shuffle != 0, seed};
    auto split = train_test_split(data, cfg);
    int k = 0;
    for (const auto& o : split.first) order[k++] = (int)o.target;
    for (const auto& o : split.second) order[k++] = (int)o.target;
    *n_train = (int)split.first.size();
  });
}

int st_fit_least_squares(const double* X, const double* y, int rows, int cols, double* beta,
                         char* err, int errlen) {
  return guarded(err, errlen, [&] {
    std::vector<Observation> obs(rows);
    for (int i = 0; i < rows; ++i) {
      obs[i].features.assign(X + (size_t)i * cols, X + (size_t)(i + 1) * cols);
      obs[i].target = y[i];
    }
    std::vector<double> b = fit_least_squares(obs);
    for (int j = 0; j < cols; ++j) beta[j] = b[j];
  });
}

int st_metrics(const double* predicted, const double* actual, int n, double* out, char* err,
               int errlen) {
  return guarded(err, errlen, [&] {
    Metrics m = metrics(std::vector<double>(predicted, predicted + n),
                        std::vector<double>(actual, actual + n));
    out[0] = m.r_squared; out[1] = m.mse; out[2] = m.rmse;
  });
}

int st_fit_model(int kind, const uint64_t* sizes, const int* streams, const double* target,
                 int rows, double train_fraction, int shuffle, uint64_t seed, double* coef,
                 double* met, int* n_train, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    SplitConfig cfg{train_fraction, shuffle != 0, seed};
    FitReport rep;
    if (kind == 0) {
      std::vector<std::pair<uint64_t, double>> r;
      for (int i = 0; i < rows; ++i) r.emplace_back(sizes[i], target[i]);
      rep = fit_sum_model(r, cfg);
    } else {
      std::vector<OverheadRow> r;
      for (int i = 0; i < rows; ++i) r.push_back({sizes[i], streams[i], target[i]});
      rep = (kind == 1) ? fit_overhead_small(r, cfg) : fit_overhead_big(r, cfg);
    }
    for (size_t j = 0; j < rep.coefficients.size(); ++j) coef[j] = rep.coefficients[j];
    const Metrics* ms[2] = {&rep.train, &rep.test};
    for (int s = 0; s < 2; ++s) {
      met[3 * s] = ms[s]->r_squared;
      met[3 * s + 1] = ms[s]->mse;
      met[3 * s + 2] = ms[s]->rmse;
    }
    if (n_train) *n_train = (int)rep.n_train;
  });
}

int st_load_stage_timings(const char* csv, pm_stage_timings* rows, int max_rows, int* n_rows,
                          char* err, int errlen) {
  return guarded(err, errlen, [&] {
    std::istringstream in(csv ? csv : "");
    StageTimingsTable t = load_stage_timings(in);
    *n_rows = (int)t.rows.size();
    for (int k = 0; k < *n_rows && k < max_rows; ++k) {
      const StageTimings& s = t.rows[k];
      rows[k] = pm_stage_timings{s.slae_size, s.t1_h2d, s.t1_comp, s.t1_d2h, s.t2_comp,
                                 s.t3_h2d,    s.t3_comp, s.t3_d2h};
    }
  });
}

int st_load_streamed_runs(const char* csv, uint64_t* sizes, int* streams, double* t_str,
                          int max_rows, int* n_rows, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    std::istringstream in(csv ? csv : "");
    StreamedRunTable t = load_streamed_runs(in);
    *n_rows = (int)t.rows.size();
    for (int k = 0; k < *n_rows && k < max_rows; ++k) {
      sizes[k] = t.rows[k].slae_size;
      streams[k] = t.rows[k].num_streams.value();
      t_str[k] = t.rows[k].t_str;
    }
  });
}

int st_derive_overhead_rows(const char* stage_csv, const char* runs_csv, uint64_t* sizes,
                            int* streams, double* overhead, int max_rows, int* n_rows, char* err,
                            int errlen) {
  return guarded(err, errlen, [&] {
    std::istringstream s1(stage_csv ? stage_csv : ""), s2(runs_csv ? runs_csv : "");
    StageTimingsTable st = load_stage_timings(s1);
    StreamedRunTable rt = load_streamed_runs(s2);
    std::vector<OverheadRow> rows = derive_overhead_rows(st, rt);
    *n_rows = (int)rows.size();
    for (int k = 0; k < *n_rows && k < max_rows; ++k) {
      sizes[k] = rows[k].slae_size;
      streams[k] = rows[k].num_streams;
      overhead[k] = rows[k].overhead_ms;
    }
  });
}

void bundle_to_c(const ModelBundle& b, pm_model_bundle* out) {
  std::memset(out, 0, sizeof(*out));
  out->sum_a = b.sum_a; out->sum_b = b.sum_b;
  out->small_a = b.small_a; out->small_b = b.small_b; out->small_c = b.small_c;
  out->big_a = b.big_a; out->big_b = b.big_b; out->big_c = b.big_c;
  out->size_threshold = b.size_threshold;
  out->num_candidates = (int32_t)std::min<size_t>(b.candidates.size(), 5);
  for (int k = 0; k < out->num_candidates; ++k) out->candidates[k] = b.candidates[k].value();
}

static int fit_bundle_c(const char* stage_csv, const char* runs_csv, uint64_t size_threshold,
                        uint64_t seed, bool anchored, pm_model_bundle* out, double* met, char* err,
                        int errlen) {
  return guarded(err, errlen, [&] {
    std::istringstream s1(stage_csv ? stage_csv : ""), s2(runs_csv ? runs_csv : "");
    StageTimingsTable st = load_stage_timings(s1);
    StreamedRunTable rt = load_streamed_runs(s2);
    BundleFit f = fit_bundle(st, rt, size_threshold, seed, anchored);
    bundle_to_c(f.bundle, out);
    if (met) {
      const FitReport* reps[3] = {&f.sum, &f.small, &f.big};
      for (int r = 0; r < 3; ++r) {
        const Metrics* ms[2] = {&reps[r]->train, &reps[r]->test};
        for (int s = 0; s < 2; ++s) {
          met[6 * r + 3 * s] = ms[s]->r_squared;
          met[6 * r + 3 * s + 1] = ms[s]->mse;
          met[6 * r + 3 * s + 2] = ms[s]->rmse;
        }
      }
    }
  });
}

int st_fit_bundle(const char* stage_csv, const char* runs_csv, uint64_t size_threshold,
                  uint64_t seed, pm_model_bundle* out, double* met, char* err, int errlen) {
  return fit_bundle_c(stage_csv, runs_csv, size_threshold, seed, false, out, met, err, errlen);
}

int st_fit_bundle_anchored(const char* stage_csv, const char* runs_csv, uint64_t size_threshold,
                           uint64_t seed, pm_model_bundle* out, double* met, char* err, int errlen) {
  return fit_bundle_c(stage_csv, runs_csv, size_threshold, seed, true, out, met, err, errlen);
}

static PipelineSpec spec_from_c(const double* stages, int n, double tau_ms, int hw_queues) {
  if (!stages) throw ValidationError("null stage durations");
  PipelineSpec p;
  p.stage1 = StageSpec{stages[0], stages[1], stages[2]};
  p.cpu_ms = stages[3];
  p.stage3 = StageSpec{stages[4], stages[5], stages[6]};
  p.num_streams = StreamCount(n);
  p.tau_ms = tau_ms;
  p.hw_queues = hw_queues;
  return p;
}

int st_simulate(const double* stages, int n, double tau_ms, int hw_queues, double* out,
                double* trace, int max_events, int* n_events, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    SimResult r = simulate(spec_from_c(stages, n, tau_ms, hw_queues));
    if (out) {
      out[0] = r.total_ms;
      out[1] = r.stage1_makespan_ms;
      out[2] = r.stage3_makespan_ms;
    }
    if (n_events) *n_events = (int)r.trace.size();
    if (trace)
      for (int k = 0; k < (int)r.trace.size() && k < max_events; ++k) {
        const TraceEvent& e = r.trace[k];
        double* row = trace + 5 * (size_t)k;
        row[0] = (double)static_cast<int>(e.engine);
        row[1] = e.stream;
        row[2] = e.stage;
        row[3] = e.start_ms;
        row[4] = e.end_ms;
      }
  });
}

int st_verify_lower_bound(const double* stages, int n, double tau_ms, int* holds, int* dominance,
                          char* err, int errlen) {
  return guarded(err, errlen, [&] {
    const PipelineSpec p = spec_from_c(stages, n, tau_ms, 32);
    if (holds) *holds = verify_lower_bound(p) ? 1 : 0;
    if (dominance) *dominance = dominance_holds(p) ? 1 : 0;
  });
}

static int copy_out(const std::string& s, char* out, int outlen, int* needed) {
  if (needed) *needed = (int)s.size() + 1;
  if (!out || outlen < (int)s.size() + 1) return 0;
  std::memcpy(out, s.c_str(), s.size() + 1);
  return 1;
}

int st_bundle_to_json(const pm_model_bundle* b, char* out, int outlen, int* needed, char* err,
                      int errlen) {
  return guarded(err, errlen, [&] {
    if (!copy_out(bundle_to_document(bundle_from_c(b)), out, outlen, needed))
      throw ValidationError("output buffer too small");
  });
}

int st_bundle_from_json(const char* doc, pm_model_bundle* out, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    if (!doc || !out) throw ValidationError("null argument");
    bundle_to_c(bundle_from_document(doc), out);
  });
}

int st_report_table(const pm_model_bundle* b, const char* table, int* passed, int* failed,
                    int* known, double* cells, int max_cells, int* n_cells, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    TableReport r = report_table(bundle_from_c(b), table ? table : "");
    if (passed) *passed = r.passed;
    if (failed) *failed = r.failed;
    if (known) *known = r.known;
    if (n_cells) *n_cells = (int)r.cells.size();
    if (cells)
      for (int k = 0; k < (int)r.cells.size() && k < max_cells; ++k) {
        double* row = cells + 4 * (size_t)k;
        row[0] = r.cells[k].expected;
        row[1] = r.cells[k].got;
        row[2] = r.cells[k].tolerance;
        row[3] = (double)static_cast<int>(r.cells[k].status);
      }
  });
}

int st_dump_reference(const char* table, char* out, int outlen, int* needed, char* err,
                      int errlen) {
  return guarded(err, errlen, [&] {
    if (!copy_out(dump_reference(table ? table : ""), out, outlen, needed))
      throw ValidationError("output buffer too small");
  });
}

}  // extern "C"
