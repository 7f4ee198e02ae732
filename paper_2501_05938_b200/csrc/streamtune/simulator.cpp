// simulator.cpp -- discrete-event model of the streamed partition-method
// pipeline; see streamtune/simulator.hpp.
#include "streamtune/simulator.hpp"

#include <algorithm>
#include <cmath>
#include <iomanip>

namespace streamtune {

namespace {

void check_duration(double v, const char* name) {
  if (!std::isfinite(v)) throw ValidationError(std::string("non-finite duration '") + name + "'");
  if (v < 0.0) throw NegativeDurationError(name);
}

// One GPU stage: n equal chunks through the three engines, chunk k on stream
// k (queue k mod hw_queues).  Engines run one chunk at a time in issue order;
// a chunk's copy-in, kernel and copy-out are ordered within its stream, and
// work of two streams that share a hardware queue is serialised.
double run_stage(const StageSpec& s, int n, int hw_queues, int stage, double t0,
                 std::vector<TraceEvent>& trace) {
  const double dur[3] = {s.h2d_ms / n, s.comp_ms / n, s.d2h_ms / n};
  double engine_free[3] = {t0, t0, t0};
  std::vector<double> queue_free((size_t)std::min(n, hw_queues), t0);
  double end = t0;
  for (int k = 0; k < n; ++k) {
    double& q = queue_free[(size_t)(k % hw_queues)];
    double ready = q;  // FIFO within the stream / queue
    for (int e = 0; e < 3; ++e) {
      const double start = std::max(engine_free[e], ready);
      const double stop = start + dur[e];
      engine_free[e] = stop;
      ready = stop;
      trace.push_back(TraceEvent{static_cast<Engine>(e), k, stage, start, stop});
    }
    q = ready;
    end = std::max(end, ready);
  }
  return end - t0;
}

}  // namespace

void PipelineSpec::validate() const {
  check_duration(stage1.h2d_ms, "stage1.h2d_ms");
  check_duration(stage1.comp_ms, "stage1.comp_ms");
  check_duration(stage1.d2h_ms, "stage1.d2h_ms");
  check_duration(cpu_ms, "cpu_ms");
  check_duration(stage3.h2d_ms, "stage3.h2d_ms");
  check_duration(stage3.comp_ms, "stage3.comp_ms");
  check_duration(stage3.d2h_ms, "stage3.d2h_ms");
  check_duration(tau_ms, "tau_ms");
  if (hw_queues < 1) throw ValidationError("hw_queues must be positive");
}

StageTimings PipelineSpec::timings(std::uint64_t slae_size) const {
  StageTimings t;
  t.slae_size = slae_size;
  t.t1_h2d = stage1.h2d_ms;
  t.t1_comp = stage1.comp_ms;
  t.t1_d2h = stage1.d2h_ms;
  t.t2_comp = cpu_ms;
  t.t3_h2d = stage3.h2d_ms;
  t.t3_comp = stage3.comp_ms;
  t.t3_d2h = stage3.d2h_ms;
  return t;
}

PipelineSpec PipelineSpec::from_timings(const StageTimings& t, StreamCount n, double tau_ms) {
  PipelineSpec s;
  s.stage1 = StageSpec{t.t1_h2d, t.t1_comp, t.t1_d2h};
  s.cpu_ms = t.t2_comp;
  s.stage3 = StageSpec{t.t3_h2d, t.t3_comp, t.t3_d2h};
  s.num_streams = n;
  s.tau_ms = tau_ms;
  return s;
}

const char* engine_name(Engine e) {
  switch (e) {
    case Engine::h2d: return "h2d";
    case Engine::comp: return "comp";
    default: return "d2h";
  }
}

SimResult simulate(const PipelineSpec& spec) {
  spec.validate();
  const int n = spec.num_streams.value();
  SimResult r;
  r.trace.reserve((size_t)6 * n);
  const double create = n * spec.tau_ms;
  r.stage1_makespan_ms = run_stage(spec.stage1, n, spec.hw_queues, 1, create, r.trace);
  const double t3 = create + r.stage1_makespan_ms + spec.cpu_ms;
  r.stage3_makespan_ms = run_stage(spec.stage3, n, spec.hw_queues, 3, t3, r.trace);
  r.total_ms = r.stage1_makespan_ms + spec.cpu_ms + r.stage3_makespan_ms + create;
  return r;
}

double stage_makespan_closed_form(const StageSpec& s, int n) {
  const double mx = std::max(s.h2d_ms, std::max(s.comp_ms, s.d2h_ms));
  return (s.h2d_ms + s.comp_ms + s.d2h_ms) / n + (n - 1) * mx / n;
}

bool verify_lower_bound(const PipelineSpec& spec) {
  const SimResult r = simulate(spec);
  const int n = spec.num_streams.value();
  const double bound = streamed_lower_bound(spec.timings(), spec.num_streams, n * spec.tau_ms);
  return r.total_ms >= bound - 1e-9;
}

bool dominance_holds(const PipelineSpec& spec) {
  const StageSpec& a = spec.stage1;
  const StageSpec& b = spec.stage3;
  return a.h2d_ms >= a.comp_ms && a.h2d_ms >= a.d2h_ms && b.d2h_ms >= b.h2d_ms &&
         b.d2h_ms >= b.comp_ms;
}

void write_trace_csv(std::ostream& out, const SimResult& r) {
  out << "engine,stream,start_ms,end_ms\n";
  const auto old = out.precision(17);
  for (const TraceEvent& e : r.trace)
    out << engine_name(e.engine) << ',' << e.stream << ',' << e.start_ms << ',' << e.end_ms << '\n';
  out.precision(old);
}

}  // namespace streamtune
