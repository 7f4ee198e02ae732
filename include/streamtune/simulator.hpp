// streamtune/simulator.hpp -- discrete-event model of the copy/compute pipeline.
//
// Follows /root/reference/SPEC.md:400-459 (module "simulator"): one H2D, one
// compute and one D2H engine per GPU; every GPU stage is split into
// num_streams equal chunks that flow H2D -> COMP -> D2H in stream order
// (per-stream FIFO, per-engine serial, unbounded buffering between engines);
// Stage 2 (the CPU solve in the paper) never overlaps a GPU
// stage; stream creation costs tau per stream.
//   total = stage1_makespan + cpu_ms + stage3_makespan + num_streams * tau
// It is the idealised model that certifies Eq. 2 (streamed_lower_bound,
// timing_model.hpp:129) as a lower bound (verify_lower_bound).
//
// On B200 the solver measures t1_d2h = t3_h2d = 0 and t2_comp = the GPU
// reduced solve; the simulator accepts those records as is.
#pragma once

#include <cstdint>
#include <ostream>
#include <string>
#include <vector>

#include "streamtune/timing_model.hpp"

namespace streamtune {

struct StageSpec {
  double h2d_ms = 0.0;
  double comp_ms = 0.0;
  double d2h_ms = 0.0;
};

// SPEC.md:407-410
struct PipelineSpec {
  StageSpec stage1;
  double cpu_ms = 0.0;
  StageSpec stage3;
  StreamCount num_streams{1};
  double tau_ms = 0.0;  // per-stream creation overhead
  int hw_queues = 32;   // Hyper-Q queues; inert for num_streams <= 32

  // Throws NegativeDurationError / ValidationError (non-finite, hw_queues < 1).
  void validate() const;
  // The StageTimings record Eq. 1/2 see for this spec (t2_comp = cpu_ms).
  StageTimings timings(std::uint64_t slae_size = 1) const;
  static PipelineSpec from_timings(const StageTimings& t, StreamCount n, double tau_ms);
};

enum class Engine { h2d = 0, comp = 1, d2h = 2 };
const char* engine_name(Engine e);

struct TraceEvent {
  Engine engine;
  int stream;  // 0-based stream (= chunk) index
  int stage;   // 1 or 3
  double start_ms;
  double end_ms;
};

// SPEC.md:412-415
struct SimResult {
  double total_ms = 0.0;
  double stage1_makespan_ms = 0.0;
  double stage3_makespan_ms = 0.0;
  std::vector<TraceEvent> trace;
};

// SPEC.md:418-427.  Stream creation (num_streams * tau) is placed first on the
// timeline, then Stage 1, the CPU Stage 2, Stage 3.
SimResult simulate(const PipelineSpec& spec);

// The closed form of one stage's makespan, (h+c+d)/n + (n-1) max(h,c,d)/n
// (SPEC.md:419), for cross-checks.
double stage_makespan_closed_form(const StageSpec& s, int n);

// simulate(spec).total >= streamed_lower_bound(t, n, n*tau) - 1e-9.
bool verify_lower_bound(const PipelineSpec& spec);

// True iff the paper's dominance regime holds (Stage 1 max is H2D, Stage 3
// max is D2H), i.e. Eq. 2 is exact.
bool dominance_holds(const PipelineSpec& spec);

// Trace export, header engine,stream,start_ms,end_ms.
void write_trace_csv(std::ostream& out, const SimResult& r);

}  // namespace streamtune
