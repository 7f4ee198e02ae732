// streamtune/dataset.hpp -- measured timing tables and the Eq. 5 batch step.
//
// Follows /root/reference/SPEC.md:326-398 (module "dataset"):
// load_stage_timings (:347), load_streamed_runs (:357), derive_overhead_rows
// (:367), ReferenceData (:341-344).  CSV schemas:
//   slae_size,t1_h2d,t1_comp,t1_d2h,t2_comp,t3_h2d,t3_comp,t3_d2h
//   slae_size,num_streams,t_str
// The B200 C2 sweep (tools/refit.py) writes exactly these two files.
#pragma once

#include <cstdint>
#include <istream>
#include <ostream>
#include <string>
#include <vector>

#include "streamtune/regression.hpp"
#include "streamtune/timing_model.hpp"

namespace streamtune {

struct StageTimingsTable {
  std::vector<StageTimings> rows;  // unique slae_size, increasing
  const StageTimings* find(std::uint64_t slae_size) const;
};

struct StreamedRunTable {
  std::vector<StreamedRun> rows;  // unique (slae_size, num_streams)
};

// Throws MalformedRowError (line, column), DuplicateSizeError,
// NegativeDurationError (line, column).
StageTimingsTable load_stage_timings(std::istream& in);
// Throws InvalidStreamCountError, MalformedRowError, DuplicateSizeError(size, n).
StreamedRunTable load_streamed_runs(std::istream& in);

void save_stage_timings(std::ostream& out, const StageTimingsTable& t);
void save_streamed_runs(std::ostream& out, const StreamedRunTable& t);

// Eq. 5 for every run with n >= 2 (n = 1 runs calibrate T_non_str only).
// Throws MissingStageTimingsError naming the size.
std::vector<OverheadRow> derive_overhead_rows(const StageTimingsTable& stage,
                                              const StreamedRunTable& runs);

// Paper tables transcribed from /root/reference/PAPER.md.
struct ReferenceData {
  struct Table1Row {
    std::uint64_t size;
    double t1_comp, t1_d2h, t3_h2d, t3_comp, sum, gomez_luna, actual;
  };
  struct Table2Row {  // PAPER.md:152-160 (size 1e6)
    int n;
    double t_str, t_non_str, sum, overhead, benefit;
  };
  struct Table4Row {
    std::uint64_t size;
    int n_act, n_pre;
  };
  struct Table5Row {  // PAPER.md:256-272 (size 0 encodes "<= 1e5")
    std::uint64_t size;
    int fp32, fp64;
    bool half;
  };
  static const std::vector<Table1Row>& table1();
  static const std::vector<Table2Row>& table2();
  static const std::vector<Table4Row>& table4();
  static const std::vector<Table5Row>& table5();
  static constexpr double tau_ms = 0.004448;
};

}  // namespace streamtune
