// oracle/ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" shim over the REFERENCE's own header-only timing model, compiled
// straight from /root/reference/proj/include (never copied) into
// oracle/_ref/libstreamtune_ref.so by oracle/Makefile.  tests/ call it to pin
// the repo's re-implementation (include/streamtune/timing_model.hpp) to the
// reference bit for bit.  Functions mirror timing_model.hpp:40-146.
#include <cstring>
#include <string>

#include "streamtune/timing_model.hpp"

using namespace streamtune;

namespace {
StageTimings mk(const double* t, unsigned long long size) {
  StageTimings s;
  s.slae_size = size;
  s.t1_h2d = t[0]; s.t1_comp = t[1]; s.t1_d2h = t[2]; s.t2_comp = t[3];
  s.t3_h2d = t[4]; s.t3_comp = t[5]; s.t3_d2h = t[6];
  return s;
}
void put(char* err, int len, const char* msg) {
  if (err && len > 0) { std::strncpy(err, msg, len - 1); err[len - 1] = 0; }
}
}  // namespace

extern "C" {
int ref_stream_count_is_valid(int n) { return StreamCount::is_valid(n) ? 1 : 0; }
double ref_total_unstreamed(const double* t) { return total_unstreamed(mk(t, 1)); }
double ref_overlap_sum(const double* t) { return overlap_sum(mk(t, 1)); }
int ref_streamed_lower_bound(const double* t, int n, double ovh, double* out) {
  try { *out = streamed_lower_bound(mk(t, 1), StreamCount(n), ovh); return 0; }
  catch (const ValidationError&) { return 1; }
}
int ref_overhead_from_measurement(double t_str, double t_non, int n, double sum, double* out) {
  try { *out = overhead_from_measurement(t_str, t_non, StreamCount(n), sum); return 0; }
  catch (const ValidationError&) { return 1; }
}
int ref_overlap_benefit(int n, double sum, double ovh, double* out) {
  try { *out = overlap_benefit(StreamCount(n), sum, ovh); return 0; }
  catch (const ValidationError&) { return 1; }
}
// 0 ok, 1 ValidationError, 3 NegativeDurationError (a ValidationError)
int ref_validate_stage_timings(const double* t, unsigned long long size, char* err, int len) {
  try { mk(t, size).validate(); return 0; }
  catch (const NegativeDurationError& e) { put(err, len, e.what()); return 3; }
  catch (const ValidationError& e) { put(err, len, e.what()); return 1; }
}
int ref_streamed_run_validate(unsigned long long size, int n, double t_str, char* err, int len) {
  try { StreamedRun r{size, StreamCount(n), t_str}; r.validate(); return 0; }
  catch (const NegativeDurationError& e) { put(err, len, e.what()); return 3; }
  catch (const InvalidStreamCountError& e) { put(err, len, e.what()); return 4; }
  catch (const ValidationError& e) { put(err, len, e.what()); return 1; }
}
}
