// examples/cpp_caller.cpp -- a C++20 caller written against the reference's
// streamtune API (timing_model.hpp / errors.hpp names) plus the solver's C ABI.
// Build:  g++ -std=c++20 examples/cpp_caller.cpp -Iinclude
//             -Lpaper_2501_05938_b200 -lpm_tridiag -Wl,-rpath,$PWD/paper_2501_05938_b200
// Run with --solve on a machine with a CUDA GPU.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include "pm_tridiag.h"
#include "streamtune/bundle_io.hpp"
#include "streamtune/dataset.hpp"
#include "streamtune/errors.hpp"
#include "streamtune/predictor.hpp"
#include "streamtune/simulator.hpp"
#include "streamtune/timing_model.hpp"

int main(int argc, char** argv) {
  using namespace streamtune;
  // --- reference API, unchanged call sites (timing_model.hpp:40-146) -------
  StageTimings t;
  t.slae_size = 1000000;
  t.t1_h2d = 4.85; t.t1_comp = 0.6; t.t1_d2h = 0.9; t.t2_comp = 0.32;
  t.t3_h2d = 0.233568; t.t3_comp = 0.7; t.t3_d2h = 1.213872;
  t.validate();
  const double sum = overlap_sum(t);
  const double ovh = overhead_from_measurement(7.401472, total_unstreamed(t), StreamCount(8), sum);
  std::printf("T_non_str %.6f  sum %.6f  T_overhead(8) %.6f  benefit(8) %.6f\n",
              total_unstreamed(t), sum, ovh, overlap_benefit(StreamCount(8), sum, ovh));
  try {
    StreamCount bad(3);
    (void)bad;
  } catch (const InvalidStreamCountError& e) {
    std::printf("caught InvalidStreamCountError(%d): %s\n", e.count(), e.what());
  }
  // --- SPEC modules (predictor) ------------------------------------------------
  const Recommendation r = recommend(ModelBundle::paper(), 1000000);
  std::printf("paper bundle: N=1e6 -> %d streams; B200 bundle: N=8e7 -> %d streams\n",
              r.chosen.value(), recommend(ModelBundle::b200(), 80000000).chosen.value());
  // --- simulator, model document, report harness ---------------
  PipelineSpec p = PipelineSpec::from_timings(t, StreamCount(8), 0.004448);
  const SimResult sr = simulate(p);
  std::printf("simulated T_str(8) %.6f ms, Eq. 2 bound holds: %s\n", sr.total_ms,
              verify_lower_bound(p) ? "yes" : "no");
  const ModelBundle back = bundle_from_document(bundle_to_document(ModelBundle::b200()));
  const TableReport t4 = report_table(ModelBundle::paper(), "table4");
  std::printf("bundle round trip exact: %s; Table 4: %d PASS, %d FAIL, %d KNOWN\n",
              back.sum_a == ModelBundle::b200().sum_a ? "yes" : "no", t4.passed, t4.failed, t4.known);
  // --- solver C ABI --------------------------------------------------------------
  if (argc > 1 && std::strcmp(argv[1], "--solve") == 0) {
    const int64_t n = 1000003;
    std::vector<double> a(n), b(n), c(n), d(n), x(n);
    for (int64_t i = 0; i < n; ++i) {
      a[i] = (i % 7) * 0.1 - 0.3;
      c[i] = (i % 5) * 0.1 - 0.2;
      b[i] = 2.0 + std::fabs(a[i]) + std::fabs(c[i]);
      d[i] = std::sin(0.001 * i);
    }
    pm_handle_t h;
    if (pm_create(&h, 0) != PM_OK) { std::printf("no GPU\n"); return 1; }
    int st = pm_solve_host_f64(h, a.data(), b.data(), c.data(), d.data(), x.data(), n, 10, 0);
    if (st != PM_OK) { std::printf("solve failed (%d): %s\n", st, pm_last_error(h)); return 1; }
    double res = 0.0, nd = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      double ri = b[i] * x[i] - d[i];
      if (i > 0) ri += a[i] * x[i - 1];
      if (i < n - 1) ri += c[i] * x[i + 1];
      res += ri * ri;
      nd += d[i] * d[i];
    }
    pm_stage_timings tm;
    double total = 0;
    int32_t used = 0;
    pm_last_stage_timings(h, &tm, &total, &used);
    std::printf("solved n=%lld with %d streams in %.3f ms, residual %.3e\n", (long long)n, used,
                total, std::sqrt(res / nd));
    // the FP32 twin and a batch of 3 copies from host memory
    std::vector<float> a32(a.begin(), a.end()), b32(b.begin(), b.end()), c32(c.begin(), c.end()),
        d32(d.begin(), d.end()), x32(n);
    st = pm_solve_host_f32(h, a32.data(), b32.data(), c32.data(), d32.data(), x32.data(), n, 10, 0);
    double err32 = 0.0, nx = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      err32 = std::fmax(err32, std::fabs(x32[i] - x[i]));
      nx = std::fmax(nx, std::fabs(x[i]));
    }
    std::vector<double> ab, bb, cb, db, xb(3 * n);
    for (int k = 0; k < 3; ++k) {
      ab.insert(ab.end(), a.begin(), a.end()); bb.insert(bb.end(), b.begin(), b.end());
      cb.insert(cb.end(), c.begin(), c.end()); db.insert(db.end(), d.begin(), d.end());
    }
    const int stb = pm_solve_batch_host_f64(h, ab.data(), bb.data(), cb.data(), db.data(), xb.data(), n,
                                            3, 10, 0, 0);
    double errb = 0.0;
    for (int64_t i = 0; i < 3 * n; ++i) errb = std::fmax(errb, std::fabs(xb[i] - x[i % n]));
    std::printf("fp32 status %d rel err %.2e; batch status %d max diff %.2e\n", st, err32 / nx, stb, errb);
    pm_destroy(h);
  }
  return 0;
}
