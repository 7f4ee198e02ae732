// streamtune/regression.hpp -- OLS fits of the paper's Eq. 4 / Eq. 7 forms.
//
// Follows /root/reference/SPEC.md:120-225 (module "regression"):
// train_test_split (:141), fit_least_squares (:151), fit_sum_model (:161),
// fit_overhead_small (:171), fit_overhead_big (:181), metrics (:191).
// Design decisions from SPEC.md:207-211: 3:1 split = train_fraction 0.75,
// exact least squares on transformed features, default seed 42, split size
// rounded half away from zero then clamped so both splits are non-empty.
// Used by the B200 re-fit (tools/refit.py -> pm_fit_bundle).
#pragma once

#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include "streamtune/errors.hpp"

namespace streamtune {

struct Observation {
  std::vector<double> features;
  double target = 0.0;
};

struct SplitConfig {
  double train_fraction = 0.75;
  bool shuffle = true;
  std::uint64_t seed = 42;
};

struct Metrics {
  double r_squared = 0.0, mse = 0.0, rmse = 0.0;
};

struct FitReport {
  std::vector<std::string> names;
  std::vector<double> coefficients;
  Metrics train, test;
  std::size_t n_train = 0, n_test = 0;
  std::uint64_t seed = 42;
};

// Deterministic for a fixed seed; |train| = round(f*|data|) clamped to
// [1, |data|-1].  Throws TooFewObservationsError for |data| < 4.
std::pair<std::vector<Observation>, std::vector<Observation>> train_test_split(
    const std::vector<Observation>& data, const SplitConfig& cfg);

// Minimises ||X beta - y||_2 (column-scaled Householder QR).
// Throws TooFewObservationsError (rows < cols) or RankDeficiencyError
// (smallest |R_ii| < 1e-10 * largest after column scaling).
std::vector<double> fit_least_squares(const std::vector<Observation>& obs);

// Throws ZeroVarianceError when `actual` is constant; ValidationError on
// length mismatch / empty input.
Metrics metrics(const std::vector<double>& predicted, const std::vector<double>& actual);

// rows: (slae_size, sum_ms) -> features [N, 1]
FitReport fit_sum_model(const std::vector<std::pair<std::uint64_t, double>>& rows,
                        const SplitConfig& cfg);

struct OverheadRow {
  std::uint64_t slae_size;
  int num_streams;
  double overhead_ms;
};
// features [N, log10 n, 1]
FitReport fit_overhead_small(const std::vector<OverheadRow>& rows, const SplitConfig& cfg);
// features [N*(4/3)log2 n, (4/3)log2 n, 1]
FitReport fit_overhead_big(const std::vector<OverheadRow>& rows, const SplitConfig& cfg);

// B200 addition (not in the SPEC, whose fits are plain OLS): the same two
// forms constrained so that T_overhead(N, n = 1) = 0 and every coefficient is
// >= 0 -- small: a = c = 0, b >= 0; big: c = 0, a, b >= 0 (exhaustive
// active-set least squares).  On B200 the overlappable work is ~1 % of the
// transfers and per-stream costs are tens of microseconds, so unconstrained
// OLS fits a negative overhead at n = 2 and predicts streaming everywhere
// (DESIGN.md §5).  Same split, seed and metrics as the OLS fits.
FitReport fit_overhead_small_anchored(const std::vector<OverheadRow>& rows, const SplitConfig& cfg);
FitReport fit_overhead_big_anchored(const std::vector<OverheadRow>& rows, const SplitConfig& cfg);

}  // namespace streamtune
