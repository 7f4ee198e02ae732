// streamtune/predictor.hpp -- stream-count recommendation from fitted models.
//
// Follows the reference spec /root/reference/SPEC.md:227-324 (module
// "predictor"): ModelBundle, Recommendation (:239-244),
// predict_sum (Eq. 4, :247), predict_overhead (Eq. 7, :257), recommend
// (Eq. 6 argmax, :267), recommend_fp32 (:278), gomez_luna_optimum (:288).
// The solver (include/pm_tridiag.h) calls recommend() when the caller passes
// num_streams = 0.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "streamtune/timing_model.hpp"

namespace streamtune {

// Coefficients of Eq. 4 (sum model) and the two Eq. 7 overhead models.
struct ModelBundle {
  double sum_a = 0.0, sum_b = 0.0;                    // sum = a*N + b
  double small_a = 0.0, small_b = 0.0, small_c = 0.0;  // a*N + b*log10(n) + c     (N <= thr)
  double big_a = 0.0, big_b = 0.0, big_c = 0.0;        // (a*N + b)*log2(n^(4/3)) + c (N > thr)
  std::uint64_t size_threshold = 1000000;             // inclusive on the small side
  std::vector<StreamCount> candidates{StreamCount(2), StreamCount(4), StreamCount(8),
                                      StreamCount(16), StreamCount(32)};
  // provenance (optional)
  std::string fitted_on;
  std::uint64_t seed = 42;

  // candidates strictly increasing, none equal to 1, threshold >= 1.
  void validate() const;

  // The RTX 2080 Ti bundle published in the paper: Eq. 4 and
  // Eq. 7.
  static ModelBundle paper();

  // The same model forms re-fitted on an NVIDIA B200 with this solver
  // (tools/refit.py, data in refit/pooled/): the C ABI's default bundle.
  static ModelBundle b200();
};

enum class OverheadModel { small, big };

struct BenefitRow {
  StreamCount n;
  double predicted_sum;
  double predicted_overhead;
  double benefit;
};

struct Recommendation {
  std::uint64_t slae_size = 0;
  StreamCount chosen{1};
  std::vector<BenefitRow> rows;
  OverheadModel model_used = OverheadModel::small;
};

// Eq. 4
double predict_sum(const ModelBundle& bundle, std::uint64_t slae_size);
// Eq. 7 (small for N <= size_threshold, else big)
double predict_overhead(const ModelBundle& bundle, std::uint64_t slae_size, StreamCount n);
// Eq. 6: argmax over candidates with benefit > 0; ties -> smaller n; none -> 1.
Recommendation recommend(const ModelBundle& bundle, std::uint64_t slae_size);
// PAPER.md:245 "divide the optimum number of streams by two" (floor at 1).
StreamCount recommend_fp32(const ModelBundle& bundle, std::uint64_t slae_size);
// Gomez-Luna: stationary point of sum/n + n*tau, i.e. sqrt(sum/tau).
// Throws NonpositiveTauError for tau <= 0.
double gomez_luna_optimum(double sum, double tau);

}  // namespace streamtune
