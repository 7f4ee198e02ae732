// Stream-count predictor: SPEC.md:227-324 (see include/streamtune/predictor.hpp).
#include "streamtune/predictor.hpp"

#include <cmath>

namespace streamtune {

void ModelBundle::validate() const {
  if (size_threshold < 1) throw ValidationError("size_threshold must be at least 1");
  if (candidates.empty()) throw ValidationError("candidate list is empty");
  int prev = 1;
  for (const StreamCount& n : candidates) {
    if (n.value() <= prev)
      throw ValidationError("candidates must be strictly increasing and exclude 1");
    prev = n.value();
  }
  const double coeffs[] = {sum_a, sum_b, small_a, small_b, small_c, big_a, big_b, big_c};
  for (double v : coeffs)
    if (!std::isfinite(v)) throw ValidationError("non-finite model coefficient");
}

ModelBundle ModelBundle::paper() {
  ModelBundle b;
  b.sum_a = 0.0000021890017149;
  b.sum_b = 0.1470644998564126;
  b.small_a = 0.0000002245645331;
  b.small_b = 0.6009426920043296;
  b.small_c = -0.0605183610625299;
  b.big_a = 0.0000000356594859;
  b.big_b = 0.0522781620855163;
  b.big_c = 0.3941472844770443;
  b.size_threshold = 1000000;
  b.fitted_on = "RTX 2080 Ti (Veneva & Imamura, arXiv 2501.05938, Eq. 4 / Eq. 7)";
  return b;
}

ModelBundle ModelBundle::b200() {
  ModelBundle b;
#include "b200_bundle.inc"
  b.fitted_on = "NVIDIA B200 re-fit (tools/refit.py; refit/pooled/)";
  return b;
}

double predict_sum(const ModelBundle& bundle, std::uint64_t slae_size) {
  return bundle.sum_a * static_cast<double>(slae_size) + bundle.sum_b;
}

double predict_overhead(const ModelBundle& bundle, std::uint64_t slae_size, StreamCount n) {
  const double size = static_cast<double>(slae_size);
  const double k = static_cast<double>(n.value());
  if (slae_size <= bundle.size_threshold)
    return bundle.small_a * size + bundle.small_b * std::log10(k) + bundle.small_c;
  const double log_term = (4.0 / 3.0) * std::log2(k);  // log2(n^(4/3))
  return (bundle.big_a * size + bundle.big_b) * log_term + bundle.big_c;
}

Recommendation recommend(const ModelBundle& bundle, std::uint64_t slae_size) {
  Recommendation rec;
  rec.slae_size = slae_size;
  rec.model_used =
      slae_size <= bundle.size_threshold ? OverheadModel::small : OverheadModel::big;
  const double sum = predict_sum(bundle, slae_size);
  double best = 0.0;
  bool any = false;
  for (const StreamCount& n : bundle.candidates) {
    const double ovh = predict_overhead(bundle, slae_size, n);
    const double ben = overlap_benefit(n, sum, ovh);
    rec.rows.push_back(BenefitRow{n, sum, ovh, ben});
    // strict '>' while scanning in increasing n: ties go to the smaller n
    if (ben > 0.0 && (!any || ben > best)) {
      best = ben;
      rec.chosen = n;
      any = true;
    }
  }
  if (!any) rec.chosen = StreamCount(1);
  return rec;
}

StreamCount recommend_fp32(const ModelBundle& bundle, std::uint64_t slae_size) {
  const int fp64 = recommend(bundle, slae_size).chosen.value();
  return StreamCount(fp64 >= 2 ? fp64 / 2 : 1);
}

double gomez_luna_optimum(double sum, double tau) {
  if (!(tau > 0.0)) throw NonpositiveTauError("tau must be positive");
  return std::sqrt(sum / tau);
}

}  // namespace streamtune
