// OLS regression and the paper's train/test protocol: SPEC.md:120-225.
#include "streamtune/regression.hpp"

#include <algorithm>
#include <cmath>
#include <numeric>

namespace streamtune {
namespace {

std::uint64_t mix64(std::uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// Fisher-Yates driven only by `seed` (never a global generator).
std::vector<std::size_t> permutation(std::size_t n, std::uint64_t seed) {
  std::vector<std::size_t> p(n);
  std::iota(p.begin(), p.end(), std::size_t{0});
  std::uint64_t state = seed;
  for (std::size_t i = n; i > 1; --i) {
    state = mix64(state);
    const std::size_t j = static_cast<std::size_t>(state % i);
    std::swap(p[i - 1], p[j]);
  }
  return p;
}

double round_half_away(double v) { return v < 0 ? -std::floor(-v + 0.5) : std::floor(v + 0.5); }

// Metrics that tolerate an undefined R^2 (reported as NaN) inside a FitReport.
Metrics report_metrics(const std::vector<double>& beta, const std::vector<Observation>& obs) {
  Metrics m{std::nan(""), std::nan(""), std::nan("")};
  if (obs.empty()) return m;
  std::vector<double> pred, act;
  for (const Observation& o : obs) {
    double p = 0.0;
    for (std::size_t k = 0; k < beta.size(); ++k) p += beta[k] * o.features[k];
    pred.push_back(p);
    act.push_back(o.target);
  }
  try {
    return metrics(pred, act);
  } catch (const ZeroVarianceError&) {
    double ss = 0.0;
    for (std::size_t i = 0; i < pred.size(); ++i) ss += (pred[i] - act[i]) * (pred[i] - act[i]);
    m.mse = ss / static_cast<double>(pred.size());
    m.rmse = std::sqrt(m.mse);
    return m;
  }
}

FitReport fit_with_split(const std::vector<Observation>& data, const SplitConfig& cfg,
                         std::vector<std::string> names) {
  auto split = train_test_split(data, cfg);
  FitReport rep;
  rep.names = std::move(names);
  rep.coefficients = fit_least_squares(split.first);
  rep.train = report_metrics(rep.coefficients, split.first);
  rep.test = report_metrics(rep.coefficients, split.second);
  rep.n_train = split.first.size();
  rep.n_test = split.second.size();
  rep.seed = cfg.seed;
  return rep;
}

// Least squares with every coefficient >= 0 and only the features in
// `allowed` free (the others fixed at 0): the minimum over the feasible
// subsets of the allowed features (<= 3 of them here, so exhaustive).
std::vector<double> fit_nonneg_subset(const std::vector<Observation>& obs, const std::vector<std::size_t>& allowed,
                                      std::size_t p) {
  std::vector<double> best(p, 0.0);
  double best_ss = 0.0;
  for (const Observation& o : obs) best_ss += o.target * o.target;  // the all-zero model
  const std::size_t k = allowed.size();
  for (std::size_t mask = 1; mask < (std::size_t{1} << k); ++mask) {
    std::vector<std::size_t> cols;
    for (std::size_t j = 0; j < k; ++j)
      if (mask & (std::size_t{1} << j)) cols.push_back(allowed[j]);
    std::vector<Observation> sub;
    sub.reserve(obs.size());
    for (const Observation& o : obs) {
      Observation q;
      q.target = o.target;
      for (std::size_t c : cols) q.features.push_back(o.features[c]);
      sub.push_back(std::move(q));
    }
    std::vector<double> beta;
    try {
      beta = fit_least_squares(sub);
    } catch (const RankDeficiencyError&) {
      continue;
    } catch (const TooFewObservationsError&) {
      continue;
    }
    if (std::any_of(beta.begin(), beta.end(), [](double v) { return v < 0.0; })) continue;
    double ss = 0.0;
    for (const Observation& o : sub) {
      double r = -o.target;
      for (std::size_t c = 0; c < cols.size(); ++c) r += beta[c] * o.features[c];
      ss += r * r;
    }
    if (ss < best_ss) {
      best_ss = ss;
      std::fill(best.begin(), best.end(), 0.0);
      for (std::size_t c = 0; c < cols.size(); ++c) best[cols[c]] = beta[c];
    }
  }
  return best;
}

FitReport fit_anchored_with_split(const std::vector<Observation>& data, const SplitConfig& cfg,
                                  std::vector<std::string> names, const std::vector<std::size_t>& allowed) {
  auto split = train_test_split(data, cfg);
  FitReport rep;
  rep.names = std::move(names);
  rep.coefficients = fit_nonneg_subset(split.first, allowed, data.front().features.size());
  rep.train = report_metrics(rep.coefficients, split.first);
  rep.test = report_metrics(rep.coefficients, split.second);
  rep.n_train = split.first.size();
  rep.n_test = split.second.size();
  rep.seed = cfg.seed;
  return rep;
}

std::vector<Observation> small_obs(const std::vector<OverheadRow>& rows) {
  std::vector<Observation> data;
  for (const auto& r : rows) {
    if (r.num_streams < 1) throw ValidationError("num_streams must be >= 1");
    data.push_back({{static_cast<double>(r.slae_size), std::log10(static_cast<double>(r.num_streams)), 1.0},
                    r.overhead_ms});
  }
  return data;
}

std::vector<Observation> big_obs(const std::vector<OverheadRow>& rows) {
  std::vector<Observation> data;
  for (const auto& r : rows) {
    if (r.num_streams < 1) throw ValidationError("num_streams must be >= 1");
    const double l = (4.0 / 3.0) * std::log2(static_cast<double>(r.num_streams));
    data.push_back({{static_cast<double>(r.slae_size) * l, l, 1.0}, r.overhead_ms});
  }
  return data;
}

}  // namespace

std::pair<std::vector<Observation>, std::vector<Observation>> train_test_split(
    const std::vector<Observation>& data, const SplitConfig& cfg) {
  if (!(cfg.train_fraction > 0.0 && cfg.train_fraction < 1.0))
    throw ValidationError("train_fraction must lie in (0, 1)");
  const std::size_t n = data.size();
  if (n < 4) throw TooFewObservationsError("train/test split needs at least 4 observations");
  double want = round_half_away(cfg.train_fraction * static_cast<double>(n));
  std::size_t n_train = static_cast<std::size_t>(std::clamp(want, 1.0, static_cast<double>(n - 1)));
  std::vector<std::size_t> order(n);
  if (cfg.shuffle)
    order = permutation(n, cfg.seed);
  else
    std::iota(order.begin(), order.end(), std::size_t{0});
  std::pair<std::vector<Observation>, std::vector<Observation>> out;
  for (std::size_t k = 0; k < n; ++k) (k < n_train ? out.first : out.second).push_back(data[order[k]]);
  return out;
}

std::vector<double> fit_least_squares(const std::vector<Observation>& obs) {
  if (obs.empty()) throw TooFewObservationsError("no observations");
  const std::size_t p = obs.front().features.size();
  const std::size_t n = obs.size();
  if (p == 0) throw ValidationError("observations have no features");
  for (const Observation& o : obs) {
    if (o.features.size() != p) throw ValidationError("ragged feature vectors");
    if (!std::isfinite(o.target)) throw ValidationError("non-finite target");
    for (double v : o.features)
      if (!std::isfinite(v)) throw ValidationError("non-finite feature");
  }
  if (n < p) throw TooFewObservationsError("fewer observations than features");

  // Column-major design matrix, columns scaled to unit 2-norm so that the
  // rank test is scale-free (features span 1 .. 1e8).
  std::vector<double> A(n * p), scale(p, 0.0), y(n);
  for (std::size_t j = 0; j < p; ++j) {
    double s = 0.0;
    for (std::size_t i = 0; i < n; ++i) s += obs[i].features[j] * obs[i].features[j];
    s = std::sqrt(s);
    if (s == 0.0) throw RankDeficiencyError("design matrix has an all-zero column");
    scale[j] = s;
    for (std::size_t i = 0; i < n; ++i) A[j * n + i] = obs[i].features[j] / s;
  }
  for (std::size_t i = 0; i < n; ++i) y[i] = obs[i].target;

  // Householder QR, applying the reflectors to y as we go.
  std::vector<double> rdiag(p);
  for (std::size_t k = 0; k < p; ++k) {
    double* col = &A[k * n];
    double norm = 0.0;
    for (std::size_t i = k; i < n; ++i) norm += col[i] * col[i];
    norm = std::sqrt(norm);
    double alpha = col[k] > 0 ? -norm : norm;
    rdiag[k] = alpha;
    if (norm == 0.0) continue;
    double vk = col[k] - alpha;
    // v = (vk, col[k+1..]); beta = 2 / v'v
    double vtv = vk * vk;
    for (std::size_t i = k + 1; i < n; ++i) vtv += col[i] * col[i];
    if (vtv == 0.0) continue;
    col[k] = vk;
    auto apply = [&](double* target) {
      double dot = 0.0;
      for (std::size_t i = k; i < n; ++i) dot += col[i] * target[i];
      const double f = 2.0 * dot / vtv;
      for (std::size_t i = k; i < n; ++i) target[i] -= f * col[i];
    };
    for (std::size_t j = k + 1; j < p; ++j) apply(&A[j * n]);
    apply(y.data());
  }
  double rmax = 0.0;
  for (double r : rdiag) rmax = std::max(rmax, std::fabs(r));
  for (double r : rdiag)
    if (!(std::fabs(r) >= 1e-10 * rmax) || rmax == 0.0)
      throw RankDeficiencyError("design matrix is rank deficient (collinear features)");
  // back substitution R beta = Q'y
  std::vector<double> beta(p);
  for (std::size_t kk = p; kk-- > 0;) {
    double s = y[kk];
    for (std::size_t j = kk + 1; j < p; ++j) s -= A[j * n + kk] * beta[j];
    beta[kk] = s / rdiag[kk];
  }
  for (std::size_t j = 0; j < p; ++j) beta[j] /= scale[j];
  return beta;
}

Metrics metrics(const std::vector<double>& predicted, const std::vector<double>& actual) {
  if (predicted.size() != actual.size() || actual.empty())
    throw ValidationError("metrics need equal, non-zero lengths");
  const double n = static_cast<double>(actual.size());
  double mean = 0.0;
  for (double a : actual) mean += a;
  mean /= n;
  double ss_res = 0.0, ss_tot = 0.0;
  for (std::size_t i = 0; i < actual.size(); ++i) {
    ss_res += (actual[i] - predicted[i]) * (actual[i] - predicted[i]);
    ss_tot += (actual[i] - mean) * (actual[i] - mean);
  }
  if (ss_tot == 0.0) throw ZeroVarianceError("R^2 undefined: actual values are all equal");
  Metrics m;
  m.r_squared = 1.0 - ss_res / ss_tot;
  m.mse = ss_res / n;
  m.rmse = std::sqrt(m.mse);
  return m;
}

FitReport fit_sum_model(const std::vector<std::pair<std::uint64_t, double>>& rows,
                        const SplitConfig& cfg) {
  std::vector<Observation> data;
  for (const auto& r : rows) data.push_back({{static_cast<double>(r.first), 1.0}, r.second});
  return fit_with_split(data, cfg, {"a", "b"});
}

FitReport fit_overhead_small(const std::vector<OverheadRow>& rows, const SplitConfig& cfg) {
  return fit_with_split(small_obs(rows), cfg, {"a", "b", "c"});
}

FitReport fit_overhead_big(const std::vector<OverheadRow>& rows, const SplitConfig& cfg) {
  return fit_with_split(big_obs(rows), cfg, {"a", "b", "c"});
}

// Anchored forms: T_overhead(N, n = 1) = 0 and never negative.  Small:
// a·N + b·log10 n + c vanishes at n = 1 for every N only with a = c = 0, so
// b >= 0 is fitted alone.  Big: (a·N + b)·(4/3)·log2 n + c with c = 0 and
// a, b >= 0.
FitReport fit_overhead_small_anchored(const std::vector<OverheadRow>& rows, const SplitConfig& cfg) {
  return fit_anchored_with_split(small_obs(rows), cfg, {"a", "b", "c"}, {1});
}

FitReport fit_overhead_big_anchored(const std::vector<OverheadRow>& rows, const SplitConfig& cfg) {
  return fit_anchored_with_split(big_obs(rows), cfg, {"a", "b", "c"}, {0, 1});
}

}  // namespace streamtune
