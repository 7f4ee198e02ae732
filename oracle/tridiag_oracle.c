/*
 * oracle/tridiag_oracle.c -- CPU ORACLE. TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load this library, and only as the checker or as the
 * timed CPU baseline.  The product path (paper_2501_05938_b200/) never
 * links or calls anything here.
 *
 * What it restates (the reference ships no solver):
 *   - the Austin et al. partition method as described in the paper
 *     (/root/reference/PAPER.md:26-30 partition into sub-systems,
 *      PAPER.md:52 sub-system size m, FP64,
 *      PAPER.md:63-68 Stage 1 on the GPU, Stage 2 reduced solve on the CPU,
 *      Stage 3 on the GPU; data flow per SURVEY.md Appendix A, algebra per
 *      SURVEY.md Appendix C): Stage 1 eliminates every m-row block to its
 *      two interface equations and keeps the spikes (y, g, h) for Stage 3;
 *      Stage 2 is a serial Thomas solve of the 2N/m-row reduced system;
 *      Stage 3 computes x_i = y_i - g_i x_s - h_i x_e.
 *      Stages 1 and 3 are OpenMP-parallel over blocks, Stage 2 serial, as
 *      in the paper (BASELINE.md "CPU baseline plan").
 *   - the sequential Thomas algorithm (the textbook reference solver).
 *   - the counter-based input generator shared bit-for-bit with the CUDA
 *     generator (SURVEY.md §8d "Inputs").
 *   - residual / relative-error checkers (SURVEY.md §8d parity bars).
 *
 * Parity pin: the reference has no solver and no solver golden vectors
 * ("parity unpinned" by the reference).  The restatement is pinned instead
 * to LAPACK dgtsv (scipy 1.18.1 / OpenBLAS) in tests/test_oracle.py and to
 * the committed fixtures in tests/golden/ (tests/golden/make_golden.py).
 *
 * Conventions (the C-ABI of the product, include/pm_tridiag.h):
 *   four length-n arrays a (sub), b (diag), c (super), d (rhs);
 *   a[0] and c[n-1] are ignored (treated as 0).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_API __attribute__((visibility("default")))

/* ------------------------------------------------------------------ */
/* Counter-based generator (identical to csrc/pm_generate.cu)          */
/* ------------------------------------------------------------------ */
static inline uint64_t orc_splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
static inline uint64_t orc_stream_key(uint64_t seed, uint64_t arr) {
  return orc_splitmix64(seed ^ (0x632BE59BD9B4E019ull * (arr + 1ull)));
}
static inline double orc_unit(uint64_t key, uint64_t i) {
  return (double)(orc_splitmix64(key + i) >> 11) * 0x1.0p-53;
}

/* Row i of the n_total-row system: a,c ~ U(-1,1) with a[0] = c[n_total-1] = 0;
 * b = +-(|a|+|c|+1+U(0,1)); d ~ U(-1,1).  Rows [row0, row0+count) are written
 * to a[0..count) etc. (a rank's slice of a row-sharded system; identical to
 * pm_generate_range_f64).  Any of the output pointers may be NULL. */
ORC_API void orc_generate_range(double* a, double* b, double* c, double* d, int64_t n_total,
                                int64_t row0, int64_t count, uint64_t seed) {
  const uint64_t ka = orc_stream_key(seed, 0), kc = orc_stream_key(seed, 1);
  const uint64_t kb = orc_stream_key(seed, 2), kd = orc_stream_key(seed, 3);
  const uint64_t ks = orc_stream_key(seed, 4);
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < count; ++k) {
    const int64_t i = row0 + k;
    double ai = (i == 0) ? 0.0 : 2.0 * orc_unit(ka, (uint64_t)i) - 1.0;
    double ci = (i == n_total - 1) ? 0.0 : 2.0 * orc_unit(kc, (uint64_t)i) - 1.0;
    double mag = ((fabs(ai) + fabs(ci)) + 1.0) + orc_unit(kb, (uint64_t)i);
    double bi = (orc_splitmix64(ks + (uint64_t)i) >> 63) ? -mag : mag;
    if (a) a[k] = ai;
    if (b) b[k] = bi;
    if (c) c[k] = ci;
    if (d) d[k] = 2.0 * orc_unit(kd, (uint64_t)i) - 1.0;
  }
}

ORC_API void orc_generate(double* a, double* b, double* c, double* d, int64_t n, uint64_t seed) {
  orc_generate_range(a, b, c, d, n, 0, n, seed);
}

/* ------------------------------------------------------------------ */
/* Sequential Thomas                                                   */
/* ------------------------------------------------------------------ */
/* Returns 0, or 2 on a zero / non-finite pivot.  work: n doubles. */
ORC_API int orc_thomas(const double* a, const double* b, const double* c, const double* d,
                       double* x, double* work, int64_t n) {
  if (n < 1) return 1;
  double* cp = work;
  double den = b[0];
  if (den == 0.0 || !isfinite(den)) return 2;
  double r = 1.0 / den;
  cp[0] = (n > 1 ? c[0] : 0.0) * r;
  x[0] = d[0] * r;
  for (int64_t i = 1; i < n; ++i) {
    den = b[i] - a[i] * cp[i - 1];
    if (den == 0.0 || !isfinite(den)) return 2;
    r = 1.0 / den;
    cp[i] = (i < n - 1 ? c[i] : 0.0) * r;
    x[i] = (d[i] - a[i] * x[i - 1]) * r;
  }
  for (int64_t i = n - 2; i >= 0; --i) x[i] -= cp[i] * x[i + 1];
  return 0;
}

/* ------------------------------------------------------------------ */
/* Partition method restatement */
/* ------------------------------------------------------------------ */
/* Block k covers rows s = k*m .. e = min(s+m, n)-1.  Interior I = s+1..e-1.
 * Stage 1: T y = d_I, T g = a_{s+1} e_1, T h = c_{e-1} e_last (one
 *          forward sweep, three right-hand sides), then two interface rows
 *   row s: [a_s,        b_s - c_s g_1,  -c_s h_1 | d_s - c_s y_1]
 *   row e: [-a_e g_L,   b_e - a_e h_L,   c_e     | d_e - a_e y_L]
 *   A one-row tail block contributes its own row unchanged.
 * Stage 2: Thomas on the reduced rows (natural order x_s0, x_e0, x_s1, ...).
 * Stage 3: x_i = y_i - g_i x_s - h_i x_e on the interior.
 *
 * ws must hold 3*n + 6*(2*nblk) doubles (orc_partition_workspace). */
ORC_API int64_t orc_partition_workspace(int64_t n, int32_t m) {
  if (n < 1 || m < 2) return 0;
  int64_t nblk = (n + m - 1) / m;
  return 3 * n + 6 * (2 * nblk);
}

ORC_API int orc_partition_solve(const double* a, const double* b, const double* c,
                                const double* d, double* x, int64_t n, int32_t m, double* ws,
                                int nthreads) {
  if (n < 1 || m < 2) return 1;
  const int64_t nblk = (n + m - 1) / m;
  double* y = ws;
  double* g = ws + n;
  double* h = ws + 2 * n;
  double* ra = ws + 3 * n;            /* reduced system, up to 2*nblk rows */
  double* rb = ra + 2 * nblk;
  double* rc = rb + 2 * nblk;
  double* rd = rc + 2 * nblk;
  double* rx = rd + 2 * nblk;
  double* rw = rx + 2 * nblk;
  int bad = 0;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#else
  (void)nthreads;
#endif

  /* ---- Stage 1: per-block elimination (parallel over blocks) ---- */
#pragma omp parallel for schedule(static) reduction(| : bad)
  for (int64_t k = 0; k < nblk; ++k) {
    const int64_t s = k * m;
    const int64_t e = (s + m < n ? s + m : n) - 1;
    const double as = (s == 0) ? 0.0 : a[s];
    const double ce = (e == n - 1) ? 0.0 : c[e];
    if (e == s) { /* one-row tail block: row passes through */
      ra[2 * k] = as; rb[2 * k] = b[s]; rc[2 * k] = ce; rd[2 * k] = d[s];
      continue;
    }
    double y1 = 0, g1 = 0, h1 = 0, yl = 0, gl = 0, hl = 0;
    if (e - s >= 2) {
      /* forward sweep over interior rows i = s+1 .. e-1, three RHS;
       * c' kept in h[] temporarily (overwritten by the backward sweep). */
      for (int64_t i = s + 1; i <= e - 1; ++i) {
        double ai = (i == s + 1) ? 0.0 : a[i];
        double den = b[i] - ai * ((i == s + 1) ? 0.0 : h[i - 1]);
        if (den == 0.0 || !isfinite(den)) bad |= 1;
        double r = 1.0 / den;
        double ci = (i == e - 1) ? 0.0 : c[i];
        h[i] = ci * r; /* c'_i */
        y[i] = (d[i] - ai * ((i == s + 1) ? 0.0 : y[i - 1])) * r;
        g[i] = ((i == s + 1) ? a[s + 1] : -ai * g[i - 1]) * r;
      }
      /* backward sweep: y, g in place; h from its single RHS entry */
      /* h: T h = c_{e-1} e_last. forward gives h'_L = c_{e-1} / den_L and 0
       * elsewhere; recompute den_L from the stored c'_{L-1}. */
      {
        int64_t L = e - 1;
        double den = b[L] - ((L == s + 1) ? 0.0 : a[L] * h[L - 1]);
        double hL = c[e - 1] / den;
        double hn = hL;
        double ynext = y[L], gnext = g[L];
        /* walk backwards; h[i] currently holds c'_i */
        for (int64_t i = L - 1; i >= s + 1; --i) {
          double cpi = h[i];
          y[i] -= cpi * ynext;
          g[i] -= cpi * gnext;
          hn = -cpi * hn;
          h[i] = hn;
          ynext = y[i];
          gnext = g[i];
        }
        h[L] = hL;
      }
      y1 = y[s + 1]; g1 = g[s + 1]; h1 = h[s + 1];
      yl = y[e - 1]; gl = g[e - 1]; hl = h[e - 1];
      ra[2 * k] = as;
      rb[2 * k] = b[s] - c[s] * g1;
      rc[2 * k] = -c[s] * h1;
      rd[2 * k] = d[s] - c[s] * y1;
      ra[2 * k + 1] = -a[e] * gl;
      rb[2 * k + 1] = b[e] - a[e] * hl;
      rc[2 * k + 1] = ce;
      rd[2 * k + 1] = d[e] - a[e] * yl;
    } else { /* two-row block: no interior, rows unchanged */
      ra[2 * k] = as;   rb[2 * k] = b[s];   rc[2 * k] = c[s];   rd[2 * k] = d[s];
      ra[2 * k + 1] = a[e]; rb[2 * k + 1] = b[e]; rc[2 * k + 1] = ce; rd[2 * k + 1] = d[e];
    }
  }
  if (bad) return 2;

  /* ---- Stage 2: serial reduced solve ("on the CPU") ---- */
  /* Compact: a one-row tail block occupies a single reduced row. */
  int64_t nr = 2 * nblk;
  const int64_t tail = n - (nblk - 1) * (int64_t)m;
  if (tail == 1) nr -= 1;
  int st = orc_thomas(ra, rb, rc, rd, rx, rw, nr);
  if (st) return st;

  /* ---- Stage 3: back-substitution (parallel over blocks) ---- */
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < nblk; ++k) {
    const int64_t s = k * m;
    const int64_t e = (s + m < n ? s + m : n) - 1;
    if (e == s) { x[s] = rx[2 * k]; continue; }
    const double xs = rx[2 * k], xe = rx[2 * k + 1];
    x[s] = xs;
    x[e] = xe;
    for (int64_t i = s + 1; i <= e - 1; ++i) x[i] = y[i] - g[i] * xs - h[i] * xe;
  }
  for (int64_t i = 0; i < n; ++i)
    if (!isfinite(x[i])) return 2;
  return 0;
}

/* ------------------------------------------------------------------ */
/* Checkers                                                            */
/* ------------------------------------------------------------------ */
/* ||Ax - d||_2 / ||d||_2 with long double accumulation. */
ORC_API double orc_residual(const double* a, const double* b, const double* c, const double* d,
                            const double* x, int64_t n) {
  long double num = 0.0L, den = 0.0L;
#pragma omp parallel for schedule(static) reduction(+ : num, den)
  for (int64_t i = 0; i < n; ++i) {
    long double r = (long double)b[i] * x[i] - (long double)d[i];
    if (i > 0) r += (long double)a[i] * x[i - 1];
    if (i < n - 1) r += (long double)c[i] * x[i + 1];
    num += r * r;
    den += (long double)d[i] * d[i];
  }
  if (den == 0.0L) return (double)sqrtl(num);
  return (double)sqrtl(num / den);
}

/* max|x - xr| / max|xr| */
ORC_API double orc_rel_err(const double* x, const double* xr, int64_t n) {
  double num = 0.0, den = 0.0;
#pragma omp parallel for schedule(static) reduction(max : num, den)
  for (int64_t i = 0; i < n; ++i) {
    double e = fabs(x[i] - xr[i]);
    if (isnan(e)) e = INFINITY;
    if (e > num) num = e;
    double v = fabs(xr[i]);
    if (v > den) den = v;
  }
  if (den == 0.0) return num;
  return num / den;
}

/* ------------------------------------------------------------------ */
/* Windowed check of a solution of the generated system               */
/* ------------------------------------------------------------------ */
/* x[0..count) claims to solve rows [row0, row0+count) of the n_total-row
 * generated system (seed); xl = x[row0-1] and xr = x[row0+count] (ignored at
 * the system's ends).  Without holding the system in memory, every window of
 * `chunk` rows is checked against sequential Thomas on the window widened by
 * `pad` rows each side (truncated at the system's ends): the synthetic
 * systems are strictly diagonally dominant with margin >= 1 and |a|+|c| < 2,
 * so the truncation perturbs the window's centre by < (2/3)^pad relative
 * (pad = 1024: < 1e-180), far below FP64 rounding -- the centre IS the
 * Thomas solution of the whole system to the last bit in practice
 * (tests/test_oracle.py compares it with a whole-system Thomas).
 * out[0] = max|x - x_thomas|, out[1] = max|x_thomas|,
 * out[2] = sum (Ax - d)^2, out[3] = sum d^2 over the rows.  Returns 0, 1 on
 * bad arguments / allocation failure, 2 on a pivot failure. */
ORC_API int orc_check_generated(const double* x, int64_t n_total, int64_t row0, int64_t count,
                                uint64_t seed, double xl, double xr, int64_t chunk, int64_t pad,
                                double* out) {
  if (count < 1 || row0 < 0 || row0 + count > n_total || chunk < 1 || pad < 0) return 1;
  const int64_t nch = (count + chunk - 1) / chunk;
  double emax = 0.0, rmax = 0.0;
  long double rsq = 0.0L, dsq = 0.0L;
  int status = 0;
#pragma omp parallel reduction(max : emax, rmax) reduction(+ : rsq, dsq) reduction(max : status)
  {
    const int64_t wmax = chunk + 2 * pad;
    double* buf = (double*)malloc(sizeof(double) * 6 * (size_t)wmax);
    if (!buf) status = 1;
#pragma omp for schedule(dynamic, 1)
    for (int64_t k = 0; k < nch; ++k) {
      if (!buf) continue;
      const int64_t lo = row0 + k * chunk;                           /* window, global rows */
      const int64_t hi = (lo + chunk < row0 + count) ? lo + chunk : row0 + count;
      const int64_t wlo = (lo - pad > 0) ? lo - pad : 0;               /* widened window */
      const int64_t whi = (hi + pad < n_total) ? hi + pad : n_total;
      const int64_t w = whi - wlo;
      double *a = buf, *b = buf + wmax, *c = buf + 2 * wmax, *d = buf + 3 * wmax;
      double *xt = buf + 4 * wmax, *work = buf + 5 * wmax;
      orc_generate_range(a, b, c, d, n_total, wlo, w, seed);
      a[0] = 0.0;       /* truncation: the window is a system of its own */
      c[w - 1] = 0.0;
      /* restore the true couplings for the residual below */
      double a_lo = 0.0, c_hi = 0.0;
      if (wlo > 0) orc_generate_range(&a_lo, NULL, NULL, NULL, n_total, wlo, 1, seed);
      if (whi < n_total) orc_generate_range(NULL, NULL, &c_hi, NULL, n_total, whi - 1, 1, seed);
      if (orc_thomas(a, b, c, d, xt, work, w) != 0) {
        status = 2;
        continue;
      }
      a[0] = a_lo;
      c[w - 1] = c_hi;
      for (int64_t i = lo; i < hi; ++i) {
        const int64_t j = i - wlo, q = i - row0;
        double e = fabs(x[q] - xt[j]);
        if (isnan(e)) e = INFINITY;
        if (e > emax) emax = e;
        if (fabs(xt[j]) > rmax) rmax = fabs(xt[j]);
        const double xm = (i == 0) ? 0.0 : (q > 0 ? x[q - 1] : xl);
        const double xp = (i == n_total - 1) ? 0.0 : (q + 1 < count ? x[q + 1] : xr);
        long double r = (long double)b[j] * x[q] - (long double)d[j];
        if (i > 0) r += (long double)a[j] * xm;
        if (i < n_total - 1) r += (long double)c[j] * xp;
        rsq += r * r;
        dsq += (long double)d[j] * d[j];
      }
    }
    free(buf);
  }
  out[0] = emax;
  out[1] = rmax;
  out[2] = (double)rsq;
  out[3] = (double)dsq;
  return status;
}

ORC_API int orc_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
