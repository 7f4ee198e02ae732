// pm_device.cuh -- device building blocks of the B200 partition-method solver.
//
// Algebra (the Austin et al. partition method cited at
// /root/reference/PAPER.md:26-30, sub-system size m at PAPER.md:52):
//
//   A "segment" covers rows f..l (l > f) and is represented by its two
//   boundary equations in the unknowns just outside / at its ends:
//     F: Fa*x[f-1] + Fb*x[f] + Fc*x[l]   = Fd
//     L: La*x[f]   + Lb*x[l] + Lc*x[l+1] = Ld
//   Stage 1 turns every m-row block into a segment by eliminating its
//   interior (block_reduce).  Stage 2 (the reduced interface system) is
//   solved by combining adjacent segments pairwise -- a tree of
//   "eliminate the two unknowns at the junction" steps (combine) inside a
//   warp (shuffles), across the warps of a CTA (shared memory), and across
//   CTA tiles by the same kernels one level up.  The downsweep recovers the
//   junction unknowns from the stored Node coefficients, and Stage 3
//   (block_interior) back-substitutes each block's interior from its two
//   boundary values.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

// One source, two precisions: the translation units compiled with
// PM_REAL_F32 (pm_kernels_f32.cu) put the FP32 solver in namespace pm32,
// the others the FP64 solver in namespace pm.
#ifdef PM_REAL_F32
#define PM_NS pm32
#else
#define PM_NS pm
#endif

namespace PM_NS {

#ifdef PM_REAL_F32
using real = float;
using real2 = float2;
__host__ __device__ __forceinline__ real2 make_real2(real x, real y) { return make_float2(x, y); }
constexpr real kTinyPivot = 1e-35f;  // continuant magnitude below which the block
                                     // falls back to the classic sweep
#else
using real = double;
using real2 = double2;
__host__ __device__ __forceinline__ real2 make_real2(real x, real y) { return make_double2(x, y); }
constexpr real kTinyPivot = 1e-280;
#endif

struct Row {
  real a, b, c, d;
};
struct Seg {
  Row F, L;
};
// Junction solve of a combine (scaled by r = 1 / (s * det)):
//   x[l1] = (p0 + p1*x[f1] + p2*x[l2]) * r
//   x[f2] = (q0 + q1*x[f1] + q2*x[l2]) * r
struct Node {
  real p0, p1, p2, q0, q1, q2, r;
};

// Reciprocal: the MUFU seed (rcp.approx.ftz) refined by Newton steps -- two
// for FP64, one for FP32 (<= 1 ulp) -- instead of the IEEE-rounded
// __drcp_rn / __frcp_rn sequences with their slow-path branch.  A zero
// argument yields inf/NaN (and is flagged separately by the callers).
__device__ __forceinline__ double drcp(double x) {
#ifdef PM_EXACT_RCP
  return __drcp_rn(x);
#else
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
#endif
}
__device__ __forceinline__ float drcp(float x) {
#ifdef PM_EXACT_RCP
  return __frcp_rn(x);
#else
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  const float e = fmaf(-x, r, 1.0f);
  return fmaf(r, e, r);
#endif
}

// 2^-(e(u) + e(v)), e = unbiased binary exponent: an exact power-of-two
// scale that keeps u*v-sized products near 1 (clamped to the normal range).
__device__ __forceinline__ double pow2_inv_scale(double u, double v) {
  const int eu = (__double2hiint(u) >> 20) & 0x7ff;
  const int ev = (__double2hiint(v) >> 20) & 0x7ff;
  int e = eu + ev - 2 * 1023;
  e = max(-1000, min(1000, e));
  return __hiloint2double((1023 - e) << 20, 0);
}
__device__ __forceinline__ float pow2_inv_scale(float u, float v) {
  const int eu = (__float_as_int(u) >> 23) & 0xff;
  const int ev = (__float_as_int(v) >> 23) & 0xff;
  int e = eu + ev - 2 * 127;
  e = max(-120, min(120, e));
  return __int_as_float((127 - e) << 23);
}

// Pivot reciprocals of a block from its continuants: inv[j] = q[j-1] / q[j],
// j = 1..L.  PM_BATCH_INV (default): one reciprocal for all L pivots
// (Montgomery's batch inversion: P_j = q_1 ... q_j, R = 1/P_L, then
// 1/q_j = R * P_{j-1} and R <- R * q_j walking down) -- 2 multiplies per
// pivot instead of a MUFU + Newton sequence each.  Returns false when the
// product leaves the safe range (the caller then takes the classic sweep).
#ifndef PM_BATCH_INV
#define PM_BATCH_INV 1
#endif
#ifdef PM_REAL_F32
constexpr real kProdLo = 1e-30f, kProdHi = 1e30f;
#else
constexpr real kProdLo = 1e-250, kProdHi = 1e250;
#endif
template <int L>
__device__ __forceinline__ bool continuant_ratios(const real (&q)[L + 1], real (&inv)[L + 1]) {
#if PM_BATCH_INV
  real P[L + 1];
  P[1] = q[1];
#pragma unroll
  for (int j = 2; j <= L; ++j) P[j] = P[j - 1] * q[j];
  const real aP = fabs(P[L]);
  if (!(aP > kProdLo && aP < kProdHi)) return false;
  real R = drcp(P[L]);
#pragma unroll
  for (int j = L; j >= 2; --j) {
    const real iq = R * P[j - 1];  // 1 / q_j
    R = R * q[j];                  // 1 / P_{j-1}
    inv[j] = q[j - 1] * iq;
  }
  inv[1] = R;  // q_0 = 1
  return true;
#else
#pragma unroll
  for (int j = 1; j <= L; ++j) inv[j] = q[j - 1] * drcp(q[j]);
  return true;
#endif
}

// Finiteness of a block's results with one compare: fma(x, 0, t) keeps t = 0
// for finite x and turns it into NaN for an inf / NaN x.
#ifndef PM_FINITE_SUM
#define PM_FINITE_SUM 1
#endif
template <int M>
__device__ __forceinline__ bool all_finite(const real (&x)[M]) {
#if PM_FINITE_SUM
  real t = 0.0;
#pragma unroll
  for (int j = 0; j < M; ++j) t = fma(x[j], real(0.0), t);
  return t == real(0.0);
#else
  bool ok = true;
#pragma unroll
  for (int j = 0; j < M; ++j) ok &= isfinite(x[j]);
  return ok;
#endif
}

// Merge segment A = [f1..l1] with its right neighbour B = [f2..l2], f2 = l1+1,
// eliminating x[l1] and x[f2].  Division-free: both output equations are
// multiplied by s*det (equations may be scaled freely), with s an exact
// power of two chosen from the operands' exponents before det is known, so
// the upsweep's dependency chain is four FP64 operations per level; the
// reciprocal the downsweep needs is computed off that chain.
__device__ __forceinline__ void combine(const Seg& A, const Seg& B, Seg& out, Node& nd,
                                        bool& bad) {
  const real s = pow2_inv_scale(A.L.b, B.F.b);
  const real det = fma(A.L.b, B.F.b, -A.L.c * B.F.a);
  bad |= (det == 0.0);
  const real ds = det * s;
  nd.p0 = fma(B.F.b, A.L.d, -A.L.c * B.F.d) * s;
  nd.p1 = -(B.F.b * A.L.a) * s;
  nd.p2 = (A.L.c * B.F.c) * s;
  nd.q0 = fma(A.L.b, B.F.d, -B.F.a * A.L.d) * s;
  nd.q1 = (B.F.a * A.L.a) * s;
  nd.q2 = -(A.L.b * B.F.c) * s;
  nd.r = drcp(ds);
  Seg o;
  o.F.a = A.F.a * ds;
  o.F.b = fma(A.F.c, nd.p1, A.F.b * ds);
  o.F.c = A.F.c * nd.p2;
  o.F.d = fma(-A.F.c, nd.p0, A.F.d * ds);
  o.L.a = B.L.a * nd.q1;
  o.L.b = fma(B.L.a, nd.q2, B.L.b * ds);
  o.L.c = B.L.c * ds;
  o.L.d = fma(-B.L.a, nd.q0, B.L.d * ds);
  out = o;
}

// Downsweep step of one node: (xf, xl) of the merged segment -> x[l1], x[f2].
__device__ __forceinline__ void split_node(const Node& nd, real xf, real xl, real& xl1,
                                           real& xf2) {
  xl1 = fma(nd.p2, xl, fma(nd.p1, xf, nd.p0)) * nd.r;
  xf2 = fma(nd.q2, xl, fma(nd.q1, xf, nd.q0)) * nd.r;
}

__device__ __forceinline__ Seg shfl_down_seg(const Seg& s, int delta) {
  Seg o;
  o.F.a = __shfl_down_sync(0xffffffffu, s.F.a, delta);
  o.F.b = __shfl_down_sync(0xffffffffu, s.F.b, delta);
  o.F.c = __shfl_down_sync(0xffffffffu, s.F.c, delta);
  o.F.d = __shfl_down_sync(0xffffffffu, s.F.d, delta);
  o.L.a = __shfl_down_sync(0xffffffffu, s.L.a, delta);
  o.L.b = __shfl_down_sync(0xffffffffu, s.L.b, delta);
  o.L.c = __shfl_down_sync(0xffffffffu, s.L.c, delta);
  o.L.d = __shfl_down_sync(0xffffffffu, s.L.d, delta);
  return o;
}

// ---------------------------------------------------------------------------
// Per-block (m rows) elimination.  Acc exposes the block's rows (with the
// boundary fix-ups already applied) as a(j), b(j), c(j), d(j), j = 0..m-1.
// Interior j = 1..L (L = m-2) is the tridiagonal T with the couplings a(1)
// (to x[s]) and c(L) (to x[e]) removed; one forward sweep serves the three
// right-hand sides y (d), g (a(1) e_1), h (c(L) e_L).  The first-interior-
// row values are accumulated on the fly: y_1 = sum_k P_k y'_k with
// P_1 = 1, P_{k+1} = -P_k c'_k, so no backward sweep is needed in Stage 1.
//   F = [a_s, b_s - c_s g_1, -c_s h_1 | d_s - c_s y_1]
//   L = [-a_e g_L, b_e - a_e h_L, c_e | d_e - a_e y_L]
// ---------------------------------------------------------------------------
template <int M, class Acc>
__device__ __forceinline__ Seg block_reduce(const Acc& r, int m_rt, bool& bad) {
  const int m = (M > 0) ? M : m_rt;
  Seg S;
  if (m == 2) {
    S.F = Row{r.a(0), r.b(0), r.c(0), r.d(0)};
    S.L = Row{r.a(1), r.b(1), r.c(1), r.d(1)};
    return S;
  }
  const int L = m - 2;
  real den = r.b(1);
  bad |= (den == 0.0);
  real inv = drcp(den);
  real cp = (L > 1) ? r.c(1) * inv : 0.0;
  real yp = r.d(1) * inv;
  real gp = r.a(1) * inv;
  real P = 1.0, Y1 = yp, G1 = gp;
  auto step = [&](int j) {
    const real aj = r.a(j);
    den = fma(-aj, cp, r.b(j));
    bad |= (den == 0.0);
    inv = drcp(den);
    P = -P * cp;
    yp = fma(-aj, yp, r.d(j)) * inv;
    gp = -aj * gp * inv;
    cp = (j < L) ? r.c(j) * inv : 0.0;
    Y1 = fma(P, yp, Y1);
    G1 = fma(P, gp, G1);
  };
  if constexpr (M > 0) {
#pragma unroll
    for (int j = 2; j <= M - 2; ++j) step(j);
  } else {
    for (int j = 2; j <= L; ++j) step(j);
  }
  const real hL = r.c(L) * inv;
  const real H1 = P * hL;
  const real as = r.a(0), bs = r.b(0), cs = r.c(0), ds = r.d(0);
  const real ae = r.a(m - 1), be = r.b(m - 1), ce = r.c(m - 1), de = r.d(m - 1);
  S.F = Row{as, fma(-cs, G1, bs), -cs * H1, fma(-cs, Y1, ds)};
  S.L = Row{-ae * gp, fma(-ae, hL, be), ce, fma(-ae, yp, de)};
  return S;
}

// Stage 1 with a short dependency chain (compile-time m, rows in registers).
// The pivots of the interior sweep are ratios of continuants,
//   den_j = q_j / q_{j-1},  q_0 = 1, q_1 = b_1,
//   q_j = b_j q_{j-1} - (a_j c_{j-1}) q_{j-2},
// an FMA-only recurrence; the reciprocals inv_j = q_{j-1} / q_j are then
// independent of each other, and the y'/g' sweeps become FMA+MUL chains.
// A zero or non-finite continuant (a zero pivot, or over/underflow for
// extreme inputs) drops the block to the classic sweep.
// KEEP (Stage 3): b(j) <- inv_j and c(j) <- c'_j for interior j < L, c(L)
// unchanged, for block_interior_kept.
template <int M, bool KEEP, class Acc>
__device__ __forceinline__ Seg block_reduce_fast(Acc& r, bool& bad) {
  static_assert(M > 0, "compile-time m only");
  Seg S;
  if constexpr (M == 2) {
    S.F = Row{r.a(0), r.b(0), r.c(0), r.d(0)};
    S.L = Row{r.a(1), r.b(1), r.c(1), r.d(1)};
    return S;
  } else {
    constexpr int L = M - 2;
    real q[L + 1], inv[L + 1];
    q[0] = 1.0;
    q[1] = r.b(1);
    bool ok = q[1] != 0.0;
#pragma unroll
    for (int j = 2; j <= L; ++j) {
      q[j] = fma(r.b(j), q[j - 1], -(r.a(j) * r.c(j - 1)) * q[j - 2]);
      ok &= (q[j] != 0.0);
    }
    ok &= isfinite(q[L]) && (fabs(q[L]) > kTinyPivot);
    if (ok) ok = continuant_ratios<L>(q, inv);
    if (!ok) {  // classic sweep (rare)
      real cprev = 0.0;
#pragma unroll
      for (int j = 1; j <= L; ++j) {
        const real den = (j == 1) ? r.b(1) : fma(-r.a(j), cprev, r.b(j));
        bad |= (den == 0.0);
        inv[j] = drcp(den);
        cprev = r.c(j) * inv[j];
      }
    }
    real cp = (L > 1) ? r.c(1) * inv[1] : 0.0;
    real yp = r.d(1) * inv[1];
    real gp = r.a(1) * inv[1];
    real P = 1.0, Y1 = yp, G1 = gp;
    if constexpr (KEEP) {
      r.set_b(1, inv[1]);
      if (L > 1) r.set_c(1, cp);
    }
#pragma unroll
    for (int j = 2; j <= L; ++j) {
      const real aj = r.a(j);
      P = -P * cp;
      yp = fma(-aj, yp, r.d(j)) * inv[j];
      gp = -aj * gp * inv[j];
      cp = (j < L) ? r.c(j) * inv[j] : 0.0;
      Y1 = fma(P, yp, Y1);
      G1 = fma(P, gp, G1);
      if constexpr (KEEP) {
        r.set_b(j, inv[j]);
        if (j < L) r.set_c(j, cp);
      }
    }
    const real hL = r.c(L) * inv[L];
    const real H1 = P * hL;
    const real as = r.a(0), bs = r.b(0), cs = r.c(0), ds = r.d(0);
    const real ae = r.a(M - 1), be = r.b(M - 1), ce = r.c(M - 1), de = r.d(M - 1);
    S.F = Row{as, fma(-cs, G1, bs), -cs * H1, fma(-cs, Y1, ds)};
    S.L = Row{-ae * gp, fma(-ae, hL, be), ce, fma(-ae, yp, de)};
    return S;
  }
}

// Stage 3 after block_reduce_fast<M, true>: forward substitution with the stored
// reciprocals (an FMA + MUL chain per row), then back-substitution; x is
// written over b(j).
template <int M, class Acc>
__device__ __forceinline__ void block_interior_kept(Acc& r, real xs, real xe) {
  if constexpr (M == 2) {
    r.set_b(0, xs);
    r.set_b(1, xe);
  } else {
    constexpr int L = M - 2;
    real dp[L + 1];
    dp[1] = fma(-r.a(1), xs, r.d(1)) * r.b(1);
#pragma unroll
    for (int j = 2; j <= L; ++j) dp[j] = fma(-r.a(j), dp[j - 1], r.d(j)) * r.b(j);
    dp[L] = fma(-(r.c(L) * r.b(L)), xe, dp[L]);  // - h_L * x_e
    real xn = dp[L];
    r.set_b(L, xn);
#pragma unroll
    for (int j = L - 1; j >= 1; --j) {
      xn = fma(-r.c(j), xn, dp[j]);
      r.set_b(j, xn);
    }
    r.set_b(0, xs);
    r.set_b(M - 1, xe);
  }
}

// Stage 3 for one block: Thomas on the interior with known x[s] = xs and
// x[e] = xe folded into the right-hand side.  Writes x(j) for j = 0..m-1
// through r.set_x.  Acc must also provide scratch set_cp/cp, set_dp/dp.
template <int M, class Acc>
__device__ __forceinline__ void block_interior(Acc& r, int m_rt, real xs, real xe,
                                               bool& bad) {
  const int m = (M > 0) ? M : m_rt;
  if (m == 2) {
    r.set_x(0, xs);
    r.set_x(1, xe);
    return;
  }
  const int L = m - 2;
  real den = r.b(1);
  bad |= (den == 0.0);
  real inv = drcp(den);
  real rhs = fma(-r.a(1), xs, r.d(1));
  if (L == 1) rhs = fma(-r.c(1), xe, rhs);
  real cp = (L > 1) ? r.c(1) * inv : 0.0;
  real dp = rhs * inv;
  r.set_cp(1, cp);
  r.set_dp(1, dp);
  auto fwd = [&](int j) {
    const real aj = r.a(j);
    den = fma(-aj, cp, r.b(j));
    bad |= (den == 0.0);
    inv = drcp(den);
    rhs = r.d(j);
    if (j == L) rhs = fma(-r.c(j), xe, rhs);
    cp = (j < L) ? r.c(j) * inv : 0.0;
    dp = fma(-aj, dp, rhs) * inv;
    r.set_cp(j, cp);
    r.set_dp(j, dp);
  };
  real xn;
  auto bwd = [&](int j) {
    xn = fma(-r.cp(j), xn, r.dp(j));
    r.set_x(j, xn);
  };
  if constexpr (M > 0) {
#pragma unroll
    for (int j = 2; j <= M - 2; ++j) fwd(j);
    xn = dp;  // x_L
    r.set_x(L, xn);
#pragma unroll
    for (int j = M - 3; j >= 1; --j) bwd(j);
  } else {
    for (int j = 2; j <= L; ++j) fwd(j);
    xn = dp;
    r.set_x(L, xn);
    for (int j = L - 1; j >= 1; --j) bwd(j);
  }
  r.set_x(0, xs);
  r.set_x(m - 1, xe);
}

}  // namespace PM_NS
