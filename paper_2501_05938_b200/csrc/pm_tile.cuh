// pm_tile.cuh -- tile-level device building blocks shared by the solver
// kernels (pm_kernels.cu: level kernels; pm_batch.cu: the cluster kernel for
// batches of independent systems): mbarrier / bulk-copy PTX, the tile
// context with its boundary fix-ups, row accessors, the Stage-3 block solve
// from the shared-memory stage, and the warp combine trees.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <mutex>
#include <utility>

#include "pm_device.cuh"

namespace PM_NS {

constexpr int kMaxStages = 4;
// Stage 3 (level 0) keeps the block rows in its shared-memory stage: ~106
// registers and a single stage per warp give 16 warps per SM, which hides
// the sweeps' FP64 latency better than the register-resident variant.
#ifndef PM_SOLVE_STAGE_ROWS
#define PM_SOLVE_STAGE_ROWS 1
#endif
// ... and reads them as 16-byte pairs, recomputing the pivots in the
// back-substitution instead of storing them (half the shared-memory traffic)
#ifndef PM_SOLVE_PAIRS
#define PM_SOLVE_PAIRS 1
#endif
#ifndef PM_REDUCE_PAIRS
#define PM_REDUCE_PAIRS 0
#endif
constexpr int kMaxWarps = 8;  // P <= 256

// ---------------------------------------------------------------------------
// PTX helpers (mbarrier + bulk copies)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(addr),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// Programmatic dependent launch: let the next kernel of the stream start its
// launch now, and wait for the previous one's results before touching them.
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// ---------------------------------------------------------------------------
// Row accessors
// ---------------------------------------------------------------------------
// Boundary fix-ups shared by both accessors (rows of one tile):
//   local row >= valid      -> identity padding row (a=c=d=0, b=1)
//   global row 0            -> a = 0   (a[0] is ignored by contract)
//   global row n-1          -> c = 0   (c[n-1] is ignored by contract)
//   tail rows not covered by the 16-byte bulk copies (the last < kBulkRows
//   rows of the level, valid not a multiple of kBulkRows) -> read from global.
constexpr int kBulkRows = 16 / (int)sizeof(real);  // rows per 16 bytes

struct TileCtx {
  const real* ga;
  const real* gb;
  const real* gc;
  const real* gd;
  int64_t row0;   // first global row of the tile
  int64_t n;      // rows of this level
  int valid;      // rows of the tile inside [0, n)
  int bulk_rows;  // rows [bulk_rows, valid) are read from global
  bool zf, zl;    // zero a[0] / c[n-1]
  int64_t sys_len;
  uint64_t sys_magic;  // batch: Lemire fastmod multiplier of sys_len (0: use %)
};

// Row index within its system (batch): g mod sys_len, by a multiply-high when
// g and sys_len fit 32 bits (the host sets sys_magic) -- a 64-bit division per
// m-block otherwise costs Stage 1 ~6 % of its instructions.
__device__ __forceinline__ int64_t sys_rem(const TileCtx& t, int64_t g) {
  if (t.sys_magic) return (int64_t)__umul64hi(t.sys_magic * (uint64_t)g, (uint64_t)t.sys_len);
  return g % t.sys_len;
}

// Does the block starting at tile row lr0 (m rows) need any fix-up?
__device__ __forceinline__ bool block_needs_fixup(const TileCtx& t, int lr0, int m) {
  const int64_t g0 = t.row0 + lr0;
  if (g0 == 0 || g0 + m > t.n - (kBulkRows - 1)) return true;
  if (t.sys_len) {
    const int64_t rem = sys_rem(t, g0);
    return rem == 0 || rem + m > t.sys_len - 1;
  }
  return false;
}

__device__ __forceinline__ void fixup_row(const TileCtx& t, int lr, real& a, real& b,
                                          real& c, real& d) {
  if (lr >= t.valid) {
    a = 0.0;
    b = 1.0;
    c = 0.0;
    d = 0.0;
    return;
  }
  const int64_t g = t.row0 + lr;
  if (lr >= t.bulk_rows) {
    a = __ldg(t.ga + g);
    b = __ldg(t.gb + g);
    c = __ldg(t.gc + g);
    d = __ldg(t.gd + g);
  }
  if (t.zf && g == 0) a = 0.0;
  if (t.zl && g == t.n - 1) c = 0.0;
  if (t.sys_len) {
    const int64_t rem = sys_rem(t, g);
    if (rem == 0) a = 0.0;
    if (rem == t.sys_len - 1) c = 0.0;
  }
}

// Compile-time m: the block's rows live in registers.
template <int M>
struct RegAcc {
  real A[M], B[M], C[M], D[M];  // C/D are reused for c'/d' in Stage 3, B for x
  __device__ __forceinline__ real a(int j) const { return A[j]; }
  __device__ __forceinline__ real b(int j) const { return B[j]; }
  __device__ __forceinline__ real c(int j) const { return C[j]; }
  __device__ __forceinline__ real d(int j) const { return D[j]; }
  __device__ __forceinline__ void set_cp(int j, real v) { C[j] = v; }
  __device__ __forceinline__ real cp(int j) const { return C[j]; }
  __device__ __forceinline__ void set_dp(int j, real v) { D[j] = v; }
  __device__ __forceinline__ real dp(int j) const { return D[j]; }
  __device__ __forceinline__ void set_x(int j, real v) { B[j] = v; }
  __device__ __forceinline__ real x(int j) const { return B[j]; }
  __device__ __forceinline__ void set_b(int j, real v) { B[j] = v; }
  __device__ __forceinline__ void set_c(int j, real v) { C[j] = v; }

  __device__ __forceinline__ void load(const real* sa, const real* sb, const real* sc,
                                       const real* sd, int r0, const TileCtx& t) {
    if constexpr ((M % 2) == 0) {
      const real2* pa = reinterpret_cast<const real2*>(sa + r0);
      const real2* pb = reinterpret_cast<const real2*>(sb + r0);
      const real2* pc = reinterpret_cast<const real2*>(sc + r0);
      const real2* pd = reinterpret_cast<const real2*>(sd + r0);
#pragma unroll
      for (int j = 0; j < M / 2; ++j) {
        real2 va = pa[j], vb = pb[j], vc = pc[j], vd = pd[j];
        A[2 * j] = va.x; A[2 * j + 1] = va.y;
        B[2 * j] = vb.x; B[2 * j + 1] = vb.y;
        C[2 * j] = vc.x; C[2 * j + 1] = vc.y;
        D[2 * j] = vd.x; D[2 * j + 1] = vd.y;
      }
    } else {
#pragma unroll
      for (int j = 0; j < M; ++j) {
        A[j] = sa[r0 + j]; B[j] = sb[r0 + j]; C[j] = sc[r0 + j]; D[j] = sd[r0 + j];
      }
    }
    // rare: only blocks touching row 0, row n-1, a system boundary or the tail
    if (block_needs_fixup(t, r0, M)) {
#pragma unroll
      for (int j = 0; j < M; ++j) fixup_row(t, r0 + j, A[j], B[j], C[j], D[j]);
    }
  }
  // all four rows arrays back to the stage / raw reload (16-byte accesses:
  // conflict-free at stride m = 10, unlike 8-byte ones)
  __device__ __forceinline__ void store_rows(real* sa, real* sb, real* sc, real* sd,
                                             int r0) const {
    if constexpr ((M % 2) == 0) {
#pragma unroll
      for (int j = 0; j < M / 2; ++j) {
        reinterpret_cast<real2*>(sa + r0)[j] = make_real2(A[2 * j], A[2 * j + 1]);
        reinterpret_cast<real2*>(sb + r0)[j] = make_real2(B[2 * j], B[2 * j + 1]);
        reinterpret_cast<real2*>(sc + r0)[j] = make_real2(C[2 * j], C[2 * j + 1]);
        reinterpret_cast<real2*>(sd + r0)[j] = make_real2(D[2 * j], D[2 * j + 1]);
      }
    } else {
#pragma unroll
      for (int j = 0; j < M; ++j) {
        sa[r0 + j] = A[j]; sb[r0 + j] = B[j]; sc[r0 + j] = C[j]; sd[r0 + j] = D[j];
      }
    }
  }
  __device__ __forceinline__ void load_raw(const real* sa, const real* sb, const real* sc,
                                           const real* sd, int r0) {
    if constexpr ((M % 2) == 0) {
#pragma unroll
      for (int j = 0; j < M / 2; ++j) {
        const real2 va = reinterpret_cast<const real2*>(sa + r0)[j];
        const real2 vb = reinterpret_cast<const real2*>(sb + r0)[j];
        const real2 vc = reinterpret_cast<const real2*>(sc + r0)[j];
        const real2 vd = reinterpret_cast<const real2*>(sd + r0)[j];
        A[2 * j] = va.x; A[2 * j + 1] = va.y; B[2 * j] = vb.x; B[2 * j + 1] = vb.y;
        C[2 * j] = vc.x; C[2 * j + 1] = vc.y; D[2 * j] = vd.x; D[2 * j + 1] = vd.y;
      }
    } else {
#pragma unroll
      for (int j = 0; j < M; ++j) {
        A[j] = sa[r0 + j]; B[j] = sb[r0 + j]; C[j] = sc[r0 + j]; D[j] = sd[r0 + j];
      }
    }
  }
  __device__ __forceinline__ void store_x(real* xbuf, int r0) const {
    if constexpr ((M % 2) == 0) {
      real2* px = reinterpret_cast<real2*>(xbuf + r0);
#pragma unroll
      for (int j = 0; j < M / 2; ++j) px[j] = make_real2(B[2 * j], B[2 * j + 1]);
    } else {
#pragma unroll
      for (int j = 0; j < M; ++j) xbuf[r0 + j] = B[j];
    }
  }
};

// Runtime m: rows stay in the shared-memory stage; c'/d' overwrite c/d in
// place and x goes to the tile's x buffer.
struct SmemAcc {
  real* sa;
  real* sb;
  real* sc;
  real* sd;
  real* sx;
  __device__ __forceinline__ real a(int j) const { return sa[j]; }
  __device__ __forceinline__ real b(int j) const { return sb[j]; }
  __device__ __forceinline__ real c(int j) const { return sc[j]; }
  __device__ __forceinline__ real d(int j) const { return sd[j]; }
  __device__ __forceinline__ void set_cp(int j, real v) { sc[j] = v; }
  __device__ __forceinline__ real cp(int j) const { return sc[j]; }
  __device__ __forceinline__ void set_dp(int j, real v) { sd[j] = v; }
  __device__ __forceinline__ real dp(int j) const { return sd[j]; }
  __device__ __forceinline__ void set_x(int j, real v) { sx[j] = v; }
  __device__ __forceinline__ real x(int j) const { return sx[j]; }

  __device__ __forceinline__ void fixup(int r0, int m, const TileCtx& t) {
    if (block_needs_fixup(t, r0, m)) {
      for (int j = 0; j < m; ++j) {
        real a0 = sa[j], b0 = sb[j], c0 = sc[j], d0 = sd[j];
        fixup_row(t, r0 + j, a0, b0, c0, d0);
        sa[j] = a0; sb[j] = b0; sc[j] = c0; sd[j] = d0;
      }
    }
  }
};

// Compile-time m, rows left in the shared-memory stage (fewer registers):
// b/c slots are overwritten with 1/den and c' by block_reduce_fast<M, true>
// and b with x by block_interior_kept.
template <int M>
struct StageAcc {
  real* sa;
  real* sb;
  real* sc;
  real* sd;
  __device__ __forceinline__ real a(int j) const { return sa[j]; }
  __device__ __forceinline__ real b(int j) const { return sb[j]; }
  __device__ __forceinline__ real c(int j) const { return sc[j]; }
  __device__ __forceinline__ real d(int j) const { return sd[j]; }
  __device__ __forceinline__ void set_b(int j, real v) { sb[j] = v; }
  __device__ __forceinline__ void set_c(int j, real v) { sc[j] = v; }
  __device__ __forceinline__ real x(int j) const { return sb[j]; }
};

// Compile-time m, rows in the shared-memory stage, read as 16-byte pairs
// (even m, pair-aligned rows): at stride m = 10 doubles a 16-byte access is
// bank-conflict free where an 8-byte one is 2-way conflicted.  Within a
// store-free stretch the compiler merges the two loads of a pair.
template <int M>
struct PairAcc {
  const real* sa;
  const real* sb;
  const real* sc;
  const real* sd;
  __device__ __forceinline__ static real pick(const real* p, int j) {
    if constexpr ((M % 2) == 0) {
      const real2 v = *reinterpret_cast<const real2*>(p + (j & ~1));
      return (j & 1) ? v.y : v.x;
    } else {
      return p[j];
    }
  }
  __device__ __forceinline__ real a(int j) const { return pick(sa, j); }
  __device__ __forceinline__ real b(int j) const { return pick(sb, j); }
  __device__ __forceinline__ real c(int j) const { return pick(sc, j); }
  __device__ __forceinline__ real d(int j) const { return pick(sd, j); }
};

// Stage 3 of one block straight from the stage: continuant pivots (as in
// block_reduce_fast), forward substitution with x[s] = xs, x[e] = xe folded
// in, back-substitution; x[0..M) returned in registers (all shared-memory
// reads precede the caller's x stores).
template <int M>
__device__ __forceinline__ void block_solve_pairs(const PairAcc<M>& r, real xs, real xe,
                                                  real (&x)[M], bool& bad) {
  if constexpr (M == 2) {
    x[0] = xs;
    x[1] = xe;
  } else {
    constexpr int L = M - 2;
    real q[L + 1], inv[L + 1], dp[L + 1];
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
    if (!ok) {
      real cprev = 0.0;
#pragma unroll
      for (int j = 1; j <= L; ++j) {
        const real den = (j == 1) ? r.b(1) : fma(-r.a(j), cprev, r.b(j));
        bad |= (den == 0.0);
        inv[j] = drcp(den);
        cprev = r.c(j) * inv[j];
      }
    }
    dp[1] = fma(-r.a(1), xs, r.d(1)) * inv[1];
#pragma unroll
    for (int j = 2; j <= L; ++j) dp[j] = fma(-r.a(j), dp[j - 1], r.d(j)) * inv[j];
    dp[L] = fma(-(r.c(L) * inv[L]), xe, dp[L]);
    x[L] = dp[L];
#pragma unroll
    for (int j = L - 1; j >= 1; --j) x[j] = fma(-(r.c(j) * inv[j]), x[j + 1], dp[j]);
    x[0] = xs;
    x[M - 1] = xe;
  }
}

__device__ __forceinline__ int warp_node_off(int k) { return 32 - (32 >> k); }

// One downsweep level inside a warp: lanes that were left operands at
// stride `stride` split their (xf, xl) with the stored node and hand the
// right half to lane + stride.
__device__ __forceinline__ void down_level(const Node* nodes, int stride, int lane, int active,
                                           bool right_nonempty, real& xf, real& xl) {
  const bool left = lane < active && (lane & (2 * stride - 1)) == 0 && right_nonempty;
  real sf = 0.0, sl = 0.0;
  if (left) {
    real xl1, xf2;
    split_node(nodes[lane / (2 * stride)], xf, xl, xl1, xf2);
    sf = xf2;
    sl = xl;
    xl = xl1;
  }
  const real rf = __shfl_up_sync(0xffffffffu, sf, stride);
  const real rl = __shfl_up_sync(0xffffffffu, sl, stride);
  if (lane < active && (lane & (2 * stride - 1)) == stride) {
    xf = rf;
    xl = rl;
  }
}

__device__ __forceinline__ Seg warp_upsweep(Seg s, Node* nodes, int lane, int nblk, bool& bad) {
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    const int stride = 1 << k;
    Seg o = shfl_down_seg(s, stride);
    if ((lane & (2 * stride - 1)) == 0 && lane + stride < nblk) {
      Node nd;
      combine(s, o, s, nd, bad);
      if (nodes) nodes[warp_node_off(k) + (lane >> (k + 1))] = nd;
    }
  }
  return s;
}

__device__ __forceinline__ void warp_downsweep(real& xf, real& xl, const Node* nodes, int lane,
                                               int nblk) {
#pragma unroll
  for (int k = 4; k >= 0; --k)
    down_level(nodes + warp_node_off(k), 1 << k, lane, 32, lane + (1 << k) < nblk, xf, xl);
}

// Raises a kernel's dynamic shared-memory limit once per (kernel, device):
// cudaFuncSetAttribute applies to the current device only, so a per-thread
// or per-process flag would miss the second GPU of a multi-device process.
template <class K>
inline cudaError_t ensure_smem_attr(K kern, size_t smem) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> configured;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const auto key = std::make_pair(reinterpret_cast<const void*>(kern), dev);
  std::lock_guard<std::mutex> lock(mu);
  auto it = configured.find(key);
  if (it != configured.end() && it->second >= smem) return cudaSuccess;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess) configured[key] = smem;
  return e;
}

}  // namespace PM_NS
