// pm_batch.h -- launch interface of the cluster kernel for batches of
// independent systems (pm_batch.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace pm {

struct BatchArgs {
  const double* a = nullptr;  // batch systems stored back to back, n_sys rows each
  const double* b = nullptr;
  const double* c = nullptr;
  const double* d = nullptr;
  double* x = nullptr;
  int64_t n_sys = 0;
  int64_t batch = 0;
  int ntiles = 0;  // tiles (32*m rows) per system
  int kmax = 0;    // max tiles per CTA
  int stages = 1;  // bulk-copy ring depth per warp
  int* flag = nullptr;
};

struct BatchPlan {
  int cluster = 1;   // CTAs per cluster (one system per cluster at a time)
  int warps = 8;     // warps per CTA
  int stages = 1;
  int kmax = 0;
  int ntiles = 0;
  int clusters = 0;  // persistent clusters launched
};

bool batch_cluster_supported(int m);
// Returns 1 and fills *out when the cluster kernel applies (compile-time m,
// even n_sys, at least two tiles per system, a CTA range of <= 256 tiles).
// force_* > 0 pin the cluster size / warps / stages (experiments).
int plan_batch(int m, int64_t n_sys, int64_t batch, int sm_count, int64_t l2_budget, int force_cluster,
               int force_warps, int force_stages, BatchPlan* out);
cudaError_t launch_batch_cluster(int m, const BatchArgs& args, const BatchPlan& plan, cudaStream_t st);

// ---- the tile-stream kernel (pm_batch_stream.cu) ----------------------------
// Per-system counters and flags sit kStreamCounterStride words apart (one
// 128-byte L2 line each): ~1000 warps poll the flags of the few systems in
// flight, and packed 32 to a line those polls, the Stage-1/Stage-3 atomics and
// the Stage-2 releases all hit one L2 slice.
constexpr int kStreamCounterStride = 32;
struct StreamArgs {
  const double* a = nullptr;  // batch systems stored back to back, n_sys rows each
  const double* b = nullptr;
  const double* c = nullptr;
  const double* d = nullptr;
  double* x = nullptr;
  int64_t n_sys = 0;
  int64_t batch = 0;
  int m = 0;
  int tps = 0;  // tiles (32*m rows) per system
  int nw = 0;   // compute warps in the grid
  int W = 0;    // compute warps per CTA (+ one control warp)
  int S = 0;    // bulk-copy stages per compute warp
  int L = 0;    // lag of Stage 3 behind Stage 1, in rounds of nw tiles (minimum)
  int Lmax = 0; // ... maximum (run-ahead while a system's Stage 2 is pending)
  int K = 0;    // ring depth in rounds (> L)
  uint64_t mg_tps = 0, mg_K = 0, mg_period = 0;  // ceil(2^64 / d) of tps, K, K*nw (0: d = 1)
  double* segs = nullptr;          // [K*nw] tile segments (8 doubles)
  double* txy = nullptr;           // [K*nw] tile boundary values (2 doubles)
  unsigned char* nodes = nullptr;  // [K*nw] tile tree nodes (1792 B)
  unsigned* cnt1 = nullptr;        // [batch][stride] Stage-1 tiles published
  unsigned* cnt3 = nullptr;        // [batch][stride] Stage-3 tiles done
  unsigned* sflag = nullptr;       // [batch][stride] Stage 2 done
  int* flag = nullptr;
  int discard = 1;  // discard.global.L2 on consumed node-ring lines
  int hints = 1;    // L2 eviction priorities on the bulk copies
  int early = 0;    // one stage per warp: issue the next tile's copies inside the current job
  int ooo = 0;      // control warp publishes ready segments out of round order
  unsigned long long* stats = nullptr;  // [15] diagnostics (PM_OPT_BATCH_STATS) or null
  unsigned long long* tl = nullptr;     // [5][batch] per-system timeline (with stats)
};

struct StreamPlan {
  int warps = 0;   // compute warps per CTA
  int stages = 0;
  int lag = 0;
  int lag_max = 0;
  int ring = 0;
  int ctas = 0;    // one per SM
  int nw = 0;
  int tps = 0;
};

// Returns 1 and fills *out when the tile-stream kernel applies (compile-time
// m, even n_sys, >= lag rounds of tiles per warp); force_* > 0 pin the plan.
// (max_ctas > 0 caps the grid: PM_OPT_MAX_CTAS)
int plan_stream(int m, int64_t n_sys, int64_t batch, int sm_count, int max_ctas, int force_warps,
                int force_stages, int force_lag, StreamPlan* out);
// device scratch: rings + per-system counters (zeroed once at allocation)
size_t stream_scratch_bytes(const StreamPlan& pl, int64_t batch);
// the division magic of StreamArgs: ceil(2^64 / d), 0 for d = 1
inline uint64_t stream_magic(uint32_t d) { return d <= 1 ? 0 : ~uint64_t{0} / d + 1; }
cudaError_t launch_batch_stream(int m, const StreamArgs& args, const StreamPlan& plan, cudaStream_t st);

}  // namespace pm
