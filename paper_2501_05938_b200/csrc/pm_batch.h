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

}  // namespace pm
