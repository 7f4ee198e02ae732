// pm_batch.cu -- batches of independent systems with one thread-block cluster
// per system (BASELINE.json config 4: 4096 systems of 1e5 rows).
//
// The level kernels (pm_kernels.cu) solve a batch as one long system whose
// couplings are cut at the system boundaries: Stage 1 streams all of it, the
// upper levels run, Stage 3 streams all of it again -- 72 B of HBM traffic
// per unknown.  Here a cluster of CL CTAs owns one system at a time (a 1e5-row
// system is 3.2 MB) and runs all three stages on it before moving on, so the
// Stage-3 re-read of a, b, c, d is served from L2 and HBM sees only the
// compulsory 40 B per unknown:
//   phase A  (Stage 1) every warp reduces its 32*M-row tiles to tile
//            segments (warp tree, pm_tile.cuh) -> shared memory;
//   CTA      warp 0 reduces the CTA's contiguous tile range: per-lane chains
//            of tiles, then the warp tree -> one segment per CTA;
//   cluster  (Stage 2) after a cluster barrier every CTA reads the CL
//            segments from its peers' shared memory (DSMEM), chains them,
//            solves the final 2x2 and walks back to its own two boundary
//            values; the downsweep recovers every tile's two values;
//   phase C  (Stage 3) the warps re-read their tiles (L2 hits), split the
//            tile trees kept in shared memory since phase A down to the
//            blocks and back-substitute, storing x with coalesced 16-byte
//            stores (no Stage-1 recomputation, unlike the level kernels).
// Every warp streams one job sequence (phase A tiles, phase C tiles, next
// system ...) through its own ring of bulk-copy stages, so the loads of the
// first phase-C tiles are in flight across the CTA and cluster barriers.
// Clusters are persistent and stride over the systems; CL and the warps per
// CTA are chosen so that tiles divide evenly over the warps and the systems
// in flight (one per cluster) fit in L2.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <map>
#include <mutex>
#include <tuple>

#include "pm_batch.h"
#include "pm_device.cuh"
#include "pm_kernels.h"
#include "pm_tile.cuh"

namespace cg = cooperative_groups;

namespace pm {

namespace {

constexpr int kBatchMaxPerLane = 8;  // tiles per lane of the CTA chain (CTA <= 256 tiles)

__host__ __device__ inline size_t batch_warp_bytes(int m, int stages) {
  const size_t T = (size_t)32 * m;
  const size_t b = (size_t)stages * 4 * T * sizeof(double) + 2 * kMaxStages * sizeof(uint64_t);
  return (b + 127) / 128 * 128;
}

// CTA region: tile boundary values, tile segments (kmax each), two cluster
// slots, per-lane chain nodes (kmax), the CTA warp-tree nodes, and the 31
// warp-tree nodes of every tile (kept from phase A for phase C).
__host__ __device__ inline size_t batch_cta_bytes(int kmax) {
  return (size_t)kmax * (sizeof(Seg) + sizeof(Node) + sizeof(double2) + 31 * sizeof(Node)) +
         31 * sizeof(Node) + 2 * sizeof(Seg);
}

template <int M>
__global__ void __launch_bounds__(512, 1) batch_cluster_kernel(BatchArgs args) {
  constexpr int T = 32 * M;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  cg::cluster_group cluster = cg::this_cluster();
  const int CL = (int)cluster.num_blocks();
  const int rank = (int)cluster.block_rank();
  const int ncl = gridDim.x / CL;
  const int cid = blockIdx.x / CL;
  const int lane = threadIdx.x & 31;
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
  const int W = blockDim.x >> 5;
  const int S = args.stages;
  const int r0 = lane * M;

  // this CTA's contiguous tile range of every system
  const int ntiles = args.ntiles;
  const int t0 = (int)((int64_t)ntiles * rank / CL);
  const int K = (int)((int64_t)ntiles * (rank + 1) / CL) - t0;
  const int cnt = (K > warp) ? (K - warp + W - 1) / W : 0;  // tiles of this warp
  const int kmax = args.kmax;

  const size_t per_warp = batch_warp_bytes(M, S);
  unsigned char* base = smem_raw + per_warp * warp;
  double* stage0 = reinterpret_cast<double*>(base);
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + per_warp - 2 * kMaxStages * sizeof(uint64_t));
  unsigned char* cta = smem_raw + per_warp * W;
  double2* txy = reinterpret_cast<double2*>(cta);  // 16-byte aligned first
  Seg* tseg = reinterpret_cast<Seg*>(txy + kmax);
  Seg* slot = tseg + kmax;  // [2]: cluster exchange, by system parity
  Node* lnode = reinterpret_cast<Node*>(slot + 2);
  Node* wnode = lnode + kmax;
  Node* tnode = wnode + 31;  // [kmax][31]: warp-tree nodes of every tile of the CTA

  const int64_t nsys = (args.batch > cid) ? (args.batch - cid + ncl - 1) / ncl : 0;
  const int64_t njobs = nsys * 2 * cnt;
  auto stage_ptr = [&](int s, int q) -> double* { return stage0 + ((size_t)s * 4 + q) * T; };
  // job k -> (system, tile): per system cnt phase-A tiles, then the same cnt tiles again
  auto job_rows = [&](int64_t k, int64_t& sys, int& tile) {
    const int64_t it = k / (2 * cnt);
    const int i = (int)(k % (2 * cnt)) % cnt;
    sys = cid + it * ncl;
    tile = t0 + warp + i * W;
  };
  auto issue = [&](int s, int64_t k) {
    int64_t sys;
    int tile;
    job_rows(k, sys, tile);
    const int64_t row0 = sys * args.n_sys + (int64_t)tile * T;
    const int64_t rem = args.n_sys - (int64_t)tile * T;
    const int64_t v = rem < T ? rem : T;
    const uint32_t bytes = static_cast<uint32_t>((v & ~int64_t(kBulkRows - 1)) * sizeof(real));
    fence_proxy_async();
    mbar_arrive_expect_tx(&bars[s], 4u * bytes);
    if (bytes) {
      bulk_g2s(stage_ptr(s, 0), args.a + row0, bytes, &bars[s]);
      bulk_g2s(stage_ptr(s, 1), args.b + row0, bytes, &bars[s]);
      bulk_g2s(stage_ptr(s, 2), args.c + row0, bytes, &bars[s]);
      bulk_g2s(stage_ptr(s, 3), args.d + row0, bytes, &bars[s]);
    }
  };
  auto make_ctx = [&](int64_t sys, int tile) {
    TileCtx ctx;
    const int64_t off = sys * args.n_sys;
    ctx.ga = args.a + off; ctx.gb = args.b + off; ctx.gc = args.c + off; ctx.gd = args.d + off;
    ctx.row0 = (int64_t)tile * T;
    ctx.n = args.n_sys;
    ctx.valid = static_cast<int>((args.n_sys - ctx.row0 < T) ? (args.n_sys - ctx.row0) : T);
    ctx.bulk_rows = ctx.valid & ~(kBulkRows - 1);
    ctx.zf = true;
    ctx.zl = true;
    ctx.sys_len = 0;
    ctx.sys_magic = 0;
    return ctx;
  };

  if (lane == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncwarp();
  pdl_wait();
  pdl_launch_dependents();
  if (lane == 0)
    for (int s = 0; s < S && s < njobs; ++s) issue(s, s);

  // per-lane chains of the CTA's tiles (warp 0)
  const int C = (K + 31) / 32;
  const int nl = C > 0 ? (K + C - 1) / C : 0;   // non-empty lanes
  const int lt0 = lane * C;
  const int lcnt = (K - lt0 < C) ? ((K - lt0 > 0) ? K - lt0 : 0) : C;

  bool bad = false;
  int64_t k = 0;
  for (int64_t it = 0; it < nsys; ++it) {
    const int64_t sys = cid + it * ncl;
    // ---- phase A: Stage 1 of this warp's tiles ------------------------------
    for (int i = 0; i < cnt; ++i, ++k) {
      const int s = static_cast<int>(k % S);
      const int tile = t0 + warp + i * W;
      const TileCtx ctx = make_ctx(sys, tile);
      double* sa = stage_ptr(s, 0);
      double* sb = stage_ptr(s, 1);
      double* sc = stage_ptr(s, 2);
      double* sd = stage_ptr(s, 3);
      mbar_wait(&bars[s], static_cast<uint32_t>((k / S) & 1));
      SmemAcc sacc{sa + r0, sb + r0, sc + r0, sd + r0, nullptr};
      sacc.fixup(r0, M, ctx);
      const PairAcc<M> pa{sa + r0, sb + r0, sc + r0, sd + r0};
      const Seg seg = block_reduce_fast<M, false>(pa, bad);
      __syncwarp();
      if (lane == 0 && k + S < njobs) issue(s, k + S);  // stage released
      const Seg top = warp_upsweep(seg, tnode + 31 * (tile - t0), lane, 32, bad);
      if (lane == 0) tseg[tile - t0] = top;
    }
    __syncthreads();
    // ---- CTA: reduce the CTA's K tile segments to one ----------------------
    const int p = static_cast<int>(it & 1);
    if (warp == 0) {
      Seg acc{};
      if (lcnt > 0) {
        acc = tseg[lt0];
        for (int j = 1; j < lcnt; ++j) combine(acc, tseg[lt0 + j], acc, lnode[lt0 + j], bad);
      }
      const Seg top = warp_upsweep(acc, wnode, lane, nl, bad);
      if (lane == 0) slot[p] = top;
    }
    // ---- cluster: Stage 2 over the CL segments (DSMEM) ---------------------
    cluster.sync();
    if (warp == 0) {
      double xf = 0.0, xl = 0.0;
      if (lane == 0) {
        Node cn[16];
        Seg acc = *cluster.map_shared_rank(&slot[p], 0);
        for (int q = 1; q < CL; ++q) combine(acc, *cluster.map_shared_rank(&slot[p], q), acc, cn[q], bad);
        // acc.F.a and acc.L.c multiply unknowns outside the system (zero)
        const double det = fma(acc.F.b, acc.L.b, -acc.F.c * acc.L.a);
        bad |= (det == 0.0);
        const double inv = drcp(det);
        const double x0 = fma(acc.F.d, acc.L.b, -acc.F.c * acc.L.d) * inv;
        double xr = fma(acc.F.b, acc.L.d, -acc.L.a * acc.F.d) * inv;
        double xfr = x0;
        for (int q = CL - 1; q >= 1 && q >= rank; --q) {
          double xl_prev, xf_q;
          split_node(cn[q], x0, xr, xl_prev, xf_q);
          if (q == rank) {
            xfr = xf_q;
            break;
          }
          xr = xl_prev;
        }
        xf = xfr;
        xl = xr;
      }
      xf = __shfl_sync(0xffffffffu, xf, 0);
      xl = __shfl_sync(0xffffffffu, xl, 0);
      warp_downsweep(xf, xl, wnode, lane, nl);
      // walk this lane's chain back to its tiles
      if (lcnt > 0) {
        double xrun = xl;
        for (int j = lcnt - 1; j >= 1; --j) {
          double xl_prev, xf_j;
          split_node(lnode[lt0 + j], xf, xrun, xl_prev, xf_j);
          txy[lt0 + j] = make_double2(xf_j, xrun);
          xrun = xl_prev;
        }
        txy[lt0] = make_double2(xf, xrun);
      }
    }
    __syncthreads();
    // ---- phase C: Stage 3 of the same tiles (L2-resident) -------------------
    for (int i = 0; i < cnt; ++i, ++k) {
      const int s = static_cast<int>(k % S);
      const int tile = t0 + warp + i * W;
      const TileCtx ctx = make_ctx(sys, tile);
      double* sa = stage_ptr(s, 0);
      double* sb = stage_ptr(s, 1);
      double* sc = stage_ptr(s, 2);
      double* sd = stage_ptr(s, 3);
      mbar_wait(&bars[s], static_cast<uint32_t>((k / S) & 1));
      SmemAcc sacc{sa + r0, sb + r0, sc + r0, sd + r0, nullptr};
      sacc.fixup(r0, M, ctx);
      const PairAcc<M> pa{sa + r0, sb + r0, sc + r0, sd + r0};
      // the tile tree was built in phase A: split it straight down to the blocks
      const double2 bv = txy[tile - t0];
      double xf = bv.x, xl = bv.y;
      warp_downsweep(xf, xl, tnode + 31 * (tile - t0), lane, 32);
      double xv[M];
      block_solve_pairs<M>(pa, xf, xl, xv, bad);
      __syncwarp();
      bad |= !all_finite<M>(xv);
      if constexpr ((M % 2) == 0) {
#pragma unroll
        for (int j = 0; j < M / 2; ++j)
          reinterpret_cast<double2*>(sb + r0)[j] = make_double2(xv[2 * j], xv[2 * j + 1]);
      } else {
#pragma unroll
        for (int j = 0; j < M; ++j) sb[r0 + j] = xv[j];
      }
      __syncwarp();
      double* gx = args.x + sys * args.n_sys + ctx.row0;
      const int v = ctx.valid;
      if ((v & 1) == 0 && ((reinterpret_cast<uintptr_t>(gx) & 15) == 0)) {
        const double2* s2 = reinterpret_cast<const double2*>(sb);
        double2* g2 = reinterpret_cast<double2*>(gx);
        for (int q = lane; q < v / 2; q += 32) g2[q] = s2[q];
      } else {
        for (int q = lane; q < v; q += 32) gx[q] = sb[q];
      }
      __syncwarp();
      if (lane == 0 && k + S < njobs) issue(s, k + S);
    }
  }
  cluster.sync();  // peers may still read this CTA's slots
  if (bad) atomicOr(args.flag, 1);
}

template <int M>
cudaError_t launch_m(const BatchArgs& a0, const BatchPlan& pl, cudaStream_t st) {
  BatchArgs a = a0;
  a.stages = pl.stages;
  a.kmax = pl.kmax;
  a.ntiles = pl.ntiles;
  auto kern = batch_cluster_kernel<M>;
  const size_t smem = batch_warp_bytes(M, pl.stages) * pl.warps + batch_cta_bytes(pl.kmax);
  cudaError_t e = ensure_smem_attr(kern, smem);
  if (e != cudaSuccess) return e;
  if (pl.cluster > 8) {  // clusters of 9-16 CTAs are a B200 opt-in
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(pl.clusters * pl.cluster);
  cfg.blockDim = dim3(32 * pl.warps);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = pl.cluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, kern, a);
}

template <int M>
int max_clusters(int cluster, int warps, int stages, int kmax) {
  static std::mutex mu;
  static std::map<std::tuple<int, int, int, int, int>, int> cache;  // + device
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_tuple(dev, cluster, warps, stages, kmax);
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  auto kern = batch_cluster_kernel<M>;
  const size_t smem = batch_warp_bytes(M, stages) * warps + batch_cta_bytes(kmax);
  int n = 0;
  if (smem <= 227 * 1024 && ensure_smem_attr(kern, smem) == cudaSuccess &&
      (cluster <= 8 ||
       cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess)) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cluster);
    cfg.blockDim = dim3(32 * warps);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cluster;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) n = 0;
  }
  cudaGetLastError();
  cache[key] = n;
  return n;
}

int max_clusters_m(int m, int cluster, int warps, int stages, int kmax) {
  switch (m) {
    case 2: return max_clusters<2>(cluster, warps, stages, kmax);
    case 8: return max_clusters<8>(cluster, warps, stages, kmax);
    case 10: return max_clusters<10>(cluster, warps, stages, kmax);
    case 16: return max_clusters<16>(cluster, warps, stages, kmax);
    default: return 0;
  }
}

}  // namespace

bool batch_cluster_supported(int m) { return m == 2 || m == 8 || m == 10 || m == 16; }

// Plan: minimise the modelled time  rounds * max_tiles_per_warp * warps
// (the kernel is instruction-issue-bound per SM; a phase lasts as long as its
// busiest warp) subject to: systems in flight (one per cluster) fit the L2
// budget, the CTA's tile range fits the per-lane chains, the CTA fits one SM.
int plan_batch(int m, int64_t n_sys, int64_t batch, int sm_count, int64_t l2_budget, int force_cluster,
               int force_warps, int force_stages, BatchPlan* out) {
  if (!batch_cluster_supported(m) || n_sys < 2 || (n_sys & 1)) return 0;
  const int64_t T = 32 * (int64_t)m;
  const int64_t nt = (n_sys + T - 1) / T;
  if (nt < 2) return 0;
  const double sys_bytes = 32.0 * (double)n_sys;
  double best = 1e300;
  BatchPlan bp{};
  for (int S = 1; S <= 2; ++S) {
    if (force_stages > 0 && S != force_stages) continue;
    // 9-16 CTA clusters only when forced: on B200 they place at most 14 (2
    // CTAs per SM) and measured slower (round 1: 8.2 ms at CL = 16 vs 6.1 ms
    // at CL = 8 for 4096 x 1e5)
    for (int CL = 1; CL <= (force_cluster > 8 ? 16 : 8); ++CL) {
      if (force_cluster > 0 && CL != force_cluster) continue;
      if (CL > nt) break;
      const int kmax = (int)((nt + CL - 1) / CL);
      if (kmax > 32 * kBatchMaxPerLane) continue;
      for (int W = 4; W <= 16; ++W) {
        if (force_warps > 0 && W != force_warps) continue;
        const int mc = max_clusters_m(m, CL, W, S, kmax);
        if (mc < 1) continue;
        int64_t ncl = std::min<int64_t>(mc, batch);
        // systems in flight must fit the L2 budget
        const int64_t fit = std::max<int64_t>(1, (int64_t)(l2_budget / sys_bytes));
        if (ncl > fit) ncl = fit;
        const int64_t rounds = (batch + ncl - 1) / ncl;
        const int64_t per_warp = (kmax + W - 1) / W;
        // issue-bound per SM: a phase lasts as long as its
        // busiest warp, and the W warps of an SM share its issue slots
        const double t = (double)rounds * (double)per_warp * W;
        // prefer more warps (latency hiding) and then fewer stages on ties
        const double score = t * (1.0 + 0.002 * (16 - W)) * (1.0 + 0.001 * S);
        if (score < best) {
          best = score;
          bp.cluster = CL;
          bp.warps = W;
          bp.stages = S;
          bp.kmax = kmax;
          bp.ntiles = (int)nt;
          bp.clusters = (int)ncl;
        }
      }
    }
  }
  if (best == 1e300) return 0;
  *out = bp;
  return 1;
}

cudaError_t launch_batch_cluster(int m, const BatchArgs& args, const BatchPlan& pl, cudaStream_t st) {
  switch (m) {
    case 2: return launch_m<2>(args, pl, st);
    case 8: return launch_m<8>(args, pl, st);
    case 10: return launch_m<10>(args, pl, st);
    case 16: return launch_m<16>(args, pl, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace pm
