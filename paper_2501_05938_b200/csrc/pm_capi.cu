// pm_capi.cu -- host orchestration behind the C ABI of include/pm_tridiag.h.
//
// Level plan.  Level 0 is the caller's system (m = the sub-system size).
// Every REDUCE launch turns each CTA tile of level L into two rows of level
// L+1, so level sizes shrink by T/2 (640x for m = 10); the level whose tiles
// number one is solved by a single ROOT launch.  Upper levels use m = 8
// (m = 2 on ranks of a row-sharded solve that are not the last, see
// pm_dist_*).  A solve is therefore
//     REDUCE(0) .. REDUCE(top-1), ROOT(top), SOLVE(top-1) .. SOLVE(0)
// e.g. N = 8e7, m = 10: 8e7 -> 125000 -> 246 rows, five launches.
//
// Streams.  pm_solve_host_f64 splits the
// level-0 tiles into num_streams chunks: per chunk H2D(a,b,c,d) -> REDUCE(0)
// on its own stream; the upper levels on the main stream after a join;
// then per chunk SOLVE(0) -> D2H(x).  The reduced system never leaves the
// device, so the paper's T1^D2H and T3^H2D are zero here.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <functional>
#include <type_traits>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "pm_batch.h"
#include "pm_kernels.h"
#include "pm_nccl.h"
#include "pm_tridiag.h"
#include "streamtune/predictor.hpp"

namespace {

// bumped whenever PM_OPT_PDL changes the process-wide launch attribute
std::atomic<uint64_t> g_pdl_gen{0};


struct Level {
  int64_t n = 0;
  int m = 10;
  int P = 128;
  int64_t T = 0;
  int64_t ntiles = 0;
  const void* a = nullptr;  // arrays of the level's precision (Prec<R>::Real)
  const void* b = nullptr;
  const void* c = nullptr;
  const void* d = nullptr;
  void* x = nullptr;
  bool bulk = true;
  int pad_mode = 1;
  int stages = 2;
  int warps_per_cta = 0;  // > 0: warp-tile kernel (P = 32 rows-blocks per tile)
  bool pair = false;      // level-0 pair-tile kernel (P = 64, two blocks per lane)
};

constexpr size_t kSmemLimit = 226 * 1024;

int choose_P(int m) {
  if (m <= 16) return 128;
  if (m <= 32) return 64;
  return 32;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// The kernels of one precision: pm (FP64, the north_star solver) and pm32
// (FP32, the paper's FP32 experiments).
template <class R>
struct Prec;
template <>
struct Prec<double> {
  using Args = pm::TileArgs;
  using Node = pm::Node;
  static cudaError_t warp(int mode, const Args& a, int w, int sm, cudaStream_t st, int* g) {
    return pm::launch_warp_tile_kernel(mode, a, w, sm, st, g);
  }
  static cudaError_t tile(int mode, const Args& a, int P, bool bulk, int sm, cudaStream_t st, int* g) {
    return pm::launch_tile_kernel(mode, a, P, bulk, sm, st, g);
  }
  static int ctas(int mode, int m, int stages, int w, bool chain) {
    return pm::warp_kernel_ctas_per_sm(mode, m, stages, w, chain);
  }
  static size_t tile_smem(int mode, int P, int m, int S) { return pm::tile_smem_bytes(mode, P, m, S); }
  static size_t warp_smem(int mode, int m, int S) { return pm::warp_smem_bytes(mode, m, S); }
  static cudaError_t pair(int mode, const Args& a, int w, int sm, cudaStream_t st, int* g) {
    return pm::launch_warp_pair_kernel(mode, a, w, sm, st, g);
  }
  static size_t pair_smem(int m, int S) { return pm::pair_smem_bytes(m, S); }
  using UpperArgs = pm::UpperArgs;
  static int upper_capacity(int sm) { return pm::upper_fused_capacity(sm); }
  static cudaError_t upper(const UpperArgs& u, int sm, cudaStream_t st, int* g) {
    return pm::launch_upper_fused(u, sm, st, g);
  }
  static cudaError_t dist_chain(const double* ia, int w, int r, double* xb, int* f, cudaStream_t st) {
    return pm::launch_dist_chain(ia, w, r, xb, f, st);
  }
  using DistUpperArgs = pm::DistUpperArgs;
  static int dist_upper_capacity(int sm) { return pm::dist_upper_capacity(sm); }
  static size_t dist_tree2_bytes() { return pm::dist_tree2_bytes(); }
  static cudaError_t dist_upper(int mode, const DistUpperArgs& u, int sm, cudaStream_t st, int* g) {
    return pm::launch_dist_upper(mode, u, sm, st, g);
  }
  static cudaError_t generate(double* a, double* b, double* c, double* d, int64_t n, int64_t r0,
                              int64_t cnt, uint64_t seed, int sm, cudaStream_t st) {
    return pm::launch_generate(a, b, c, d, n, r0, cnt, seed, sm, st);
  }
};
template <>
struct Prec<float> {
  using Args = pm32::TileArgs;
  using Node = pm32::Node;
  static cudaError_t warp(int mode, const Args& a, int w, int sm, cudaStream_t st, int* g) {
    return pm32::launch_warp_tile_kernel(mode, a, w, sm, st, g);
  }
  static cudaError_t tile(int mode, const Args& a, int P, bool bulk, int sm, cudaStream_t st, int* g) {
    return pm32::launch_tile_kernel(mode, a, P, bulk, sm, st, g);
  }
  static int ctas(int mode, int m, int stages, int w, bool chain) {
    return pm32::warp_kernel_ctas_per_sm(mode, m, stages, w, chain);
  }
  static size_t tile_smem(int mode, int P, int m, int S) { return pm32::tile_smem_bytes(mode, P, m, S); }
  static size_t warp_smem(int mode, int m, int S) { return pm32::warp_smem_bytes(mode, m, S); }
  static cudaError_t pair(int mode, const Args& a, int w, int sm, cudaStream_t st, int* g) {
    return pm32::launch_warp_pair_kernel(mode, a, w, sm, st, g);
  }
  static size_t pair_smem(int m, int S) { return pm32::pair_smem_bytes(m, S); }
  using UpperArgs = pm32::UpperArgs;
  static int upper_capacity(int sm) { return pm32::upper_fused_capacity(sm); }
  static cudaError_t upper(const UpperArgs& u, int sm, cudaStream_t st, int* g) {
    return pm32::launch_upper_fused(u, sm, st, g);
  }
  static cudaError_t dist_chain(const float* ia, int w, int r, float* xb, int* f, cudaStream_t st) {
    return pm32::launch_dist_chain(ia, w, r, xb, f, st);
  }
  using DistUpperArgs = pm32::DistUpperArgs;
  static int dist_upper_capacity(int sm) { return pm32::dist_upper_capacity(sm); }
  static size_t dist_tree2_bytes() { return pm32::dist_tree2_bytes(); }
  static cudaError_t dist_upper(int mode, const DistUpperArgs& u, int sm, cudaStream_t st, int* g) {
    return pm32::launch_dist_upper(mode, u, sm, st, g);
  }
  static cudaError_t generate(float* a, float* b, float* c, float* d, int64_t n, int64_t r0,
                              int64_t cnt, uint64_t seed, int sm, cudaStream_t st) {
    return pm32::launch_generate(a, b, c, d, n, r0, cnt, seed, sm, st);
  }
};

}  // namespace

struct pm_handle_s {
  int device = 0;
  int sm_count = 148;
  std::string err;
  // options
  int stages = 2;
  int stream_mode = 0;
  int reverse = 1;
  int max_ctas = 0;
  int timings = 0;
  int warp_tiles = 1;
  int solve_stages = 1;   // level-0 Stage 3 ring depth (0 = same as `stages`)
  int warps_per_cta = 4;
  int pair_tiles = -1;  // PM_OPT_PAIR_TILES: -1 auto (FP32 on, FP64 off)
  int pair_stages = 1;  // PM_OPT_PAIR_STAGES: ring depth of the pair-tile Stage 1
  // batch cluster kernel
  int batch_cluster = 0;
  int batch_l2_mb = 64;
  int batch_force_cluster = 0;
  int batch_force_warps = 0;
  int batch_force_stages = 0;
  pm::BatchPlan last_batch_plan{0, 0, 0, 0, 0, 0};
  // tile-stream batch kernel (PM_OPT_BATCH_CLUSTER = 2)
  int batch_lag = 0;       // PM_OPT_BATCH_LAG (0 = plan)
  int batch_discard = 15;  // PM_OPT_BATCH_DISCARD: bit 0 discard, 1 L2 hints, 2 early issue, 3 out-of-order publish
  char* bscr = nullptr;    // node / segment / boundary-value rings
  size_t bscr_bytes = 0;
  char* bcnt = nullptr;    // per-system counters and flags, zero between launches
  size_t bcnt_bytes = 0;
  pm::StreamPlan last_stream_plan{};
  int batch_stats = 0;                    // PM_OPT_BATCH_STATS
  unsigned long long* dstats = nullptr;   // [15] tile-stream diagnostics + [5][batch] timeline
  size_t dstats_words = 0;
  int64_t dstats_batch = 0;
  // device scratch for upper levels (+ dist boundary values)
  char* scratch = nullptr;  // level arrays of the current solve's precision
  size_t scratch_bytes = 0;
  int* dflag = nullptr;
  unsigned long long* dsync = nullptr;  // counters of the fused upper-level kernel
  int upper_fused = 1;                  // PM_OPT_UPPER_FUSED
  int upper_cap[2] = {-1, -1};          // its co-resident CTAs (FP64, FP32; -1: not queried)
  // row-sharded ranks: level 1 + the chain of its tile segments in two
  // launches (pm::launch_dist_upper); set by build_plan
  bool dist_fused = false;
  int dist_chain = 1;                   // level-2 segments per thread
  void* dist_seg2 = nullptr;            // [G][8] | [G][8] nodes | [G][2] x, in the level scratch
  int dist_cap[2] = {-1, -1};
  // device staging for the host path: a, b, c, d, x
  char* hbuf = nullptr;
  size_t hbuf_bytes = 0;
  std::vector<cudaStream_t> pool;
  cudaStream_t main = nullptr;
  cudaStream_t last_stream = nullptr;
  streamtune::ModelBundle bundle = streamtune::ModelBundle::b200();
  pm_stage_timings last_t{};
  double last_total_ms = 0.0;
  int last_streams = 0;
  int launches = 0;
  std::vector<Level> levels;
  // chain mode (level 0 warp tiles): per part (stream chunk) chunk counts
  bool chain = false;
  int nparts = 1;
  int opt_chain = 0;
  int upper_m = 0;   // warp-tile m of the upper levels (0: CTA tiles, m = 8)
  int root_m = 8;    // ROOT tile: 128 * root_m rows
  int upper_cta_m = 8;    // CTA-tile upper levels: rows per thread
  int upper_cta_p = 128;  // ... and threads per CTA tile
  std::vector<int64_t> part_chunks, part_base;
  void* chain_nodes = nullptr;
  // P2P interface exchange (pm_dist_*_p2p): this rank's exchange buffer,
  // the peers' buffers (device array), the rank's interface equations
  char* xbuf = nullptr;
  int xbuf_world = 0;
  void** d_peers = nullptr;
  int xworld = 0, xrank = -1;
  uint64_t epoch = 0;
  void* iface_local = nullptr;
  void* coll_buf = nullptr;  // pm_solve_dist_*: [8 | 8*world] reals (iface, iface_all)
  size_t coll_bytes = 0;
  // set while a pm_dist_*_p2p call enqueues its top level: that launch
  // publishes (REDUCE) or acquires and chains (SOLVE) the interface rows itself
  struct P2PTop {
    bool active = false;
    uint64_t epoch = 0;
  } p2p_top;
  // CUDA graphs of device-resident solves (PM_OPT_GRAPHS): one executable
  // graph per (precision, arrays, sizes, plan generation, scratch) key
  int use_graphs = 0;
  uint64_t plan_gen = 0;  // bumped by every pm_set_option
  struct GraphEntry {
    size_t esz;
    const void* p[5];
    int64_t n, nps;
    int m;
    uint64_t gen, pdl_gen;
    const void* scratch;
    cudaGraphExec_t exec;
    int launches;
    uint64_t last_use;
  };
  std::vector<GraphEntry> graphs;
  uint64_t graph_clock = 0;
  // pivot-failure retry: a solve whose fast (continuant) pivots leave the
  // FP range for extremely scaled rows is re-run once with classic sweeps
  int robust_mode = 0;
  std::function<int()> retry;  // re-enqueues the last device-resident solve
  cudaStream_t retry_stream = nullptr;
  // per-launch CUDA-event timing (PM_OPT_KERNEL_TIMES)
  int ktimes = 0;
  std::vector<cudaEvent_t> kev;
  struct KRec { int mode, level; size_t ev; };
  std::vector<KRec> krec;
};

namespace {

int fail(pm_handle_t h, int code, const std::string& msg) {
  if (h) h->err = msg;
  return code;
}

int cuda_fail(pm_handle_t h, cudaError_t e, const char* what) {
  return fail(h, PM_ERR_RUNTIME, std::string(what) + ": " + cudaGetErrorString(e));
}

#define PM_CUDA(h, call)                                     \
  do {                                                       \
    cudaError_t e_ = (call);                                 \
    if (e_ != cudaSuccess) return cuda_fail((h), e_, #call); \
  } while (0)

int ensure_scratch(pm_handle_t h, size_t bytes) {
  if (bytes <= h->scratch_bytes) return PM_OK;
  if (h->scratch) {
    PM_CUDA(h, cudaDeviceSynchronize());
    PM_CUDA(h, cudaFree(h->scratch));
    h->scratch = nullptr;
    h->scratch_bytes = 0;
  }
  const size_t want = std::max(bytes, (size_t)1 << 20);
  PM_CUDA(h, cudaMalloc(&h->scratch, want));
  h->scratch_bytes = want;
  return PM_OK;
}

template <class R>
int pick_stages(int want, int P, int m) {
  int S = std::max(1, std::min(want, 4));
  while (S > 1 && Prec<R>::tile_smem(pm::kModeSolve, P, m, S) > kSmemLimit) --S;
  return S;
}

// Warp-tile configuration of a level: ring depth and as many warps per CTA
// (<= PM_OPT_WARPS_PER_CTA) as the shared memory allows.
template <class R>
void set_warp_tiles(pm_handle_t h, Level& L) {
  int S = std::max(1, std::min(std::max(h->stages, h->solve_stages), 4));
  int W = 0;
  while (S >= 1) {
    W = (int)std::min<size_t>(h->warps_per_cta,
                              kSmemLimit / Prec<R>::warp_smem(pm::kModeReduce, L.m, S));
    W = (int)std::min<size_t>(W, kSmemLimit / Prec<R>::warp_smem(pm::kModeSolve, L.m, 1));
    if (W >= 1) break;
    --S;
  }
  if (W >= 1) {
    L.P = 32;
    L.stages = S;
    L.warps_per_cta = W;
  }
}

// Builds h->levels for a level-0 system; allocates scratch for levels >= 1.
// ragged0: the caller's last tile must not be padded (row-sharded ranks that
// are not the last one); then m must divide n and upper levels use m = 2.
template <class R>
int build_plan(pm_handle_t h, int64_t n, int m, const R* a, const R* b, const R* c,
               const R* d, R* x, bool ragged0, size_t extra_elems,
               bool allow_chain = true, int nparts = 1, int dist_world = 0) {
  std::vector<Level> lv;
  Level L0;
  L0.n = n;
  L0.m = m;
  L0.a = a; L0.b = b; L0.c = c; L0.d = d; L0.x = x;
  L0.pad_mode = ragged0 ? 0 : 1;
  L0.bulk = aligned16(a) && aligned16(b) && aligned16(c) && aligned16(d) && aligned16(x);
  // a system that fits one CTA tile is solved by a single ROOT launch
  const bool one_tile = n <= (int64_t)choose_P(m) * m;
  if (L0.bulk && h->warp_tiles && !one_tile) set_warp_tiles<R>(h, L0);
  if (L0.warps_per_cta == 0) {
    L0.P = choose_P(m);
    L0.stages = pick_stages<R>(h->stages, L0.P, m);
    if (Prec<R>::tile_smem(pm::kModeSolve, L0.P, m, 1) > kSmemLimit)
      return fail(h, PM_ERR_VALIDATION, "sub-system size m too large for shared memory");
  }
  // pair tiles: two m-blocks per lane, 64*m rows per warp tile (not with
  // chain mode, whose chunks are cut in 32-block tiles)
  const bool want_pair = !h->robust_mode && (h->pair_tiles > 0 || (h->pair_tiles < 0 && sizeof(R) == 4));
  if (L0.warps_per_cta > 0 && want_pair && pm::m_is_specialised(m) && !(h->opt_chain && allow_chain)) {
    // Stage 1 rings h->pair_stages stages per warp, Stage 3 one (solve_stages)
    const int S = std::max(1, std::min(h->pair_stages, 4));
    const int W = (int)std::min<size_t>(2, kSmemLimit / Prec<R>::pair_smem(m, S));
    if (W >= 1) {
      L0.pair = true;
      L0.P = 64;
      L0.stages = S;
      L0.warps_per_cta = W;
    }
  }
  L0.T = (int64_t)L0.P * m;
  L0.ntiles = (n + L0.T - 1) / L0.T;
  // a ragged rank whose rows fill whole tiles never pads: it runs the padded
  // (single-system) kernel variants, whose tree bounds are constants
  if (ragged0 && n % L0.T == 0) L0.pad_mode = 1;
  lv.push_back(L0);
  // Chain mode (single system / batch on warp tiles): level 0's tiles form C
  // contiguous chunks (C = the Stage-3 kernel's resident warps); each warp
  // chains its chunk's tile segments, so level 1 has 2C rows and is solved by
  // one ROOT launch.  Otherwise every upper level is a CTA-tile REDUCE/SOLVE
  // launch pair and the top a ROOT launch (m_up = 8, or 2 for the ragged
  // levels of a row-sharded rank).
  h->chain = h->opt_chain && allow_chain && !ragged0 && L0.warps_per_cta > 0 && L0.ntiles > 1;
  nparts = (int)std::max<int64_t>(1, std::min<int64_t>(nparts, L0.ntiles));
  h->nparts = nparts;
  h->part_chunks.clear();
  h->part_base.clear();
  if (h->chain) {
    const int ctas = Prec<R>::ctas(pm::kModeSolve, m, std::max(1, std::min(h->solve_stages > 0 ? h->solve_stages : L0.stages, L0.stages)),
                                                 L0.warps_per_cta, true);
    int64_t C = (int64_t)std::max(1, ctas) * L0.warps_per_cta * h->sm_count;
    C = std::min<int64_t>(C, 8192);
    int64_t total = 0;
    for (int k = 0; k < nparts; ++k) {
      const int64_t t0 = L0.ntiles * k / nparts, t1 = L0.ntiles * (k + 1) / nparts;
      int64_t ck = std::max<int64_t>(1, C * (t1 - t0) / L0.ntiles);
      ck = std::min<int64_t>(ck, t1 - t0);
      if (t1 == t0) ck = 0;
      h->part_base.push_back(total);
      h->part_chunks.push_back(ck);
      total += ck;
    }
    Level U;
    U.n = 2 * total;
    U.m = (int)std::max<int64_t>(8, (U.n + 127) / 128);
    U.P = 128;
    U.T = (int64_t)U.P * U.m;
    U.ntiles = 1;
    U.pad_mode = 1;
    U.bulk = true;
    U.stages = 1;
    if (U.m > PM_MAX_M) return fail(h, PM_ERR_RUNTIME, "chain root too large");
    lv.push_back(U);
  }
  // Row-sharded rank (dist_world > 0): level 1 of 128 x 8 CTA tiles, one
  // co-resident CTA each, and the chain of their G segments (two launches,
  // pm::launch_dist_upper) when level 1 holds whole 8-row blocks (a non-last
  // rank cannot pad), G fits the chain and the device, and G > 1.
  h->dist_fused = false;
  if (dist_world > 0 && dist_world <= pm::kDistMaxWorld && h->upper_fused >= 2 && !h->robust_mode && !h->chain &&
      L0.warps_per_cta > 0 && L0.ntiles > 1) {
    const int64_t n1 = 2 * L0.ntiles;
    const int64_t T1 = (int64_t)pm::kUpperP * pm::kUpperM;
    const int64_t G = (n1 + T1 - 1) / T1;
    int& cap = h->dist_cap[sizeof(R) == 4];
    if (cap < 0) cap = Prec<R>::dist_upper_capacity(h->sm_count);
    if (G > 1 && G <= (int64_t)pm::kUpperP * pm::kDistChainMax && G <= cap && !(ragged0 && n1 % pm::kUpperM)) {
      Level U;
      U.n = n1;
      U.m = pm::kUpperM;
      U.P = pm::kUpperP;
      U.T = T1;
      U.ntiles = G;
      U.pad_mode = ragged0 ? 0 : 1;
      U.bulk = true;
      U.stages = 1;
      lv.push_back(U);
      h->dist_fused = true;
      h->dist_chain = (int)((G + pm::kUpperP - 1) / pm::kUpperP);
    }
  }
  // Upper levels: warp tiles of 32*upper_m rows while the level exceeds one
  // ROOT tile (128*root_m rows), then the ROOT; ragged ranks use CTA tiles
  // with m = 2.
  const int m_up = ragged0 ? 2 : h->upper_cta_m;
  while (!h->dist_fused && lv.back().ntiles > 1) {
    const Level& prev = lv.back();
    Level U;
    U.n = 2 * prev.ntiles;
    U.pad_mode = ragged0 ? 0 : 1;
    U.bulk = true;
    U.P = ragged0 ? 128 : h->upper_cta_p;
    if (!ragged0 && h->upper_m > 0) {
      U.m = h->root_m;
      if (U.n > (int64_t)128 * h->root_m && h->warp_tiles) {
        U.m = h->upper_m;
        set_warp_tiles<R>(h, U);
      }
    } else {
      U.m = m_up;
    }
    if (U.warps_per_cta == 0) U.stages = pick_stages<R>(h->stages, U.P, U.m);
    U.T = (int64_t)U.P * U.m;
    U.ntiles = (U.n + U.T - 1) / U.T;
    lv.push_back(U);
  }
  // scratch: levels >= 1 hold a, b, c, d, x (n_L each); 256-byte aligned
  size_t total = extra_elems;  // in elements of R
  std::vector<size_t> off(lv.size(), 0);
  for (size_t k = 1; k < lv.size(); ++k) {
    off[k] = total;
    total += 5 * (size_t)((lv[k].n + 31) / 32 * 32);
  }
  size_t nodes_off = 0;
  if (h->chain) {
    nodes_off = (total + 31) / 32 * 32;
    total = nodes_off + (size_t)L0.ntiles * 8;  // 7 reals per Node, padded to 8
  }
  size_t seg2_off = 0;
  if (h->dist_fused) {
    seg2_off = (total + 31) / 32 * 32;
    // segments, chain nodes, boundary pairs | level 2's CTA tree
    total = seg2_off + ((size_t)lv[1].ntiles * 18 + 3) / 4 * 4 + (Prec<R>::dist_tree2_bytes() + 2 * sizeof(R)) / sizeof(R);
  }
  int st = ensure_scratch(h, total * sizeof(R));
  if (st) return st;
  R* scr = reinterpret_cast<R*>(h->scratch);
  h->chain_nodes = h->chain ? (void*)(scr + nodes_off) : nullptr;
  h->dist_seg2 = h->dist_fused ? (void*)(scr + seg2_off) : nullptr;
  for (size_t k = 1; k < lv.size(); ++k) {
    const size_t stride = (size_t)((lv[k].n + 31) / 32 * 32);
    R* base = scr + off[k];
    lv[k].a = base;
    lv[k].b = base + stride;
    lv[k].c = base + 2 * stride;
    lv[k].d = base + 3 * stride;
    lv[k].x = base + 4 * stride;
    lv[k].bulk = true;
  }
  h->levels = std::move(lv);
  return PM_OK;
}

// Batch system length of a launch, with the fast-modulo multiplier when the
// rows and the length fit 32 bits.
template <class Args>
void set_sys(Args& A, int64_t sys_len) {
  A.sys_len = sys_len;
  A.sys_magic = (sys_len > 0 && A.n < (int64_t(1) << 32) && sys_len < (int64_t(1) << 32))
                    ? UINT64_MAX / (uint64_t)sys_len + 1
                    : 0;
}

template <class R>
typename Prec<R>::Args args_for(pm_handle_t h, const Level& L, int64_t t0, int64_t t1) {
  typename Prec<R>::Args A;
  A.a = static_cast<const R*>(L.a); A.b = static_cast<const R*>(L.b);
  A.c = static_cast<const R*>(L.c); A.d = static_cast<const R*>(L.d); A.x = static_cast<R*>(L.x);
  A.n = L.n;
  A.tile_begin = t0;
  A.tile_end = t1;
  A.m = L.m;
  A.stages = L.stages;
  A.max_ctas = h->max_ctas;
  A.flag = h->dflag;
  A.pad_mode = L.pad_mode;
  A.robust = h->robust_mode;
  return A;
}

cudaEvent_t next_kevent(pm_handle_t h) {
  const size_t k = h->krec.size() * 2 + 2;
  while (h->kev.size() < k) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
    h->kev.push_back(e);
  }
  return h->kev[k - 2];
}

template <class R>
int launch(pm_handle_t h, int mode, const typename Prec<R>::Args& A, const Level& L, cudaStream_t st) {
  int grid = 0;
  const int level = (int)(&L - h->levels.data());
  const bool timed = h->ktimes && next_kevent(h) != nullptr;
  const size_t ev = h->krec.size() * 2;
  if (timed) cudaEventRecord(h->kev[ev], st);
  cudaError_t e;
  if (L.pair && mode != pm::kModeRoot)
    e = Prec<R>::pair(mode, A, L.warps_per_cta, h->sm_count, st, &grid);
  else if (L.warps_per_cta > 0 && mode != pm::kModeRoot)
    e = Prec<R>::warp(mode, A, L.warps_per_cta, h->sm_count, st, &grid);
  else
    e = Prec<R>::tile(mode, A, L.P, L.bulk, h->sm_count, st, &grid);
  if (e != cudaSuccess) return cuda_fail(h, e, "tile kernel launch");
  if (timed) {
    cudaEventRecord(h->kev[ev + 1], st);
    h->krec.push_back({mode, level, ev});
  }
  if (grid > 0) ++h->launches;
  return PM_OK;
}


// REDUCE of level k over tiles [t0, t1): writes rows into level k+1 (or `out4`).
template <class R>
void set_chain(pm_handle_t h, typename Prec<R>::Args& A, int part) {
  A.nchunks = h->part_chunks[part];
  A.chunk_base = h->part_base[part];
  A.chain_nodes = static_cast<typename Prec<R>::Node*>(h->chain_nodes);
}

template <class R>
void set_p2p(pm_handle_t h, typename Prec<R>::Args& A) {
  A.xpeers = h->d_peers;
  A.xlocal = h->xbuf;
  A.xworld = h->xworld;
  A.xrank = h->xrank;
  A.xepoch = h->p2p_top.epoch;
  A.xtimeout_ns = 20ull * 1000 * 1000 * 1000;  // 20 s
}

template <class R>
int enq_reduce(pm_handle_t h, size_t k, int64_t t0, int64_t t1, cudaStream_t st, bool zf, bool zl,
               int64_t sys_len, R* const* out4, int part = 0) {
  const Level& L = h->levels[k];
  typename Prec<R>::Args A = args_for<R>(h, L, t0, t1);
  if (out4) {
    A.ra = out4[0]; A.rb = out4[1]; A.rc = out4[2]; A.rd = out4[3];
  } else {
    const Level& U = h->levels[k + 1];
    A.ra = static_cast<R*>(const_cast<void*>(U.a)); A.rb = static_cast<R*>(const_cast<void*>(U.b));
    A.rc = static_cast<R*>(const_cast<void*>(U.c)); A.rd = static_cast<R*>(const_cast<void*>(U.d));
  }
  A.zero_first = zf;
  A.zero_last = zl;
  set_sys(A, (k == 0) ? sys_len : 0);
  if (k == 0 && h->chain) set_chain<R>(h, A, part);
  if (h->p2p_top.active && k + 1 == h->levels.size()) set_p2p<R>(h, A);
  return launch<R>(h, pm::kModeReduce, A, L, st);
}

template <class R>
int enq_solve(pm_handle_t h, size_t k, int64_t t0, int64_t t1, cudaStream_t st, bool zf, bool zl,
              int64_t sys_len, const R* xb, int part = 0) {
  const Level& L = h->levels[k];
  typename Prec<R>::Args A = args_for<R>(h, L, t0, t1);
  A.xb = xb ? xb : static_cast<const R*>(h->levels[k + 1].x);
  if (L.warps_per_cta > 0 && h->solve_stages > 0) A.stages = std::min(h->solve_stages, L.stages);
  A.zero_first = zf;
  A.zero_last = zl;
  set_sys(A, (k == 0) ? sys_len : 0);
  A.reverse = h->reverse;
  if (k == 0 && h->chain) set_chain<R>(h, A, part);
  if (h->p2p_top.active && k + 1 == h->levels.size()) set_p2p<R>(h, A);
  return launch<R>(h, pm::kModeSolve, A, L, st);
}

template <class R>
int enq_root(pm_handle_t h, size_t k, cudaStream_t st, int64_t sys_len) {
  const Level& L = h->levels[k];
  typename Prec<R>::Args A = args_for<R>(h, L, 0, 1);
  set_sys(A, (k == 0) ? sys_len : 0);
  return launch<R>(h, pm::kModeRoot, A, L, st);
}


// The top two levels in one launch (pm::launch_upper_fused): a plan of three
// or more levels whose top level is one 128 x 8 CTA tile fed by a level of
// 128 x 8 CTA tiles with every tile's CTA co-resident (N = 8e7, m = 10:
// levels 1-2; N = 1e9: levels 2-3).  Not in robust mode (classic sweeps).
template <class R>
bool upper_fusable(pm_handle_t h) {
  if (!h->upper_fused || h->robust_mode || h->chain || h->p2p_top.active || h->levels.size() < 3)
    return false;
  auto cta8 = [](const Level& L) {
    return L.warps_per_cta == 0 && !L.pair && L.P == pm::kUpperP && L.m == pm::kUpperM && L.pad_mode == 1;
  };
  const size_t top = h->levels.size() - 1;
  const Level& Lk = h->levels[top - 1];
  const Level& Lt = h->levels[top];
  if (!cta8(Lk) || !cta8(Lt) || Lt.ntiles != 1 || Lt.n != 2 * Lk.ntiles) return false;
  int& cap = h->upper_cap[sizeof(R) == 4];
  if (cap < 0) cap = Prec<R>::upper_capacity(h->sm_count);
  return Lk.ntiles <= cap;
}

// Levels k and k+1 (the top) in one launch.
template <class R>
int enq_upper_fused(pm_handle_t h, size_t k, cudaStream_t st) {
  const Level& L1 = h->levels[k];
  const Level& L2 = h->levels[k + 1];
  typename Prec<R>::UpperArgs u;
  u.a1 = static_cast<const R*>(L1.a); u.b1 = static_cast<const R*>(L1.b);
  u.c1 = static_cast<const R*>(L1.c); u.d1 = static_cast<const R*>(L1.d);
  u.x1 = static_cast<R*>(L1.x);
  u.n1 = L1.n;
  u.a2 = static_cast<R*>(const_cast<void*>(L2.a)); u.b2 = static_cast<R*>(const_cast<void*>(L2.b));
  u.c2 = static_cast<R*>(const_cast<void*>(L2.c)); u.d2 = static_cast<R*>(const_cast<void*>(L2.d));
  u.x2 = static_cast<R*>(L2.x);
  u.n2 = L2.n;
  u.sync = h->dsync;
  u.flag = h->dflag;
  const bool timed = h->ktimes && next_kevent(h) != nullptr;
  const size_t ev = h->krec.size() * 2;
  if (timed) cudaEventRecord(h->kev[ev], st);
  int grid = 0;
  const cudaError_t e = Prec<R>::upper(u, h->sm_count, st, &grid);
  if (e != cudaSuccess) return cuda_fail(h, e, "fused upper-level kernel launch");
  if (timed) {
    cudaEventRecord(h->kev[ev + 1], st);
    h->krec.push_back({3, (int)k, ev});
  }
  if (grid > 0) ++h->launches;
  return PM_OK;
}

// Row-sharded rank, fused plan: level 1 + the level-2 chain in one launch
// (mode kModeReduce: -> iface or the P2P publish; kModeSolve: iface_all or
// the P2P acquire -> level 1's x).
template <class R>
int enq_dist_upper(pm_handle_t h, int mode, bool zf, bool zl, int rank, int world, R* iface,
                   const R* iface_all, bool p2p, cudaStream_t st) {
  const Level& L1 = h->levels[1];
  typename Prec<R>::DistUpperArgs u;
  u.a1 = static_cast<const R*>(L1.a); u.b1 = static_cast<const R*>(L1.b);
  u.c1 = static_cast<const R*>(L1.c); u.d1 = static_cast<const R*>(L1.d);
  u.x1 = static_cast<R*>(L1.x);
  u.n1 = L1.n;
  const size_t G = (size_t)L1.ntiles;
  R* base = static_cast<R*>(h->dist_seg2);
  u.seg2 = base;
  u.node2 = base + 8 * G;
  u.x2 = base + 16 * G;
  u.tree2 = base + (18 * G + 3) / 4 * 4;  // 16-byte aligned for both precisions
  u.chain = h->dist_chain;
  u.ragged = L1.pad_mode == 0;
  u.zero_first = zf;
  u.zero_last = zl;
  u.iface = iface;
  u.iface_all = iface_all;
  u.rank = rank;
  u.world = world;
  if (p2p) {
    u.xpeers = h->d_peers;
    u.xlocal = h->xbuf;
    u.xepoch = h->p2p_top.epoch;
    u.xtimeout_ns = 20ull * 1000 * 1000 * 1000;  // 20 s
  }
  u.sync = h->dsync;
  u.flag = h->dflag;
  const bool timed = h->ktimes && next_kevent(h) != nullptr;
  const size_t ev = h->krec.size() * 2;
  if (timed) cudaEventRecord(h->kev[ev], st);
  int grid = 0;
  const cudaError_t e = Prec<R>::dist_upper(mode, u, h->sm_count, st, &grid);
  if (e != cudaSuccess) return cuda_fail(h, e, "row-sharded upper-level kernel launch");
  if (timed) {
    cudaEventRecord(h->kev[ev + 1], st);
    h->krec.push_back({mode == pm::kModeReduce ? 5 : 6, 1, ev});
  }
  if (grid > 0) ++h->launches;
  return PM_OK;
}

// Upper levels (1..top) on one stream: REDUCE 1..top-1, ROOT top, SOLVE
// top-1..1 (chain mode: level 1 is the top, a single ROOT); the top two
// levels in one launch when that applies.
template <class R>
int enq_upper(pm_handle_t h, cudaStream_t st) {
  const size_t top = h->levels.size() - 1;
  int r;
  if (upper_fusable<R>(h)) {
    for (size_t k = 1; k + 1 < top; ++k)
      if ((r = enq_reduce<R>(h, k, 0, h->levels[k].ntiles, st, true, true, 0, nullptr))) return r;
    if ((r = enq_upper_fused<R>(h, top - 1, st))) return r;
    for (size_t k = top - 1; k-- > 1;)
      if ((r = enq_solve<R>(h, k, 0, h->levels[k].ntiles, st, true, true, 0, nullptr))) return r;
    return PM_OK;
  }
  for (size_t k = 1; k < top; ++k)
    if ((r = enq_reduce<R>(h, k, 0, h->levels[k].ntiles, st, true, true, 0, nullptr))) return r;
  if (top >= 1 && (r = enq_root<R>(h, top, st, 0))) return r;
  for (size_t k = top; k-- > 1;)
    if ((r = enq_solve<R>(h, k, 0, h->levels[k].ntiles, st, true, true, 0, nullptr))) return r;
  return PM_OK;
}

// Whole solve of the planned system on one stream.
template <class R>
int enq_full(pm_handle_t h, cudaStream_t st, int64_t sys_len) {
  int r;
  if (h->levels.size() == 1) return enq_root<R>(h, 0, st, sys_len);
  if ((r = enq_reduce<R>(h, 0, 0, h->levels[0].ntiles, st, true, true, sys_len, nullptr))) return r;
  if ((r = enq_upper<R>(h, st))) return r;
  return enq_solve<R>(h, 0, 0, h->levels[0].ntiles, st, true, true, sys_len, nullptr);
}

int validate_common(pm_handle_t h, const void* a, const void* b, const void* c, const void* d,
                    const void* x, int64_t n, int32_t m) {
  if (!h) return PM_ERR_VALIDATION;
  if (!a || !b || !c || !d || !x) return fail(h, PM_ERR_VALIDATION, "null array pointer");
  if (n < 1) return fail(h, PM_ERR_VALIDATION, "SLAE size must be at least 1");
  if (m < 2 || m > PM_MAX_M)
    return fail(h, PM_ERR_VALIDATION,
                "sub-system size m must lie in [2, " + std::to_string(PM_MAX_M) + "]");
  return PM_OK;
}

streamtune::ModelBundle from_c(const pm_model_bundle& c) {
  streamtune::ModelBundle b;
  b.sum_a = c.sum_a; b.sum_b = c.sum_b;
  b.small_a = c.small_a; b.small_b = c.small_b; b.small_c = c.small_c;
  b.big_a = c.big_a; b.big_b = c.big_b; b.big_c = c.big_c;
  b.size_threshold = c.size_threshold;
  b.candidates.clear();
  for (int k = 0; k < c.num_candidates && k < 5; ++k)
    b.candidates.push_back(streamtune::StreamCount(c.candidates[k]));
  return b;
}

void to_c(const streamtune::ModelBundle& b, pm_model_bundle* c) {
  std::memset(c, 0, sizeof(*c));
  c->sum_a = b.sum_a; c->sum_b = b.sum_b;
  c->small_a = b.small_a; c->small_b = b.small_b; c->small_c = b.small_c;
  c->big_a = b.big_a; c->big_b = b.big_b; c->big_c = b.big_c;
  c->size_threshold = b.size_threshold;
  c->num_candidates = (int32_t)std::min<size_t>(b.candidates.size(), 5);
  for (int k = 0; k < c->num_candidates; ++k) c->candidates[k] = b.candidates[k].value();
}

int read_flag(pm_handle_t h, cudaStream_t st) {
  int flag = 0;
  PM_CUDA(h, cudaMemcpyAsync(&flag, h->dflag, sizeof(int), cudaMemcpyDeviceToHost, st));
  PM_CUDA(h, cudaStreamSynchronize(st));
  if (flag == 1 && h->retry && !h->robust_mode) {
    // a zero / non-finite pivot in the fast path: redo the last solve with
    // classic sweeps (continuant products can leave the FP range for rows
    // scaled over many orders of magnitude); report only if that fails too
    PM_CUDA(h, cudaMemsetAsync(h->dflag, 0, sizeof(int), st));
    PM_CUDA(h, cudaStreamSynchronize(st));
    h->robust_mode = 1;
    const int r = h->retry();
    h->robust_mode = 0;
    cudaStream_t rs = h->retry_stream;
    if (r) return r;
    PM_CUDA(h, cudaStreamSynchronize(rs));
    PM_CUDA(h, cudaMemcpyAsync(&flag, h->dflag, sizeof(int), cudaMemcpyDeviceToHost, rs));
    PM_CUDA(h, cudaStreamSynchronize(rs));
  }
  if (flag) {
    PM_CUDA(h, cudaMemsetAsync(h->dflag, 0, sizeof(int), st));
    PM_CUDA(h, cudaStreamSynchronize(st));
    if (flag & 4) return fail(h, PM_ERR_RUNTIME, "P2P interface exchange timed out (a peer never published)");
    if (flag & 16) {
      // counters and flags of the tile-stream kernel are inconsistent now
      if (h->bcnt) PM_CUDA(h, cudaMemset(h->bcnt, 0, h->bcnt_bytes));
      return fail(h, PM_ERR_RUNTIME, "batch tile-stream kernel: a Stage-3 wait for its system timed out");
    }
    if (flag & 8) {
      PM_CUDA(h, cudaMemset(h->dsync, 0, 8 * sizeof(unsigned long long)));
      return fail(h, PM_ERR_RUNTIME, "fused upper-level kernel: level-2 flag wait timed out");
    }
    return fail(h, PM_ERR_COMPUTATION, "zero or non-finite pivot (system not solvable without pivoting)");
  }
  return PM_OK;
}

}  // namespace

// ---- the solver entry points, one instantiation per precision -------------

// Runs `enqueue` (which enqueues the solve on `st`) through a cached CUDA
// graph when PM_OPT_GRAPHS is on: the first call with a key records the
// launches with stream capture and instantiates them; later calls replay
// one cudaGraphLaunch.  The plan (and its scratch) is built before, outside
// the capture.  Kernel-time recording bypasses graphs.  A capture the driver
// rejects falls back to direct launches.
template <class F>
int run_maybe_graph(pm_handle_t h, cudaStream_t st, size_t esz, const void* const* ptrs, int64_t n,
                    int64_t nps, int m, F&& enqueue) {
  if (!h->use_graphs || h->ktimes || h->robust_mode || st == nullptr) return enqueue();
  for (auto& g : h->graphs) {
    if (g.esz == esz && g.n == n && g.nps == nps && g.m == m && g.gen == h->plan_gen &&
        g.pdl_gen == g_pdl_gen.load(std::memory_order_relaxed) &&
        g.scratch == h->scratch && std::equal(ptrs, ptrs + 5, g.p)) {
      g.last_use = ++h->graph_clock;
      h->launches = g.launches;
      PM_CUDA(h, cudaGraphLaunch(g.exec, st));
      return PM_OK;
    }
  }
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return enqueue();
  PM_CUDA(h, cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
  const int r = enqueue();
  cudaGraph_t graph = nullptr;
  const cudaError_t ee = cudaStreamEndCapture(st, &graph);
  if (r != PM_OK) {
    if (graph) cudaGraphDestroy(graph);
    return r;
  }
  cudaGraphExec_t exec = nullptr;
  if (ee != cudaSuccess || cudaGraphInstantiate(&exec, graph, 0) != cudaSuccess) {
    if (graph) cudaGraphDestroy(graph);
    cudaGetLastError();
    return enqueue();  // direct launches
  }
  cudaGraphDestroy(graph);
  if (h->graphs.size() >= 8) {  // evict the least recently used
    auto lru = std::min_element(h->graphs.begin(), h->graphs.end(),
                                [](const auto& x, const auto& y) { return x.last_use < y.last_use; });
    cudaGraphExecDestroy(lru->exec);
    h->graphs.erase(lru);
  }
  pm_handle_s::GraphEntry g{};
  g.esz = esz;
  std::copy(ptrs, ptrs + 5, g.p);
  g.n = n;
  g.nps = nps;
  g.m = m;
  g.gen = h->plan_gen;
  g.pdl_gen = g_pdl_gen.load(std::memory_order_relaxed);
  g.scratch = h->scratch;
  g.exec = exec;
  g.launches = h->launches;
  g.last_use = ++h->graph_clock;
  h->graphs.push_back(g);
  PM_CUDA(h, cudaGraphLaunch(exec, st));
  return PM_OK;
}

template <class R>
int solve_device_impl(pm_handle_t h, const R* a, const R* b, const R* c,
                        const R* d, R* x, int64_t n, int32_t m, void* stream) {
  int r = validate_common(h, a, b, c, d, x, n, m);
  if (r) return r;
  PM_CUDA(h, cudaSetDevice(h->device));
  h->launches = 0;
  if ((r = build_plan<R>(h, n, m, a, b, c, d, x, false, 0))) return r;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  h->last_stream = st;
  const void* ptrs[5] = {a, b, c, d, x};
  h->retry = nullptr;  // (x aliasing an input: the inputs are gone, no retry)
  if (x != a && x != b && x != c && x != d) {
    h->retry = [h, a, b, c, d, x, n, m, st]() {
      int rr = build_plan<R>(h, n, m, a, b, c, d, x, false, 0);
      return rr ? rr : enq_full<R>(h, st, 0);
    };
    h->retry_stream = st;
  }
  return run_maybe_graph(h, st, sizeof(R), ptrs, n, 0, m, [&] { return enq_full<R>(h, st, 0); });
}

template <class R>
int solve_batch_impl(pm_handle_t h, const R* a, const R* b, const R* c,
                              const R* d, R* x, int64_t n_per_system, int64_t batch,
                              int32_t m, void* stream) {
  if (batch < 1) return fail(h, PM_ERR_VALIDATION, "batch must be at least 1");
  if (n_per_system < 1) return fail(h, PM_ERR_VALIDATION, "SLAE size must be at least 1");
  if (n_per_system > INT64_MAX / batch) return fail(h, PM_ERR_VALIDATION, "batch too large");
  const int64_t n = n_per_system * batch;
  int r = validate_common(h, a, b, c, d, x, n, m);
  if (r) return r;
  PM_CUDA(h, cudaSetDevice(h->device));
  h->launches = 0;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  h->last_stream = st;
  if (!h->robust_mode) {
    h->retry = nullptr;
    if (x != a && x != b && x != c && x != d) {
      h->retry = [h, a, b, c, d, x, n_per_system, batch, m, stream]() {
        return solve_batch_impl<R>(h, a, b, c, d, x, n_per_system, batch, m, stream);
      };
      h->retry_stream = st;
    }
  }
  h->last_stream_plan = pm::StreamPlan{};
  pm::StreamPlan sp{};
  if (std::is_same<R, double>::value && batch > 1 && h->batch_cluster == 2 && !h->robust_mode && aligned16(a) &&
      aligned16(b) && aligned16(c) && aligned16(d) && aligned16(x) &&
      pm::plan_stream(m, n_per_system, batch, h->sm_count, h->max_ctas, h->batch_force_warps, h->batch_force_stages,
                      h->batch_lag, &sp)) {
    // rings (no initial state) and the per-system counters (zero between
    // launches) live in separate allocations: the counters must never
    // overlap a previous launch's ring data when the batch size changes
    const size_t need = pm::stream_scratch_bytes(sp, batch);
    if (need > h->bscr_bytes) {
      if (h->bscr) {
        PM_CUDA(h, cudaStreamSynchronize(st));
        PM_CUDA(h, cudaFree(h->bscr));
        h->bscr = nullptr;
        h->bscr_bytes = 0;
      }
      PM_CUDA(h, cudaMalloc(&h->bscr, need));
      h->bscr_bytes = need;
    }
    const size_t cneed = (size_t)batch * 3 * pm::kStreamCounterStride * sizeof(unsigned);
    if (cneed > h->bcnt_bytes) {
      if (h->bcnt) {
        PM_CUDA(h, cudaStreamSynchronize(st));
        PM_CUDA(h, cudaFree(h->bcnt));
        h->bcnt = nullptr;
        h->bcnt_bytes = 0;
      }
      PM_CUDA(h, cudaMalloc(&h->bcnt, cneed));
      PM_CUDA(h, cudaMemset(h->bcnt, 0, cneed));
      h->bcnt_bytes = cneed;
    }
    pm::StreamArgs A;  // FP64-only, like the cluster kernel
    A.a = reinterpret_cast<const double*>(a); A.b = reinterpret_cast<const double*>(b);
    A.c = reinterpret_cast<const double*>(c); A.d = reinterpret_cast<const double*>(d);
    A.x = reinterpret_cast<double*>(x);
    A.n_sys = n_per_system;
    A.batch = batch;
    A.m = m;
    A.tps = sp.tps;
    A.nw = sp.nw;
    A.W = sp.warps;
    A.S = sp.stages;
    A.L = sp.lag;
    A.Lmax = sp.lag_max;
    A.K = sp.ring;
    A.mg_tps = pm::stream_magic((uint32_t)sp.tps);
    A.mg_K = pm::stream_magic((uint32_t)sp.ring);
    A.mg_period = pm::stream_magic((uint32_t)sp.ring * (uint32_t)sp.nw);
    const size_t slots = (size_t)sp.ring * sp.nw;
    A.cnt1 = reinterpret_cast<unsigned*>(h->bcnt);  // [3][batch][stride], zero between launches
    A.cnt3 = A.cnt1 + batch * pm::kStreamCounterStride;
    A.sflag = A.cnt3 + batch * pm::kStreamCounterStride;
    char* p = h->bscr;
    A.nodes = reinterpret_cast<unsigned char*>(p);
    p += slots * 1792;
    A.segs = reinterpret_cast<double*>(p);
    p += slots * 8 * sizeof(double);
    A.txy = reinterpret_cast<double*>(p);
    A.flag = h->dflag;
    A.discard = h->batch_discard & 1;
    A.hints = (h->batch_discard >> 1) & 1;
    A.early = (h->batch_discard >> 2) & 1;
    A.ooo = (h->batch_discard >> 3) & 1;
    if (h->batch_stats) {
      // counters + per-system timeline + job traces of 8 warps + control trace of CTA 0
      const size_t words = 16 + 5 * (size_t)batch + 8 * 2400 * 4 + 1200 * 2 + 4096 * 12;
      if (words > h->dstats_words) {
        if (h->dstats) cudaFree(h->dstats);
        h->dstats = nullptr;
        PM_CUDA(h, cudaMalloc(&h->dstats, words * sizeof(unsigned long long)));
        h->dstats_words = words;
      }
      PM_CUDA(h, cudaMemsetAsync(h->dstats, 0, 16 * sizeof(unsigned long long), st));
      PM_CUDA(h, cudaMemsetAsync(h->dstats + 16, 0xff, 5 * (size_t)batch * sizeof(unsigned long long), st));
      PM_CUDA(h, cudaMemsetAsync(h->dstats + 16 + batch, 0, (size_t)batch * sizeof(unsigned long long), st));
      PM_CUDA(h, cudaMemsetAsync(h->dstats + 16 + 5 * batch, 0, (8 * 2400 * 4 + 1200 * 2 + 4096 * 12) * sizeof(unsigned long long), st));
      A.stats = h->dstats;
      A.tl = h->dstats + 16;
      h->dstats_batch = batch;
    }
    h->levels.clear();
    h->last_batch_plan = pm::BatchPlan{0, 0, 0, 0, 0, 0};
    h->last_stream_plan = sp;
    const bool timed = h->ktimes && next_kevent(h) != nullptr;
    const size_t ev = h->krec.size() * 2;
    if (timed) cudaEventRecord(h->kev[ev], st);
    PM_CUDA(h, pm::launch_batch_stream(m, A, sp, st));
    if (timed) {
      cudaEventRecord(h->kev[ev + 1], st);
      h->krec.push_back({4, 0, ev});
    }
    ++h->launches;
    return PM_OK;
  }
  pm::BatchPlan pl{};
  if (std::is_same<R, double>::value && batch > 1 && h->batch_cluster == 1 && !h->robust_mode && aligned16(a) && aligned16(b) && aligned16(c) &&
      aligned16(d) && aligned16(x) &&
      pm::plan_batch(m, n_per_system, batch, h->sm_count, (int64_t)h->batch_l2_mb << 20,
                     h->batch_force_cluster, h->batch_force_warps, h->batch_force_stages, &pl)) {
    pm::BatchArgs A;  // the cluster kernel is FP64-only
    A.a = reinterpret_cast<const double*>(a); A.b = reinterpret_cast<const double*>(b);
    A.c = reinterpret_cast<const double*>(c); A.d = reinterpret_cast<const double*>(d);
    A.x = reinterpret_cast<double*>(x);
    A.n_sys = n_per_system;
    A.batch = batch;
    A.flag = h->dflag;
    h->levels.clear();
    h->last_batch_plan = pl;
    const bool timed = h->ktimes && next_kevent(h) != nullptr;
    const size_t ev = h->krec.size() * 2;
    if (timed) cudaEventRecord(h->kev[ev], st);
    PM_CUDA(h, pm::launch_batch_cluster(m, A, pl, st));
    if (timed) {
      cudaEventRecord(h->kev[ev + 1], st);
      h->krec.push_back({4, 0, ev});
    }
    ++h->launches;
    return PM_OK;
  }
  h->last_batch_plan = pm::BatchPlan{0, 0, 0, 0, 0, 0};
  if ((r = build_plan<R>(h, n, m, a, b, c, d, x, false, 0))) return r;
  const void* ptrs[5] = {a, b, c, d, x};
  return run_maybe_graph(h, st, sizeof(R), ptrs, n, n_per_system, m,
                         [&] { return enq_full<R>(h, st, batch > 1 ? n_per_system : 0); });
}

template <class R>
int solve_host_impl(pm_handle_t h, const R* a, const R* b, const R* c,
                      const R* d, R* x, int64_t n, int32_t m, int32_t num_streams) {
  int r = validate_common(h, a, b, c, d, x, n, m);
  if (r) return r;
  h->retry = nullptr;
  if (num_streams != 0 && !streamtune::StreamCount::is_valid(num_streams))
    return fail(h, PM_ERR_VALIDATION,
                streamtune::InvalidStreamCountError(num_streams).what());
  PM_CUDA(h, cudaSetDevice(h->device));
  int ns = num_streams;
  if (ns == 0) {
    try {
      ns = streamtune::recommend(h->bundle, (uint64_t)n).chosen.value();
    } catch (const std::exception& ex) {
      return fail(h, PM_ERR_VALIDATION, ex.what());
    }
  }
  // device staging: a, b, c, d, x (x separate so the caller may alias d)
  const size_t stride = (size_t)((n + 31) / 32 * 32);
  const size_t need = 5 * stride * sizeof(R);
  if (need > h->hbuf_bytes) {
    if (h->hbuf) {
      PM_CUDA(h, cudaDeviceSynchronize());
      PM_CUDA(h, cudaFree(h->hbuf));
      h->hbuf = nullptr;
      h->hbuf_bytes = 0;
    }
    PM_CUDA(h, cudaMalloc(&h->hbuf, need));
    h->hbuf_bytes = need;
  }
  R* da = reinterpret_cast<R*>(h->hbuf);
  R* db = da + stride;
  R* dc = db + stride;
  R* dd = dc + stride;
  R* dx = dd + stride;
  h->launches = 0;
  {
    // parts = the stream chunks, so that chain chunks never straddle them
    const int parts_hint = ns > 1 ? ns : 1;
    if ((r = build_plan<R>(h, n, m, da, db, dc, dd, dx, false, 0, true, parts_hint))) return r;
  }
  const Level& L0 = h->levels[0];
  const bool single_tile = h->levels.size() == 1;
  int chunks = single_tile ? 1 : h->nparts;

  cudaStream_t main = h->main;
  std::vector<cudaStream_t> streams;
  std::vector<cudaEvent_t> evs;
  auto cleanup = [&]() {
    for (cudaEvent_t e : evs) cudaEventDestroy(e);
    if (h->stream_mode == 1)
      for (cudaStream_t s : streams) cudaStreamDestroy(s);
  };
  cudaEvent_t tev[6];
  for (int k = 0; k < 6; ++k) {
    cudaError_t e = cudaEventCreate(&tev[k]);
    if (e != cudaSuccess) { cleanup(); return cuda_fail(h, e, "cudaEventCreate"); }
    evs.push_back(tev[k]);
  }
  // The stream set: created inside the timed region in stream mode 1 (the
  // paper's T_overhead includes creating them).
  cudaEventRecord(tev[0], main);
  if (ns > 1) {
    if (h->stream_mode == 1) {
      for (int k = 0; k < ns; ++k) {
        cudaStream_t s;
        cudaError_t e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
        if (e != cudaSuccess) { cleanup(); return cuda_fail(h, e, "cudaStreamCreate"); }
        streams.push_back(s);
      }
    } else {
      while ((int)h->pool.size() < ns) {
        cudaStream_t s;
        cudaError_t e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
        if (e != cudaSuccess) { cleanup(); return cuda_fail(h, e, "cudaStreamCreate"); }
        h->pool.push_back(s);
      }
      streams.assign(h->pool.begin(), h->pool.begin() + ns);
    }
  }
  const bool record = h->timings && ns == 1;
  auto bytes_of = [](int64_t rows) { return (size_t)rows * sizeof(R); };
  cudaError_t e = cudaSuccess;
  auto h2d = [&](int64_t r0, int64_t r1, cudaStream_t s) {
    const size_t bytes = bytes_of(r1 - r0);
    if (e == cudaSuccess) e = cudaMemcpyAsync(da + r0, a + r0, bytes, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(db + r0, b + r0, bytes, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dc + r0, c + r0, bytes, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dd + r0, d + r0, bytes, cudaMemcpyHostToDevice, s);
  };
  auto d2h = [&](int64_t r0, int64_t r1, cudaStream_t s) {
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(x + r0, dx + r0, bytes_of(r1 - r0), cudaMemcpyDeviceToHost, s);
  };

  if (ns == 1 || chunks <= 1) {
    h2d(0, n, main);
    if (record) cudaEventRecord(tev[1], main);
    if (single_tile) {
      if (e == cudaSuccess && (r = enq_root<R>(h, 0, main, 0))) { cleanup(); return r; }
      if (record) { cudaEventRecord(tev[2], main); cudaEventRecord(tev[3], main); }
    } else {
      if (e == cudaSuccess && (r = enq_reduce<R>(h, 0, 0, L0.ntiles, main, true, true, 0, nullptr))) { cleanup(); return r; }
      if (record) cudaEventRecord(tev[2], main);
      if (e == cudaSuccess && (r = enq_upper<R>(h, main))) { cleanup(); return r; }
      if (record) cudaEventRecord(tev[3], main);
      if (e == cudaSuccess && (r = enq_solve<R>(h, 0, 0, L0.ntiles, main, true, true, 0, nullptr))) { cleanup(); return r; }
    }
    if (record) cudaEventRecord(tev[4], main);
    d2h(0, n, main);
  } else {
    // fork
    cudaEvent_t fork, join;
    cudaEventCreateWithFlags(&fork, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&join, cudaEventDisableTiming);
    evs.push_back(fork);
    evs.push_back(join);
    std::vector<cudaEvent_t> done(chunks);
    for (int k = 0; k < chunks; ++k) {
      cudaEventCreateWithFlags(&done[k], cudaEventDisableTiming);
      evs.push_back(done[k]);
    }
    cudaEventRecord(fork, main);
    for (int k = 0; k < chunks; ++k) {
      const int64_t t0 = L0.ntiles * k / chunks, t1 = L0.ntiles * (k + 1) / chunks;
      const int64_t r0 = t0 * L0.T, r1 = std::min(n, t1 * L0.T);
      cudaStream_t s = streams[k];
      cudaStreamWaitEvent(s, fork, 0);
      h2d(r0, r1, s);
      if (e == cudaSuccess && (r = enq_reduce<R>(h, 0, t0, t1, s, true, true, 0, nullptr, k))) { cleanup(); return r; }
      cudaEventRecord(done[k], s);
    }
    for (int k = 0; k < chunks; ++k) cudaStreamWaitEvent(main, done[k], 0);
    if (e == cudaSuccess && (r = enq_upper<R>(h, main))) { cleanup(); return r; }
    cudaEventRecord(join, main);
    for (int k = 0; k < chunks; ++k) {
      const int64_t t0 = L0.ntiles * k / chunks, t1 = L0.ntiles * (k + 1) / chunks;
      const int64_t r0 = t0 * L0.T, r1 = std::min(n, t1 * L0.T);
      cudaStream_t s = streams[k];
      cudaStreamWaitEvent(s, join, 0);
      if (e == cudaSuccess && (r = enq_solve<R>(h, 0, t0, t1, s, true, true, 0, nullptr, k))) { cleanup(); return r; }
      d2h(r0, r1, s);
      cudaEventRecord(done[k], s);
    }
    for (int k = 0; k < chunks; ++k) cudaStreamWaitEvent(main, done[k], 0);
  }
  if (h->stream_mode == 1) {
    for (cudaStream_t s : streams) cudaStreamDestroy(s);
    streams.clear();
  }
  cudaEventRecord(tev[5], main);
  if (e != cudaSuccess) { cleanup(); return cuda_fail(h, e, "cudaMemcpyAsync"); }
  cudaError_t se = cudaEventSynchronize(tev[5]);
  if (se != cudaSuccess) { cleanup(); return cuda_fail(h, se, "solve"); }
  float ms = 0.f;
  cudaEventElapsedTime(&ms, tev[0], tev[5]);
  h->last_total_ms = ms;
  h->last_streams = ns;
  std::memset(&h->last_t, 0, sizeof(h->last_t));
  h->last_t.slae_size = (uint64_t)n;
  if (record) {
    float t[5];
    for (int k = 0; k < 5; ++k) cudaEventElapsedTime(&t[k], tev[k], tev[k + 1]);
    h->last_t.t1_h2d = t[0];
    h->last_t.t1_comp = t[1];
    h->last_t.t2_comp = t[2];
    h->last_t.t3_comp = t[3];
    h->last_t.t3_d2h = t[4];
  }
  cleanup();
  h->last_stream = main;
  // retry on the staged device copies (separate from x, so host aliasing is fine)
  h->retry = [h, da, db, dc, dd, dx, x, n, m, main]() {
    int rr = build_plan<R>(h, n, m, da, db, dc, dd, dx, false, 0);
    if (!rr) rr = enq_full<R>(h, main, 0);
    if (!rr) PM_CUDA(h, cudaMemcpyAsync(x, dx, (size_t)n * sizeof(R), cudaMemcpyDeviceToHost, main));
    return rr;
  };
  h->retry_stream = main;
  return read_flag(h, main);
}

template <class R>
int generate_range_impl(pm_handle_t h, R* a, R* b, R* c, R* d,
                          int64_t n_total, int64_t row0, int64_t count, uint64_t seed,
                          void* stream) {
  if (!h) return PM_ERR_VALIDATION;
  if (n_total < 1 || count < 1 || row0 < 0 || row0 + count > n_total)
    return fail(h, PM_ERR_VALIDATION, "row range outside [0, n_total)");
  PM_CUDA(h, cudaSetDevice(h->device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  PM_CUDA(h, Prec<R>::generate(a, b, c, d, n_total, row0, count, seed, h->sm_count, st));
  h->last_stream = st;
  return PM_OK;
}

template <class R>
int dist_reduce_impl(pm_handle_t h, const R* a, const R* b, const R* c,
                       const R* d, int64_t n_local, int32_t m, int32_t rank, int32_t world,
                       R* iface, void* stream) {
  if (h) h->retry = nullptr;  // collective: no single-rank retry
  // x is not used by the reduce; pass d so the plan's alignment test sees a real pointer
  int r = validate_common(h, a, b, c, d, d, n_local, m);
  if (r) return r;
  if (!iface) return fail(h, PM_ERR_VALIDATION, "null iface pointer");
  if (world < 1 || rank < 0 || rank >= world)
    return fail(h, PM_ERR_VALIDATION, "rank must lie in [0, world)");
  const bool last = rank == world - 1;
  if (!last && n_local % m != 0)
    return fail(h, PM_ERR_VALIDATION, "n_local must be a multiple of m on every rank but the last");
  PM_CUDA(h, cudaSetDevice(h->device));
  h->launches = 0;
  // same plan (and the same 32-R prefix) as pm_dist_solve_f64
  if ((r = build_plan<R>(h, n_local, m, a, b, c, d, const_cast<R*>(d), !last, 32, false, 1, world))) return r;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  h->last_stream = st;
  const bool zf = rank == 0, zl = last;
  if (h->dist_fused) {
    if ((r = enq_reduce<R>(h, 0, 0, h->levels[0].ntiles, st, zf, zl, 0, nullptr))) return r;
    return enq_dist_upper<R>(h, pm::kModeReduce, zf, zl, rank, world, iface, nullptr, h->p2p_top.active, st);
  }
  const size_t top = h->levels.size() - 1;
  for (size_t k = 0; k < top; ++k)
    if ((r = enq_reduce<R>(h, k, 0, h->levels[k].ntiles, st, zf, zl, 0, nullptr))) return r;
  R* out4[4] = {iface, iface + 2, iface + 4, iface + 6};
  return enq_reduce<R>(h, top, 0, 1, st, zf, zl, 0, out4);
}

template <class R>
int dist_solve_impl(pm_handle_t h, const R* a, const R* b, const R* c,
                      const R* d, R* x, int64_t n_local, int32_t m, int32_t rank,
                      int32_t world, const R* iface_all, void* stream,
                      const uint64_t* flags = nullptr, uint64_t epoch = 0) {
  if (h) h->retry = nullptr;  // collective: no single-rank retry
  int r = validate_common(h, a, b, c, d, x, n_local, m);
  if (r) return r;
  if (!iface_all) return fail(h, PM_ERR_VALIDATION, "null iface_all pointer");
  if (world < 1 || rank < 0 || rank >= world)
    return fail(h, PM_ERR_VALIDATION, "rank must lie in [0, world)");
  const bool last = rank == world - 1;
  if (!last && n_local % m != 0)
    return fail(h, PM_ERR_VALIDATION, "n_local must be a multiple of m on every rank but the last");
  PM_CUDA(h, cudaSetDevice(h->device));
  h->launches = 0;
  // two extra doubles in front of the level scratch hold this rank's (xf, xl)
  if ((r = build_plan<R>(h, n_local, m, a, b, c, d, x, !last, 32, false, 1, world))) return r;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  h->last_stream = st;
  R* xb = reinterpret_cast<R*>(h->scratch);  // extra_elems region
  const bool zf = rank == 0, zl = last;
  if (h->dist_fused) {
    if (flags) {
      h->p2p_top.active = true;
      h->p2p_top.epoch = epoch;
    }
    r = enq_dist_upper<R>(h, pm::kModeSolve, zf, zl, rank, world, nullptr, iface_all, flags != nullptr, st);
    h->p2p_top.active = false;
    if (r) return r;
    return enq_solve<R>(h, 0, 0, h->levels[0].ntiles, st, zf, zl, 0, nullptr);
  }
  const size_t top = h->levels.size() - 1;
  if (flags) {  // P2P: the top-level SOLVE acquires and chains the interface rows itself
    h->p2p_top.active = true;
    h->p2p_top.epoch = epoch;
    r = enq_solve<R>(h, top, 0, 1, st, zf, zl, 0, xb);
    h->p2p_top.active = false;
    if (r) return r;
  } else {
    PM_CUDA(h, Prec<R>::dist_chain(iface_all, world, rank, xb, h->dflag, st));
    ++h->launches;
    if ((r = enq_solve<R>(h, top, 0, 1, st, zf, zl, 0, xb))) return r;
  }
  for (size_t k = top; k-- > 0;)
    if ((r = enq_solve<R>(h, k, 0, h->levels[k].ntiles, st, zf, zl, 0, nullptr))) return r;
  return PM_OK;
}

// ---- batch of independent systems from host memory (config 4 end to end) --
// Chunks of whole systems flow through a ring of `depth` device staging
// slots: H2D of chunk k on the copy-in stream, the batch solve of chunk k on
// the main stream (chunks serialised there: they share the level scratch),
// D2H of chunk k on the copy-out stream.  PCIe is full duplex, so the
// copy-in of chunk k+1 overlaps the copy-out of chunk k-1: e2e time tends to
// max(H2D, D2H) instead of their sum (a single system cannot do this: its
// Stage 3 needs all of Stage 1).
template <class R>
int solve_batch_host_impl(pm_handle_t h, const R* a, const R* b, const R* c, const R* d, R* x,
                          int64_t n_per_system, int64_t batch, int32_t m, int32_t depth,
                          int64_t systems_per_chunk) {
  if (!h) return PM_ERR_VALIDATION;
  if (batch < 1 || n_per_system < 1) return fail(h, PM_ERR_VALIDATION, "batch and n_per_system must be >= 1");
  if (n_per_system > INT64_MAX / batch) return fail(h, PM_ERR_VALIDATION, "batch too large");
  int r = validate_common(h, a, b, c, d, x, n_per_system * batch, m);
  if (r) return r;
  if (depth == 0) depth = 3;
  if (depth < 1 || depth > 32) return fail(h, PM_ERR_VALIDATION, "depth must lie in [1, 32] (0 = 3)");
  // ~256 MB of a, b, c, d per chunk: config 4 end to end 255.6 ms with 64 MB
  // chunks, 246 ms from 256 MB up (0.96-0.97 of the pinned H2D bound;
  // tools/batch_host_probe.py, profiles/round2/batch_host_probe.json)
  if (systems_per_chunk <= 0)
    systems_per_chunk = std::max<int64_t>(1, ((int64_t)256 << 20) / (4 * (int64_t)sizeof(R) * n_per_system));
  systems_per_chunk = std::min<int64_t>(systems_per_chunk, batch);
  const int64_t nchunks = (batch + systems_per_chunk - 1) / systems_per_chunk;
  depth = (int)std::min<int64_t>(depth, nchunks);
  PM_CUDA(h, cudaSetDevice(h->device));
  const int64_t rows = systems_per_chunk * n_per_system;
  const size_t stride = (size_t)((rows + 31) / 32 * 32);
  const size_t need = (size_t)depth * 5 * stride * sizeof(R);
  if (need > h->hbuf_bytes) {
    if (h->hbuf) {
      PM_CUDA(h, cudaDeviceSynchronize());
      PM_CUDA(h, cudaFree(h->hbuf));
      h->hbuf = nullptr;
      h->hbuf_bytes = 0;
    }
    PM_CUDA(h, cudaMalloc(&h->hbuf, need));
    h->hbuf_bytes = need;
  }
  while ((int)h->pool.size() < 2) {
    cudaStream_t sn;
    PM_CUDA(h, cudaStreamCreateWithFlags(&sn, cudaStreamNonBlocking));
    h->pool.push_back(sn);
  }
  cudaStream_t s_in = h->pool[0], s_out = h->pool[1], s_comp = h->main;
  std::vector<cudaEvent_t> evs;
  auto cleanup = [&]() {
    for (cudaEvent_t e : evs) cudaEventDestroy(e);
  };
  auto mk = [&](cudaEvent_t* e) {
    cudaError_t err = cudaEventCreateWithFlags(e, cudaEventDisableTiming);
    if (err == cudaSuccess) evs.push_back(*e);
    return err;
  };
  std::vector<cudaEvent_t> in_done(depth), comp_done(depth), out_done(depth);
  for (int k = 0; k < depth; ++k) {
    cudaError_t e1 = mk(&in_done[k]), e2 = mk(&comp_done[k]), e3 = mk(&out_done[k]);
    if (e1 != cudaSuccess || e2 != cudaSuccess || e3 != cudaSuccess) {
      cleanup();
      return cuda_fail(h, e1 != cudaSuccess ? e1 : (e2 != cudaSuccess ? e2 : e3), "cudaEventCreate");
    }
  }
  cudaEvent_t start;
  if (mk(&start) != cudaSuccess) { cleanup(); return cuda_fail(h, cudaErrorUnknown, "cudaEventCreate"); }
  // order the three streams after everything the caller enqueued before
  cudaEventRecord(start, s_comp);
  cudaStreamWaitEvent(s_in, start, 0);
  cudaStreamWaitEvent(s_out, start, 0);
  int launches = 0;
  cudaError_t e = cudaSuccess;
  for (int64_t k = 0; k < nchunks && e == cudaSuccess; ++k) {
    const int slot = (int)(k % depth);
    const int64_t s0 = k * systems_per_chunk;
    const int64_t ns = std::min<int64_t>(systems_per_chunk, batch - s0);
    const int64_t r0 = s0 * n_per_system, nr = ns * n_per_system;
    R* base = reinterpret_cast<R*>(h->hbuf) + (size_t)slot * 5 * stride;
    R* da = base;
    R* db = base + stride;
    R* dc = base + 2 * stride;
    R* dd = base + 3 * stride;
    R* dx = base + 4 * stride;
    const size_t bytes = (size_t)nr * sizeof(R);
    if (k >= depth) cudaStreamWaitEvent(s_in, out_done[slot], 0);  // slot free again
    if (e == cudaSuccess) e = cudaMemcpyAsync(da, a + r0, bytes, cudaMemcpyHostToDevice, s_in);
    if (e == cudaSuccess) e = cudaMemcpyAsync(db, b + r0, bytes, cudaMemcpyHostToDevice, s_in);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dc, c + r0, bytes, cudaMemcpyHostToDevice, s_in);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dd, d + r0, bytes, cudaMemcpyHostToDevice, s_in);
    cudaEventRecord(in_done[slot], s_in);
    cudaStreamWaitEvent(s_comp, in_done[slot], 0);
    if (e != cudaSuccess) break;
    if ((r = solve_batch_impl<R>(h, da, db, dc, dd, dx, n_per_system, ns, m, s_comp))) {
      cleanup();
      return r;
    }
    launches += h->launches;
    cudaEventRecord(comp_done[slot], s_comp);
    cudaStreamWaitEvent(s_out, comp_done[slot], 0);
    e = cudaMemcpyAsync(x + r0, dx, bytes, cudaMemcpyDeviceToHost, s_out);
    cudaEventRecord(out_done[slot], s_out);
  }
  if (e != cudaSuccess) { cleanup(); return cuda_fail(h, e, "cudaMemcpyAsync"); }
  cudaError_t se = cudaStreamSynchronize(s_out);
  if (se == cudaSuccess) se = cudaStreamSynchronize(s_comp);
  cleanup();
  h->retry = nullptr;  // the per-chunk retries are gone with the staging slots
  if (se != cudaSuccess) return cuda_fail(h, se, "batch solve");
  h->launches = launches;
  h->last_stream = s_comp;
  return read_flag(h, s_comp);
}

// ---- P2P interface exchange (NVLink peer memory instead of the all-gather) --

size_t exchange_bytes(int world) {
  // [2][world][8] reals (sized for FP64; FP32 uses the first half) | [2][world] uint64
  return (size_t)2 * world * 8 * sizeof(double) + (size_t)2 * world * sizeof(uint64_t);
}

template <class R>
int dist_reduce_p2p_impl(pm_handle_t h, const R* a, const R* b, const R* c, const R* d,
                         int64_t n_local, int32_t m, void* stream) {
  if (!h) return PM_ERR_VALIDATION;
  if (!h->d_peers || h->xworld < 1) return fail(h, PM_ERR_VALIDATION, "pm_dist_set_peers not called");
  if (!h->iface_local) PM_CUDA(h, cudaMalloc(&h->iface_local, 8 * sizeof(double)));
  // the rank's top-level REDUCE publishes its two rows to every peer itself
  h->p2p_top.active = true;
  h->p2p_top.epoch = h->epoch + 1;
  const int r = dist_reduce_impl<R>(h, a, b, c, d, n_local, m, h->xrank, h->xworld,
                                    static_cast<R*>(h->iface_local), stream);
  h->p2p_top.active = false;
  if (r) return r;
  ++h->epoch;
  return PM_OK;
}

template <class R>
int dist_solve_p2p_impl(pm_handle_t h, const R* a, const R* b, const R* c, const R* d, R* x,
                        int64_t n_local, int32_t m, void* stream) {
  if (!h) return PM_ERR_VALIDATION;
  if (!h->d_peers || !h->xbuf || h->xworld < 1)
    return fail(h, PM_ERR_VALIDATION, "pm_dist_exchange_alloc / pm_dist_set_peers not called");
  if (h->epoch == 0) return fail(h, PM_ERR_VALIDATION, "pm_dist_reduce_p2p must precede the solve");
  const R* slots = reinterpret_cast<const R*>(h->xbuf);
  // flags at a fixed byte offset for both precisions (exchange_bytes)
  const uint64_t* flags = reinterpret_cast<const uint64_t*>(static_cast<const char*>(h->xbuf) +
                                                            (size_t)2 * h->xworld * 8 * sizeof(double));
  return dist_solve_impl<R>(h, a, b, c, d, x, n_local, m, h->xrank, h->xworld, slots, stream, flags,
                            h->epoch);
}

// ---- one-call collective solve (pm_solve_dist_*): reduce, exchange, solve --
// The exchange is the caller's all-gather (callback) or NCCL's (dlopen).
// Both halves and the exchange are ordered on `stream`; the handle's
// coll_buf holds this rank's 8 interface reals and the gathered 8*world.
template <class R, class Gather>
int solve_dist_impl(pm_handle_t h, const R* a, const R* b, const R* c, const R* d, R* x, int64_t n_local,
                    int32_t m, int32_t rank, int32_t world, void* stream, Gather&& gather) {
  if (!h) return PM_ERR_VALIDATION;
  if (world < 1 || rank < 0 || rank >= world) return fail(h, PM_ERR_VALIDATION, "rank must lie in [0, world)");
  const size_t need = (size_t)(8 + 8 * (size_t)world) * sizeof(R);
  if (h->coll_bytes < need) {
    PM_CUDA(h, cudaSetDevice(h->device));
    if (h->coll_buf) {
      PM_CUDA(h, cudaDeviceSynchronize());  // an earlier solve may still read it
      cudaFree(h->coll_buf);
      h->coll_buf = nullptr;
      h->coll_bytes = 0;
    }
    PM_CUDA(h, cudaMalloc(&h->coll_buf, need));
    h->coll_bytes = need;
  }
  R* iface = static_cast<R*>(h->coll_buf);
  R* iface_all = iface + 8;
  int r = dist_reduce_impl<R>(h, a, b, c, d, n_local, m, rank, world, iface, stream);
  if (r) return r;
  const int reduce_launches = h->launches;
  std::string why;
  if (gather(static_cast<const void*>(iface), static_cast<void*>(iface_all), why) != 0)
    return fail(h, PM_ERR_RUNTIME, why);
  r = dist_solve_impl<R>(h, a, b, c, d, x, n_local, m, rank, world, iface_all, stream);
  h->launches += reduce_launches;
  return r;
}

template <class R>
int solve_dist_cb_impl(pm_handle_t h, const R* a, const R* b, const R* c, const R* d, R* x, int64_t n_local,
                       int32_t m, int32_t rank, int32_t world, pm_allgather_fn allgather, void* user,
                       void* stream) {
  if (h && !allgather) return fail(h, PM_ERR_VALIDATION, "null all-gather callback");
  return solve_dist_impl<R>(h, a, b, c, d, x, n_local, m, rank, world, stream,
                            [&](const void* send, void* recv, std::string& why) {
                              const int st = allgather(send, recv, (int64_t)(8 * sizeof(R)), stream, user);
                              if (st != 0) why = "all-gather callback returned " + std::to_string(st);
                              return st;
                            });
}

template <class R>
int solve_dist_nccl_impl(pm_handle_t h, const R* a, const R* b, const R* c, const R* d, R* x,
                         int64_t n_local, int32_t m, void* comm, void* stream) {
  if (!h) return PM_ERR_VALIDATION;
  if (!comm) return fail(h, PM_ERR_VALIDATION, "null NCCL communicator");
  std::string why;
  int world = 0, rank = 0;
  if (pmnccl::comm_count(comm, &world, &why) != 0 || pmnccl::comm_user_rank(comm, &rank, &why) != 0)
    return fail(h, PM_ERR_RUNTIME, why);
  return solve_dist_impl<R>(h, a, b, c, d, x, n_local, m, rank, world, stream,
                            [&](const void* send, void* recv, std::string& w) {
                              return pmnccl::all_gather(send, recv, 8, sizeof(R) == 8, comm, stream, &w);
                            });
}

extern "C" {

int pm_get_version(void) { return 100; }

int pm_create(pm_handle_t* out, int device) {
  if (!out) return PM_ERR_VALIDATION;
  *out = nullptr;
  pm_handle_t h = new pm_handle_s();
  h->device = device;
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&h->sm_count, cudaDevAttrMultiProcessorCount, device);
  if (e == cudaSuccess) e = cudaMalloc(&h->dflag, sizeof(int));
  if (e == cudaSuccess) e = cudaMemset(h->dflag, 0, sizeof(int));
  if (e == cudaSuccess) e = cudaMalloc(&h->dsync, 8 * sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMemset(h->dsync, 0, 8 * sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&h->main, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete h;
    return PM_ERR_RUNTIME;
  }
  *out = h;
  return PM_OK;
}

int pm_destroy(pm_handle_t h) {
  if (!h) return PM_OK;
  cudaSetDevice(h->device);
  cudaDeviceSynchronize();
  for (cudaStream_t s : h->pool) cudaStreamDestroy(s);
  for (cudaEvent_t e : h->kev) cudaEventDestroy(e);
  if (h->main) cudaStreamDestroy(h->main);
  if (h->scratch) cudaFree(h->scratch);
  if (h->bscr) cudaFree(h->bscr);
  if (h->bcnt) cudaFree(h->bcnt);
  if (h->dstats) cudaFree(h->dstats);
  if (h->hbuf) cudaFree(h->hbuf);
  if (h->dflag) cudaFree(h->dflag);
  if (h->dsync) cudaFree(h->dsync);
  if (h->xbuf) cudaFree(h->xbuf);
  if (h->d_peers) cudaFree(h->d_peers);
  if (h->iface_local) cudaFree(h->iface_local);
  if (h->coll_buf) cudaFree(h->coll_buf);
  for (auto& g : h->graphs) cudaGraphExecDestroy(g.exec);
  delete h;
  return PM_OK;
}

const char* pm_last_error(pm_handle_t h) { return h ? h->err.c_str() : "null handle"; }

int pm_set_option(pm_handle_t h, int option, int64_t value) {
  if (!h) return PM_ERR_VALIDATION;
  ++h->plan_gen;  // recorded graphs of earlier settings are not reused
  switch (option) {
    case PM_OPT_GRAPHS:
      h->use_graphs = value ? 1 : 0;
      return PM_OK;
    case PM_OPT_STAGES:
      if (value < 1 || value > 4) return fail(h, PM_ERR_VALIDATION, "stages must lie in [1, 4]");
      h->stages = (int)value;
      return PM_OK;
    case PM_OPT_STREAM_MODE:
      if (value != 0 && value != 1) return fail(h, PM_ERR_VALIDATION, "stream mode is 0 or 1");
      h->stream_mode = (int)value;
      return PM_OK;
    case PM_OPT_REVERSE_SOLVE:
      h->reverse = value ? 1 : 0;
      return PM_OK;
    case PM_OPT_MAX_CTAS:
      if (value < 0) return fail(h, PM_ERR_VALIDATION, "max_ctas must be >= 0");
      h->max_ctas = (int)value;
      return PM_OK;
    case PM_OPT_TIMINGS:
      h->timings = value ? 1 : 0;
      return PM_OK;
    case PM_OPT_WARP_TILES:
      h->warp_tiles = value ? 1 : 0;
      return PM_OK;
    case PM_OPT_SOLVE_STAGES:
      if (value < 0 || value > 4) return fail(h, PM_ERR_VALIDATION, "solve stages must lie in [0, 4]");
      h->solve_stages = (int)value;
      return PM_OK;
    case PM_OPT_PDL:
      // process-wide launch attribute: every handle's recorded graphs carry
      // the old attribute, so the global generation invalidates them all
      pm::set_pdl(value != 0);
      pm32::set_pdl(value != 0);
      g_pdl_gen.fetch_add(1, std::memory_order_relaxed);
      return PM_OK;
    case PM_OPT_CHAIN:
      h->opt_chain = value ? 1 : 0;
      return PM_OK;
    case PM_OPT_UPPER_M:
      if (value != 0 && (value < 2 || value > 16))
        return fail(h, PM_ERR_VALIDATION, "upper m must be 0 or lie in [2, 16]");
      h->upper_m = (int)value;
      return PM_OK;
    case PM_OPT_ROOT_M:
      if (value < 2 || value > PM_MAX_M) return fail(h, PM_ERR_VALIDATION, "root m out of range");
      h->root_m = (int)value;
      return PM_OK;
    case PM_OPT_WARPS_PER_CTA:
      if (value < 1 || value > 4) return fail(h, PM_ERR_VALIDATION, "warps per CTA must lie in [1, 4]");
      h->warps_per_cta = (int)value;
      return PM_OK;
    case PM_OPT_BATCH_CLUSTER:
      if (value < 0 || value > 2) return fail(h, PM_ERR_VALIDATION, "batch kernel must be 0, 1 or 2");
      h->batch_cluster = (int)value;
      return PM_OK;
    case PM_OPT_BATCH_LAG:
      if (value < 0 || (value & 0xff) > 64 || (value >> 8) > 65)
        return fail(h, PM_ERR_VALIDATION, "batch lag must be L + 256 * (extra + 1), L in [0, 64], extra in [0, 64]");
      h->batch_lag = (int)value;
      return PM_OK;
    case PM_OPT_BATCH_DISCARD:
      if (value < 0 || value > 15) return fail(h, PM_ERR_VALIDATION, "batch discard must lie in [0, 15]");
      h->batch_discard = (int)value;
      return PM_OK;
    case PM_OPT_BATCH_STATS:
      h->batch_stats = value ? 1 : 0;
      return PM_OK;
    case PM_OPT_BATCH_L2_MB:
      if (value < 1 || value > 1024) return fail(h, PM_ERR_VALIDATION, "L2 budget must lie in [1, 1024] MB");
      h->batch_l2_mb = (int)value;
      return PM_OK;
    case PM_OPT_BATCH_CLUSTER_SIZE:
      if (value < 0 || value > 16) return fail(h, PM_ERR_VALIDATION, "cluster size must lie in [0, 16]");
      h->batch_force_cluster = (int)value;
      return PM_OK;
    case PM_OPT_BATCH_WARPS:
      if (value != 0 && (value < 2 || value > 16))
        return fail(h, PM_ERR_VALIDATION, "batch warps must be 0 or lie in [2, 16]");
      h->batch_force_warps = (int)value;
      return PM_OK;
    case PM_OPT_BATCH_STAGES:
      if (value < 0 || value > 2) return fail(h, PM_ERR_VALIDATION, "batch stages must lie in [0, 2]");
      h->batch_force_stages = (int)value;
      return PM_OK;
    case PM_OPT_UPPER_CTA_M:
      if (value < 2 || value > 32) return fail(h, PM_ERR_VALIDATION, "upper CTA m must lie in [2, 32]");
      h->upper_cta_m = (int)value;
      return PM_OK;
    case PM_OPT_UPPER_CTA_P:
      if (value != 64 && value != 128 && value != 256)
        return fail(h, PM_ERR_VALIDATION, "upper CTA threads must be 64, 128 or 256");
      h->upper_cta_p = (int)value;
      return PM_OK;
    case PM_OPT_UPPER_FUSED:
      if (value < 0 || value > 2) return fail(h, PM_ERR_VALIDATION, "upper fused must be 0, 1 or 2");
      h->upper_fused = (int)value;
      return PM_OK;
    case PM_OPT_PAIR_STAGES:
      if (value < 1 || value > 4) return fail(h, PM_ERR_VALIDATION, "pair stages must lie in [1, 4]");
      h->pair_stages = (int)value;
      return PM_OK;
    case PM_OPT_PAIR_TILES:
      if (value < -1 || value > 1) return fail(h, PM_ERR_VALIDATION, "pair tiles is -1 (auto), 0 or 1");
      h->pair_tiles = (int)value;
      return PM_OK;
    case PM_OPT_KERNEL_TIMES:
      h->ktimes = value ? 1 : 0;
      h->krec.clear();
      return PM_OK;
    default:
      return fail(h, PM_ERR_VALIDATION, "unknown option");
  }
}

int pm_solve_device_f64(pm_handle_t h, const double* a, const double* b, const double* c,
                        const double* d, double* x, int64_t n, int32_t m, void* stream) {
  return solve_device_impl<double>(h, a, b, c, d, x, n, m, stream);
}
int pm_solve_device_f32(pm_handle_t h, const float* a, const float* b, const float* c,
                        const float* d, float* x, int64_t n, int32_t m, void* stream) {
  return solve_device_impl<float>(h, a, b, c, d, x, n, m, stream);
}

int pm_solve_batch_device_f64(pm_handle_t h, const double* a, const double* b, const double* c,
                              const double* d, double* x, int64_t n_per_system, int64_t batch,
                              int32_t m, void* stream) {
  return solve_batch_impl<double>(h, a, b, c, d, x, n_per_system, batch, m, stream);
}
int pm_solve_batch_device_f32(pm_handle_t h, const float* a, const float* b, const float* c,
                              const float* d, float* x, int64_t n_per_system, int64_t batch,
                              int32_t m, void* stream) {
  return solve_batch_impl<float>(h, a, b, c, d, x, n_per_system, batch, m, stream);
}

int pm_last_batch_plan(pm_handle_t h, int32_t* out6) {
  if (!h || !out6) return PM_ERR_VALIDATION;
  const pm::BatchPlan& p = h->last_batch_plan;
  out6[0] = p.cluster; out6[1] = p.warps; out6[2] = p.stages;
  out6[3] = p.kmax; out6[4] = p.ntiles; out6[5] = p.clusters;
  return PM_OK;
}

int pm_last_stream_plan(pm_handle_t h, int32_t* out8) {
  if (!h || !out8) return PM_ERR_VALIDATION;
  const pm::StreamPlan& p = h->last_stream_plan;
  out8[0] = p.ctas > 0; out8[1] = p.warps; out8[2] = p.stages; out8[3] = p.lag;
  out8[4] = p.ring; out8[5] = p.ctas; out8[6] = p.nw; out8[7] = p.tps;
  return PM_OK;
}

int pm_batch_stream_stats(pm_handle_t h, uint64_t* out15) {
  if (!h || !out15) return PM_ERR_VALIDATION;
  if (!h->dstats) {
    std::memset(out15, 0, 15 * sizeof(uint64_t));
    return PM_OK;
  }
  PM_CUDA(h, cudaSetDevice(h->device));
  PM_CUDA(h, cudaDeviceSynchronize());
  PM_CUDA(h, cudaMemcpy(out15, h->dstats, 15 * sizeof(uint64_t), cudaMemcpyDeviceToHost));
  return PM_OK;
}

int pm_batch_stream_timeline(pm_handle_t h, uint64_t* out, int64_t n) {
  if (!h || !out || n < 0) return PM_ERR_VALIDATION;
  std::memset(out, 0, (size_t)n * sizeof(uint64_t));
  const int64_t have = 5 * h->dstats_batch + 8 * 2400 * 4 + 1200 * 2 + 4096 * 12;
  if (n > have) n = have;
  if (!h->dstats || n == 0) return PM_OK;
  PM_CUDA(h, cudaSetDevice(h->device));
  PM_CUDA(h, cudaDeviceSynchronize());
  PM_CUDA(h, cudaMemcpy(out, h->dstats + 16, (size_t)n * sizeof(uint64_t), cudaMemcpyDeviceToHost));
  return PM_OK;
}

int pm_batch_stream_counters(pm_handle_t h, uint32_t* out, int64_t n) {
  if (!h || !out || n < 0) return PM_ERR_VALIDATION;
  const int64_t have = (int64_t)(h->bcnt_bytes / sizeof(uint32_t));
  std::memset(out, 0, (size_t)n * sizeof(uint32_t));
  if (n > have) n = have;
  if (!h->bcnt || n == 0) return PM_OK;
  PM_CUDA(h, cudaSetDevice(h->device));
  PM_CUDA(h, cudaDeviceSynchronize());
  PM_CUDA(h, cudaMemcpy(out, h->bcnt, (size_t)n * sizeof(uint32_t), cudaMemcpyDeviceToHost));
  return PM_OK;
}

int pm_check(pm_handle_t h) {
  if (!h) return PM_ERR_VALIDATION;
  PM_CUDA(h, cudaSetDevice(h->device));
  cudaStream_t st = h->last_stream;
  cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(h, e, "solve");
  return read_flag(h, h->main);
}

int pm_solve_host_f64(pm_handle_t h, const double* a, const double* b, const double* c,
                      const double* d, double* x, int64_t n, int32_t m, int32_t num_streams) {
  return solve_host_impl<double>(h, a, b, c, d, x, n, m, num_streams);
}
int pm_solve_host_f32(pm_handle_t h, const float* a, const float* b, const float* c,
                      const float* d, float* x, int64_t n, int32_t m, int32_t num_streams) {
  return solve_host_impl<float>(h, a, b, c, d, x, n, m, num_streams);
}

int pm_last_stage_timings(pm_handle_t h, pm_stage_timings* out, double* total_ms,
                          int32_t* streams_used) {
  if (!h) return PM_ERR_VALIDATION;
  if (out) *out = h->last_t;
  if (total_ms) *total_ms = h->last_total_ms;
  if (streams_used) *streams_used = h->last_streams;
  return PM_OK;
}

int pm_host_register(void* ptr, uint64_t bytes) {
  if (!ptr || bytes == 0) return PM_ERR_VALIDATION;
  return cudaHostRegister(ptr, bytes, cudaHostRegisterDefault) == cudaSuccess ? PM_OK : PM_ERR_RUNTIME;
}
int pm_host_unregister(void* ptr) {
  if (!ptr) return PM_ERR_VALIDATION;
  return cudaHostUnregister(ptr) == cudaSuccess ? PM_OK : PM_ERR_RUNTIME;
}

int pm_set_model_bundle(pm_handle_t h, const pm_model_bundle* bundle) {
  if (!h || !bundle) return PM_ERR_VALIDATION;
  try {
    streamtune::ModelBundle b = from_c(*bundle);
    b.validate();
    h->bundle = b;
  } catch (const std::exception& ex) {
    return fail(h, PM_ERR_VALIDATION, ex.what());
  }
  return PM_OK;
}

int pm_get_model_bundle(pm_handle_t h, pm_model_bundle* out) {
  if (!h || !out) return PM_ERR_VALIDATION;
  to_c(h->bundle, out);
  return PM_OK;
}

int pm_paper_bundle(pm_model_bundle* out) {
  if (!out) return PM_ERR_VALIDATION;
  to_c(streamtune::ModelBundle::paper(), out);
  return PM_OK;
}

int pm_b200_bundle(pm_model_bundle* out) {
  if (!out) return PM_ERR_VALIDATION;
  to_c(streamtune::ModelBundle::b200(), out);
  return PM_OK;
}

int pm_recommend_streams(int64_t n, const pm_model_bundle* bundle) {
  if (n < 1) return -1;
  try {
    streamtune::ModelBundle b = bundle ? from_c(*bundle) : streamtune::ModelBundle::paper();
    b.validate();
    return streamtune::recommend(b, (uint64_t)n).chosen.value();
  } catch (...) {
    return -1;
  }
}

int pm_generate_f64(pm_handle_t h, double* a, double* b, double* c, double* d, int64_t n,
                    uint64_t seed, void* stream) {
  return pm_generate_range_f64(h, a, b, c, d, n, 0, n, seed, stream);
}
int pm_generate_f32(pm_handle_t h, float* a, float* b, float* c, float* d, int64_t n,
                    uint64_t seed, void* stream) {
  return pm_generate_range_f32(h, a, b, c, d, n, 0, n, seed, stream);
}

int pm_generate_range_f64(pm_handle_t h, double* a, double* b, double* c, double* d,
                          int64_t n_total, int64_t row0, int64_t count, uint64_t seed,
                          void* stream) {
  return generate_range_impl<double>(h, a, b, c, d, n_total, row0, count, seed, stream);
}
int pm_generate_range_f32(pm_handle_t h, float* a, float* b, float* c, float* d,
                          int64_t n_total, int64_t row0, int64_t count, uint64_t seed,
                          void* stream) {
  return generate_range_impl<float>(h, a, b, c, d, n_total, row0, count, seed, stream);
}

int pm_dist_reduce_f64(pm_handle_t h, const double* a, const double* b, const double* c,
                       const double* d, int64_t n_local, int32_t m, int32_t rank, int32_t world,
                       double* iface, void* stream) {
  return dist_reduce_impl<double>(h, a, b, c, d, n_local, m, rank, world, iface, stream);
}
int pm_dist_reduce_f32(pm_handle_t h, const float* a, const float* b, const float* c,
                       const float* d, int64_t n_local, int32_t m, int32_t rank, int32_t world,
                       float* iface, void* stream) {
  return dist_reduce_impl<float>(h, a, b, c, d, n_local, m, rank, world, iface, stream);
}

int pm_dist_solve_f64(pm_handle_t h, const double* a, const double* b, const double* c,
                      const double* d, double* x, int64_t n_local, int32_t m, int32_t rank,
                      int32_t world, const double* iface_all, void* stream) {
  return dist_solve_impl<double>(h, a, b, c, d, x, n_local, m, rank, world, iface_all, stream);
}
int pm_dist_solve_f32(pm_handle_t h, const float* a, const float* b, const float* c,
                      const float* d, float* x, int64_t n_local, int32_t m, int32_t rank,
                      int32_t world, const float* iface_all, void* stream) {
  return dist_solve_impl<float>(h, a, b, c, d, x, n_local, m, rank, world, iface_all, stream);
}

int pm_solve_batch_host_f64(pm_handle_t h, const double* a, const double* b, const double* c,
                            const double* d, double* x, int64_t n_per_system, int64_t batch, int32_t m,
                            int32_t depth, int64_t systems_per_chunk) {
  return solve_batch_host_impl<double>(h, a, b, c, d, x, n_per_system, batch, m, depth, systems_per_chunk);
}
int pm_solve_batch_host_f32(pm_handle_t h, const float* a, const float* b, const float* c,
                            const float* d, float* x, int64_t n_per_system, int64_t batch, int32_t m,
                            int32_t depth, int64_t systems_per_chunk) {
  return solve_batch_host_impl<float>(h, a, b, c, d, x, n_per_system, batch, m, depth, systems_per_chunk);
}

int pm_solve_dist_f64(pm_handle_t h, const double* a, const double* b, const double* c, const double* d,
                      double* x, int64_t n_local, int32_t m, int32_t rank, int32_t world,
                      pm_allgather_fn allgather, void* user, void* stream) {
  return solve_dist_cb_impl<double>(h, a, b, c, d, x, n_local, m, rank, world, allgather, user, stream);
}
int pm_solve_dist_f32(pm_handle_t h, const float* a, const float* b, const float* c, const float* d,
                      float* x, int64_t n_local, int32_t m, int32_t rank, int32_t world,
                      pm_allgather_fn allgather, void* user, void* stream) {
  return solve_dist_cb_impl<float>(h, a, b, c, d, x, n_local, m, rank, world, allgather, user, stream);
}
int pm_solve_dist_nccl_f64(pm_handle_t h, const double* a, const double* b, const double* c,
                           const double* d, double* x, int64_t n_local, int32_t m, void* nccl_comm,
                           void* stream) {
  return solve_dist_nccl_impl<double>(h, a, b, c, d, x, n_local, m, nccl_comm, stream);
}
int pm_solve_dist_nccl_f32(pm_handle_t h, const float* a, const float* b, const float* c, const float* d,
                           float* x, int64_t n_local, int32_t m, void* nccl_comm, void* stream) {
  return solve_dist_nccl_impl<float>(h, a, b, c, d, x, n_local, m, nccl_comm, stream);
}

int pm_nccl_version(void) { return pmnccl::load(nullptr) ? pmnccl::version() : -1; }

int pm_nccl_get_unique_id(pm_handle_t h, void* id_out) {
  if (!h) return PM_ERR_VALIDATION;
  if (!id_out) return fail(h, PM_ERR_VALIDATION, "null id buffer");
  std::string why;
  if (pmnccl::get_unique_id(id_out, &why) != 0) return fail(h, PM_ERR_RUNTIME, why);
  return PM_OK;
}

int pm_nccl_comm_init(pm_handle_t h, void** comm_out, int32_t world, const void* id, int32_t rank) {
  if (!h) return PM_ERR_VALIDATION;
  if (!comm_out || !id) return fail(h, PM_ERR_VALIDATION, "null communicator / id pointer");
  if (world < 1 || rank < 0 || rank >= world) return fail(h, PM_ERR_VALIDATION, "rank must lie in [0, world)");
  PM_CUDA(h, cudaSetDevice(h->device));
  std::string why;
  if (pmnccl::comm_init_rank(comm_out, world, id, rank, &why) != 0) return fail(h, PM_ERR_RUNTIME, why);
  return PM_OK;
}

int pm_nccl_comm_destroy(pm_handle_t h, void* comm) {
  if (!h) return PM_ERR_VALIDATION;
  if (!comm) return PM_OK;
  PM_CUDA(h, cudaSetDevice(h->device));
  std::string why;
  if (pmnccl::comm_destroy(comm, &why) != 0) return fail(h, PM_ERR_RUNTIME, why);
  return PM_OK;
}

int64_t pm_dist_exchange_bytes(int32_t world) {
  return world < 1 ? -1 : (int64_t)exchange_bytes(world);
}

int pm_dist_exchange_alloc(pm_handle_t h, int32_t world, void** out) {
  if (!h || !out || world < 1) return h ? fail(h, PM_ERR_VALIDATION, "world must be >= 1") : PM_ERR_VALIDATION;
  PM_CUDA(h, cudaSetDevice(h->device));
  if (h->xbuf) {
    PM_CUDA(h, cudaDeviceSynchronize());
    PM_CUDA(h, cudaFree(h->xbuf));
    h->xbuf = nullptr;
  }
  PM_CUDA(h, cudaMalloc(&h->xbuf, exchange_bytes(world)));
  PM_CUDA(h, cudaMemset(h->xbuf, 0, exchange_bytes(world)));
  h->xbuf_world = world;
  h->epoch = 0;
  *out = h->xbuf;
  return PM_OK;
}

int pm_dist_set_peers(pm_handle_t h, void* const* peer_bufs, int32_t world, int32_t rank) {
  if (!h || !peer_bufs) return PM_ERR_VALIDATION;
  if (world < 1 || rank < 0 || rank >= world) return fail(h, PM_ERR_VALIDATION, "rank must lie in [0, world)");
  if (world > 64) return fail(h, PM_ERR_VALIDATION, "the P2P exchange supports at most 64 ranks");
  if (!h->xbuf || h->xbuf_world != world)
    return fail(h, PM_ERR_VALIDATION, "pm_dist_exchange_alloc(world) must precede pm_dist_set_peers");
  for (int k = 0; k < world; ++k)
    if (!peer_bufs[k]) return fail(h, PM_ERR_VALIDATION, "null peer buffer");
  PM_CUDA(h, cudaSetDevice(h->device));
  // a new session: forget the previous epochs (callers barrier after this on
  // every rank before the first pm_dist_reduce_p2p)
  PM_CUDA(h, cudaMemset(h->xbuf, 0, exchange_bytes(world)));
  if (h->d_peers) PM_CUDA(h, cudaFree(h->d_peers));
  PM_CUDA(h, cudaMalloc(&h->d_peers, sizeof(void*) * world));
  PM_CUDA(h, cudaMemcpy(h->d_peers, peer_bufs, sizeof(void*) * world, cudaMemcpyHostToDevice));
  h->xworld = world;
  h->xrank = rank;
  h->epoch = 0;
  return PM_OK;
}

int pm_ipc_get_handle(const void* dptr, void* handle_out) {
  if (!dptr || !handle_out) return PM_ERR_VALIDATION;
  cudaIpcMemHandle_t hd;
  if (cudaIpcGetMemHandle(&hd, const_cast<void*>(dptr)) != cudaSuccess) return PM_ERR_RUNTIME;
  static_assert(sizeof(hd) == PM_IPC_HANDLE_BYTES, "CUDA IPC handle size");
  std::memcpy(handle_out, &hd, sizeof(hd));
  return PM_OK;
}

int pm_ipc_open_handle(const void* handle, void** dptr_out) {
  if (!handle || !dptr_out) return PM_ERR_VALIDATION;
  cudaIpcMemHandle_t hd;
  std::memcpy(&hd, handle, sizeof(hd));
  if (cudaIpcOpenMemHandle(dptr_out, hd, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess)
    return PM_ERR_RUNTIME;
  return PM_OK;
}

int pm_ipc_close_handle(void* dptr) {
  if (!dptr) return PM_ERR_VALIDATION;
  return cudaIpcCloseMemHandle(dptr) == cudaSuccess ? PM_OK : PM_ERR_RUNTIME;
}

int pm_dist_reduce_p2p_f64(pm_handle_t h, const double* a, const double* b, const double* c,
                           const double* d, int64_t n_local, int32_t m, void* stream) {
  return dist_reduce_p2p_impl<double>(h, a, b, c, d, n_local, m, stream);
}
int pm_dist_reduce_p2p_f32(pm_handle_t h, const float* a, const float* b, const float* c,
                           const float* d, int64_t n_local, int32_t m, void* stream) {
  return dist_reduce_p2p_impl<float>(h, a, b, c, d, n_local, m, stream);
}
int pm_dist_solve_p2p_f64(pm_handle_t h, const double* a, const double* b, const double* c,
                          const double* d, double* x, int64_t n_local, int32_t m, void* stream) {
  return dist_solve_p2p_impl<double>(h, a, b, c, d, x, n_local, m, stream);
}
int pm_dist_solve_p2p_f32(pm_handle_t h, const float* a, const float* b, const float* c,
                          const float* d, float* x, int64_t n_local, int32_t m, void* stream) {
  return dist_solve_p2p_impl<float>(h, a, b, c, d, x, n_local, m, stream);
}

int pm_last_launch_count(pm_handle_t h) { return h ? h->launches : -1; }

int pm_kernel_times(pm_handle_t h, int32_t* modes, int32_t* levels, float* ms, int32_t max) {
  if (!h) return -1;
  int k = 0;
  for (const auto& r : h->krec) {
    if (k >= max) break;
    float t = 0.f;
    if (cudaEventSynchronize(h->kev[r.ev + 1]) != cudaSuccess ||
        cudaEventElapsedTime(&t, h->kev[r.ev], h->kev[r.ev + 1]) != cudaSuccess)
      return fail(h, -1, "event timing failed"), -1;
    if (modes) modes[k] = r.mode;
    if (levels) levels[k] = r.level;
    if (ms) ms[k] = t;
    ++k;
  }
  h->krec.clear();
  return k;
}

int pm_last_plan(pm_handle_t h, int64_t* rows_per_level, int32_t max_levels) {
  if (!h) return -1;
  const int nl = (int)h->levels.size();
  for (int k = 0; k < nl && k < max_levels; ++k)
    if (rows_per_level) rows_per_level[k] = h->levels[k].n;
  return nl;
}

}  // extern "C"
