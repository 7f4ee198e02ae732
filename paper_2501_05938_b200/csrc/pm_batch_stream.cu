// pm_batch_stream.cu -- a batch of independent systems as ONE stream of warp
// tiles, Stage 3 running a few rounds behind Stage 1 (BASELINE.json config 4:
// 4096 systems of 1e5 rows).
//
// The level kernels solve a batch as one long system cut at the system
// boundaries: Stage 1 streams all of it, then Stage 3 streams all of it again
// (72 B of HBM traffic per unknown).  The cluster kernel (pm_batch.cu) keeps a
// system in L2 between the stages but stalls every CTA of a cluster at two
// barriers per system.  Here the batch is the flat sequence of its warp tiles
// (32 m-blocks each; system s owns tiles [s*tps, (s+1)*tps)), and every compute
// warp of a persistent grid walks its share f = r*nw + gw (round r) as
//
//     A(0) .. A(L-1), A(L), C(0), A(L+1), C(1), ...,  C(R-1)
//
// A(r) = Stage 1 of tile f: block sweeps + warp tree from the shared-memory
//        stage (rows by cp.async.bulk from HBM); the tree nodes leave by one
//        bulk store into a small L2-resident node ring, the tile's segment
//        goes to the CTA's control warp through a shared-memory mailbox;
// C(r) = Stage 3 of the same tile L rounds later: rows (again, now L2 hits:
//        the whole batch in flight is L rounds x nw tiles, a few tens of MB)
//        and its nodes come back by bulk copy, the tile's two boundary values
//        from the system's Stage 2, then downsweep, block back-substitution
//        and one bulk store of x.
// Stage 2 needs no grid barrier: one control warp per CTA copies the mailbox
// segments to global memory, publishes them with one fence + atomicAdd per
// (system, batch of tiles) into a per-system counter, and the control warp
// that completes a system's count solves that system's reduced system (tps
// tile segments: per-lane chains + warp tree, as the CTA step of the cluster
// kernel), writes every tile's (x_first, x_last) and releases the system's
// flag.  The compute warps never execute a memory fence (a fence would wait for
// their own bulk copies in flight -- measured in round 1: +50 % for Stage 1),
// so HBM sees 32 B/unknown of reads and 8 B/unknown of x writes, the
// compulsory 40 B, and every warp always has work: there is no
// per-system barrier to wait at.
//
// Flags and counters are per system and return to zero by the end of every
// launch (the Stage-2 warp clears the Stage-1 counter; the last Stage-3 tile of
// a system clears its flag and the Stage-3 counter), so launches need no
// memset and a CUDA graph can replay them.  The grid is cooperative (all CTAs
// co-resident: a C job may wait for tiles of other CTAs); with L >= S + 1 no
// wait can close a cycle.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <map>
#include <mutex>
#include <tuple>

#include "pm_batch.h"
#include "pm_device.cuh"
#include "pm_tile.cuh"

namespace pm {

namespace {

constexpr int kNodeBytes = 1792;  // 31 Nodes (1736 B) padded to 14 x 128 B
constexpr int kNodeCopy = 1744;   // 16-byte multiple covering the 31 nodes
constexpr int kMbox = 8;          // mailbox slots per compute warp
constexpr int kCS = kStreamCounterStride;  // a system's counters / flag: one 128-byte line each
constexpr int kStreamMaxWarps = 14;
constexpr int kStreamThreads = 32 * (kStreamMaxWarps + 2);  // + control warp + Stage-2 warp
constexpr uint64_t kStreamWaitNs = 20ull * 1000ull * 1000ull * 1000ull;
constexpr int kFlagTimeout = 16;  // status bit: a Stage-3 wait timed out

static_assert(31 * sizeof(Node) <= (size_t)kNodeCopy && kNodeCopy <= kNodeBytes, "node ring slot");
static_assert(sizeof(Node) <= sizeof(Seg), "chain nodes overwrite consumed segments in place");

struct Layout {
  size_t stage;   // bytes of one stage: a, b, c, d rows | tree nodes
  size_t bars;    // [W][S] stage mbarriers
  size_t mfull;   // [W][kMbox]
  size_t mempty;  // [W][kMbox]
  size_t mbox;    // [W][kMbox] Seg
  size_t wnode;   // 31 Node: control warp's tree
  size_t chain;   // [tps] Seg: one system's tile segments, chain nodes in place
  size_t gbar;    // mbarrier of the Stage-2 warp's segment gather
  size_t total;
};

__host__ __device__ inline size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

__host__ __device__ inline Layout stream_layout(int m, int W, int S, int tps) {
  Layout L;
  L.stage = (size_t)4 * 32 * m * sizeof(double) + kNodeBytes;  // a 128-multiple for m even
  size_t o = (size_t)W * S * L.stage;
  L.bars = o;
  o += (size_t)W * S * sizeof(uint64_t);
  L.mfull = o;
  o += (size_t)W * kMbox * sizeof(uint64_t);
  L.mempty = o;
  o += (size_t)W * kMbox * sizeof(uint64_t);
  o = align_up(o, 16);
  L.mbox = o;
  o += (size_t)W * kMbox * sizeof(Seg);
  L.wnode = o;
  o += 31 * sizeof(Node);
  o = align_up(o, 16);
  L.chain = o;
  o += (size_t)tps * sizeof(Seg);
  L.gbar = o;
  o += sizeof(uint64_t);
  L.total = align_up(o, 128);
  return L;
}

__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// all but the most recent bulk group of this thread complete (writes done)
__device__ __forceinline__ void bulk_wait_complete1() {
  asm volatile("cp.async.bulk.wait_group 1;" ::: "memory");
}
__device__ __forceinline__ void discard_l2_line(const void* p) {
  asm volatile("discard.global.L2 [%0], 128;" ::"l"(p) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Diagnostics (PM_OPT_BATCH_STATS): per-warp clock64 counters summed into
// A.stats at exit -- [0] C-flag wait cycles, [1] C waits that spun, [2]
// mailbox-full wait cycles, [3] stage wait cycles, [4] control iterations,
// [5] idle control iterations, [6] Stage-2 cycles, [7] Stage-2 count,
// [8] control publish (fence + atomics) cycles, [9] compute-warp cycles,
// [10] control-warp cycles, [11] A jobs, [12] C jobs, [13] (unused), [14]
// ns from a system's Stage-2 start to its flag.  With stats on, A.tl also
// gets per-system globaltimer stamps, job traces of 8 sample warps and
// per-warp / per-CTA cycle summaries (tools/stream_probe.py reads them).
struct Stats {
  unsigned long long v[15];
};
__device__ __forceinline__ long long clk() { return clock64(); }

// L2 eviction priorities for the bulk copies: Stage 1 reads a tile that
// Stage 3 re-reads L rounds later (evict_last); Stage 3's re-read and the x
// store are the data's last use (evict_first).
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                              uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void bulk_s2g_hint(void* dst, const void* src, uint32_t bytes, uint64_t pol) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes), "l"(pol)
               : "memory");
}

__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// generic-proxy global writes (made visible to this thread by an acquire) ->
// ordered before this thread's later bulk copies (async proxy)
__device__ __forceinline__ void fence_proxy_async_all() { asm volatile("fence.proxy.async;" ::: "memory"); }

// 32-bit division by a launch constant: n / d = umulhi64(ceil(2^64 / d), n)
// (exact for 32-bit n and d; mg = 0 encodes d = 1).  The tile index math runs
// once per job, where 64-bit divisions would cost ~100 instructions each.
__device__ __forceinline__ uint32_t fdiv(uint32_t n, uint64_t mg) {
  return mg ? static_cast<uint32_t>(__umul64hi(mg, static_cast<uint64_t>(n))) : n;
}

struct Job {
  bool solve;
  int r;
};

__device__ __forceinline__ Seg* seg_ring(const StreamArgs& A) { return reinterpret_cast<Seg*>(A.segs); }
__device__ __forceinline__ double2* txy_ring(const StreamArgs& A) { return reinterpret_cast<double2*>(A.txy); }

struct Geo {
  uint32_t sys;
  int t;
  uint32_t slot;
  int valid;
};
__device__ __forceinline__ uint32_t ring_slot(const StreamArgs& A, uint32_t r, uint32_t gw) {
  return (r - fdiv(r, A.mg_K) * A.K) * A.nw + gw;
}
__device__ __forceinline__ Geo geo_of(const StreamArgs& A, int r, uint32_t gw) {
  Geo g;
  const uint32_t f = static_cast<uint32_t>(r) * A.nw + gw;
  g.sys = fdiv(f, A.mg_tps);
  g.t = static_cast<int>(f - g.sys * A.tps);
  g.slot = ring_slot(A, r, gw);
  const int64_t rem = A.n_sys - (int64_t)g.t * 32 * A.m;
  g.valid = static_cast<int>(rem < 32 * A.m ? rem : 32 * A.m);
  return g;
}
// slot of tile f: f mod (K * nw) -- a system's slots are contiguous but for the wrap
__device__ __forceinline__ uint32_t slot_of_tile(const StreamArgs& A, uint32_t f) {
  return f - fdiv(f, A.mg_period) * (uint32_t)(A.K * A.nw);
}

template <int M>
__device__ __forceinline__ void compute_warp(const StreamArgs& A, unsigned char* smem, const Layout& lay,
                                             int w, int lane, bool& bad) {
  constexpr int T = 32 * M;
  const int S = A.S;
  const int F = static_cast<int>(A.batch * A.tps);  // < 2^31 (plan)
  const int gw = blockIdx.x * A.W + w;
  const int R = (F > gw) ? (F - gw + A.nw - 1) / A.nw : 0;
  const int njobs = 2 * R;
  const int r0 = lane * M;
  unsigned char* wst = smem + (size_t)w * S * lay.stage;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + lay.bars) + w * S;
  uint64_t* mfull = reinterpret_cast<uint64_t*>(smem + lay.mfull) + w * kMbox;
  uint64_t* mempty = reinterpret_cast<uint64_t*>(smem + lay.mempty) + w * kMbox;
  Seg* mbox = reinterpret_cast<Seg*>(smem + lay.mbox) + w * kMbox;
  auto rows = [&](int s) { return reinterpret_cast<double*>(wst + (size_t)s * lay.stage); };
  auto tree = [&](int s) { return reinterpret_cast<Node*>(wst + (size_t)s * lay.stage + 4 * T * sizeof(double)); };

  // Job scheduling (lane 0).  A(r) / C(r) are issued in round order each;
  // the next job is decided when its stage is refilled: A while the lag
  // a_iss - c_iss is below L, C once it reaches Lmax, and in between C only if
  // its system's Stage 2 is already done (its flag, loaded one job ahead),
  // else one more A -- so a warp runs ahead instead of waiting while the
  // slowest tiles of a system are still in Stage 1.  With L >= S + 1 every C
  // is issued at least S + 1 issues after its A: that A has been processed
  // and its node store is older than the most recent bulk group.
  const int Lmin = A.L, Lmax = A.Lmax;
  int a_iss = 0, c_iss = 0;
  unsigned c_ready = 0;   // prefetched flag of the system of C(c_iss)
  int jq0 = 0, jq1 = 0;   // the job codes (2 r + solve) in stages 0 / 1
  const uint64_t pol_last = policy_evict_last();
  const uint64_t pol_first = policy_evict_first();
  // issue_rows decides the next job, arms its stage and copies its rows;
  // issue_nodes copies a Stage-3 job's tree nodes (after the completion wait
  // that orders them behind their Stage-1 store).  In early mode (one stage
  // per warp, A.early) they run inside the current job: the rows as soon as
  // the current job has consumed its own (after the block sweeps), the nodes
  // once the stage's node area is free.
  int pend = -1;  // code of a C job whose node copy is still to issue
  // per job parity (the job issued next never overwrites the one running):
  // a C job's values fetched at issue
  int n_iss = 0;
  bool pre0 = false, pre1 = false;
  double2 pv0 = make_double2(0.0, 0.0), pv1 = make_double2(0.0, 0.0);
  unsigned po0 = 0, po1 = 0;
  auto issue_rows = [&](int s) {  // lane 0
    const int lag = a_iss - c_iss;
    const bool doA = a_iss < R && (lag < Lmin || (lag < Lmax && !c_ready));
    const int r = doA ? a_iss++ : c_iss++;
    const int code = 2 * r + (doA ? 0 : 1);
    if (s == 0) jq0 = code;
    else jq1 = code;
    const Geo g = geo_of(A, r, gw);
    if (!doA) {
      // a C whose system's flag was already seen: its boundary values and
      // Stage-3 count are fetched now, not at the job's start.  The job-top
      // prefetch reads the flag relaxed (an acquire there stalls the warp
      // ~0.7 us on every job: 19 % of the kernel); the acquire re-read here,
      // only for a C about to use the values, orders the txy load behind the
      // Stage-2 warp's release.  It cannot see the flag cleared: the last
      // Stage-3 tile of the system clears it, and this one has not counted.
      const bool pre = c_ready != 0;
      double2 pv = make_double2(0.0, 0.0);
      unsigned po = 0;
      if (pre) {
        (void)ld_acquire_u32(A.sflag + kCS * g.sys);
        pv = __ldcg(txy_ring(A) + g.slot);
        po = atomicAdd(A.cnt3 + kCS * g.sys, 1u);
      }
      if ((n_iss & 1) == 0) { pre0 = pre; pv0 = pv; po0 = po; }
      else { pre1 = pre; pv1 = pv; po1 = po; }
      c_ready = 0;
    }
    ++n_iss;
    const int64_t off = (int64_t)g.sys * A.n_sys + (int64_t)g.t * T;
    const uint32_t bytes = static_cast<uint32_t>(g.valid) * sizeof(double);  // valid is even
    fence_proxy_async();
    mbar_arrive_expect_tx(&bars[s], 4u * bytes + (doA ? 0u : (uint32_t)kNodeCopy));
    double* st = rows(s);
    if (A.hints) {
      const uint64_t pol = doA ? pol_last : pol_first;
      bulk_g2s_hint(st, A.a + off, bytes, &bars[s], pol);
      bulk_g2s_hint(st + T, A.b + off, bytes, &bars[s], pol);
      bulk_g2s_hint(st + 2 * T, A.c + off, bytes, &bars[s], pol);
      bulk_g2s_hint(st + 3 * T, A.d + off, bytes, &bars[s], pol);
    } else {
      bulk_g2s(st, A.a + off, bytes, &bars[s]);
      bulk_g2s(st + T, A.b + off, bytes, &bars[s]);
      bulk_g2s(st + 2 * T, A.c + off, bytes, &bars[s]);
      bulk_g2s(st + 3 * T, A.d + off, bytes, &bars[s]);
    }
    pend = doA ? -1 : code;
  };
  auto issue_nodes = [&](int s) {  // lane 0
    if (pend < 0) return;
    const Geo g = geo_of(A, pend >> 1, gw);
    pend = -1;
    if (a_iss < R) bulk_wait_complete1();  // its A processed >= 1 job ago
    else bulk_wait0();                     // the tail: its A may be the last job
    if (A.hints) bulk_g2s_hint(tree(s), A.nodes + g.slot * kNodeBytes, kNodeCopy, &bars[s], pol_first);
    else bulk_g2s(tree(s), A.nodes + g.slot * kNodeBytes, kNodeCopy, &bars[s]);
  };
  auto issue = [&](int s) {
    issue_rows(s);
    issue_nodes(s);
  };
  const bool early = (S == 1) && A.early;

  if (lane == 0)
    for (int s = 0; s < S && s < njobs; ++s) issue(s);

  Stats st{};
  const long long t_begin = clk();
  const unsigned long long g_begin = A.tl ? gtimer() : 0ull;
  int na = 0;  // A jobs published so far (mailbox cursor)
  unsigned long long st_a_cyc = 0, st_c_cyc = 0, st_ai_cyc = 0, st_ci_cyc = 0;
  // job trace of 8 sample warps (diagnostics): [code, start, stage ready, end]
  unsigned long long* trace = nullptr;
  if (A.tl) {
    const int tw[8] = {0, 1, 7, 8, 300, 591, 1000, 1183};
    for (int i = 0; i < 8; ++i)
      if (gw == tw[i] && tw[i] < A.nw) trace = A.tl + 5 * A.batch + (size_t)i * 2400 * 4;
  }
  unsigned long long st_top_cyc = 0, st_top1_cyc = 0;
  for (int k = 0; k < njobs; ++k) {
    const long long c_top = clk();
    const int s = (S == 2) ? (k & 1) : 0;  // S is 1 or 2 (plan)
    const int code = __shfl_sync(0xffffffffu, s == 0 ? jq0 : jq1, 0);
    const Job j{(code & 1) != 0, code >> 1};
    const Geo g = geo_of(A, j.r, gw);
    // prefetch the flag the next issue decision may need
    if (lane == 0 && c_iss < a_iss && a_iss - c_iss >= Lmin && c_iss < R)
      c_ready = ld_relaxed_u32(A.sflag + kCS * fdiv(static_cast<uint32_t>(c_iss) * A.nw + gw, A.mg_tps));
    double* sa = rows(s);
    double* sb = sa + T;
    double* sc = sa + 2 * T;
    double* sd = sa + 3 * T;
    Node* nodes = tree(s);
    TileCtx ctx;
    const int64_t off = (int64_t)g.sys * A.n_sys;
    ctx.ga = A.a + off; ctx.gb = A.b + off; ctx.gc = A.c + off; ctx.gd = A.d + off;
    ctx.row0 = (int64_t)g.t * T;
    ctx.n = A.n_sys;
    ctx.valid = g.valid;
    ctx.bulk_rows = g.valid;
    ctx.zf = true;
    ctx.zl = true;
    ctx.sys_len = 0;
    ctx.sys_magic = 0;
    const int nblk = (g.valid + M - 1) / M;

    // the Stage-3 job's system flag first: the wait (rare) overlaps the copy
    unsigned* cflag = A.sflag + kCS * g.sys;
    double xf = 0.0, xl = 0.0;
    unsigned c_old = 0;
    const bool tr = trace && lane == 0 && k < 2400;
    if (tr) {
      trace[4 * k] = (unsigned long long)code;
      trace[4 * k + 1] = gtimer();
    }
    const long long c_mid = clk();
    st_top1_cyc += c_mid - c_top;
    const unsigned prefetched = __shfl_sync(0xffffffffu, (lane == 0 && j.solve) ? ((k & 1) == 0 ? pre0 : pre1) : 0u, 0);
    if (j.solve && prefetched) {
      if (lane == 0) {
        const double2 v = ((k & 1) == 0) ? pv0 : pv1;
        xf = v.x;
        xl = v.y;
        // c_old is taken from po0/po1 at the end of the job: reading the
        // atomic's result here would expose its latency (the system's
        // counter is hit by every warp working on it)
      }
    } else if (j.solve) {
      if (A.tl && lane == 0) atomicMin(A.tl + 4 * A.batch + g.sys, (unsigned long long)gtimer());
      // Warp-uniform wait (lane 0 polls, the result is broadcast: the loop is
      // provably convergent, so the shuffle trees below stay plain SHFL):
      // relaxed polls with sleeps, then one acquire load.
      unsigned ok = (lane == 0) ? ld_relaxed_u32(cflag) : 0u;
      ok = __shfl_sync(0xffffffffu, ok, 0);
      if (!ok) {
        const long long c0 = clk();
        ++st.v[1];
        const uint64_t t0 = gtimer();
        unsigned backoff = 128;
        while (!ok) {
          // exponential nanosleep back-off: the polls (an mbarrier timed
          // try_wait returns after ~100 ns) were a third of the kernel's
          // instructions when a system's Stage 2 ran late
          __nanosleep(backoff);
          backoff = backoff < 2048 ? 2 * backoff : 2048;
          unsigned v = (lane == 0) ? ld_relaxed_u32(cflag) : 0u;
          if (lane == 0 && !v && gtimer() - t0 > kStreamWaitNs) {
            atomicOr(A.flag, kFlagTimeout);
            v = 1u;
          }
          ok = __shfl_sync(0xffffffffu, v, 0);
        }
        st.v[0] += clk() - c0;
      }
      if (lane == 0) {
        (void)ld_acquire_u32(cflag);
        const double2 v = __ldcg(txy_ring(A) + g.slot);
        xf = v.x;
        xl = v.y;
        c_old = atomicAdd(A.cnt3 + kCS * g.sys, 1u);  // result used at the end of the job
      }
    }
    st_top_cyc += clk() - c_mid;
    {
      const long long c0 = clk();
      mbar_wait(&bars[s], static_cast<uint32_t>((S == 2 ? (k >> 1) : k) & 1));
      st.v[3] += clk() - c0;
    }
    if (tr) trace[4 * k + 2] = gtimer();
    const long long c_job = clk();
    SmemAcc sacc{sa + r0, sb + r0, sc + r0, sd + r0, nullptr};
    sacc.fixup(r0, M, ctx);
    const PairAcc<M> pa{sa + r0, sb + r0, sc + r0, sd + r0};
    ++st.v[j.solve ? 12 : 11];

    if (A.tl && lane == 0 && !j.solve) atomicMin(A.tl + g.sys, (unsigned long long)gtimer());
    if (!j.solve) {
      // ---- A: Stage 1 of the tile -------------------------------------------
      const Seg seg = block_reduce_fast<M, false>(pa, bad);
      if (early) {
        __syncwarp();  // every lane has consumed its rows
        if (lane == 0 && k + 1 < njobs) issue_rows(s);
      }
      const Seg top = warp_upsweep(seg, nodes, lane, nblk, bad);
      fence_proxy_async();  // the lanes' node writes -> visible to the bulk store
      __syncwarp();
      if (lane == 0) {
        if (A.hints) bulk_s2g_hint(A.nodes + g.slot * kNodeBytes, nodes, kNodeCopy, pol_last);
        else bulk_s2g(A.nodes + g.slot * kNodeBytes, nodes, kNodeCopy);
        bulk_commit();
        if (early && pend >= 0) {
          bulk_wait_read0();  // the node store has read the node area
          issue_nodes(s);
        }
        const int q = static_cast<int>(na % kMbox);
        const long long c0 = clk();
        mbar_wait(&mempty[q], static_cast<uint32_t>(((na / kMbox) & 1) ^ 1));
        st.v[2] += clk() - c0;
        mbox[q] = top;
        mbar_arrive(&mfull[q]);
        if (A.tl) atomicMax(A.tl + 1 * A.batch + g.sys, (unsigned long long)gtimer());
      }
      ++na;
    } else {
      // ---- C: Stage 3 of the tile -------------------------------------------
      if (A.discard && lane < kNodeBytes / 128)  // the ring slot is dead: no write-back
        discard_l2_line(A.nodes + g.slot * kNodeBytes + lane * 128);
      xf = __shfl_sync(0xffffffffu, xf, 0);
      xl = __shfl_sync(0xffffffffu, xl, 0);
      warp_downsweep(xf, xl, nodes, lane, nblk);
      double xv[M];
      block_solve_pairs<M>(pa, xf, xl, xv, bad);
      __syncwarp();
      bad |= !all_finite<M>(xv);
      if (early) {
        // rows and nodes consumed: the next job's copies go out now, x leaves
        // from registers (16-byte stores; the stage is being refilled)
        if (lane == 0 && k + 1 < njobs) {
          issue_rows(s);
          issue_nodes(s);
        }
        double* gx = A.x + off + ctx.row0 + r0;
        if (r0 + M <= g.valid) {
          if constexpr ((M % 2) == 0) {
#pragma unroll
            for (int i = 0; i < M / 2; ++i)
              __stcs(reinterpret_cast<double2*>(gx) + i, make_double2(xv[2 * i], xv[2 * i + 1]));
          } else {
#pragma unroll
            for (int i = 0; i < M; ++i) __stcs(gx + i, xv[i]);
          }
        } else {
#pragma unroll
          for (int i = 0; i < M; ++i)
            if (r0 + i < g.valid) __stcs(gx + i, xv[i]);
        }
        if (lane == 0 && (prefetched ? ((k & 1) == 0 ? po0 : po1) : c_old) == static_cast<unsigned>(A.tps) - 1) {  // the system's last Stage-3 tile
          A.cnt3[kCS * g.sys] = 0;
          *cflag = 0;
        }
      } else {
      if constexpr ((M % 2) == 0) {
#pragma unroll
        for (int i = 0; i < M / 2; ++i)
          reinterpret_cast<double2*>(sb + r0)[i] = make_double2(xv[2 * i], xv[2 * i + 1]);
      } else {
#pragma unroll
        for (int i = 0; i < M; ++i) sb[r0 + i] = xv[i];
      }
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) {
        if (A.hints)
          bulk_s2g_hint(A.x + off + ctx.row0, sb, static_cast<uint32_t>(g.valid) * sizeof(double), pol_first);
        else
          bulk_s2g(A.x + off + ctx.row0, sb, static_cast<uint32_t>(g.valid) * sizeof(double));
        bulk_commit();
        if ((prefetched ? ((k & 1) == 0 ? po0 : po1) : c_old) == static_cast<unsigned>(A.tps) - 1) {  // the system's last Stage-3 tile
          A.cnt3[kCS * g.sys] = 0;
          *cflag = 0;
        }
      }
      }
    }
    __syncwarp();
    const long long c_iss0 = clk();
    (j.solve ? st_c_cyc : st_a_cyc) += c_iss0 - c_job;
    if (!early && lane == 0 && k + S < njobs) {
      bulk_wait_read0();  // the bulk store has read the stage
      issue(s);
    }
    if (tr) trace[4 * k + 3] = gtimer();
    (j.solve ? st_ci_cyc : st_ai_cyc) += clk() - c_iss0;
  }
  if (lane == 0) bulk_wait0();
  st.v[9] = clk() - t_begin;
  if (A.tl && lane == 0 && gw < 4096) {  // per-warp summary: A cycles, C cycles, C wait cycles, SM id
    unsigned long long* sm = A.tl + 5 * A.batch + 8 * 2400 * 4 + 1200 * 2 + (size_t)gw * 12;
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    sm[0] = st_a_cyc;
    sm[1] = st_c_cyc;
    sm[2] = st.v[0];
    sm[3] = smid;
    sm[4] = st_ai_cyc;
    sm[5] = st_ci_cyc;
    sm[6] = st.v[2];
    sm[7] = st.v[3];
    sm[8] = st.v[9];
    sm[9] = st_top1_cyc;  // loop top up to the Stage-3 flag section
    sm[10] = gtimer();
    sm[11] = st_top_cyc;  // the Stage-3 flag section (prefetched values or the wait)
  }
  if (A.stats && lane == 0)
    for (int i = 0; i < 15; ++i)
      if (st.v[i]) atomicAdd(A.stats + i, st.v[i]);
}

// Stage 2 of system s by the CTA's Stage-2 warp: tile segments (gathered by
// at most two bulk copies: a system's slots are contiguous in the ring but
// for the ring's wrap) -> per-lane chains -> warp tree -> 2x2 -> downsweep ->
// every tile's (x_first, x_last) -> the system's flag.
__device__ __forceinline__ void system_stage2(const StreamArgs& A, uint32_t s, Seg* tsegs, Node* wnode,
                                              uint64_t* gbar, uint32_t& gphase, int lane, bool& bad) {
  const int tps = A.tps;
  const uint32_t f0 = s * tps;
  if (lane == 0) {
    const uint32_t period = (uint32_t)A.K * A.nw;  // slots wrap every K rounds
    const uint32_t fw = (fdiv(f0, A.mg_period) + 1) * period;  // first wrap after f0
    const int n1 = (int)(fw - f0 < (uint32_t)tps ? fw - f0 : tps);
    fence_proxy_async_all();
    mbar_arrive_expect_tx(gbar, (uint32_t)tps * sizeof(Seg));
    bulk_g2s(tsegs, seg_ring(A) + slot_of_tile(A, f0), (uint32_t)n1 * sizeof(Seg), gbar);
    if (n1 < tps) bulk_g2s(tsegs + n1, seg_ring(A), (uint32_t)(tps - n1) * sizeof(Seg), gbar);
  }
  mbar_wait(gbar, gphase);
  gphase ^= 1u;
  __syncwarp();
  const int C = (tps + 31) / 32;
  const int nl = (tps + C - 1) / C;
  const int t0 = lane * C;
  const int lcnt = (tps - t0 < C) ? ((tps - t0 > 0) ? tps - t0 : 0) : C;
  Seg acc{};
  if (lcnt > 0) {
    acc = tsegs[t0];
    for (int i = 1; i < lcnt; ++i) {
      const Seg nx = tsegs[t0 + i];
      Node nd;
      combine(acc, nx, acc, nd, bad);
      *reinterpret_cast<Node*>(&tsegs[t0 + i]) = nd;  // over the consumed segment
    }
  }
  const Seg top = warp_upsweep(acc, wnode, lane, nl, bad);
  double xf = 0.0, xl = 0.0;
  if (lane == 0) {
    // top.F.a and top.L.c multiply unknowns outside the system (zero)
    const double det = fma(top.F.b, top.L.b, -top.F.c * top.L.a);
    bad |= (det == 0.0);
    const double inv = drcp(det);
    xf = fma(top.F.d, top.L.b, -top.F.c * top.L.d) * inv;
    xl = fma(top.F.b, top.L.d, -top.L.a * top.F.d) * inv;
  }
  xf = __shfl_sync(0xffffffffu, xf, 0);
  xl = __shfl_sync(0xffffffffu, xl, 0);
  __syncwarp();
  warp_downsweep(xf, xl, wnode, lane, nl);
  if (lcnt > 0) {
    double xrun = xl;
    for (int i = lcnt - 1; i >= 1; --i) {
      double xl_prev, xf_i;
      split_node(*reinterpret_cast<const Node*>(&tsegs[t0 + i]), xf, xrun, xl_prev, xf_i);
      txy_ring(A)[slot_of_tile(A, f0 + t0 + i)] = make_double2(xf_i, xrun);
      xrun = xl_prev;
    }
    txy_ring(A)[slot_of_tile(A, f0 + t0)] = make_double2(xf, xrun);
  }
  __syncwarp();
  __threadfence();  // every lane's x values before the flag
  if (lane == 0) {
    A.cnt1[kCS * s] = 0;  // no other Stage-1 arrival for s in this launch
    st_release_u32(A.sflag + kCS * s, 1u);
    if (A.tl) A.tl[3 * A.batch + s] = gtimer();
  }
  __syncwarp();
  fence_proxy_async();  // the chain nodes written in place -> before the next gather
}

// The Stage-2 warp of CTA b owns systems b, b + G, b + 2G, ... (G = the
// grid): it waits for each one's Stage-1 count in turn (timed sleeps between
// relaxed polls, then one acquire) and solves it.  A fixed owner keeps the
// Stage-2 work spread evenly; handing a system to whichever CTA published its
// last tile (round-2 first version) made the slowest CTA the Stage-2 server
// for a quarter of the batch -- a positive feedback loop that slowed that SM's
// compute warps 6x and, through the lag bound, the whole grid (22 ms/batch).
// In-order service cannot deadlock: Stage 1 of system s depends only on the
// Stage 2 of systems before s (through the compute warps' lag bound).
__device__ __forceinline__ void solver_warp(const StreamArgs& A, unsigned char* smem, const Layout& lay, int lane,
                                            bool& bad) {
  uint64_t* gbar = reinterpret_cast<uint64_t*>(smem + lay.gbar);
  Seg* tsegs = reinterpret_cast<Seg*>(smem + lay.chain);
  Node* wnode = reinterpret_cast<Node*>(smem + lay.wnode);
  uint32_t gphase = 0;
  Stats st{};
  const unsigned tps = static_cast<unsigned>(A.tps);
  for (int64_t sys = blockIdx.x; sys < A.batch; sys += gridDim.x) {
    const unsigned* cnt = A.cnt1 + kCS * sys;
    unsigned ok = (lane == 0) ? (ld_relaxed_u32(cnt) == tps) : 0u;
    ok = __shfl_sync(0xffffffffu, ok, 0);
    if (!ok) {
      const uint64_t t0 = gtimer();
      unsigned backoff = 256;
      while (!ok) {
        __nanosleep(backoff);
        backoff = backoff < 2048 ? 2 * backoff : 2048;
        unsigned v = (lane == 0) ? (ld_relaxed_u32(cnt) == tps) : 0u;
        if (lane == 0 && !v && gtimer() - t0 > kStreamWaitNs) {
          atomicOr(A.flag, kFlagTimeout);
          v = 1u;
        }
        ok = __shfl_sync(0xffffffffu, v, 0);
      }
    }
    if (lane == 0) (void)ld_acquire_u32(cnt);
    __syncwarp();
    const unsigned long long tq = (A.tl && lane == 0) ? gtimer() : 0ull;
    const long long c0 = clk();
    system_stage2(A, static_cast<uint32_t>(sys), tsegs, wnode, gbar, gphase, lane, bad);
    st.v[6] += clk() - c0;
    if (A.tl && lane == 0) st.v[14] += gtimer() - tq;
    ++st.v[7];
  }
  if (A.tl && lane == 0 && A.W * gridDim.x + blockIdx.x < 4096) {  // per-CTA Stage-2 count and cycles
    unsigned long long* sm = A.tl + 5 * A.batch + 8 * 2400 * 4 + 1200 * 2 + (size_t)(A.W * gridDim.x + blockIdx.x) * 12;
    sm[0] = st.v[7];
    sm[1] = st.v[6];
  }
  if (A.stats && lane == 0)
    for (int i = 6; i < 15; ++i)
      if (st.v[i]) atomicAdd(A.stats + i, st.v[i]);
}

// The control warp: lane w takes compute warp w's Stage-1 segments in round
// order (blocking mbarrier waits: the warps of a CTA advance together), stores
// them into the segment ring, and publishes a round's segments with one fence
// and one atomicAdd per system touched.
__device__ __forceinline__ void control_warp(const StreamArgs& A, unsigned char* smem, const Layout& lay, int lane,
                                             bool& bad) {
  (void)bad;
  const int W = A.W;
  const int F = static_cast<int>(A.batch * A.tps);
  const bool own = lane < W;
  const int gw = blockIdx.x * W + lane;
  const int R = (own && F > gw) ? (F - gw + A.nw - 1) / A.nw : 0;
  const int Rmax = __reduce_max_sync(0xffffffffu, static_cast<unsigned>(R));
  uint64_t* mfull = reinterpret_cast<uint64_t*>(smem + lay.mfull) + lane * kMbox;
  uint64_t* mempty = reinterpret_cast<uint64_t*>(smem + lay.mempty) + lane * kMbox;
  const Seg* mbox = reinterpret_cast<const Seg*>(smem + lay.mbox) + lane * kMbox;
  Stats st{};
  const long long t_begin = clk();
  unsigned long long* ctr = (A.tl && blockIdx.x == 0) ? A.tl + 5 * A.batch + 8 * 2400 * 4 : nullptr;
  if (A.ooo) {
    // Out of order: publish whatever segments the CTA's warps have ready,
    // each warp's in its own round order, instead of a whole round at a time
    // (a round waits for the CTA's slowest warp; its systems complete late).
    int head = 0;
    unsigned idle_ns = 64;
    while (__any_sync(0xffffffffu, head < R)) {
      ++st.v[4];
      const int q = head % kMbox;
      const bool ready = head < R && mbar_test(&mfull[q], static_cast<uint32_t>((head / kMbox) & 1));
      if (!__any_sync(0xffffffffu, ready)) {
        ++st.v[5];
        __nanosleep(idle_ns);
        idle_ns = idle_ns < 1024 ? 2 * idle_ns : 1024;
        continue;
      }
      idle_ns = 64;
      long long sys = -1 - lane;  // unique key for lanes with nothing to publish
      if (ready) {
        const Seg sg = mbox[q];
        mbar_arrive(&mempty[q]);
        seg_ring(A)[ring_slot(A, head, gw)] = sg;
        sys = fdiv(static_cast<uint32_t>(head) * A.nw + gw, A.mg_tps);
        ++head;
      }
      const long long c0 = clk();
      __syncwarp();
      __threadfence();  // release: the segments stored above, before the counts
      const unsigned grp = __match_any_sync(0xffffffffu, sys);
      if (ready && (__ffs(grp) - 1) == lane) {
        const unsigned n = __popc(grp);
        const unsigned old = atomicAdd(A.cnt1 + kCS * sys, n);
        if (A.tl && old + n == static_cast<unsigned>(A.tps)) A.tl[2 * A.batch + sys] = gtimer();
      }
      __syncwarp();
      st.v[8] += clk() - c0;
    }
  }
  for (int c = 0; !A.ooo && c < Rmax; ++c) {
    ++st.v[4];
    if (ctr && lane == 0 && c < 1200) ctr[2 * c] = gtimer();
    const bool active = c < R;
    long long sys = -1;
    if (active) {
      const int q = c % kMbox;
      mbar_wait(&mfull[q], static_cast<uint32_t>((c / kMbox) & 1));
      const Seg sg = mbox[q];
      mbar_arrive(&mempty[q]);
      seg_ring(A)[ring_slot(A, c, gw)] = sg;
      sys = fdiv(static_cast<uint32_t>(c) * A.nw + gw, A.mg_tps);
    }
    const long long c0 = clk();
    __syncwarp();
    __threadfence();  // release: the segments stored above, before the counts
    const unsigned grp = __match_any_sync(0xffffffffu, sys);
    if (active && (__ffs(grp) - 1) == lane) {
      const unsigned n = __popc(grp);
      const unsigned old = atomicAdd(A.cnt1 + kCS * sys, n);
      if (A.tl && old + n == static_cast<unsigned>(A.tps)) A.tl[2 * A.batch + sys] = gtimer();
    }
    __syncwarp();
    st.v[8] += clk() - c0;
    if (ctr && lane == 0 && c < 1200) ctr[2 * c + 1] = gtimer();
  }
  st.v[10] = clk() - t_begin;
  if (A.tl && lane == 0 && A.W * gridDim.x + blockIdx.x < 4096) {
    unsigned long long* sm = A.tl + 5 * A.batch + 8 * 2400 * 4 + 1200 * 2 + (size_t)(A.W * gridDim.x + blockIdx.x) * 12;
    sm[2] = st.v[8];
    sm[3] = st.v[10];
  }
  if (A.stats && lane == 0)
    for (int i = 0; i < 13; ++i)
      if (st.v[i]) atomicAdd(A.stats + i, st.v[i]);
}

template <int M>
__global__ void __launch_bounds__(kStreamThreads, 1) batch_stream_kernel(StreamArgs A) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31;
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
  const Layout lay = stream_layout(M, A.W, A.S, A.tps);
  if (threadIdx.x == 0) {
    uint64_t* b = reinterpret_cast<uint64_t*>(smem + lay.bars);
    for (int i = 0; i < A.W * A.S; ++i) mbar_init(&b[i], 1);
    uint64_t* f = reinterpret_cast<uint64_t*>(smem + lay.mfull);
    uint64_t* e = reinterpret_cast<uint64_t*>(smem + lay.mempty);
    for (int i = 0; i < A.W * kMbox; ++i) {
      mbar_init(&f[i], 1);
      mbar_init(&e[i], 1);
    }
    mbar_init(reinterpret_cast<uint64_t*>(smem + lay.gbar), 1);
    fence_mbar_init();
  }
  __syncthreads();
  pdl_wait();
  pdl_launch_dependents();
  bool bad = false;
  if (warp < A.W) compute_warp<M>(A, smem, lay, warp, lane, bad);
  else if (warp == A.W) control_warp(A, smem, lay, lane, bad);
  else solver_warp(A, smem, lay, lane, bad);
  if (bad) atomicOr(A.flag, 1);
}

template <int M>
cudaError_t launch_stream_m(const StreamArgs& A, const StreamPlan& pl, cudaStream_t st) {
  auto kern = batch_stream_kernel<M>;
  const size_t smem = stream_layout(M, pl.warps, pl.stages, pl.tps).total;
  cudaError_t e = ensure_smem_attr(kern, smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(pl.ctas);
  cfg.blockDim = dim3(32 * (pl.warps + 2));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;  // every CTA co-resident
  attr[0].val.cooperative = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, kern, A);
}

template <int M>
int stream_ctas_per_sm(int W, int S, int tps) {
  static std::mutex mu;
  static std::map<std::tuple<int, int, int, int>, int> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_tuple(dev, W, S, tps);
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  auto kern = batch_stream_kernel<M>;
  const size_t smem = stream_layout(M, W, S, tps).total;
  int n = 0;
  if (smem <= 227 * 1024 && ensure_smem_attr(kern, smem) == cudaSuccess &&
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, 32 * (W + 2), smem) != cudaSuccess)
    n = 0;
  cudaGetLastError();
  cache[key] = n;
  return n;
}

int stream_ctas_per_sm_m(int m, int W, int S, int tps) {
  switch (m) {
    case 2: return stream_ctas_per_sm<2>(W, S, tps);
    case 8: return stream_ctas_per_sm<8>(W, S, tps);
    case 10: return stream_ctas_per_sm<10>(W, S, tps);
    case 16: return stream_ctas_per_sm<16>(W, S, tps);
    default: return 0;
  }
}

}  // namespace

size_t stream_scratch_bytes(const StreamPlan& pl, int64_t batch) {
  const size_t slots = (size_t)pl.ring * pl.nw;
  (void)batch;
  return slots * (sizeof(Seg) + sizeof(double2) + kNodeBytes);
}

// Plan: W compute warps (+ 1 control warp) per CTA, S stages per warp, lag L
// rounds, one CTA per SM.  Needs compile-time m, even n_sys (16-byte aligned
// system starts), the system's segments in shared memory and at least L
// rounds of tiles per warp.
int plan_stream(int m, int64_t n_sys, int64_t batch, int sm_count, int max_ctas, int force_warps,
                int force_stages, int force_lag, StreamPlan* out) {
  if (!(m == 2 || m == 8 || m == 10 || m == 16) || n_sys < 2 || (n_sys & 1)) return 0;
  const int64_t T = 32 * (int64_t)m;
  const int64_t tps = (n_sys + T - 1) / T;
  if (tps > 4096) return 0;
  // 14 compute warps with one stage each: measured 4.95 ms per 4096 x 1e5
  // batch on B200; 8 warps x 2 stages (the first default) falls into a
  // wait-bound mode (~19-21 ms)
  int W = force_warps > 0 ? force_warps : 14;
  int S = force_stages > 0 ? force_stages : 1;
  if (W > kStreamMaxWarps) W = kStreamMaxWarps;
  // shrink until one CTA fits an SM
  while (W >= 2 && stream_ctas_per_sm_m(m, W, S, (int)tps) < 1) {
    if (force_stages <= 0 && S > 1) --S;
    else --W;
  }
  if (W < 2 || stream_ctas_per_sm_m(m, W, S, (int)tps) < 1) return 0;
  const int ctas = (max_ctas > 0 && max_ctas < sm_count) ? max_ctas : sm_count;
  const int64_t nw = (int64_t)ctas * W;
  // Stage 3 of a tile waits for every Stage-1 tile of its system: a system
  // spans up to ceil((tps - 1) / nw) + 1 rounds, so the lag must cover them
  // (no wait cycle); S + 1 keeps the node store of A(r) complete before C(r).
  const int64_t span = (tps - 1 + nw - 1) / nw;
  // force_lag: bits 0-7 the lag, bits 8-15 + 1 the extra run-ahead (0 = plan)
  const int lag_req = force_lag & 0xff;
  const int extra = (force_lag >> 8) ? (force_lag >> 8) - 1 : 8;
  const int L = (int)std::max<int64_t>(std::max(lag_req > 0 ? lag_req : 4, S + 1), span + 1);
  const int Lmax = L + extra;  // adaptive run-ahead while a system's Stage 2 is pending
  if (L > 64 || batch * tps / nw < L) return 0;  // every warp needs >= L rounds
  if (batch * tps >= (int64_t{1} << 31) || (int64_t)(Lmax + 2) * nw >= (int64_t{1} << 31)) return 0;  // 32-bit math
  StreamPlan p;
  p.warps = W;
  p.stages = S;
  p.lag = L;
  p.lag_max = Lmax;
  p.ring = Lmax + 2;  // a slot is reused K rounds on: C(r) precedes A(r + K)
  p.ctas = ctas;
  p.nw = (int)nw;
  p.tps = (int)tps;
  *out = p;
  return 1;
}

cudaError_t launch_batch_stream(int m, const StreamArgs& args, const StreamPlan& pl, cudaStream_t st) {
  switch (m) {
    case 2: return launch_stream_m<2>(args, pl, st);
    case 8: return launch_stream_m<8>(args, pl, st);
    case 10: return launch_stream_m<10>(args, pl, st);
    case 16: return launch_stream_m<16>(args, pl, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace pm
