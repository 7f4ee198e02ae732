/*
 * pm_tridiag.h -- C ABI of the B200-native partition-method tridiagonal solver.
 *
 * Drop-in boundary.  The reference ships no solver
 * (/root/reference/SPEC.md:12 puts "the CUDA solver itself" out of scope);
 * its only code is the header-only streamtune API
 * (/root/reference/proj/include/streamtune/timing_model.hpp,
 *  /root/reference/proj/include/streamtune/errors.hpp).  The north_star
 * names the solver API the paper's C++ code exposes: "coefficient arrays
 * a/b/c/d in, x out, sub-system size m, num_streams" (PAPER.md:52 m = 10,
 * FP64; PAPER.md:54-60 streams are powers of two up to 32).  This header is
 * that API as a plain C ABI (no torch types, no exceptions):
 *
 *   pm_solve_host_f64    <- the paper's whole pipeline:
 *                           host a,b,c,d -> x with H2D / kernels / D2H
 *                           overlapped over num_streams CUDA streams;
 *                           num_streams == 0 asks the streamtune predictor
 *                           (SPEC.md:267 recommend) for the count.
 *   pm_solve_device_f64  <- Stages 1-3 on device-resident arrays
 *                           (PAPER.md:80 Stage 1 / Stage 3 kernels; Stage 2
 *                           runs on the GPU here instead of PAPER.md:63's CPU).
 *   pm_solve_batch_device_f64, pm_dist_*  <- B200 additions (BASELINE.json
 *                           configs 4 and 5).
 *   *_f32                <- FP32 variants of the above.
 *   pm_recommend_streams <- streamtune::recommend.
 *
 * Conventions
 *   - a: sub-diagonal, b: diagonal, c: super-diagonal, d: right-hand side,
 *     all length n; a[0] and c[n-1] are ignored (treated as 0).  x may alias d.
 *   - 2 <= m <= PM_MAX_M.  Sub-system size of Stage 1.
 *   - The caller owns every buffer; the library never frees caller memory.
 *   - Status codes: PM_OK; PM_ERR_VALIDATION (streamtune::ValidationError,
 *     errors.hpp:9-14: n < 1, m out of range, bad stream count -- the
 *     InvalidStreamCountError of errors.hpp:75-86 --, null pointers);
 *     PM_ERR_COMPUTATION (streamtune::ComputationError, errors.hpp:16-21:
 *     zero or non-finite pivot); PM_ERR_RUNTIME (CUDA / NCCL failure).
 *     The message is in pm_last_error(h).
 *   - A handle is single-threaded: one handle per host thread / per GPU.
 *   - Systems must be solvable without pivoting (e.g. diagonally dominant),
 *     as for the paper's method.
 */
#ifndef PM_TRIDIAG_H
#define PM_TRIDIAG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PM_OK 0
#define PM_ERR_VALIDATION 1
#define PM_ERR_COMPUTATION 2
#define PM_ERR_RUNTIME 3

#define PM_MAX_M 128

typedef struct pm_handle_s* pm_handle_t;

/* Mirrors streamtune::StageTimings (timing_model.hpp:77-85).  ms. */
typedef struct pm_stage_timings {
  uint64_t slae_size;
  double t1_h2d, t1_comp, t1_d2h, t2_comp, t3_h2d, t3_comp, t3_d2h;
} pm_stage_timings;

/* Mirrors streamtune::ModelBundle. */
typedef struct pm_model_bundle {
  double sum_a, sum_b;
  double small_a, small_b, small_c;
  double big_a, big_b, big_c;
  uint64_t size_threshold;
  int32_t num_candidates;
  int32_t candidates[5];
} pm_model_bundle;

/* Options for pm_set_option. */
#define PM_OPT_STAGES 1        /* bulk-copy ring depth per CTA, 1..4 (default 2)   */
#define PM_OPT_STREAM_MODE 2   /* 0: pooled streams (default); 1: create and destroy
                                  the streams inside every solve, as the paper's
                                  T_overhead measures      */
#define PM_OPT_REVERSE_SOLVE 3 /* 1 (default): Stage 3 walks tiles last-to-first so
                                  the tail Stage 1 left in L2 is re-read from L2   */
#define PM_OPT_MAX_CTAS 4      /* cap on persistent CTAs per launch (0 = none)     */
#define PM_OPT_TIMINGS 5       /* 1: record StageTimings with CUDA events in
                                  pm_solve_host_f64 (num_streams == 1 only)        */
#define PM_OPT_KERNEL_TIMES 6  /* 1: bracket every kernel launch with CUDA events;
                                  read them with pm_kernel_times                   */
#define PM_OPT_WARP_TILES 7    /* 1 (default): level 0 uses warp-owned tiles of
                                  32*m rows; 0: CTA tiles (P*m rows, P <= 128)     */
#define PM_OPT_SOLVE_STAGES 8  /* ring depth of the level-0 Stage-3 kernel
                                  (default 1; 0 = PM_OPT_STAGES)                   */
#define PM_OPT_WARPS_PER_CTA 9 /* warps per CTA of the warp-tile kernels (1..4)    */
#define PM_OPT_CHAIN 10        /* 1: level-0 warps chain contiguous tile chunks, so
                                  level 1 is a single ROOT tile (default 0)        */
#define PM_OPT_UPPER_M 11      /* rows per thread of the warp-tile upper levels
                                  (default 0 = CTA tiles with m = 8)               */
#define PM_OPT_ROOT_M 12       /* ROOT tile = 128 * root_m rows (default 8)        */
#define PM_OPT_PDL 13          /* programmatic dependent launch (process-wide;
                                  default on; 0 disables it for both precisions)   */
#define PM_OPT_BATCH_CLUSTER 14 /* batch kernel of pm_solve_batch_device_f64:
                                  0: one long system through the level kernels
                                  (72 B/unknown); 1: one thread-block cluster per
                                  system (all stages while the system is L2-
                                  resident); 2: the tile-stream kernel (Stage 3 a
                                  few rounds behind Stage 1 over one stream of
                                  warp tiles, per-system Stage 2 by control warps,
                                  40 B/unknown).  1 and 2 apply to m in
                                  {2, 8, 10, 16}, even n_per_system, 16-byte
                                  aligned arrays (else the level kernels run);
                                  DESIGN.md §6                                     */
#define PM_OPT_BATCH_L2_MB 15  /* L2 budget for the systems in flight (default 64) */
#define PM_OPT_BATCH_CLUSTER_SIZE 16 /* force CTAs per cluster, 1..16 (0 = plan)  */
#define PM_OPT_BATCH_WARPS 17  /* force warps per CTA, 4..16 (0 = plan)           */
#define PM_OPT_BATCH_STAGES 18 /* force bulk-copy stages per warp, 1..2 (0 = plan) */
#define PM_OPT_UPPER_CTA_M 20  /* rows per thread of the CTA-tile upper levels (8) */
#define PM_OPT_UPPER_CTA_P 21  /* threads per CTA tile of the upper levels (128)   */
#define PM_OPT_GRAPHS 22       /* 1: device-resident solves (pm_solve_device_*,
                                  level-kernel batches) replay a cached CUDA graph
                                  per (arrays, sizes, options); stream must not be
                                  the legacy default stream (default 0)            */
#define PM_OPT_PAIR_STAGES 23  /* bulk-copy ring depth of the pair-tile Stage 1 (1) */
#define PM_OPT_UPPER_FUSED 24  /* 1 (default): levels 1-2 of a three-level plan
                                  (both of 128 x 8 CTA tiles, level 2 one tile)
                                  in one launch, one co-resident CTA per level-1
                                  tile: reduce, last CTA solves level 2, each
                                  back-solves its tile (3 launches -> 1); 0: off;
                                  2: also a row-sharded rank's upper levels in
                                  two launches (level 1 of 8-row blocks + the
                                  chain of its tile segments; pm_dist_*)        */
#define PM_OPT_BATCH_LAG 25    /* tile-stream kernel: rounds Stage 3 trails Stage 1
                                  (0 = plan, >= stages + 1)                        */
#define PM_OPT_BATCH_DISCARD 26 /* tile-stream kernel: bit 0 discards consumed
                                  node-ring lines from L2 instead of writing them
                                  back; bit 1 sets L2 eviction priorities on its
                                  bulk copies (Stage-1 reads evict_last, Stage-3
                                  re-reads and x stores evict_first); bit 2 (one
                                  stage per warp) issues the next tile's copies
                                  inside the current job; bit 3 lets the control
                                  warp publish ready segments out of round order;
                                  default 15                                      */
#define PM_OPT_BATCH_STATS 27  /* tile-stream kernel: accumulate clock64 wait /
                                  work counters (pm_batch_stream_stats; off)      */
#define PM_OPT_PAIR_TILES 19   /* level-0 pair tiles (two m-blocks per lane, 64*m
                                  rows per warp tile; m in {2, 8, 10, 16}):
                                  -1 (default) = on for FP32, off for FP64; 0; 1  */

int pm_create(pm_handle_t* out, int device);
int pm_destroy(pm_handle_t h);
const char* pm_last_error(pm_handle_t h);
int pm_set_option(pm_handle_t h, int option, int64_t value);
int pm_get_version(void); /* major*10000 + minor*100 + patch */

/* Device-resident solve (stream-ordered, asynchronous; stream NULL = default
 * stream).  Pivot failures are reported by the next pm_check(). */
int pm_solve_device_f64(pm_handle_t h, const double* a, const double* b, const double* c,
                        const double* d, double* x, int64_t n, int32_t m, void* stream);

/* Batch of independent systems stored back to back (system k occupies rows
 * [k*n_per_system, (k+1)*n_per_system)); each system's first a and last c
 * are ignored.  Asynchronous like pm_solve_device_f64.  See
 * PM_OPT_BATCH_CLUSTER for the cluster-per-system kernel. */
int pm_solve_batch_device_f64(pm_handle_t h, const double* a, const double* b, const double* c,
                              const double* d, double* x, int64_t n_per_system, int64_t batch,
                              int32_t m, void* stream);

/* Configuration of the last batch solve's cluster kernel: {CTAs per cluster,
 * warps per CTA, stages, max tiles per CTA, tiles per system, clusters}; all
 * zero when the last batch solve used the level kernels. */
int pm_last_batch_plan(pm_handle_t h, int32_t* out6);
/* Tile-stream kernel plan of the last batch solve: [used (0/1), compute warps
 * per CTA, stages, lag, ring rounds, CTAs, compute warps in the grid, tiles
 * per system]. */
int pm_last_stream_plan(pm_handle_t h, int32_t* out8);
/* Diagnostics of the last tile-stream launch with PM_OPT_BATCH_STATS on (SM
 * cycles summed over warps): [0] Stage-3 flag waits, [1] waits that spun,
 * [2] mailbox waits, [3] stage (bulk copy) waits, [4] control iterations,
 * [5] idle ones, [6] Stage-2 cycles, [7] Stage-2 solves, [8] publish (fence +
 * atomics) cycles, [9] compute-warp cycles, [10] control-warp cycles,
 * [11] Stage-1 jobs, [12] Stage-3 jobs, [13] unused, [14] Stage-2 ns (start
 * to flag, summed).  Synchronises the device. */
int pm_batch_stream_stats(pm_handle_t h, uint64_t* out15);
/* Diagnostics: the first n words of the tile-stream kernel's per-system
 * counters (Stage-1 counts | Stage-3 counts | Stage-2 flags, 32 * batch words
 * each -- one 128-byte line per system -- as laid out by the last launch); all
 * zero between launches. */
int pm_batch_stream_counters(pm_handle_t h, uint32_t* out, int64_t n);
/* Diagnostics (PM_OPT_BATCH_STATS): the first n words of the last tile-stream
 * launch's trace buffer: per-system globaltimer stamps, [5][batch] words
 * (first Stage-1 start | last Stage-1 end | Stage-1 count complete | Stage-2
 * flag | first Stage-3 wait start), then job traces of 8 sample warps
 * [8][2400][4] (job code, start, stage ready, end), the control warp of CTA 0
 * [1200][2], and per-warp / per-CTA cycle summaries [4096][8]. */
int pm_batch_stream_timeline(pm_handle_t h, uint64_t* out, int64_t n);

/* Batch of independent systems from host memory, end to end (config 4):
 * chunks of `systems_per_chunk` systems (0 = ~256 MB of inputs per chunk) flow
 * H2D -> batch solve -> D2H through a ring of `depth` device staging slots
 * (0 = 3) on separate copy-in / compute / copy-out streams, so the copy-in of
 * one chunk overlaps the copy-out of an earlier one (PCIe is full duplex).
 * Synchronous; page-locked host arrays required for the overlap. */
int pm_solve_batch_host_f64(pm_handle_t h, const double* a, const double* b, const double* c,
                            const double* d, double* x, int64_t n_per_system, int64_t batch, int32_t m,
                            int32_t depth, int64_t systems_per_chunk);
int pm_solve_batch_host_f32(pm_handle_t h, const float* a, const float* b, const float* c,
                            const float* d, float* x, int64_t n_per_system, int64_t batch, int32_t m,
                            int32_t depth, int64_t systems_per_chunk);

/* Waits for the handle's last stream; PM_ERR_COMPUTATION if any solve since
 * the previous check met a zero or non-finite pivot (the flag is cleared).
 * After a flagged device-resident solve (pm_solve_device_*, pm_solve_batch_
 * device_*; x not aliasing an input) pm_check first re-runs that solve once
 * with classic pivot sweeps -- the fast continuant pivots can leave the FP
 * range for rows scaled over >~1e60 -- and reports only if that fails too;
 * so the inputs must be unchanged until pm_check. */
int pm_check(pm_handle_t h);

/* End-to-end solve from host memory (synchronous).  num_streams in
 * {0, 1, 2, 4, 8, 16, 32}; 0 = predictor.  Page-locked buffers (cudaHostAlloc
 * or pm_host_register) are required for copy/compute overlap. */
int pm_solve_host_f64(pm_handle_t h, const double* a, const double* b, const double* c,
                      const double* d, double* x, int64_t n, int32_t m, int32_t num_streams);

/* StageTimings of the last pm_solve_host_f64 (components are filled when it
 * ran with one stream and PM_OPT_TIMINGS=1), its total time and stream count. */
int pm_last_stage_timings(pm_handle_t h, pm_stage_timings* out, double* total_ms,
                          int32_t* streams_used);

int pm_host_register(void* ptr, uint64_t bytes);
int pm_host_unregister(void* ptr);

/* Stream-count model used when num_streams == 0. */
int pm_set_model_bundle(pm_handle_t h, const pm_model_bundle* bundle);
int pm_get_model_bundle(pm_handle_t h, pm_model_bundle* out);
/* streamtune::recommend; bundle NULL = the paper's RTX 2080 Ti bundle.
 * Returns the stream count (>= 1) or -1 on a validation error. */
int pm_recommend_streams(int64_t n, const pm_model_bundle* bundle);
int pm_paper_bundle(pm_model_bundle* out);
/* The B200 re-fit (tools/refit.py): a new handle's default bundle. */
int pm_b200_bundle(pm_model_bundle* out);

/* Counter-based synthetic system (bit-identical to the CPU oracle's
 * generator): a, c ~ U(-1,1) with a[0] = c[n-1] = 0, b = +-(|a|+|c|+1+U(0,1)),
 * d ~ U(-1,1).  Any output may be NULL. */
int pm_generate_f64(pm_handle_t h, double* a, double* b, double* c, double* d, int64_t n,
                    uint64_t seed, void* stream);
/* Rows [row0, row0 + count) of the same n_total-row system, written to
 * a[0..count) etc. (a rank's slice of a row-sharded system). */
int pm_generate_range_f64(pm_handle_t h, double* a, double* b, double* c, double* d,
                          int64_t n_total, int64_t row0, int64_t count, uint64_t seed,
                          void* stream);

/* Row-sharded single system over `world` ranks (BASELINE.json config 5).
 * Rank r holds rows [offset_r, offset_r + n_local) in a,b,c,d.
 *   1. pm_dist_reduce_f64: Stage 1 + local levels; writes the rank's two
 *      interface equations (8 doubles) to iface (device memory).
 *   2. caller all-gathers iface over ranks into iface_all (8*world doubles,
 *      rank order), e.g. ncclAllGather / torch.distributed.
 *   3. pm_dist_solve_f64: solves the 2*world-row interface system
 *      redundantly, then Stages 3 of all local levels; writes x.
 * Both calls are asynchronous on `stream` and must use the same n_local, m. */
int pm_dist_reduce_f64(pm_handle_t h, const double* a, const double* b, const double* c,
                       const double* d, int64_t n_local, int32_t m, int32_t rank, int32_t world,
                       double* iface, void* stream);
int pm_dist_solve_f64(pm_handle_t h, const double* a, const double* b, const double* c,
                      const double* d, double* x, int64_t n_local, int32_t m, int32_t rank,
                      int32_t world, const double* iface_all, void* stream);

/* One-call collective solve of a row-sharded system (every rank calls it
 * with its rows; BASELINE.json config 5, SURVEY.md §8b pm_solve_dist_f64):
 * Stage 1 + local levels -> the rank's 8 interface reals, the all-gather of
 * those 8 reals over the ranks, the 2*world-row interface solve + Stage 3 of
 * every local level -> x.  Stream-ordered on `stream`; pivot failures are
 * reported by pm_check.  Same row split rules as pm_dist_*: every rank but
 * the last holds a multiple of m rows.
 *
 * The exchange is the caller's:
 *   pm_solve_dist_*       `allgather(send, recv, bytes_per_rank, stream, user)`
 *                         must gather bytes_per_rank (64 FP64 / 32 FP32) from
 *                         every rank's device buffer `send` into `recv` in
 *                         rank order, ordered after the work already on
 *                         `stream` and before anything enqueued on it later
 *                         (e.g. ncclAllGather / MPI_Allgather of a staged copy);
 *                         non-zero return -> PM_ERR_RUNTIME.
 *   pm_solve_dist_nccl_*  NCCL's ncclAllGather on `nccl_comm` (an ncclComm_t;
 *                         rank and world are the communicator's).  NCCL is
 *                         loaded at run time (PM_NCCL_LIB, else libnccl.so.2:
 *                         the copy already in the process if any); the library
 *                         does not link it.
 * pm_nccl_* create a communicator without including nccl.h:
 * pm_nccl_get_unique_id on one rank (PM_NCCL_ID_BYTES bytes, sent to the
 * others by any side channel), pm_nccl_comm_init on every rank (on the
 * handle's device).  pm_nccl_version: NCCL_VERSION_CODE, -1 if unloadable. */
typedef int (*pm_allgather_fn)(const void* send, void* recv, int64_t bytes_per_rank, void* stream,
                               void* user);
int pm_solve_dist_f64(pm_handle_t h, const double* a, const double* b, const double* c, const double* d,
                      double* x, int64_t n_local, int32_t m, int32_t rank, int32_t world,
                      pm_allgather_fn allgather, void* user, void* stream);
int pm_solve_dist_f32(pm_handle_t h, const float* a, const float* b, const float* c, const float* d,
                      float* x, int64_t n_local, int32_t m, int32_t rank, int32_t world,
                      pm_allgather_fn allgather, void* user, void* stream);
int pm_solve_dist_nccl_f64(pm_handle_t h, const double* a, const double* b, const double* c,
                           const double* d, double* x, int64_t n_local, int32_t m, void* nccl_comm,
                           void* stream);
int pm_solve_dist_nccl_f32(pm_handle_t h, const float* a, const float* b, const float* c, const float* d,
                           float* x, int64_t n_local, int32_t m, void* nccl_comm, void* stream);
#define PM_NCCL_ID_BYTES 128
int pm_nccl_version(void);
int pm_nccl_get_unique_id(pm_handle_t h, void* id_out);
int pm_nccl_comm_init(pm_handle_t h, void** comm_out, int32_t world, const void* id, int32_t rank);
int pm_nccl_comm_destroy(pm_handle_t h, void* comm);

/* Peer-memory (NVLink P2P) exchange of the interface equations -- the
 * all-gather of pm_dist_* done by the solver's own kernels.  Each rank
 * allocates an exchange buffer (pm_dist_exchange_alloc; owned by the handle),
 * exports it with pm_ipc_get_handle, receives the peers' handles by any
 * side channel (e.g. torch.distributed), maps them with pm_ipc_open_handle
 * and calls pm_dist_set_peers with every rank's buffer in rank order (its
 * own included).  Then per solve, on every rank:
 *   pm_dist_reduce_p2p_*  Stage 1 + local levels; the top-level kernel that
 *                         produces the rank's 8 interface reals stores them
 *                         into every peer's buffer and releases an epoch
 *                         flag (system scope) itself;
 *   pm_dist_solve_p2p_*   the top-level Stage-3 kernel acquires all ranks'
 *                         flags, solves the 2*world-row interface system,
 *                         then every level's Stage 3 (at most 64 ranks).
 * No host synchronisation or collective call on the data path.  A peer that
 * never publishes makes the wait time out after 20 s (PM_ERR_RUNTIME from
 * pm_check).  Ranks must call the pair in lockstep (collective semantics). */
#define PM_IPC_HANDLE_BYTES 64
int64_t pm_dist_exchange_bytes(int32_t world);
int pm_dist_exchange_alloc(pm_handle_t h, int32_t world, void** out);
int pm_dist_set_peers(pm_handle_t h, void* const* peer_bufs, int32_t world, int32_t rank);
int pm_ipc_get_handle(const void* dptr, void* handle_out);
int pm_ipc_open_handle(const void* handle, void** dptr_out);
int pm_ipc_close_handle(void* dptr);
int pm_dist_reduce_p2p_f64(pm_handle_t h, const double* a, const double* b, const double* c,
                           const double* d, int64_t n_local, int32_t m, void* stream);
int pm_dist_solve_p2p_f64(pm_handle_t h, const double* a, const double* b, const double* c,
                          const double* d, double* x, int64_t n_local, int32_t m, void* stream);
int pm_dist_reduce_p2p_f32(pm_handle_t h, const float* a, const float* b, const float* c,
                           const float* d, int64_t n_local, int32_t m, void* stream);
int pm_dist_solve_p2p_f32(pm_handle_t h, const float* a, const float* b, const float* c,
                          const float* d, float* x, int64_t n_local, int32_t m, void* stream);

/* FP32 variants (the paper's FP32 experiments; Table 5 and
 * streamtune::recommend_fp32): the same pipeline, plan, options and status
 * codes on float arrays -- half the HBM and host-link bytes per unknown.
 * The FP32 generator writes the round-to-nearest FP32 images of the FP64
 * generator's values.  Accuracy is FP32's: see DESIGN.md (relative error vs
 * the FP64 solution of the same FP32 inputs <= 1e-4 on the synthetic
 * diagonally dominant systems). */
int pm_solve_device_f32(pm_handle_t h, const float* a, const float* b, const float* c,
                        const float* d, float* x, int64_t n, int32_t m, void* stream);
int pm_solve_batch_device_f32(pm_handle_t h, const float* a, const float* b, const float* c,
                              const float* d, float* x, int64_t n_per_system, int64_t batch,
                              int32_t m, void* stream);
int pm_solve_host_f32(pm_handle_t h, const float* a, const float* b, const float* c,
                      const float* d, float* x, int64_t n, int32_t m, int32_t num_streams);
int pm_generate_f32(pm_handle_t h, float* a, float* b, float* c, float* d, int64_t n,
                    uint64_t seed, void* stream);
int pm_generate_range_f32(pm_handle_t h, float* a, float* b, float* c, float* d,
                          int64_t n_total, int64_t row0, int64_t count, uint64_t seed,
                          void* stream);
int pm_dist_reduce_f32(pm_handle_t h, const float* a, const float* b, const float* c,
                       const float* d, int64_t n_local, int32_t m, int32_t rank, int32_t world,
                       float* iface, void* stream);
int pm_dist_solve_f32(pm_handle_t h, const float* a, const float* b, const float* c,
                      const float* d, float* x, int64_t n_local, int32_t m, int32_t rank,
                      int32_t world, const float* iface_all, void* stream);

/* Diagnostics: number of kernel launches the last solve call enqueued, and
 * the level plan (rows per level) of the last plan. */
int pm_last_launch_count(pm_handle_t h);
/* Per-launch durations (ms) recorded since the last call while
 * PM_OPT_KERNEL_TIMES is on; mode 0 = Stage-1 reduce, 1 = Stage-3 solve,
 * 2 = root, 3 = fused upper levels (recorded as level 1), 4 = batch cluster
 * kernel; level 0 = the caller's system.  Synchronises; returns the count. */
int pm_kernel_times(pm_handle_t h, int32_t* modes, int32_t* levels, float* ms, int32_t max);
int pm_last_plan(pm_handle_t h, int64_t* rows_per_level, int32_t max_levels);

#ifdef __cplusplus
}
#endif

#endif /* PM_TRIDIAG_H */
