// pm_kernels.h -- host-visible launch interface of the solver kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace pm {

struct Node;

constexpr int kModeReduce = 0;  // Stage 1 of one level: tile -> 2 interface rows
constexpr int kModeSolve = 1;   // Stage 3 of one level: boundary values -> x
constexpr int kModeRoot = 2;    // whole (single-tile) top level

struct TileArgs {
  // the level's tridiagonal system (SoA, n rows)
  const double* a = nullptr;
  const double* b = nullptr;
  const double* c = nullptr;
  const double* d = nullptr;
  double* x = nullptr;         // SOLVE/ROOT: solution of this level
  const double* xb = nullptr;  // SOLVE: solution of the level above (2 per tile)
  double* ra = nullptr;        // REDUCE: system of the level above (2 rows per tile)
  double* rb = nullptr;
  double* rc = nullptr;
  double* rd = nullptr;
  int64_t n = 0;
  int64_t tile_begin = 0, tile_end = 0;  // tiles handled by this launch
  int m = 10;                            // rows per thread block (sub-system size)
  int stages = 2;                        // bulk-copy ring depth (1..4)
  int reverse = 0;                       // walk tiles from the end (L2 reuse)
  int max_ctas = 0;                      // cap on the persistent grid (0 = none)
  int* flag = nullptr;                   // set to 1 on a zero / non-finite pivot
  int zero_first = 1;                    // treat a[0] as 0 (global first row)
  int zero_last = 1;                     // treat c[n-1] as 0 (global last row)
  int pad_mode = 1;                      // 1: pad the last tile with identity rows
                                         // 0: ragged last tile (n % m == 0 required);
                                         //    its trailing blocks are empty segments
  int64_t sys_len = 0;                   // batch: rows per independent system (0 = one)
  // chain mode (warp-tile kernels): the launch's tiles form `nchunks`
  // contiguous chunks; Stage 1 combines each chunk's tile segments in order
  // (one Node per tile -> chain_nodes[tile]) and writes two rows per chunk
  // at 2*(chunk_base + j); Stage 3 reads xb[2*(chunk_base + j) .. +1] and
  // walks the chunk backwards.
  int64_t nchunks = 0;
  int64_t chunk_base = 0;
  struct Node* chain_nodes = nullptr;
};

// CTAs per SM of a warp-tile kernel variant (occupancy query).
int warp_kernel_ctas_per_sm(int mode, int m, int stages, int warps_per_cta, bool chain);

// Row-sharded solve: combine the ranks' interface segments (8 doubles each,
// rank order) and write this rank's two boundary values to xb[0..1].
cudaError_t launch_dist_chain(const double* iface_all, int world, int rank, double* xb, int* flag,
                              cudaStream_t st);

size_t tile_smem_bytes(int mode, int P, int m, int stages);
// Level-0 warp-tile kernel: a tile is 32*m rows owned by one warp (REDUCE or
// SOLVE; 16-byte aligned arrays only).  Shared memory per warp:
__host__ __device__ size_t warp_smem_bytes(int mode, int m, int stages);
cudaError_t launch_warp_tile_kernel(int mode, const TileArgs& args, int warps_per_cta,
                                    int sm_count, cudaStream_t st, int* grid_out);
bool m_is_specialised(int m);
// Programmatic dependent launch for the solver kernels (default on).
void set_pdl(bool on);
cudaError_t launch_tile_kernel(int mode, const TileArgs& args, int P, bool bulk, int sm_count,
                               cudaStream_t st, int* grid_out);
// rows [row0, row0 + count) of the n_total-row synthetic system, stored at a[0..count)
cudaError_t launch_generate(double* a, double* b, double* c, double* d, int64_t n_total,
                            int64_t row0, int64_t count, uint64_t seed, int sm_count,
                            cudaStream_t st);

}  // namespace pm
