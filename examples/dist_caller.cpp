// dist_caller.cpp -- a C++ caller of the row-sharded solve through the C ABI
// alone (no Python, no torch): BASELINE.json config 5's decomposition, the
// MPI-style partition of PAPER.md:29-30, with the interface exchange supplied
// by the caller.
//
//   dist_caller [world] [n]           `world` ranks as threads sharing one GPU,
//                                     one pm handle and stream each; the
//                                     all-gather is a host-staged callback
//                                     (D2H of 64 bytes, barrier, H2D of
//                                     64*world bytes) -- what an MPI program
//                                     would do with MPI_Allgather.
//   dist_caller --nccl [n]            one rank, ncclAllGather on a 1-rank
//                                     communicator made by pm_nccl_* (NCCL
//                                     loaded at run time by the library).
//
// Prints the max |x - x_single| / max |x_single| against the single-system
// solve of the same rows and the relative residual of the gathered x.
#include <cuda_runtime.h>

#include <barrier>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "pm_tridiag.h"

namespace {

#define CK(call)                                                                        \
  do {                                                                                  \
    const int st_ = (call);                                                             \
    if (st_ != 0) {                                                                     \
      std::fprintf(stderr, "%s:%d %s -> %d\n", __FILE__, __LINE__, #call, st_);         \
      std::exit(1);                                                                     \
    }                                                                                   \
  } while (0)

// Host-staged all-gather shared by the rank threads.
struct HostGather {
  int world = 1;
  std::vector<double> slots;  // 8 * world
  std::barrier<>* arrive = nullptr;
};
struct RankCtx {
  HostGather* g = nullptr;
  int rank = 0;
};

int host_allgather(const void* send, void* recv, int64_t bytes_per_rank, void* stream, void* user) {
  auto* rc = static_cast<RankCtx*>(user);
  HostGather* g = rc->g;
  auto st = static_cast<cudaStream_t>(stream);
  char* mine = reinterpret_cast<char*>(g->slots.data()) + rc->rank * bytes_per_rank;
  if (cudaMemcpyAsync(mine, send, bytes_per_rank, cudaMemcpyDeviceToHost, st) != cudaSuccess) return 1;
  if (cudaStreamSynchronize(st) != cudaSuccess) return 2;  // the reduce's 8 reals are in
  g->arrive->arrive_and_wait();                            // every rank published
  if (cudaMemcpyAsync(recv, g->slots.data(), bytes_per_rank * g->world, cudaMemcpyHostToDevice, st) !=
      cudaSuccess)
    return 3;
  if (cudaStreamSynchronize(st) != cudaSuccess) return 4;  // slots may be rewritten next solve
  g->arrive->arrive_and_wait();
  return 0;
}

// rows per rank: every rank but the last a multiple of m (dist.split_rows)
std::vector<int64_t> split_rows(int64_t n, int world, int m) {
  if (world == 1) return {n};
  int64_t q = std::max<int64_t>(m, (n / world) / m * m);
  std::vector<int64_t> r(world, q);
  r[world - 1] = n - q * (world - 1);
  return r;
}

}  // namespace

int main(int argc, char** argv) {
  bool use_nccl = argc > 1 && std::strcmp(argv[1], "--nccl") == 0;
  const int world = use_nccl ? 1 : (argc > 1 ? std::atoi(argv[1]) : 2);
  const int64_t n = argc > 2 ? std::atoll(argv[2]) : 1000003;
  const int m = 10;
  const uint64_t seed = 77;
  const auto rows = split_rows(n, world, m);
  if (rows.back() < 1) {
    std::fprintf(stderr, "n too small for %d ranks\n", world);
    return 1;
  }

  // the whole system once, and its single-system solution (the comparison)
  double *a, *b, *c, *d, *x, *xs;
  for (double** p : {&a, &b, &c, &d, &x, &xs}) CK(cudaMalloc(p, n * sizeof(double)));
  pm_handle_t h0;
  CK(pm_create(&h0, 0));
  CK(pm_generate_f64(h0, a, b, c, d, n, seed, nullptr));
  CK(pm_solve_device_f64(h0, a, b, c, d, xs, n, m, nullptr));
  CK(pm_check(h0));

  std::vector<int64_t> off(world + 1, 0);
  for (int r = 0; r < world; ++r) off[r + 1] = off[r] + rows[r];

  if (use_nccl) {
    std::printf("nccl version %d\n", pm_nccl_version());
    pm_handle_t h;
    CK(pm_create(&h, 0));
    char id[PM_NCCL_ID_BYTES];
    void* comm = nullptr;
    CK(pm_nccl_get_unique_id(h, id));
    CK(pm_nccl_comm_init(h, &comm, 1, id, 0));
    cudaStream_t st;
    cudaStreamCreate(&st);
    for (int rep = 0; rep < 2; ++rep) CK(pm_solve_dist_nccl_f64(h, a, b, c, d, x, n, m, comm, st));
    CK(pm_check(h));
    CK(pm_nccl_comm_destroy(h, comm));
    cudaStreamDestroy(st);
    CK(pm_destroy(h));
  } else {
    HostGather g;
    g.world = world;
    g.slots.assign(8 * world, 0.0);
    std::barrier<> bar(world);
    g.arrive = &bar;
    std::vector<std::thread> th;
    std::vector<int> status(world, 0);
    for (int r = 0; r < world; ++r) {
      th.emplace_back([&, r] {
        cudaSetDevice(0);
        pm_handle_t h;
        if (pm_create(&h, 0)) {
          status[r] = 1;
          return;
        }
        cudaStream_t st;
        cudaStreamCreate(&st);
        RankCtx rc{&g, r};
        const int64_t o = off[r];
        for (int rep = 0; rep < 3 && status[r] == 0; ++rep)  // consecutive solves reuse the buffers
          status[r] = pm_solve_dist_f64(h, a + o, b + o, c + o, d + o, x + o, rows[r], m, r, world,
                                        host_allgather, &rc, st);
        if (status[r] == 0) status[r] = pm_check(h);
        if (status[r]) std::fprintf(stderr, "rank %d: %s\n", r, pm_last_error(h));
        std::printf("rank %d rows %lld launches %d status %d\n", r, (long long)rows[r],
                    pm_last_launch_count(h), status[r]);
        cudaStreamDestroy(st);
        pm_destroy(h);
      });
    }
    for (auto& t : th) t.join();
    for (int s : status)
      if (s) return 1;
  }

  std::vector<double> ha(n), hb(n), hc(n), hd(n), hx(n), hxs(n);
  for (auto [dst, src] : {std::pair{&ha, a}, {&hb, b}, {&hc, c}, {&hd, d}, {&hx, x}, {&hxs, xs}})
    CK(cudaMemcpy(dst->data(), src, n * sizeof(double), cudaMemcpyDeviceToHost));
  double emax = 0, rmax = 0, rs = 0, ds = 0;
  for (int64_t i = 0; i < n; ++i) {
    emax = std::max(emax, std::fabs(hx[i] - hxs[i]));
    rmax = std::max(rmax, std::fabs(hxs[i]));
    double r = hb[i] * hx[i] - hd[i];
    if (i > 0) r += ha[i] * hx[i - 1];
    if (i + 1 < n) r += hc[i] * hx[i + 1];
    rs += r * r;
    ds += hd[i] * hd[i];
  }
  std::printf("dist world %d n %lld rel_vs_single %.3e residual %.3e\n", world, (long long)n, emax / rmax,
              std::sqrt(rs / ds));
  for (double* p : {a, b, c, d, x, xs}) cudaFree(p);
  pm_destroy(h0);
  return 0;
}
