// bw_probe.cu -- HBM ceilings of the solver's two level-0 access patterns on
// this GPU (measurement tool, not product code):
//   read4        read a, b, c, d (Stage 1's 32 B/unknown)
//   read4write1  read a, b, c, d, write x (Stage 3's 40 B/unknown)
// Grid-stride loops with 16-byte loads/stores, persistent grid of
// ctas_per_sm x #SMs CTAs; nvcc -O3 -gencode arch=compute_100a,code=sm_100a
// -shared -Xcompiler -fPIC tools/bw_probe.cu -o build/libbw_probe.so
#include <cuda_runtime.h>

#include <cstdint>

__global__ void read4(const double2* __restrict__ a, const double2* __restrict__ b,
                      const double2* __restrict__ c, const double2* __restrict__ d, int64_t n2,
                      double* sink) {
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n2;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double2 va = __ldcs(a + i), vb = __ldcs(b + i), vc = __ldcs(c + i), vd = __ldcs(d + i);
    acc += va.x + va.y + vb.x + vb.y + vc.x + vc.y + vd.x + vd.y;
  }
  if (acc == 12345.678) *sink = acc;  // keep the loads
}

__global__ void read4write1(const double2* __restrict__ a, const double2* __restrict__ b,
                            const double2* __restrict__ c, const double2* __restrict__ d,
                            double2* __restrict__ x, int64_t n2) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n2;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double2 va = __ldcs(a + i), vb = __ldcs(b + i), vc = __ldcs(c + i), vd = __ldcs(d + i);
    __stcs(x + i, make_double2(va.x + vb.x + vc.x + vd.x, va.y + vb.y + vc.y + vd.y));
  }
}

// one buffer read with L2-cached loads (ld.global.cg): repeated passes over a
// buffer that L2 retains run at L2 bandwidth (tools/l2_probe.py)
__global__ void read1cg(const double2* __restrict__ a, int64_t n2, double* sink) {
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n2;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double2 v = __ldcg(a + i);
    acc += v.x + v.y;
  }
  if (acc == 12345.678) *sink = acc;
}

extern "C" float l2_probe(const double* a, double* sink, int64_t n, int ctas_per_sm, int threads, int reps) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = sms * ctas_per_sm;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  read1cg<<<grid, threads>>>((const double2*)a, n / 2, sink);  // first pass
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) read1cg<<<grid, threads>>>((const double2*)a, n / 2, sink);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return cudaGetLastError() == cudaSuccess ? ms / reps : -1.f;
}

extern "C" float bw_probe(int kind, const double* a, const double* b, const double* c, const double* d,
                          double* x, int64_t n, int ctas_per_sm, int threads, int reps) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = sms * ctas_per_sm;
  const int64_t n2 = n / 2;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&]() {
    if (kind == 0)
      read4<<<grid, threads>>>((const double2*)a, (const double2*)b, (const double2*)c,
                               (const double2*)d, n2, x);
    else
      read4write1<<<grid, threads>>>((const double2*)a, (const double2*)b, (const double2*)c,
                                     (const double2*)d, (double2*)x, n2);
  };
  run();
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) run();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return cudaGetLastError() == cudaSuccess ? ms / reps : -1.f;
}
