// pm_kernels_f32.cu -- the FP32 solver kernels (namespace pm32): the same
// sources as pm_kernels.cu compiled with real = float (pm_device.cuh).
// FP32 rows need fewer registers, so the level-0 kernels run more CTAs per
// SM than the FP64 build (B200 sweep, round 1: Stage 1 0.233 -> 0.214 ms,
// Stage 3 0.344 -> 0.340 ms at N = 8e7).
#define PM_REAL_F32 1
#define PM_SOLVE_MINB 6
#define PM_REDUCE_MINB 4
#include "pm_kernels.cu"
