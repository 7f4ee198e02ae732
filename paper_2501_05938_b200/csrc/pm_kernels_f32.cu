// pm_kernels_f32.cu -- the FP32 solver kernels (namespace pm32): the same
// sources as pm_kernels.cu compiled with real = float (pm_device.cuh).
#define PM_REAL_F32 1
#include "pm_kernels.cu"
