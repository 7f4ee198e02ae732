// pm_kernels.h -- host-visible launch interface of the solver kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#define PM_API_NS pm
#define PM_API_REAL double
#include "pm_kernels_api.inc"
#undef PM_API_NS
#undef PM_API_REAL
#define PM_API_NS pm32
#define PM_API_REAL float
#include "pm_kernels_api.inc"
#undef PM_API_NS
#undef PM_API_REAL
