// hb_common.cuh -- shared helpers of the sm_100a heat-BEM kernels.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "heatbem_b200.h"

namespace hb {

constexpr int kWarps = 8;              // warps per CTA of the pair kernels
constexpr unsigned kFull = 0xffffffffu;
constexpr double kPi = 3.141592653589793;
constexpr double kInvPi = 0.3183098861837907;

// error reporting (thread-local message, set by the C-ABI layer)
void set_error(const char *fmt, ...);
int cuda_check(cudaError_t err, const char *what);

__host__ __device__ inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace hb
