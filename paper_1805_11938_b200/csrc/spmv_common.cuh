// Helpers shared by the SpMV kernel files.
#pragma once

#include "prims.cuh"

namespace spmvb {

__device__ __forceinline__ double ldx(const double* __restrict__ x, int32_t j) { return __ldg(x + j); }

__device__ __forceinline__ double load_scale(const double* scale) { return scale ? *scale : 1.0; }

// Butterfly sum: every lane gets the same, order-fixed result.
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
  return v;
}

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

}  // namespace spmvb
