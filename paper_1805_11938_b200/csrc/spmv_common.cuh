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
inline bool aligned32(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 31u) == 0; }

// 256-bit streaming loads (sm_100: LDG.256), L1 bypass, L2 evict-first:
// eight int32 / four fp64 per instruction, 32-byte aligned addresses.
__device__ __forceinline__ void ld_stream8(const int32_t* p, int32_t (&v)[8]) {
  asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "l"(p));
}
__device__ __forceinline__ void ld_stream4(const double* p, double* v) {
  asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3])
               : "l"(p));
}

}  // namespace spmvb
