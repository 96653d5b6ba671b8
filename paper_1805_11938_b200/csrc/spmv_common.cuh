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

// Calls f(r) for every empty row r (ptr[r] == ptr[r+1]) in grid-stride
// order; each ptr entry is loaded once (ptr[r+1] comes from the next lane).
template <typename F>
__device__ __forceinline__ void for_each_empty_row(int64_t n_rows, const int32_t* __restrict__ ptr, F f) {
  const int lane = threadIdx.x & 31;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t base = blockIdx.x * static_cast<int64_t>(blockDim.x) + (threadIdx.x & ~31); base < n_rows;
       base += stride) {  // warp-uniform trip count (shuffles below)
    const int64_t r = base + lane;
    const int32_t p0 = r <= n_rows ? ld_stream(ptr + r) : 0;
    int32_t p1 = __shfl_down_sync(0xffffffffu, p0, 1);
    if (lane == 31) p1 = r + 1 <= n_rows ? ld_stream(ptr + r + 1) : 0;
    if (r < n_rows && p0 == p1) f(r);
  }
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
