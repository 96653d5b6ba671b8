// Bulk asynchronous copies (TMA, cp.async.bulk) global -> shared with an
// mbarrier completion and L2 eviction-priority cache hints (sm_90+/sm_100a).
#pragma once

#include <cstdint>

namespace spmvb {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_MBAR:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_MBAR;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// Global -> shared bulk copy; dst/src 16-byte aligned, bytes % 16 == 0.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// Read-only gather with an L2 eviction policy (x vectors: evict_last).
__device__ __forceinline__ double ld_hint(const double* p, uint64_t policy) {
  double v;
  asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(policy));
  return v;
}

// Plan of a staged element range [lo, hi) of an array of n elements of
// `esz` bytes: the 16-byte-aligned middle goes through one bulk copy, the
// unaligned tail (at the end of the array only) is loaded by threads.
struct StageRange {
  int64_t base;     // first element held in shared memory (aligned down)
  int64_t bulk_hi;  // end of the bulk-copied part
  int64_t hi;       // end of the needed range
  __device__ __forceinline__ uint32_t bulk_bytes(int esz) const {
    return bulk_hi > base ? static_cast<uint32_t>((bulk_hi - base) * esz) : 0u;
  }
};

__device__ __forceinline__ StageRange plan_stage(int64_t lo, int64_t hi, int64_t n, int esz) {
  const int64_t al = 16 / esz;
  StageRange s;
  s.base = lo & ~(al - 1);
  int64_t up = (hi + al - 1) & ~(al - 1);
  int64_t cap = n & ~(al - 1);
  s.bulk_hi = up < cap ? up : cap;
  if (s.bulk_hi < s.base) s.bulk_hi = s.base;
  s.hi = hi;
  return s;
}

}  // namespace spmvb
