// Helpers shared by the SpMV kernel files.
#pragma once

#include "prims.cuh"

namespace spmvb {

#ifndef SPMVB_LDX_NOALLOC
#define SPMVB_LDX_NOALLOC 0  // 1: x gathers bypass L1 allocation (A/B knob)
#endif
#ifndef SPMVB_LDX_HOT
#define SPMVB_LDX_HOT 0  // > 0: columns >= this gather without L1 allocation (A/B knob)
#endif
#ifndef SPMVB_LDX_HOT_MODE
// 0: cold no_allocate; 1: hot evict_last + cold evict_first (per lane: the
// two loads diverge); 2: every gather evict_last; 3: every gather
// evict_first; 4-6: ONE load per warp instruction, chosen by a vote -- when
// at least SPMVB_LDX_VOTE active lanes gather a cold column the whole warp
// uses evict_first (4) / no_allocate (5) / the default policy (6), else
// evict_last (4, 6) / the default (5).  All A/B knobs; every variant was
// slower than the plain __ldg (profiles/r02_l1_hot_split_ab.txt,
// profiles/r02_l1_vote_ab.txt).
#define SPMVB_LDX_HOT_MODE 0
#endif
#ifndef SPMVB_LDX_VOTE
#define SPMVB_LDX_VOTE 24
#endif
__device__ __forceinline__ double ldx_el(const double* p) {
  double v;
  asm("ld.global.nc.L1::evict_last.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ double ldx_ef(const double* p) {
  double v;
  asm("ld.global.nc.L1::evict_first.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ double ldx_na(const double* p) {
  double v;
  asm("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ double ldx(const double* __restrict__ x, int32_t j) {
#if SPMVB_LDX_HOT_MODE == 2
  return ldx_el(x + j);
#elif SPMVB_LDX_HOT_MODE == 3
  return ldx_ef(x + j);
#elif SPMVB_LDX_HOT > 0 && SPMVB_LDX_HOT_MODE >= 4
  const unsigned am = __activemask();
  const bool cold = __popc(__ballot_sync(am, j >= SPMVB_LDX_HOT)) >= min(SPMVB_LDX_VOTE, __popc(am));
#if SPMVB_LDX_HOT_MODE == 4
  return cold ? ldx_ef(x + j) : ldx_el(x + j);
#elif SPMVB_LDX_HOT_MODE == 5
  return cold ? ldx_na(x + j) : __ldg(x + j);
#else
  return cold ? __ldg(x + j) : ldx_el(x + j);
#endif
#elif SPMVB_LDX_HOT > 0
  if (j < SPMVB_LDX_HOT) {
#if SPMVB_LDX_HOT_MODE == 1
    return ldx_el(x + j);
#else
    return __ldg(x + j);
#endif
  }
#if SPMVB_LDX_HOT_MODE == 1
  return ldx_ef(x + j);
#else
  return ldx_na(x + j);
#endif
#elif SPMVB_LDX_NOALLOC
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(x + j));
  return v;
#else
  return __ldg(x + j);
#endif
}

__device__ __forceinline__ double load_scale(const double* scale) { return scale ? *scale : 1.0; }

// Butterfly sum: every lane gets the same, order-fixed result.
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
  return v;
}

// Calls f(r) for every empty row r (ptr[r] == ptr[r+1]) of [0, n_rows);
// block `bid` of `nb` blocks, warp-strided.  Each ptr entry is loaded once
// (ptr[r+1] comes from the next lane) and four strides are loaded before any
// is used, so a warp keeps four loads in flight.
template <typename F>
__device__ __forceinline__ void for_each_empty_row(int64_t n_rows, const int32_t* __restrict__ ptr, F f, int64_t bid,
                                                   int64_t nb) {
  const int lane = threadIdx.x & 31;
  const int64_t stride = nb * blockDim.x;
  constexpr int U = 4;
  for (int64_t base = bid * blockDim.x + (threadIdx.x & ~31); base < n_rows; base += U * stride) {
    int32_t p0[U], p1[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {  // warp-uniform bounds (shuffles below)
      const int64_t r = base + u * stride + lane;
      p0[u] = r <= n_rows ? ld_stream(ptr + r) : 0;
      p1[u] = (lane == 31 && r + 1 <= n_rows) ? ld_stream(ptr + r + 1) : 0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t r = base + u * stride + lane;
      const int32_t nx = __shfl_down_sync(0xffffffffu, p0[u], 1);
      if (lane != 31) p1[u] = nx;
      if (r < n_rows && p0[u] == p1[u]) f(r);
    }
  }
}
template <typename F>
__device__ __forceinline__ void for_each_empty_row(int64_t n_rows, const int32_t* __restrict__ ptr, F f) {
  for_each_empty_row(n_rows, ptr, f, blockIdx.x, gridDim.x);
}

// Folds chains of equal non-negative keys over items [begin, end): a chain is
// a maximal run of consecutive items with the same key; apply(key, sum) gets
// the chain's sum.  The sum is defined independently of how items map to
// warps (so any split of the items into ranges gives the same bits): lane i
// of a virtual warp sums items start+i, start+i+32, ... sequentially from
// 0.0, and the 32 lane sums are combined by the xor butterfly of warp_sum.
// One warp per 32-item window; the window holding a chain's first item owns
// it.  Chains ending inside their window are evaluated by the start lane
// alone (the same butterfly replayed in registers; one round of independent
// loads); chains running past it are summed by the whole warp.
template <typename Key, typename Val, typename Apply>
__device__ __forceinline__ void fold_chains(int64_t begin, int64_t end, Key key_of, Val val_of, Apply apply) {
  const int lane = threadIdx.x & 31;
  const int64_t warp_id = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  auto key = [&](int64_t t) -> int32_t { return (t >= begin && t < end) ? key_of(t) : -1; };
  for (int64_t w0 = begin + warp_id * 32; w0 < end; w0 += nwarps * 32) {
    const int64_t t = w0 + lane;
    const int32_t r = key(t);
    int32_t rp = __shfl_up_sync(0xffffffffu, r, 1);
    if (lane == 0) rp = key(t - 1);
    const bool start = r >= 0 && rp != r;
    const unsigned cont = __ballot_sync(0xffffffffu, r >= 0 && rp == r);
    // lanes after this one that do NOT continue its chain
    const unsigned breaks = lane == 31 ? 0u : (~cont) >> (lane + 1);
    const int len = breaks ? __ffs(breaks) : 32 - lane;  // chain items inside the window
    const bool spills = start && !breaks && key(w0 + 32) == r;
    if (start && !spills) {
      double u[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) u[i] = i < len ? 0.0 + val_of(t + i) : 0.0;
#pragma unroll
      for (int d = 16; d >= 1; d >>= 1) {
#pragma unroll
        for (int i = 0; i < d; ++i) u[i] = u[i] + u[i + d];
      }
      apply(r, u[0]);
    }
    unsigned longs = __ballot_sync(0xffffffffu, spills);
    while (longs) {
      const int l = __ffs(longs) - 1;
      longs &= longs - 1;
      const int32_t k = __shfl_sync(0xffffffffu, r, l);
      double acc = 0.0;
      bool done = false;
      for (int64_t b = w0 + l; !done; b += 4 * 32) {  // four 32-item blocks per round trip
        bool in[4];
        double cv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) in[u] = key(b + u * 32 + lane) == k;
#pragma unroll
        for (int u = 0; u < 4; ++u) cv[u] = in[u] ? val_of(b + u * 32 + lane) : 0.0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (done) break;
          const unsigned m = __ballot_sync(0xffffffffu, in[u]);
          const int n = (m == 0xffffffffu) ? 32 : __ffs(~m) - 1;
          if (lane < n) acc += cv[u];
          done = n < 32;
        }
      }
      acc = warp_sum(acc);
      if (lane == 0) apply(k, acc);
    }
  }
}

// Sequential row sum over k slots at base + j*stride (ELL/SELL column-major
// grids): acc = ((0 + v0*x[c0]) + v1*x[c1]) + ..., separately rounded
// products, exactly the reference recurrence (kernels.py:101-104).  Four
// slots per step; the next four slots' loads are issued before this step's
// x gathers are consumed (unpredicated full steps, then a scalar tail).
// Two alternating buffers: C3 ELL back-to-back 37.5 -> 35.1 us, L2-flushed
// 43.3 -> 43.1 us, against one buffer copied forward each step.
template <bool CACHED = false, int D = 4>
__device__ __forceinline__ double seq_slots(int64_t k, int64_t stride, int64_t base, const int32_t* __restrict__ idx,
                                            const double* __restrict__ val, const double* __restrict__ x) {
  // CACHED: slot loads through L1 (narrow SELL slices, see seq_slots4).
  // D: slots per step (the prefetch depth; D gathers in flight per thread)
  auto li = [](const int32_t* p) { return CACHED ? __ldg(p) : ld_stream(p); };
  auto lv = [](const double* p) { return CACHED ? __ldg(p) : ld_stream(p); };
  // two D-slot buffers used alternately (a 2x-unrolled loop) so that no
  // register is copied while its prefetched load is still pending: a
  // copy would wait for the load and end the overlap
  auto load = [&](int64_t j, int32_t (&c)[D], double (&v)[D]) {
#pragma unroll
    for (int u = 0; u < D; ++u) {
      c[u] = li(idx + base + (j + u) * stride);
      v[u] = lv(val + base + (j + u) * stride);
    }
  };
  double acc = 0.0;
  auto consume = [&](const int32_t (&c)[D], const double (&v)[D]) {
    double xv[D];
#pragma unroll
    for (int u = 0; u < D; ++u) xv[u] = ldx(x, c[u]);
#pragma unroll
    for (int u = 0; u < D; ++u) acc = __dadd_rn(acc, __dmul_rn(v[u], xv[u]));
  };
  int64_t j = 0;
  if (k >= D) {
    int32_t ca[D], cb[D];
    double va[D], vb[D];
    load(0, ca, va);
    for (;;) {  // ca/va hold slots j..j+D-1
      if (j + 2 * D <= k) {
        load(j + D, cb, vb);
        consume(ca, va);
        j += D;
      } else {
        consume(ca, va);
        j += D;
        break;
      }
      // cb/vb hold slots j..j+D-1
      if (j + 2 * D <= k) {
        load(j + D, ca, va);
        consume(cb, vb);
        j += D;
      } else {
        consume(cb, vb);
        j += D;
        break;
      }
    }
  }
  for (; j < k; ++j) {
    const int64_t o = base + j * stride;
    acc = __dadd_rn(acc, __dmul_rn(lv(val + o), ldx(x, li(idx + o))));
  }
  return acc;
}

// The same recurrence four slots at a time without the prefetch: fewer
// registers, so more resident threads -- better for short rows (k <= 8).
// CACHED: slot loads through L1 (narrow SELL slices: the 16-byte index pieces
// of consecutive slots share 32-byte sectors, which L1 then serves).
template <bool CACHED = false>
__device__ __forceinline__ double seq_slots4(int64_t k, int64_t stride, int64_t base, const int32_t* __restrict__ idx,
                                             const double* __restrict__ val, const double* __restrict__ x) {
  auto li = [](const int32_t* p) { return CACHED ? __ldg(p) : ld_stream(p); };
  auto lv = [](const double* p) { return CACHED ? __ldg(p) : ld_stream(p); };
  double acc = 0.0;
  int64_t j = 0;
  for (; j + 4 <= k; j += 4) {
    const int64_t o = base + j * stride;
    const double v0 = lv(val + o), v1 = lv(val + o + stride);
    const double v2 = lv(val + o + 2 * stride), v3 = lv(val + o + 3 * stride);
    const int32_t c0 = li(idx + o), c1 = li(idx + o + stride);
    const int32_t c2 = li(idx + o + 2 * stride), c3 = li(idx + o + 3 * stride);
    acc = __dadd_rn(acc, __dmul_rn(v0, ldx(x, c0)));
    acc = __dadd_rn(acc, __dmul_rn(v1, ldx(x, c1)));
    acc = __dadd_rn(acc, __dmul_rn(v2, ldx(x, c2)));
    acc = __dadd_rn(acc, __dmul_rn(v3, ldx(x, c3)));
  }
  for (; j < k; ++j) {
    const int64_t o = base + j * stride;
    acc = __dadd_rn(acc, __dmul_rn(lv(val + o), ldx(x, li(idx + o))));
  }
  return acc;
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
