// Device-wide primitives used by the conversion kernels: block scans,
// a reduce-then-scan exclusive prefix sum over integer sequences, and a
// stable LSD radix sort of (uint64 key, 4- or 8-byte value) pairs.
//
// Everything here is integer arithmetic, so results are independent of the
// reduction order and therefore deterministic.
#pragma once

#include "common.cuh"

namespace spmvb {

// ---------------------------------------------------------------------------
// Block-level scans (blockDim.x == THREADS, multiple of 32)
// ---------------------------------------------------------------------------
template <typename T, int THREADS, typename Op>
__device__ __forceinline__ T block_exclusive_scan(T v, Op op, T identity, T* warp_tmp /*[THREADS/32+1]*/,
                                                  T* block_total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int NW = THREADS / 32;
  T inc = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    T o = __shfl_up_sync(0xffffffffu, inc, d);
    if (lane >= d) inc = op(o, inc);
  }
  if (lane == 31) warp_tmp[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    T w = (lane < NW) ? warp_tmp[lane] : identity;
    T winc = w;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      T o = __shfl_up_sync(0xffffffffu, winc, d);
      if (lane >= d) winc = op(o, winc);
    }
    if (lane < NW) warp_tmp[lane] = op(winc, identity);  // inclusive per warp
    if (lane == NW - 1) warp_tmp[NW] = winc;
  }
  __syncthreads();
  T warp_prefix = (warp == 0) ? identity : warp_tmp[warp - 1];
  T excl = __shfl_up_sync(0xffffffffu, inc, 1);
  if (lane == 0) excl = identity;
  T result = op(warp_prefix, excl);
  if (block_total) *block_total = warp_tmp[NW];
  return result;
}

template <typename T, int THREADS, typename Op>
__device__ __forceinline__ T block_reduce(T v, Op op, T identity, T* warp_tmp) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int NW = THREADS / 32;
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) v = op(v, __shfl_down_sync(0xffffffffu, v, d));
  if (lane == 0) warp_tmp[warp] = v;
  __syncthreads();
  T r = identity;
  if (warp == 0) {
    r = (lane < NW) ? warp_tmp[lane] : identity;
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) r = op(r, __shfl_down_sync(0xffffffffu, r, d));
  }
  __syncthreads();
  return r;  // valid in thread 0
}

struct OpSum {
  template <typename T>
  __host__ __device__ T operator()(T a, T b) const { return a + b; }
};
struct OpMin {
  template <typename T>
  __host__ __device__ T operator()(T a, T b) const { return b < a ? b : a; }
};
struct OpMax {
  template <typename T>
  __host__ __device__ T operator()(T a, T b) const { return a < b ? b : a; }
};

// ---------------------------------------------------------------------------
// Device-wide exclusive scan: out(i) = op(in(0..i-1)), total written to
// *total (device pointer, may be null).  `load(i)` and `store(i, v)` are
// device functors so inputs/outputs can be fused transforms.
// ---------------------------------------------------------------------------
constexpr int SCAN_THREADS = 256;
constexpr int SCAN_ITEMS = 8;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

template <typename T, typename Load, typename Op>
__global__ void __launch_bounds__(SCAN_THREADS) k_scan_tile_reduce(int64_t n, Load load, Op op, T identity,
                                                                   T* tile_out) {
  pdl_wait();
  __shared__ T tmp[SCAN_THREADS / 32 + 1];
  int64_t base = static_cast<int64_t>(blockIdx.x) * SCAN_TILE;
  T acc = identity;
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; ++i) {
    int64_t idx = base + i * SCAN_THREADS + threadIdx.x;
    if (idx < n) acc = op(acc, load(idx));
  }
  T r = block_reduce<T, SCAN_THREADS>(acc, op, identity, tmp);
  if (threadIdx.x == 0) tile_out[blockIdx.x] = r;
}

template <typename T, typename Load, typename Store, typename Op>
__global__ void __launch_bounds__(SCAN_THREADS) k_scan_tile(int64_t n, Load load, Store store, Op op,
                                                            T identity, const T* tile_prefix, T* total) {
  __shared__ T buf[SCAN_TILE];
  __shared__ T tmp[SCAN_THREADS / 32 + 1];
  __shared__ T btotal;
  int64_t base = static_cast<int64_t>(blockIdx.x) * SCAN_TILE;
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; ++i) {
    int j = i * SCAN_THREADS + threadIdx.x;
    int64_t idx = base + j;
    buf[j] = (idx < n) ? load(idx) : identity;
  }
  __syncthreads();
  T local[SCAN_ITEMS];
  T run = identity;
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; ++i) {
    local[i] = run;
    run = op(run, buf[threadIdx.x * SCAN_ITEMS + i]);
  }
  T prefix = block_exclusive_scan<T, SCAN_THREADS>(run, op, identity, tmp, threadIdx.x == 0 ? &btotal : nullptr);
  T tp = tile_prefix ? tile_prefix[blockIdx.x] : identity;
  prefix = op(tp, prefix);
  __syncthreads();
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; ++i) buf[threadIdx.x * SCAN_ITEMS + i] = op(prefix, local[i]);
  __syncthreads();
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; ++i) {
    int j = i * SCAN_THREADS + threadIdx.x;
    int64_t idx = base + j;
    if (idx < n) store(idx, buf[j]);
  }
  if (total && threadIdx.x == 0 && blockIdx.x == gridDim.x - 1) *total = op(tp, btotal);
}

template <typename T>
struct ArrayLoad {
  const T* p;
  __device__ T operator()(int64_t i) const { return p[i]; }
};
template <typename T>
struct ArrayStore {
  T* p;
  __device__ void operator()(int64_t i, T v) const { p[i] = v; }
};

template <typename T, typename Load, typename Store, typename Op>
void exclusive_scan(int64_t n, Load load, Store store, Op op, T identity, T* total, cudaStream_t s) {
  if (n <= 0) {
    if (total) SPMVB_CUDA(cudaMemcpyAsync(total, &identity, sizeof(T), cudaMemcpyHostToDevice, s));
    if (total) SPMVB_CUDA(cudaStreamSynchronize(s));  // identity lives on the host stack
    return;
  }
  int64_t tiles = (n + SCAN_TILE - 1) / SCAN_TILE;
  if (tiles == 1) {
    k_scan_tile<T><<<1, SCAN_THREADS, 0, s>>>(n, load, store, op, identity, nullptr, total);
    SPMVB_LAUNCHED("k_scan_tile");
    return;
  }
  DevBuf<T> tile_sums(tiles, s);
  k_scan_tile_reduce<T><<<grid_for(tiles * SCAN_TILE, SCAN_TILE), SCAN_THREADS, 0, s>>>(n, load, op, identity,
                                                                                        tile_sums.get());
  SPMVB_LAUNCHED("k_scan_tile_reduce");
  exclusive_scan<T>(tiles, ArrayLoad<T>{tile_sums.get()}, ArrayStore<T>{tile_sums.get()}, op, identity,
                    static_cast<T*>(nullptr), s);
  k_scan_tile<T><<<static_cast<unsigned>(tiles), SCAN_THREADS, 0, s>>>(n, load, store, op, identity,
                                                                       tile_sums.get(), total);
  SPMVB_LAUNCHED("k_scan_tile");
}

// Device-wide reduction to a device scalar.
template <typename T, typename Load, typename Op>
__global__ void __launch_bounds__(SCAN_THREADS) k_reduce_final(int64_t n, Load load, Op op, T identity, T* out) {
  pdl_wait();
  __shared__ T tmp[SCAN_THREADS / 32 + 1];
  T acc = identity;
  for (int64_t i = threadIdx.x; i < n; i += SCAN_THREADS) acc = op(acc, load(i));
  T r = block_reduce<T, SCAN_THREADS>(acc, op, identity, tmp);
  if (threadIdx.x == 0) *out = r;
}

// pdl: launch as programmatic dependents of the preceding kernel (see
// launch_pdl); the kernels wait for it before reading.
template <typename T, typename Load, typename Op>
void device_reduce(int64_t n, Load load, Op op, T identity, T* out, cudaStream_t s, bool pdl = false) {
  if (n <= SCAN_TILE) {
    if (pdl) launch_pdl(k_reduce_final<T, Load, Op>, dim3(1), dim3(SCAN_THREADS), 0, s, n, load, op, identity, out);
    else k_reduce_final<T><<<1, SCAN_THREADS, 0, s>>>(n, load, op, identity, out);
    SPMVB_LAUNCHED("k_reduce_final");
    return;
  }
  int64_t tiles = (n + SCAN_TILE - 1) / SCAN_TILE;
  DevBuf<T> part(tiles, s);
  if (pdl)
    launch_pdl(k_scan_tile_reduce<T, Load, Op>, dim3(static_cast<unsigned>(tiles)), dim3(SCAN_THREADS), 0, s, n,
               load, op, identity, part.get());
  else
    k_scan_tile_reduce<T><<<static_cast<unsigned>(tiles), SCAN_THREADS, 0, s>>>(n, load, op, identity, part.get());
  SPMVB_LAUNCHED("k_scan_tile_reduce");
  device_reduce<T>(tiles, ArrayLoad<T>{part.get()}, op, identity, out, s, pdl);
}

// ---------------------------------------------------------------------------
// Long rows.  Thread-per-row loops serialise power-law rows (R-MAT rows reach
// ~4e5 entries), so per-row copy kernels skip rows longer than LONG_ROW and a
// second launch gives each of those rows a whole CTA.
// ---------------------------------------------------------------------------
constexpr int64_t LONG_ROW = 512;

template <typename F>
__global__ void k_per_long_row(const int32_t* __restrict__ list, F f) {
  f(static_cast<int64_t>(list[blockIdx.x]), static_cast<int64_t>(threadIdx.x), static_cast<int64_t>(blockDim.x));
}

// Runs f(row, first, stride) with one 256-thread CTA for every row whose
// count(row) > LONG_ROW (ascending row list built by scan compaction).
template <typename Count, typename F>
void for_long_rows(Count count, int64_t n, F f, cudaStream_t s) {
  if (n <= 0) return;
  DevBuf<int32_t> list(n, s);
  DevBuf<int32_t> total(1, s);
  int32_t* lp = list.get();
  exclusive_scan<int32_t>(
      n, [=] __device__(int64_t i) { return count(i) > LONG_ROW ? 1 : 0; },
      [=] __device__(int64_t i, int32_t v) {
        if (count(i) > LONG_ROW) lp[v] = static_cast<int32_t>(i);
      },
      OpSum{}, 0, total.get(), s);
  int32_t h = 0;
  copy_to_host(&h, total.get(), 1, s);
  if (h > 0) {
    k_per_long_row<<<static_cast<unsigned>(h), 256, 0, s>>>(lp, f);
    SPMVB_LAUNCHED("k_per_long_row");
  }
}

// ---------------------------------------------------------------------------
// Stable LSD radix sort of (uint64 key, value) pairs over the low `key_bits`
// bits, 8-bit digits.  Below 2^30 items each pass is one kernel (digit
// histograms of all passes from one read of the keys, then per pass a tile
// ranking + decoupled look-back + shared-memory-staged scatter, so global
// writes are coalesced per digit run); above, reduce-then-scan passes.
// ---------------------------------------------------------------------------
constexpr int RS_THREADS = 256;
constexpr int RS_WARPS = RS_THREADS / 32;
#ifndef SPMVB_RS_LANE_ITEMS
#define SPMVB_RS_LANE_ITEMS 16
#endif
constexpr int RS_LANE_ITEMS = SPMVB_RS_LANE_ITEMS;       // per lane
constexpr int RS_WARP_ITEMS = 32 * RS_LANE_ITEMS;        // 512
constexpr int RS_TILE = RS_WARPS * RS_WARP_ITEMS;        // 4096
constexpr int RS_RADIX = 256;

struct RadixSortResult {
  uint64_t* keys;
  uint32_t* vals;
};
struct RadixSortResult64 {
  uint64_t* keys;
  uint64_t* vals;
};

// Sorts keys_a/vals_a (vals_a may be null: identity 0..n-1) using keys_b /
// vals_b as ping-pong storage. Returns the buffers that hold the result.
RadixSortResult radix_sort_pairs(uint64_t* keys_a, uint32_t* vals_a, uint64_t* keys_b, uint32_t* vals_b,
                                 uint32_t* vals_scratch, int64_t n, int key_bits, cudaStream_t s);

// Sorts keys_a carrying 8-byte values read from vals_in (left unmodified);
// keys_b, vals_a and vals_b are ping-pong storage.  Returns the buffers that
// hold the result (keys_a or keys_b; vals_a or vals_b).
// digit_hist (optional, device): the digit counts of every pass already
// taken by the caller while building the keys, hist[p*256 + d] for the
// ceil(key_bits/8) passes (saves the sort its own read of the keys).
RadixSortResult64 radix_sort_pairs64(uint64_t* keys_a, uint64_t* keys_b, const uint64_t* vals_in, uint64_t* vals_a,
                                     uint64_t* vals_b, int64_t n, int key_bits, cudaStream_t s,
                                     const uint32_t* digit_hist = nullptr);

}  // namespace spmvb
