// Stable LSD radix sort of (uint64 key, value) pairs; see prims.cuh.
//
// Below 2^30 items every pass is ONE kernel (single-pass "onesweep" scheme):
// the digit histograms of all passes come from one read of the keys up
// front, and each tile finds the global position of its digit runs by a
// decoupled look-back over its predecessors' published counts, so a pass
// reads and writes every (key, value) pair once.  Larger inputs use the
// reduce-then-scan scheme (per-pass tile histogram, scan, scatter).
#include <cstdlib>
#include <utility>

#include "prims.cuh"

#ifndef SPMVB_RS_MIN_BLOCKS
#define SPMVB_RS_MIN_BLOCKS 4
#endif

namespace spmvb {

// resident blocks per SM the tile kernels are compiled for (registers)
constexpr int RS_MIN_BLOCKS = SPMVB_RS_MIN_BLOCKS;

__device__ __forceinline__ unsigned rs_digit(uint64_t key, int shift, unsigned mask) {
  return static_cast<unsigned>(key >> shift) & mask;
}

// Lanes of the warp holding the same digit (warp multi-split by ballots: one
// ballot per digit bit, constant time however many distinct digits the warp
// holds -- __match_any_sync slows down with every distinct value).  Only
// meaningful for valid lanes; invalid lanes are excluded from every mask.
__device__ __forceinline__ unsigned rs_peers(unsigned d, bool valid) {
  unsigned peers = __ballot_sync(0xffffffffu, valid);
#pragma unroll
  for (int b = 0; b < 8; ++b) {  // RS_RADIX = 256: 8 digit bits
    const bool bit = (d >> b) & 1u;
    const unsigned bal = __ballot_sync(0xffffffffu, bit);
    peers &= bit ? bal : ~bal;
  }
  return peers;
}

// ------------------------------------------------------------------------
// Tile ranking shared by both schemes: loads the tile's keys (lane-strided
// per warp, so item order = warp, then r, then lane), ranks each item among
// the equal digits of its warp that precede it, and leaves per-warp digit
// counts in wcnt.  Stable by construction.  Values are not held across the
// ranking (registers decide the occupancy of these kernels): they are read
// when the tile is written out.
// ------------------------------------------------------------------------
struct RsTileSmem {
  uint64_t buf[RS_TILE];  // the tile in digit order: keys, then values
  uint8_t dig[RS_TILE];   // digit of each slot (for the value round)
  uint32_t wcnt[RS_WARPS][RS_RADIX];
  uint32_t dstart[RS_RADIX];
  uint32_t gbase[RS_RADIX];
  uint32_t tmp[RS_THREADS / 32 + 1];
  uint32_t thist[RS_RADIX];  // the tile's digit counts (onesweep: published before the ranking)
  uint32_t tile;
};

__device__ __forceinline__ void rs_load_tile(const uint64_t* __restrict__ keys_in, int64_t n, int64_t tile_base,
                                             uint64_t (&key)[RS_LANE_ITEMS]) {
  const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t warp_base = tile_base + static_cast<int64_t>(warp) * RS_WARP_ITEMS;
#pragma unroll
  for (int r = 0; r < RS_LANE_ITEMS; ++r) {
    const int64_t idx = warp_base + r * 32 + lane;
    key[r] = idx < n ? keys_in[idx] : 0;
  }
}

__device__ __forceinline__ void rs_rank_loaded(RsTileSmem& sm, int64_t n, int64_t tile_base, int shift, unsigned mask,
                                               const uint64_t (&key)[RS_LANE_ITEMS],
                                               uint32_t (&rank)[RS_LANE_ITEMS]) {
  const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t warp_base = tile_base + static_cast<int64_t>(warp) * RS_WARP_ITEMS;
#pragma unroll
  for (int r = 0; r < RS_LANE_ITEMS; ++r) {
    const int64_t idx = warp_base + r * 32 + lane;
    const bool valid = idx < n;
    const unsigned d = valid ? rs_digit(key[r], shift, mask) : 0u;
    const unsigned peers = rs_peers(d, valid);
    uint32_t before = 0;
    if (valid) before = sm.wcnt[warp][d];
    __syncwarp();
    if (valid && lane == static_cast<unsigned>(__ffs(peers) - 1)) sm.wcnt[warp][d] = before + __popc(peers);
    __syncwarp();
    // the item's position in the tile's digit order once wcnt holds the
    // per-warp exclusive prefixes (rs_write_tile adds dstart and wcnt)
    rank[r] = before + __popc(peers & lanemask_lt());
  }
}

__device__ __forceinline__ void rs_rank_tile(RsTileSmem& sm, const uint64_t* __restrict__ keys_in, int64_t n,
                                             int64_t tile_base, int shift, unsigned mask,
                                             uint64_t (&key)[RS_LANE_ITEMS], uint32_t (&rank)[RS_LANE_ITEMS]) {
  rs_load_tile(keys_in, n, tile_base, key);
  rs_rank_loaded(sm, n, tile_base, shift, mask, key, rank);
}

// Writes the ranked tile out: keys through shared memory in digit order
// (consecutive threads write consecutive positions of each digit run), then
// the values the same way through the same buffer (read from global here;
// vals_in == nullptr: the identity, item index).
template <typename V>
__device__ __forceinline__ void rs_write_tile(RsTileSmem& sm, int64_t n, int64_t tile_base, int shift,
                                              unsigned mask, const uint64_t (&key)[RS_LANE_ITEMS],
                                              uint32_t (&rank)[RS_LANE_ITEMS], const V* __restrict__ vals_in,
                                              uint64_t* __restrict__ keys_out, V* __restrict__ vals_out) {
  const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t warp_base = tile_base + static_cast<int64_t>(warp) * RS_WARP_ITEMS;
#pragma unroll
  for (int r = 0; r < RS_LANE_ITEMS; ++r) {
    const int64_t idx = warp_base + r * 32 + lane;
    if (idx < n) {
      const unsigned d = rs_digit(key[r], shift, mask);
      rank[r] += sm.dstart[d] + sm.wcnt[warp][d];
      sm.buf[rank[r]] = key[r];
    }
  }
  // the values' loads are issued now (the key registers are dead) and land
  // while the keys are written out
  V vv[RS_LANE_ITEMS];
#pragma unroll
  for (int r = 0; r < RS_LANE_ITEMS; ++r) {
    const int64_t idx = warp_base + r * 32 + lane;
    vv[r] = idx < n ? (vals_in ? vals_in[idx] : static_cast<V>(idx)) : V(0);
  }
  __syncthreads();
  int64_t count = n - tile_base;
  if (count > RS_TILE) count = RS_TILE;
  // tile slot i goes to gbase[d] + (i - dstart[d]), d = the slot's digit
  for (int i = threadIdx.x; i < count; i += RS_THREADS) {
    const uint64_t k = sm.buf[i];
    const unsigned d = rs_digit(k, shift, mask);
    sm.dig[i] = static_cast<uint8_t>(d);
    keys_out[static_cast<int64_t>(sm.gbase[d]) + (i - static_cast<int64_t>(sm.dstart[d]))] = k;
  }
  __syncthreads();
  V* vbuf = reinterpret_cast<V*>(sm.buf);
#pragma unroll
  for (int r = 0; r < RS_LANE_ITEMS; ++r) {
    const int64_t idx = warp_base + r * 32 + lane;
    if (idx < n) vbuf[rank[r]] = vv[r];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < count; i += RS_THREADS) {
    const unsigned d = sm.dig[i];
    vals_out[static_cast<int64_t>(sm.gbase[d]) + (i - static_cast<int64_t>(sm.dstart[d]))] = vbuf[i];
  }
}

// Per digit (thread d): exclusive prefix of the per-warp counts in place;
// returns the tile's count of digit d.
__device__ __forceinline__ uint32_t rs_warp_prefix(RsTileSmem& sm) {
  const int d = threadIdx.x;  // RS_THREADS == RS_RADIX
  uint32_t run = 0;
#pragma unroll
  for (int w = 0; w < RS_WARPS; ++w) {
    const uint32_t t = sm.wcnt[w][d];
    sm.wcnt[w][d] = run;
    run += t;
  }
  return run;
}

// ------------------------------------------------------------ onesweep ----
constexpr uint32_t RS_FLAG_AGG = 1u << 30;     // tile's own count published
constexpr uint32_t RS_FLAG_PRE = 2u << 30;     // inclusive prefix published
constexpr uint32_t RS_VAL_MASK = (1u << 30) - 1;
constexpr int RS_MAX_PASSES = 8;

__device__ __forceinline__ uint32_t ld_relaxed_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_gpu(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Digit histograms of every pass in one read of the keys: hist[p*256 + d]
// (zeroed by the caller).  Each warp counts into its own shared-memory copy
// (plain atomics: conflicts only among a warp's lanes), merged at the end.
constexpr int RS_HIST_WARPS = 4;
__global__ void __launch_bounds__(RS_HIST_WARPS * 32) k_rs_hist_all(const uint64_t* __restrict__ keys, int64_t n,
                                                                    int passes, int key_bits,
                                                                    uint32_t* __restrict__ hist) {
  __shared__ uint32_t cnt[RS_HIST_WARPS][RS_MAX_PASSES * RS_RADIX];
  for (int i = threadIdx.x; i < RS_HIST_WARPS * RS_MAX_PASSES * RS_RADIX; i += blockDim.x) (&cnt[0][0])[i] = 0;
  __syncthreads();
  uint32_t* mine = cnt[threadIdx.x >> 5];
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  constexpr int U = 4;
  for (int64_t base = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; base < n; base += U * stride) {
    uint64_t k[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + u * stride;
      k[u] = i < n ? keys[i] : ~0ull;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (base + u * stride >= n) break;
      for (int p = 0, shift = 0; p < passes; ++p, shift += 8) {
        const int nb = key_bits - shift < 8 ? key_bits - shift : 8;
        atomicAdd(&mine[p * RS_RADIX + rs_digit(k[u], shift, (1u << nb) - 1u)], 1u);
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < passes * RS_RADIX; i += blockDim.x) {
    uint32_t t = 0;
#pragma unroll
    for (int w = 0; w < RS_HIST_WARPS; ++w) t += cnt[w][i];
    if (t) atomicAdd(&hist[i], t);
  }
}

// hist[p*256 + d] -> exclusive prefix over d, in place (one block per pass).
__global__ void __launch_bounds__(RS_RADIX) k_rs_digit_offsets(uint32_t* hist) {
  __shared__ uint32_t tmp[RS_RADIX / 32 + 1];
  uint32_t* h = hist + blockIdx.x * RS_RADIX;
  const uint32_t v = h[threadIdx.x];
  const uint32_t e = block_exclusive_scan<uint32_t, RS_RADIX>(v, OpSum{}, 0u, tmp, nullptr);
  h[threadIdx.x] = e;
}

// One pass.  Tiles are numbered in the order their blocks start (atomic
// counter), so every predecessor a tile looks back at is running or done:
// the look-back always terminates.
template <typename V>
__global__ void __launch_bounds__(RS_THREADS, RS_MIN_BLOCKS) k_rs_onesweep(const uint64_t* __restrict__ keys_in,
                                                            const V* __restrict__ vals_in,
                                                            uint64_t* __restrict__ keys_out,
                                                            V* __restrict__ vals_out, int64_t n, int shift,
                                                            unsigned mask, const uint32_t* __restrict__ digit_off,
                                                            uint32_t* __restrict__ status,
                                                            uint32_t* __restrict__ tile_counter) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  RsTileSmem& sm = *reinterpret_cast<RsTileSmem*>(smem_raw);
  const int d = threadIdx.x;
  if (threadIdx.x == 0) sm.tile = atomicAdd(tile_counter, 1u);
  for (int i = threadIdx.x; i < RS_WARPS * RS_RADIX; i += RS_THREADS) (&sm.wcnt[0][0])[i] = 0;
  sm.thist[d] = 0;
  __syncthreads();
  const int64_t t = sm.tile;
  const int64_t tile_base = t * RS_TILE;
  uint64_t key[RS_LANE_ITEMS];
  uint32_t rank[RS_LANE_ITEMS];
  rs_load_tile(keys_in, n, tile_base, key);
  // the tile's digit counts first, published at once so that successors'
  // look-backs find them while this tile is still ranking
  {
    const int64_t warp_base = tile_base + static_cast<int64_t>(threadIdx.x >> 5) * RS_WARP_ITEMS + (threadIdx.x & 31);
#pragma unroll
    for (int r = 0; r < RS_LANE_ITEMS; ++r)
      if (warp_base + r * 32 < n) atomicAdd(&sm.thist[rs_digit(key[r], shift, mask)], 1u);
  }
  __syncthreads();
  const uint32_t total = sm.thist[d];
  uint32_t* mine = status + t * RS_RADIX + d;
  st_relaxed_gpu(mine, (t == 0 ? RS_FLAG_PRE : RS_FLAG_AGG) | total);
  rs_rank_loaded(sm, n, tile_base, shift, mask, key, rank);
  __syncthreads();
  rs_warp_prefix(sm);
  // look back for the exclusive prefix
  uint32_t excl = 0;
  if (t > 0) {
    for (int64_t j = t - 1;;) {
      const uint32_t w = ld_relaxed_gpu(status + j * RS_RADIX + d);
      if ((w & ~RS_VAL_MASK) == 0) continue;  // predecessor not there yet
      excl += w & RS_VAL_MASK;
      if (w & RS_FLAG_PRE) break;
      --j;
    }
    st_relaxed_gpu(mine, RS_FLAG_PRE | (excl + total));
  }
  sm.gbase[d] = digit_off[d] + excl;
  const uint32_t start = block_exclusive_scan<uint32_t, RS_THREADS>(total, OpSum{}, 0u, sm.tmp, nullptr);
  sm.dstart[d] = start;
  __syncthreads();
  rs_write_tile(sm, n, tile_base, shift, mask, key, rank, vals_in, keys_out, vals_out);
}

// ------------------------------------------------------ reduce-then-scan ----
// Per-tile digit histogram, written digit-major: hist[d * num_tiles + tile].
__global__ void __launch_bounds__(RS_THREADS) k_rs_hist(const uint64_t* __restrict__ keys, int64_t n, int shift,
                                                        unsigned mask, uint32_t* __restrict__ hist,
                                                        int64_t num_tiles) {
  __shared__ uint32_t cnt[RS_RADIX];
  for (int d = threadIdx.x; d < RS_RADIX; d += RS_THREADS) cnt[d] = 0;
  __syncthreads();
  int64_t base = static_cast<int64_t>(blockIdx.x) * RS_TILE;
  const unsigned lane = threadIdx.x & 31;
  // all of this thread's keys in flight first (the loop below is latency
  // bound otherwise), then warp-aggregated shared-memory counts
  constexpr int PER = RS_TILE / RS_THREADS;
  uint64_t k[PER];
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int64_t idx = base + static_cast<int64_t>(i) * RS_THREADS + threadIdx.x;
    k[i] = idx < n ? keys[idx] : 0;
  }
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int64_t idx = base + static_cast<int64_t>(i) * RS_THREADS + threadIdx.x;
    bool valid = idx < n;
    unsigned d = valid ? rs_digit(k[i], shift, mask) : 0u;
    unsigned peers = rs_peers(d, valid);
    if (valid && lane == static_cast<unsigned>(__ffs(peers) - 1)) atomicAdd(&cnt[d], __popc(peers));
  }
  __syncthreads();
  for (int d = threadIdx.x; d < RS_RADIX; d += RS_THREADS) hist[static_cast<int64_t>(d) * num_tiles + blockIdx.x] = cnt[d];
}

template <typename V>
__global__ void __launch_bounds__(RS_THREADS, RS_MIN_BLOCKS) k_rs_scatter(const uint64_t* __restrict__ keys_in,
                                                           const V* __restrict__ vals_in,
                                                           uint64_t* __restrict__ keys_out, V* __restrict__ vals_out,
                                                           int64_t n, int shift, unsigned mask,
                                                           const uint32_t* __restrict__ offsets, int64_t num_tiles) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  RsTileSmem& sm = *reinterpret_cast<RsTileSmem*>(smem_raw);
  for (int i = threadIdx.x; i < RS_WARPS * RS_RADIX; i += RS_THREADS) (&sm.wcnt[0][0])[i] = 0;
  __syncthreads();
  const int64_t tile_base = static_cast<int64_t>(blockIdx.x) * RS_TILE;
  uint64_t key[RS_LANE_ITEMS];
  uint32_t rank[RS_LANE_ITEMS];
  rs_rank_tile(sm, keys_in, n, tile_base, shift, mask, key, rank);
  __syncthreads();
  const int d = threadIdx.x;
  const uint32_t total = rs_warp_prefix(sm);
  sm.gbase[d] = offsets[static_cast<int64_t>(d) * num_tiles + blockIdx.x];
  const uint32_t start = block_exclusive_scan<uint32_t, RS_THREADS>(total, OpSum{}, 0u, sm.tmp, nullptr);
  sm.dstart[d] = start;
  __syncthreads();
  rs_write_tile(sm, n, tile_base, shift, mask, key, rank, vals_in, keys_out, vals_out);
}

__global__ void k_iota_u32(uint32_t* v, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    v[i] = static_cast<uint32_t>(i);
}

namespace {

// The passes: the first reads vin (or the identity), writes b; later passes
// ping-pong b <-> a.  Returns the buffers holding the result.
template <typename V>
std::pair<uint64_t*, V*> sort_passes(uint64_t* keys_a, uint64_t* keys_b, const V* vin, V* vals_a, V* vals_b, int64_t n,
                                     int key_bits, cudaStream_t s, const uint32_t* hist_in = nullptr) {
  const int64_t tiles = (n + RS_TILE - 1) / RS_TILE;
  const int passes = (key_bits + 7) / 8;
  const size_t smem = sizeof(RsTileSmem);
  uint64_t* kin = keys_a;
  uint64_t* kout = keys_b;
  const V* vcur = vin;
  V* vout = vals_b;
  auto advance = [&] {
    std::swap(kin, kout);
    vcur = vout;
    vout = (vout == vals_b) ? vals_a : vals_b;
  };
  // SPMVB_RADIX_RTS=1 forces the reduce-then-scan passes (tests of that path
  // without a 2^30-item input)
  const char* force = getenv("SPMVB_RADIX_RTS");
  const bool onesweep = !(force && force[0] == '1') && n < (1ll << 30) && passes <= RS_MAX_PASSES;
  if (onesweep) {
    SPMVB_CUDA(cudaFuncSetAttribute(k_rs_onesweep<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    DevBuf<uint32_t> hist(static_cast<size_t>(passes) * RS_RADIX, s);
    DevBuf<uint32_t> status(static_cast<size_t>(tiles) * RS_RADIX, s);
    DevBuf<uint32_t> counters(passes, s);
    SPMVB_CUDA(cudaMemsetAsync(counters.get(), 0, passes * sizeof(uint32_t), s));
    if (hist_in) {
      SPMVB_CUDA(cudaMemcpyAsync(hist.get(), hist_in, passes * RS_RADIX * sizeof(uint32_t), cudaMemcpyDeviceToDevice,
                                 s));
    } else {
      SPMVB_CUDA(cudaMemsetAsync(hist.get(), 0, passes * RS_RADIX * sizeof(uint32_t), s));
      k_rs_hist_all<<<grid_for(n, RS_HIST_WARPS * 32, 148 * 8), RS_HIST_WARPS * 32, 0, s>>>(keys_a, n, passes,
                                                                                          key_bits, hist.get());
      SPMVB_LAUNCHED("k_rs_hist_all");
    }
    k_rs_digit_offsets<<<passes, RS_RADIX, 0, s>>>(hist.get());
    SPMVB_LAUNCHED("k_rs_digit_offsets");
    for (int p = 0; p < passes; ++p) {
      const int shift = 8 * p;
      const int nb = key_bits - shift < 8 ? key_bits - shift : 8;
      SPMVB_CUDA(cudaMemsetAsync(status.get(), 0, tiles * RS_RADIX * sizeof(uint32_t), s));
      k_rs_onesweep<V><<<static_cast<unsigned>(tiles), RS_THREADS, smem, s>>>(
          kin, vcur, kout, vout, n, shift, (1u << nb) - 1u, hist.get() + p * RS_RADIX, status.get(),
          counters.get() + p);
      SPMVB_LAUNCHED("k_rs_onesweep");
      advance();
    }
  } else {
    SPMVB_CUDA(cudaFuncSetAttribute(k_rs_scatter<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    DevBuf<uint32_t> hist(static_cast<size_t>(tiles) * RS_RADIX, s);
    for (int p = 0; p < passes; ++p) {
      const int shift = 8 * p;
      const int nb = key_bits - shift < 8 ? key_bits - shift : 8;
      const unsigned mask = (1u << nb) - 1u;
      k_rs_hist<<<static_cast<unsigned>(tiles), RS_THREADS, 0, s>>>(kin, n, shift, mask, hist.get(), tiles);
      SPMVB_LAUNCHED("k_rs_hist");
      uint32_t* h = hist.get();
      exclusive_scan<uint32_t>(tiles * RS_RADIX, ArrayLoad<uint32_t>{h}, ArrayStore<uint32_t>{h}, OpSum{}, 0u,
                               static_cast<uint32_t*>(nullptr), s);
      k_rs_scatter<V><<<static_cast<unsigned>(tiles), RS_THREADS, smem, s>>>(kin, vcur, kout, vout, n, shift, mask,
                                                                             h, tiles);
      SPMVB_LAUNCHED("k_rs_scatter");
      advance();
    }
  }
  return {kin, const_cast<V*>(vcur)};
}

}  // namespace

RadixSortResult radix_sort_pairs(uint64_t* keys_a, uint32_t* vals_a, uint64_t* keys_b, uint32_t* vals_b,
                                 uint32_t* vals_scratch, int64_t n, int key_bits, cudaStream_t s) {
  // vals_a == nullptr means "identity values"; vals_scratch must then be a
  // buffer of n entries that can hold the ping-pong copy.
  if (n >= (1ll << 32)) fail(SPMVB_INVALID_ARG, "radix sort supports fewer than 2^32 items");
  if (n == 0) return {keys_a, vals_a ? vals_a : vals_scratch};
  if (key_bits <= 0) {
    if (!vals_a) {
      k_iota_u32<<<grid_for(n, 256, 4096), 256, 0, s>>>(vals_scratch, n);
      SPMVB_LAUNCHED("k_iota_u32");
      return {keys_a, vals_scratch};
    }
    return {keys_a, vals_a};
  }
  // values ping-pong between vals_b and the other buffer: vals_a itself, or
  // the scratch buffer for identity values
  auto r = sort_passes<uint32_t>(keys_a, keys_b, vals_a, vals_a ? vals_a : vals_scratch, vals_b, n, key_bits, s);
  return {r.first, r.second};
}

RadixSortResult64 radix_sort_pairs64(uint64_t* keys_a, uint64_t* keys_b, const uint64_t* vals_in, uint64_t* vals_a,
                                     uint64_t* vals_b, int64_t n, int key_bits, cudaStream_t s,
                                     const uint32_t* digit_hist) {
  if (n >= (1ll << 32)) fail(SPMVB_INVALID_ARG, "radix sort supports fewer than 2^32 items");
  if (n == 0) return {keys_a, vals_a};
  if (key_bits <= 0) {
    SPMVB_CUDA(cudaMemcpyAsync(vals_a, vals_in, n * sizeof(uint64_t), cudaMemcpyDeviceToDevice, s));
    return {keys_a, vals_a};
  }
  auto r = sort_passes<uint64_t>(keys_a, keys_b, vals_in, vals_a, vals_b, n, key_bits, s, digit_hist);
  return {r.first, r.second};
}

}  // namespace spmvb
