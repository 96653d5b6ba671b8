// Stable LSD radix sort of (uint64 key, uint32 value) pairs; see prims.cuh.
#include "prims.cuh"

namespace spmvb {

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

struct RsScatterSmem {
  uint64_t keys[RS_TILE];
  uint32_t vals[RS_TILE];
  uint32_t wcnt[RS_WARPS][RS_RADIX];
  uint32_t dstart[RS_RADIX];
  uint32_t gbase[RS_RADIX];
  uint32_t tmp[RS_THREADS / 32 + 1];
};

__global__ void __launch_bounds__(RS_THREADS) k_rs_scatter(const uint64_t* __restrict__ keys_in,
                                                           const uint32_t* __restrict__ vals_in,
                                                           uint64_t* __restrict__ keys_out,
                                                           uint32_t* __restrict__ vals_out, int64_t n, int shift,
                                                           unsigned mask, const uint32_t* __restrict__ offsets,
                                                           int64_t num_tiles) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  RsScatterSmem& sm = *reinterpret_cast<RsScatterSmem*>(smem_raw);
  const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < RS_WARPS * RS_RADIX; i += RS_THREADS) (&sm.wcnt[0][0])[i] = 0;
  __syncthreads();

  const int64_t tile_base = static_cast<int64_t>(blockIdx.x) * RS_TILE;
  const int64_t warp_base = tile_base + static_cast<int64_t>(warp) * RS_WARP_ITEMS;
  uint64_t key[RS_LANE_ITEMS];
  uint32_t val[RS_LANE_ITEMS];
  uint32_t rank[RS_LANE_ITEMS];
#pragma unroll
  for (int r = 0; r < RS_LANE_ITEMS; ++r) {
    int64_t idx = warp_base + r * 32 + lane;
    bool valid = idx < n;
    key[r] = valid ? keys_in[idx] : 0;
    val[r] = valid ? (vals_in ? vals_in[idx] : static_cast<uint32_t>(idx)) : 0;
  }
#pragma unroll
  for (int r = 0; r < RS_LANE_ITEMS; ++r) {
    int64_t idx = warp_base + r * 32 + lane;
    bool valid = idx < n;
    unsigned d = valid ? rs_digit(key[r], shift, mask) : 0u;
    unsigned peers = rs_peers(d, valid);
    uint32_t before = 0;
    if (valid) before = sm.wcnt[warp][d];
    __syncwarp();
    if (valid && lane == static_cast<unsigned>(__ffs(peers) - 1)) sm.wcnt[warp][d] = before + __popc(peers);
    __syncwarp();
    rank[r] = before + __popc(peers & lanemask_lt());
  }
  __syncthreads();
  // Per digit: exclusive prefix over warps, then block-wide digit starts.
  uint32_t total = 0;
  {
    const int d = threadIdx.x;  // RS_THREADS == RS_RADIX
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < RS_WARPS; ++w) {
      uint32_t t = sm.wcnt[w][d];
      sm.wcnt[w][d] = run;
      run += t;
    }
    total = run;
    sm.gbase[d] = offsets[static_cast<int64_t>(d) * num_tiles + blockIdx.x];
  }
  uint32_t start = block_exclusive_scan<uint32_t, RS_THREADS>(total, OpSum{}, 0u, sm.tmp, nullptr);
  sm.dstart[threadIdx.x] = start;
  __syncthreads();
#pragma unroll
  for (int r = 0; r < RS_LANE_ITEMS; ++r) {
    int64_t idx = warp_base + r * 32 + lane;
    if (idx < n) {
      unsigned d = rs_digit(key[r], shift, mask);
      uint32_t pos = sm.dstart[d] + sm.wcnt[warp][d] + rank[r];
      sm.keys[pos] = key[r];
      sm.vals[pos] = val[r];
    }
  }
  __syncthreads();
  int64_t count = n - tile_base;
  if (count > RS_TILE) count = RS_TILE;
  for (int i = threadIdx.x; i < count; i += RS_THREADS) {
    uint64_t k = sm.keys[i];
    unsigned d = rs_digit(k, shift, mask);
    int64_t g = static_cast<int64_t>(sm.gbase[d]) + (i - static_cast<int64_t>(sm.dstart[d]));
    keys_out[g] = k;
    vals_out[g] = sm.vals[i];
  }
}

__global__ void k_iota_u32(uint32_t* v, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    v[i] = static_cast<uint32_t>(i);
}

RadixSortResult radix_sort_pairs(uint64_t* keys_a, uint32_t* vals_a, uint64_t* keys_b, uint32_t* vals_b,
                                 uint32_t* vals_scratch, int64_t n, int key_bits, cudaStream_t s) {
  // vals_a == nullptr means "identity values"; vals_scratch must then be a
  // buffer of n entries that can hold the ping-pong copy.
  if (n >= (1ll << 32)) fail(SPMVB_INVALID_ARG, "radix sort supports fewer than 2^32 items");
  uint64_t* kin = keys_a;
  uint32_t* vin = vals_a;
  uint64_t* kout = keys_b;
  uint32_t* vout = vals_b;
  if (n == 0) return {keys_a, vals_a ? vals_a : vals_scratch};
  if (key_bits <= 0) {
    if (!vals_a) {
      k_iota_u32<<<grid_for(n, 256, 4096), 256, 0, s>>>(vals_scratch, n);
      SPMVB_LAUNCHED("k_iota_u32");
      return {keys_a, vals_scratch};
    }
    return {keys_a, vals_a};
  }
  const int64_t tiles = (n + RS_TILE - 1) / RS_TILE;
  DevBuf<uint32_t> hist(static_cast<size_t>(tiles) * RS_RADIX, s);
  const size_t smem = sizeof(RsScatterSmem);
  SPMVB_CUDA(cudaFuncSetAttribute(k_rs_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  bool first = true;
  for (int shift = 0; shift < key_bits; shift += 8) {
    int nbits = key_bits - shift < 8 ? key_bits - shift : 8;
    unsigned mask = (1u << nbits) - 1u;
    k_rs_hist<<<static_cast<unsigned>(tiles), RS_THREADS, 0, s>>>(kin, n, shift, mask, hist.get(), tiles);
    SPMVB_LAUNCHED("k_rs_hist");
    uint32_t* h = hist.get();
    exclusive_scan<uint32_t>(tiles * RS_RADIX, ArrayLoad<uint32_t>{h}, ArrayStore<uint32_t>{h}, OpSum{}, 0u,
                             static_cast<uint32_t*>(nullptr), s);
    if (first && !vals_a) vout = vals_b;  // identity values generated on the fly
    k_rs_scatter<<<static_cast<unsigned>(tiles), RS_THREADS, smem, s>>>(kin, first ? vals_a : vin, kout, vout, n,
                                                                        shift, mask, h, tiles);
    SPMVB_LAUNCHED("k_rs_scatter");
    // ping-pong
    uint64_t* tk = kin; kin = kout; kout = tk;
    if (first && !vals_a) {
      vin = vout;
      vout = vals_scratch;
    } else {
      uint32_t* tv = vin; vin = vout; vout = tv;
    }
    first = false;
  }
  return {kin, vin};
}

}  // namespace spmvb
