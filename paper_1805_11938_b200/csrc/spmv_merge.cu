// Merge-path CSR SpMV (reference kernels.py:76-95 spmv_csr) and the fused
// HYB kernel (kernels.py:177-199 spmv_hyb: ELL part + COO tail reduced
// through the tail's row pointer).  Deterministic: no floating-point
// atomics; rows crossing tiles are folded by k_merge_fixup in a fixed order.
#include "spmv_common.cuh"

using namespace spmvb;

namespace {

// =========================================================================
// Merge-path CSR (Merrill & Garland style), optional fused ELL part (HYB).
// The merge list is (row ends ptr[1..n], nonzero indices 0..nnz-1); each CTA
// consumes MP_TILE consecutive merge items whose start coordinates are
// precomputed by k_merge_plan (the "analysis" step).
// =========================================================================
constexpr int MP_THREADS = 256;
constexpr int MP_IPT = 8;
constexpr int MP_TILE = MP_THREADS * MP_IPT;

__global__ void k_merge_plan(int64_t n_rows, int64_t nnz, const int32_t* __restrict__ ptr, int64_t num_tiles,
                             int32_t* __restrict__ tile_row, int32_t* __restrict__ tile_nz) {
  for (int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; c <= num_tiles;
       c += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t d = c * MP_TILE;
    if (d > n_rows + nnz) d = n_rows + nnz;
    int64_t lo = d - nnz > 0 ? d - nnz : 0;
    int64_t hi = d < n_rows ? d : n_rows;
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (static_cast<int64_t>(ptr[mid + 1]) <= d - mid - 1) lo = mid + 1; else hi = mid;
    }
    tile_row[c] = static_cast<int32_t>(lo);
    tile_nz[c] = static_cast<int32_t>(d - lo);
  }
}

struct KeyVal {
  int key;
  double val;
};

struct ReduceByKeyOp {
  __device__ KeyVal operator()(const KeyVal& a, const KeyVal& b) const {
    return KeyVal{b.key, a.key == b.key ? a.val + b.val : b.val};
  }
};

__device__ __forceinline__ KeyVal shfl_up_kv(KeyVal v, int d) {
  KeyVal o;
  o.key = __shfl_up_sync(0xffffffffu, v.key, d);
  o.val = __shfl_up_sync(0xffffffffu, v.val, d);
  return o;
}

struct MergeSmem {
  int32_t row_end[MP_TILE + 1];
  double prod[MP_TILE];
  double yv[MP_TILE];
  KeyVal warp_kv[MP_THREADS / 32];
};

template <bool HAS_ELL>
__global__ void __launch_bounds__(MP_THREADS) k_spmv_merge(
    int64_t n_rows, int64_t nnz, const int32_t* __restrict__ ptr, const int32_t* __restrict__ col,
    const double* __restrict__ val, const int32_t* __restrict__ tile_row, const int32_t* __restrict__ tile_nz,
    int32_t* __restrict__ carry_row, double* __restrict__ carry_val, const double* __restrict__ x,
    double* __restrict__ y, const double* __restrict__ scale_p, int64_t ell_k, const int32_t* __restrict__ ell_idx,
    const double* __restrict__ ell_val) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  MergeSmem& sm = *reinterpret_cast<MergeSmem*>(smem_raw);
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int c = blockIdx.x;
  const int r0 = tile_row[c], z0 = tile_nz[c];
  const int r1 = tile_row[c + 1], z1 = tile_nz[c + 1];
  const int R = r1 - r0, Z = z1 - z0;

  // Stage row ends (R + 1 of them; the last is the row in progress at the
  // tile end) and the products of this tile's nonzeros.
  {
    // all loads of the tile issued back to back (8 column/value pairs and
    // 8 row ends per thread), then 8 independent gathers of x
    int32_t cc[MP_IPT];
    double vv[MP_IPT];
#pragma unroll
    for (int it = 0; it < MP_IPT; ++it) {
      const int j = tid + it * MP_THREADS;
      const int64_t k = static_cast<int64_t>(z0) + j;
      cc[it] = j < Z ? ld_stream(col + k) : 0;
      vv[it] = j < Z ? ld_stream(val + k) : 0.0;
      const int64_t r = static_cast<int64_t>(r0) + j;
      if (j <= R) sm.row_end[j] = r < n_rows ? ld_stream(ptr + r + 1) : INT32_MAX;
    }
    if (tid == 0 && R == MP_TILE) {
      const int64_t r = static_cast<int64_t>(r0) + R;
      sm.row_end[R] = r < n_rows ? ptr[r + 1] : INT32_MAX;
    }
#pragma unroll
    for (int it = 0; it < MP_IPT; ++it) {
      const int j = tid + it * MP_THREADS;
      if (j < Z) sm.prod[j] = vv[it] * ldx(x, cc[it]);
    }
  }
  __syncthreads();

  // Thread-level merge-path search inside the tile.
  const int items = R + Z;
  int td = tid * MP_IPT;
  if (td > items) td = items;
  int lo = td - Z > 0 ? td - Z : 0;
  int hi = td < R ? td : R;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (sm.row_end[mid] <= z0 + td - mid - 1) lo = mid + 1; else hi = mid;
  }
  int row = lo, nz = td - lo;
  double running = 0.0;
  int first_row = -1;
#pragma unroll
  for (int it = 0; it < MP_IPT; ++it) {
    if (td + it < items) {
      if (z0 + nz < sm.row_end[row]) {
        running += sm.prod[nz];
        ++nz;
      } else {
        sm.yv[row] = running;
        if (first_row < 0) first_row = row;
        running = 0.0;
        ++row;
      }
    }
  }
  // Block-wide exclusive reduce-by-key over the threads' carry-outs.
  KeyVal kv{row, running};
  KeyVal inc = kv;
  ReduceByKeyOp op;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    KeyVal o = shfl_up_kv(inc, d);
    if (lane >= d) inc = op(o, inc);
  }
  if (lane == 31) sm.warp_kv[warp] = inc;
  __syncthreads();
  KeyVal excl = shfl_up_kv(inc, 1);
  KeyVal wprefix{-1, 0.0};
  for (int w = 0; w < warp; ++w) wprefix = (w == 0) ? sm.warp_kv[0] : op(wprefix, sm.warp_kv[w]);
  KeyVal prefix;
  if (lane == 0) prefix = wprefix;
  else prefix = (warp == 0) ? excl : op(wprefix, excl);
  if (tid == 0) prefix = KeyVal{-1, 0.0};
  if (first_row >= 0 && prefix.key == first_row) sm.yv[first_row] += prefix.val;
  if (tid == MP_THREADS - 1) {
    KeyVal total = (warp == 0) ? inc : op(wprefix, inc);
    // Tile carry-out: the partial of the row in progress at the tile end.
    int64_t gr = static_cast<int64_t>(r0) + total.key;
    carry_row[c] = gr < n_rows ? static_cast<int32_t>(gr) : -1;
    carry_val[c] = total.val;
  }
  __syncthreads();
  const double s = load_scale(scale_p);
  for (int i = tid; i < R; i += MP_THREADS) {
    int64_t r = static_cast<int64_t>(r0) + i;
    double v = sm.yv[i];
    if (HAS_ELL) {
      double e = 0.0;
      for (int64_t j = 0; j < ell_k; ++j) {
        int64_t o = j * n_rows + r;
        e = __dadd_rn(e, __dmul_rn(ld_stream(ell_val + o), ldx(x, ld_stream(ell_idx + o))));
      }
      v = e + v;
    }
    y[r] = s * v;
  }
}

// Folds every chain of tile carry-outs (consecutive tiles whose carry row is
// the same) into its row.  One warp per 32 tiles finds the chain starts; each
// chain is then summed by the whole warp, 32 tiles per step, with a fixed
// reduction tree (deterministic), so a row spanning thousands of tiles costs
// tens of steps instead of thousands.
__global__ void k_merge_fixup(int64_t num_tiles, const int32_t* __restrict__ carry_row,
                              const double* __restrict__ carry_val, double* __restrict__ y,
                              const double* __restrict__ scale_p) {
  const int lane = threadIdx.x & 31;
  const int64_t warp_id = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t w0 = warp_id * 32; w0 < num_tiles; w0 += nwarps * 32) {
    const int64_t c = w0 + lane;
    const int32_t r = c < num_tiles ? carry_row[c] : -1;
    const bool start = r >= 0 && !(c > 0 && carry_row[c - 1] == r);
    unsigned starts = __ballot_sync(0xffffffffu, start);
    while (starts) {
      const int l = __ffs(starts) - 1;
      starts &= starts - 1;
      const int32_t key = __shfl_sync(0xffffffffu, r, l);
      double acc = 0.0;
      for (int64_t b = w0 + l;; b += 32) {
        const int64_t cc = b + lane;
        const bool in = cc < num_tiles && carry_row[cc] == key;
        const unsigned m = __ballot_sync(0xffffffffu, in);
        const int len = (m == 0xffffffffu) ? 32 : __ffs(~m) - 1;
        if (lane < len) acc += carry_val[cc];
        if (len < 32) break;
      }
      acc = warp_sum(acc);
      if (lane == 0) y[key] += load_scale(scale_p) * acc;
    }
  }
}

// -------------------------------------------------------------------------
// TMA-staged merge-path kernel: one elected thread moves the tile's values,
// column indices and row ends into shared memory with three bulk copies
// (L2 evict_first: each byte is read once), all threads then form the
// products with L2-evict_last gathers of x (up to 8 independent gathers in
// flight per thread), and the merge consumption runs out of shared memory.
// -------------------------------------------------------------------------
struct MergeTmaSmem {
  double vals[MP_TILE + 8];  // values, then products in place
  int32_t cols[MP_TILE + 8];
  int32_t rend[MP_TILE + 8];
  double yv[MP_TILE];
  KeyVal warp_kv[MP_THREADS / 32];
  uint64_t bar;
};

template <bool HAS_ELL>
__global__ void __launch_bounds__(MP_THREADS) k_spmv_merge_tma(
    int64_t n_rows, int64_t nnz, const int32_t* __restrict__ ptr, const int32_t* __restrict__ col,
    const double* __restrict__ val, const int32_t* __restrict__ tile_row, const int32_t* __restrict__ tile_nz,
    int32_t* __restrict__ carry_row, double* __restrict__ carry_val, const double* __restrict__ x,
    double* __restrict__ y, const double* __restrict__ scale_p, int64_t ell_k, const int32_t* __restrict__ ell_idx,
    const double* __restrict__ ell_val) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  MergeTmaSmem& sm = *reinterpret_cast<MergeTmaSmem*>(smem_raw);
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int c = blockIdx.x;
  const int r0 = tile_row[c], z0 = tile_nz[c];
  const int R = tile_row[c + 1] - r0, Z = tile_nz[c + 1] - z0;
  const int64_t rhi = static_cast<int64_t>(r0) + R + 2 < n_rows + 1 ? static_cast<int64_t>(r0) + R + 2 : n_rows + 1;
  const StageRange sv = plan_stage(z0, static_cast<int64_t>(z0) + Z, nnz, 8);
  const StageRange sc = plan_stage(z0, static_cast<int64_t>(z0) + Z, nnz, 4);
  const StageRange sr = plan_stage(static_cast<int64_t>(r0) + 1, rhi, n_rows + 1, 4);
  const uint32_t bytes = sv.bulk_bytes(8) + sc.bulk_bytes(4) + sr.bulk_bytes(4);
  if (tid == 0) {
    mbar_init(&sm.bar, 1);
    if (bytes) {
      const uint64_t pol = policy_evict_first();
      mbar_arrive_expect_tx(&sm.bar, bytes);
      if (sv.bulk_bytes(8)) bulk_g2s(sm.vals, val + sv.base, sv.bulk_bytes(8), &sm.bar, pol);
      if (sc.bulk_bytes(4)) bulk_g2s(sm.cols, col + sc.base, sc.bulk_bytes(4), &sm.bar, pol);
      if (sr.bulk_bytes(4)) bulk_g2s(sm.rend, ptr + sr.base, sr.bulk_bytes(4), &sm.bar, pol);
    }
  }
  // unaligned tails at the very end of the arrays, and the end sentinel
  for (int64_t e = (sv.bulk_hi > z0 ? sv.bulk_hi : z0) + tid; e < sv.hi; e += MP_THREADS)
    sm.vals[e - sv.base] = val[e];
  for (int64_t e = (sc.bulk_hi > z0 ? sc.bulk_hi : z0) + tid; e < sc.hi; e += MP_THREADS)
    sm.cols[e - sc.base] = col[e];
  for (int64_t e = (sr.bulk_hi > r0 + 1 ? sr.bulk_hi : r0 + 1) + tid; e < sr.hi; e += MP_THREADS)
    sm.rend[e - sr.base] = ptr[e];
  if (tid == 0 && static_cast<int64_t>(r0) + R + 1 > n_rows) sm.rend[static_cast<int64_t>(r0) + R + 1 - sr.base] = INT32_MAX;
  __syncthreads();  // barrier init + tails visible
  if (bytes) mbar_wait(&sm.bar, 0);

  const int dv = static_cast<int>(z0 - sv.base), dc = static_cast<int>(z0 - sc.base);
  const int dr = static_cast<int>(static_cast<int64_t>(r0) + 1 - sr.base);
  {
    const uint64_t pol_x = policy_evict_last();
    double p[MP_IPT];
#pragma unroll
    for (int it = 0; it < MP_IPT; ++it) {
      const int j = tid + it * MP_THREADS;
      p[it] = j < Z ? ld_hint(x + sm.cols[j + dc], pol_x) : 0.0;
    }
#pragma unroll
    for (int it = 0; it < MP_IPT; ++it) {
      const int j = tid + it * MP_THREADS;
      if (j < Z) sm.vals[j + dv] *= p[it];
    }
  }
  __syncthreads();

  const int items = R + Z;
  int td = tid * MP_IPT;
  if (td > items) td = items;
  int lo = td - Z > 0 ? td - Z : 0;
  int hi = td < R ? td : R;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (sm.rend[mid + dr] <= z0 + td - mid - 1) lo = mid + 1; else hi = mid;
  }
  int row = lo, nz = td - lo;
  double running = 0.0;
  int first_row = -1;
#pragma unroll
  for (int it = 0; it < MP_IPT; ++it) {
    if (td + it < items) {
      if (z0 + nz < sm.rend[row + dr]) {
        running += sm.vals[nz + dv];
        ++nz;
      } else {
        sm.yv[row] = running;
        if (first_row < 0) first_row = row;
        running = 0.0;
        ++row;
      }
    }
  }
  KeyVal inc{row, running};
  ReduceByKeyOp op;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    KeyVal o = shfl_up_kv(inc, d);
    if (lane >= d) inc = op(o, inc);
  }
  if (lane == 31) sm.warp_kv[warp] = inc;
  __syncthreads();
  KeyVal excl = shfl_up_kv(inc, 1);
  KeyVal wprefix{-1, 0.0};
  for (int w = 0; w < warp; ++w) wprefix = (w == 0) ? sm.warp_kv[0] : op(wprefix, sm.warp_kv[w]);
  KeyVal prefix = (lane == 0) ? wprefix : ((warp == 0) ? excl : op(wprefix, excl));
  if (tid == 0) prefix = KeyVal{-1, 0.0};
  if (first_row >= 0 && prefix.key == first_row) sm.yv[first_row] += prefix.val;
  if (tid == MP_THREADS - 1) {
    KeyVal total = (warp == 0) ? inc : op(wprefix, inc);
    int64_t gr = static_cast<int64_t>(r0) + total.key;
    carry_row[c] = gr < n_rows ? static_cast<int32_t>(gr) : -1;
    carry_val[c] = total.val;
  }
  __syncthreads();
  const double s = load_scale(scale_p);
  for (int i = tid; i < R; i += MP_THREADS) {
    int64_t r = static_cast<int64_t>(r0) + i;
    double v = sm.yv[i];
    if (HAS_ELL) {
      double e = 0.0;
      for (int64_t j = 0; j < ell_k; ++j) {
        int64_t o = j * n_rows + r;
        e = __dadd_rn(e, __dmul_rn(ld_stream(ell_val + o), ldx(x, ld_stream(ell_idx + o))));
      }
      v = e + v;
    }
    y[r] = s * v;
  }
}


void launch_merge_plain(int64_t n_rows, int64_t nnz, const int32_t* ptr, const int32_t* col, const double* val,
                        const int32_t* tile_row, const int32_t* tile_nz, int32_t* carry_row, double* carry_val,
                        const double* x, double* y, const double* scale, int64_t ell_k, const int32_t* ell_idx,
                        const double* ell_val, cudaStream_t s);

void launch_merge(int64_t n_rows, int64_t nnz, const int32_t* ptr, const int32_t* col, const double* val,
                  const int32_t* tile_row, const int32_t* tile_nz, int32_t* carry_row, double* carry_val,
                  const double* x, double* y, const double* scale, int64_t ell_k, const int32_t* ell_idx,
                  const double* ell_val, cudaStream_t s) {
  if (n_rows <= 0) return;
  const int64_t tiles = (n_rows + nnz + MP_TILE - 1) / MP_TILE;
  // Kernel variant (experiments): SPMVB_MERGE_KERNEL=tma selects the
  // TMA-staged kernel, anything else the register-unrolled one.
  const char* variant = getenv("SPMVB_MERGE_KERNEL");
  const bool tma = variant && variant[0] == 't' && aligned16(ptr) && (nnz == 0 || (aligned16(col) && aligned16(val)));
  if (tma) {
    const size_t smem = sizeof(MergeTmaSmem);
    if (ell_k > 0) {
      SPMVB_CUDA(cudaFuncSetAttribute(k_spmv_merge_tma<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      k_spmv_merge_tma<true><<<static_cast<unsigned>(tiles), MP_THREADS, smem, s>>>(
          n_rows, nnz, ptr, col, val, tile_row, tile_nz, carry_row, carry_val, x, y, scale, ell_k, ell_idx, ell_val);
    } else {
      SPMVB_CUDA(cudaFuncSetAttribute(k_spmv_merge_tma<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      k_spmv_merge_tma<false><<<static_cast<unsigned>(tiles), MP_THREADS, smem, s>>>(
          n_rows, nnz, ptr, col, val, tile_row, tile_nz, carry_row, carry_val, x, y, scale, 0, nullptr, nullptr);
    }
    SPMVB_LAUNCHED("k_spmv_merge_tma");
  } else {
    launch_merge_plain(n_rows, nnz, ptr, col, val, tile_row, tile_nz, carry_row, carry_val, x, y, scale, ell_k,
                       ell_idx, ell_val, s);
  }
  if (tiles > 1) {
    k_merge_fixup<<<grid_for(tiles, 256, 148 * 8), 256, 0, s>>>(tiles, carry_row, carry_val, y, scale);
    SPMVB_LAUNCHED("k_merge_fixup");
  }
}

void launch_merge_plain(int64_t n_rows, int64_t nnz, const int32_t* ptr, const int32_t* col, const double* val,
                        const int32_t* tile_row, const int32_t* tile_nz, int32_t* carry_row, double* carry_val,
                        const double* x, double* y, const double* scale, int64_t ell_k, const int32_t* ell_idx,
                        const double* ell_val, cudaStream_t s) {
  const int64_t tiles = (n_rows + nnz + MP_TILE - 1) / MP_TILE;
  const size_t smem = sizeof(MergeSmem);
  if (ell_k > 0) {
    SPMVB_CUDA(cudaFuncSetAttribute(k_spmv_merge<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_spmv_merge<true><<<static_cast<unsigned>(tiles), MP_THREADS, smem, s>>>(
        n_rows, nnz, ptr, col, val, tile_row, tile_nz, carry_row, carry_val, x, y, scale, ell_k, ell_idx, ell_val);
  } else {
    SPMVB_CUDA(cudaFuncSetAttribute(k_spmv_merge<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_spmv_merge<false><<<static_cast<unsigned>(tiles), MP_THREADS, smem, s>>>(
        n_rows, nnz, ptr, col, val, tile_row, tile_nz, carry_row, carry_val, x, y, scale, 0, nullptr, nullptr);
  }
  SPMVB_LAUNCHED("k_spmv_merge");
}

}  // namespace

extern "C" int64_t spmvb_csr_merge_tiles(int64_t n_rows, int64_t nnz) {
  if (n_rows <= 0) return 0;
  return (n_rows + nnz + MP_TILE - 1) / MP_TILE;
}

extern "C" int spmvb_csr_merge_plan(int64_t n_rows, int64_t nnz, const int32_t* ptr, int32_t* tile_row,
                                    int32_t* tile_nz, void* stream) {
  return guard([&] {
    cudaStream_t s = as_stream(stream);
    int64_t tiles = spmvb_csr_merge_tiles(n_rows, nnz);
    if (tiles == 0) return;
    if (n_rows + nnz > INT32_MAX) fail(SPMVB_INVALID_ARG, "n_rows + nnz exceeds the int32 merge-path range");
    k_merge_plan<<<grid_for(tiles + 1, 256, 148 * 16), 256, 0, s>>>(n_rows, nnz, ptr, tiles, tile_row, tile_nz);
    SPMVB_LAUNCHED("k_merge_plan");
  });
}

extern "C" int spmvb_spmv_csr(int64_t n_rows, int64_t nnz, const int32_t* ptr, const int32_t* col, const double* val,
                              const int32_t* tile_row, const int32_t* tile_nz, int32_t* carry_row,
                              double* carry_val, const double* x, double* y, const double* scale, void* stream) {
  return guard([&] {
    launch_merge(n_rows, nnz, ptr, col, val, tile_row, tile_nz, carry_row, carry_val, x, y, scale, 0, nullptr,
                 nullptr, as_stream(stream));
  });
}

extern "C" int spmvb_spmv_hyb(int64_t n_rows, int64_t k, const int32_t* ell_idx, const double* ell_val,
                              int64_t tail_nnz, const int32_t* tail_ptr, const int32_t* tail_col,
                              const double* tail_val, const int32_t* tile_row, const int32_t* tile_nz,
                              int32_t* carry_row, double* carry_val, const double* x, double* y, const double* scale,
                              void* stream) {
  return guard([&] {
    launch_merge(n_rows, tail_nnz, tail_ptr, tail_col, tail_val, tile_row, tile_nz, carry_row, carry_val, x, y,
                 scale, k, ell_idx, ell_val, as_stream(stream));
  });
}

