// fp64 SpMV kernels, one per storage format (reference kernels.py:76-219).
//
// All kernels are deterministic: no floating-point atomics; partial sums of
// rows that cross work units (CSR merge tiles, CSR5 tiles, HYB tail tiles)
// are folded by a fix-up kernel in ascending tile order, mirroring the
// reference's ascending-task fold (kernels.py:5-9, 172-173, 197-198).
// ELL and SELL accumulate each row sequentially over all slots with
// separately rounded products, which is bit-identical to the reference
// kernels (kernels.py:101-104, 122-125).
#include "prims.cuh"
#include "tma.cuh"

using namespace spmvb;

namespace {

__device__ __forceinline__ double ldx(const double* __restrict__ x, int32_t j) { return __ldg(x + j); }

__device__ __forceinline__ double load_scale(const double* scale) { return scale ? *scale : 1.0; }

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

// Butterfly sum: every lane gets the same, order-fixed result.
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
  return v;
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

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

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

// =========================================================================
// CSR5.  Segment ordinal s inside tile t maps to the g-th non-empty row with
// g = rank(tile_ptr[t]) + s (tile_aux bits 0-30); bit 31 marks a tile whose
// head continues a row begun earlier: that first segment is a carry.
// Writing the start segment of non-empty row g also zero-fills the empty
// rows between non-empty rows g-1 and g (and after the last one).
// =========================================================================
struct Csr5Ctx {
  int64_t n_rows, nnz, n_nonempty;
  int omega, sigma;
  const int32_t* tile_ptr;
  const uint8_t* bit_flag;
  const int32_t* col;
  const double* val;
  const uint32_t* aux;
  const int32_t* nonempty;
  double* carry;
  const double* x;
  double* y;
  const double* scale_p;
};

__device__ __forceinline__ int64_t csr5_row_of(const Csr5Ctx& C, int64_t g) {
  return C.nonempty ? static_cast<int64_t>(C.nonempty[g]) : g;
}

__device__ __forceinline__ void csr5_emit(const Csr5Ctx& C, double sc, int64_t t, uint32_t aux, int64_t s, double v) {
  const bool cont = (aux & 0x80000000u) != 0;
  if (s == 0 && cont) {
    C.carry[t] = sc * v;
    return;
  }
  const int64_t g = static_cast<int64_t>(aux & 0x7fffffffu) + s;
  const int64_t r = csr5_row_of(C, g);
  C.y[r] = sc * v;
  if (C.nonempty) {
    const int64_t prev = g > 0 ? csr5_row_of(C, g - 1) : -1;
    for (int64_t z = prev + 1; z < r; ++z) C.y[z] = 0.0;
    if (g == C.n_nonempty - 1)
      for (int64_t z = r + 1; z < C.n_rows; ++z) C.y[z] = 0.0;
  }
}

// Generic: one thread per tile, CSR order recovered from the stored layout.
__global__ void k_csr5_generic(Csr5Ctx C, int64_t t_begin, int64_t t_end) {
  const int64_t tile = static_cast<int64_t>(C.omega) * C.sigma;
  const double sc = load_scale(C.scale_p);
  for (int64_t t = t_begin + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < t_end;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t base = t * tile;
    const int64_t m = C.nnz - base < tile ? C.nnz - base : tile;
    const int64_t q = m / C.sigma, rem = m % C.sigma;
    const uint32_t aux = C.aux[t];
    int64_t seg = -1;
    double sum = 0.0;
    for (int64_t p = 0; p < m; ++p) {
      const int64_t gi = p % C.sigma, gj = p / C.sigma;
      const int64_t pos = base + gi * q + (gi < rem ? gi : rem) + gj;
      if (C.bit_flag[pos]) {
        if (seg >= 0) csr5_emit(C, sc, t, aux, seg, sum);
        ++seg;
        sum = 0.0;
      }
      sum += C.val[pos] * ldx(C.x, C.col[pos]);
    }
    if (seg >= 0) csr5_emit(C, sc, t, aux, seg, sum);
  }
}

// Fast path: W lanes per full tile (omega == W), lane j owns tile column j
// (sigma consecutive CSR-order entries stored at base + i*W + j).
template <int W>
__global__ void __launch_bounds__(256) k_csr5_warp(Csr5Ctx C, int64_t full_tiles) {
  const int lane = threadIdx.x & 31;
  const int j = lane % W;
  const int64_t group = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) / W;
  const bool active = group < full_tiles;
  const int64_t t = active ? group : 0;
  const int sigma = C.sigma;
  const int64_t base = t * static_cast<int64_t>(W) * sigma;
  const uint32_t aux = active ? C.aux[t] : 0u;
  const double sc = load_scale(C.scale_p);

  double head = 0.0, sum = 0.0;
  int nflags = 0;
  // First pass: count this lane's flags so segment ordinals are known while
  // streaming; flags are 1 byte/entry and re-read from L1.
  for (int i = 0; i < sigma && active; ++i) nflags += C.bit_flag[base + static_cast<int64_t>(i) * W + j] ? 1 : 0;
  // Exclusive prefix of flag counts across the group's lanes.
  int incl = nflags;
#pragma unroll
  for (int d = 1; d < W; d <<= 1) {
    int o = __shfl_up_sync(0xffffffffu, incl, d, W);
    if (j >= d) incl += o;
  }
  const int seg_base = incl - nflags;
  int seen = 0;
  if (active) {
    for (int i = 0; i < sigma; ++i) {
      const int64_t pos = base + static_cast<int64_t>(i) * W + j;
      const bool f = C.bit_flag[pos] != 0;
      const double v = ld_stream(C.val + pos) * ldx(C.x, ld_stream(C.col + pos));
      if (f) {
        if (seen == 0) head = sum;
        else csr5_emit(C, sc, t, aux, seg_base + seen - 1, sum);
        ++seen;
        sum = 0.0;
      }
      sum += v;
    }
  }
  const bool F = seen > 0;
  if (!F) head = sum;
  // R_j = H_j + (F_j ? 0 : R_{j+1}): segmented suffix sum of heads.
  double rv = head;
  bool stop = F;
#pragma unroll
  for (int d = 1; d < W; d <<= 1) {
    double ov = __shfl_down_sync(0xffffffffu, rv, d, W);
    bool ostop = __shfl_down_sync(0xffffffffu, stop ? 1 : 0, d, W) != 0;
    if (!stop && j + d < W) {
      rv += ov;
      stop = ostop;
    }
  }
  double right = __shfl_down_sync(0xffffffffu, rv, 1, W);
  if (j == W - 1) right = 0.0;
  if (active && F) csr5_emit(C, sc, t, aux, seg_base + seen - 1, sum + right);
}

// Same algorithm with a compile-time sigma: each lane issues its S flag,
// column and value loads back to back, then S independent x gathers, so a
// warp keeps 32*S gathers in flight (random-column matrices are bound by the
// L1TEX wavefront rate of these gathers, ~2 cycles per distinct line).
template <int W, int S, bool PARTIAL>
__global__ void __launch_bounds__(256) k_csr5_warp_s(Csr5Ctx C, int64_t t_begin, int64_t t_end) {
  const int lane = threadIdx.x & 31;
  const int j = lane % W;
  const int64_t group = t_begin + (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) / W;
  const bool active = group < t_end;
  const int64_t t = active ? group : t_begin;
  const int64_t tile0 = t * static_cast<int64_t>(W) * S;
  const double sc = load_scale(C.scale_p);
  uint32_t fmask = 0;
  int32_t cidx[S];
  double v[S];
  if (!PARTIAL) {
    const int64_t base = tile0 + j;
    if (active) {
#pragma unroll
      for (int i = 0; i < S; ++i) {
        fmask |= (C.bit_flag[base + i * W] ? 1u : 0u) << i;
        cidx[i] = ld_stream(C.col + base + i * W);
        v[i] = ld_stream(C.val + base + i * W);
      }
#pragma unroll
      for (int i = 0; i < S; ++i) v[i] *= ldx(C.x, cidx[i]);
    }
  } else {
    // trailing partial tile: row-major over occupied cells (formats.py:24-25)
    const int64_t m = C.nnz - tile0;
    const int q = static_cast<int>(m / S), rem = static_cast<int>(m % S);
#pragma unroll
    for (int i = 0; i < S; ++i) {
      const bool ok = active && static_cast<int64_t>(j) * S + i < m;
      const int64_t pos = tile0 + static_cast<int64_t>(i) * q + (i < rem ? i : rem) + j;
      fmask |= (ok && C.bit_flag[pos] ? 1u : 0u) << i;
      v[i] = ok ? C.val[pos] * ldx(C.x, C.col[pos]) : 0.0;
    }
  }
  const uint32_t aux = active ? C.aux[t] : 0u;
  const int nflags = __popc(fmask);
  int incl = nflags;
#pragma unroll
  for (int d = 1; d < W; d <<= 1) {
    int o = __shfl_up_sync(0xffffffffu, incl, d, W);
    if (j >= d) incl += o;
  }
  const int seg_base = incl - nflags;
  double head = 0.0, sum = 0.0;
  int seen = 0;
  if (active) {
#pragma unroll
    for (int i = 0; i < S; ++i) {
      if ((fmask >> i) & 1u) {
        if (seen == 0) head = sum;
        else csr5_emit(C, sc, t, aux, seg_base + seen - 1, sum);
        ++seen;
        sum = 0.0;
      }
      sum += v[i];
    }
  }
  const bool F = seen > 0;
  if (!F) head = sum;
  double rv = head;
  bool stop = F;
#pragma unroll
  for (int d = 1; d < W; d <<= 1) {
    double ov = __shfl_down_sync(0xffffffffu, rv, d, W);
    bool ostop = __shfl_down_sync(0xffffffffu, stop ? 1 : 0, d, W) != 0;
    if (!stop && j + d < W) {
      rv += ov;
      stop = ostop;
    }
  }
  double right = __shfl_down_sync(0xffffffffu, rv, 1, W);
  if (j == W - 1) right = 0.0;
  if (active && F) csr5_emit(C, sc, t, aux, seg_base + seen - 1, sum + right);
}

// TMA-staged fast path for omega == 32, sigma <= 16: a CTA of 8 warps owns 8
// consecutive full tiles, which are contiguous in stored order, so three bulk
// copies (values, columns, flags; L2 evict_first) stage them; products are
// formed CTA-wide with 16 independent x gathers per thread (L2 evict_last);
// each warp then runs the column-segmented sum of one tile from shared memory.
constexpr int C5_TPB = 8;
constexpr int C5_MAX_ENTRIES = C5_TPB * 32 * 16;

struct Csr5TmaSmem {
  double vals[C5_MAX_ENTRIES];
  int32_t cols[C5_MAX_ENTRIES];
  uint8_t flags[C5_MAX_ENTRIES];
  uint64_t bar;
};

__global__ void __launch_bounds__(256) k_csr5_tma(Csr5Ctx C, int64_t full_tiles) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Csr5TmaSmem& sm = *reinterpret_cast<Csr5TmaSmem*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int sigma = C.sigma;
  const int tile = 32 * sigma;
  const int64_t t0 = static_cast<int64_t>(blockIdx.x) * C5_TPB;
  const int ntile = full_tiles - t0 < C5_TPB ? static_cast<int>(full_tiles - t0) : C5_TPB;
  const int cnt = ntile * tile;
  const int64_t e0 = t0 * tile;
  if (tid == 0) {
    mbar_init(&sm.bar, 1);
    const uint64_t pol = policy_evict_first();
    mbar_arrive_expect_tx(&sm.bar, static_cast<uint32_t>(cnt) * 13u);
    bulk_g2s(sm.vals, C.val + e0, cnt * 8u, &sm.bar, pol);
    bulk_g2s(sm.cols, C.col + e0, cnt * 4u, &sm.bar, pol);
    bulk_g2s(sm.flags, C.bit_flag + e0, static_cast<uint32_t>(cnt), &sm.bar, pol);
  }
  __syncthreads();
  mbar_wait(&sm.bar, 0);
  {
    const uint64_t pol_x = policy_evict_last();
    constexpr int PER = C5_MAX_ENTRIES / 256;
    double p[PER];
#pragma unroll
    for (int it = 0; it < PER; ++it) {
      const int e = tid + it * 256;
      p[it] = e < cnt ? ld_hint(C.x + sm.cols[e], pol_x) : 0.0;
    }
#pragma unroll
    for (int it = 0; it < PER; ++it) {
      const int e = tid + it * 256;
      if (e < cnt) sm.vals[e] *= p[it];
    }
  }
  __syncthreads();
  if (warp >= ntile) return;  // whole warps only: shuffles below stay full-mask
  const int64_t t = t0 + warp;
  const uint32_t aux = C.aux[t];
  const double sc = load_scale(C.scale_p);
  const int base = warp * tile;
  int nflags = 0;
  for (int i = 0; i < sigma; ++i) nflags += sm.flags[base + i * 32 + lane] ? 1 : 0;
  int incl = nflags;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    int o = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += o;
  }
  const int seg_base = incl - nflags;
  double head = 0.0, sum = 0.0;
  int seen = 0;
  for (int i = 0; i < sigma; ++i) {
    const int idx = base + i * 32 + lane;
    if (sm.flags[idx]) {
      if (seen == 0) head = sum;
      else csr5_emit(C, sc, t, aux, seg_base + seen - 1, sum);
      ++seen;
      sum = 0.0;
    }
    sum += sm.vals[idx];
  }
  const bool F = seen > 0;
  if (!F) head = sum;
  double rv = head;
  bool stop = F;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    double ov = __shfl_down_sync(0xffffffffu, rv, d);
    bool ostop = __shfl_down_sync(0xffffffffu, stop ? 1 : 0, d) != 0;
    if (!stop && lane + d < 32) {
      rv += ov;
      stop = ostop;
    }
  }
  double right = __shfl_down_sync(0xffffffffu, rv, 1);
  if (lane == 31) right = 0.0;
  if (F) csr5_emit(C, sc, t, aux, seg_base + seen - 1, sum + right);
}

__global__ void k_csr5_fixup(int64_t num_tiles, const int32_t* __restrict__ tile_ptr, const uint32_t* __restrict__ aux,
                             const double* __restrict__ carry, double* __restrict__ y) {
  // chains of continuation tiles, folded warp-cooperatively as in k_merge_fixup
  const int lane = threadIdx.x & 31;
  const int64_t warp_id = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t w0 = warp_id * 32; w0 < num_tiles; w0 += nwarps * 32) {
    const int64_t t = w0 + lane;
    const bool cont = t < num_tiles && (aux[t] & 0x80000000u);
    const int32_t r = cont ? tile_ptr[t] : -1;
    const bool start = cont && !(t > 0 && (aux[t - 1] & 0x80000000u) && tile_ptr[t - 1] == r);
    unsigned starts = __ballot_sync(0xffffffffu, start);
    while (starts) {
      const int l = __ffs(starts) - 1;
      starts &= starts - 1;
      const int32_t key = __shfl_sync(0xffffffffu, r, l);
      double acc = 0.0;
      for (int64_t b = w0 + l;; b += 32) {
        const int64_t tt = b + lane;
        const bool in = tt < num_tiles && (aux[tt] & 0x80000000u) && tile_ptr[tt] == key;
        const unsigned m = __ballot_sync(0xffffffffu, in);
        const int len = (m == 0xffffffffu) ? 32 : __ffs(~m) - 1;
        if (lane < len) acc += carry[tt];
        if (len < 32) break;
      }
      acc = warp_sum(acc);
      if (lane == 0) y[key] = y[key] + acc;
    }
  }
}

// ================================================================ ELL ====
__global__ void k_spmv_ell(int64_t n_rows, int64_t k, const int32_t* __restrict__ idx, const double* __restrict__ val,
                           const double* __restrict__ x, double* __restrict__ y, const double* __restrict__ scale_p) {
  const double s = load_scale(scale_p);
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < n_rows;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double acc = 0.0;
    int64_t j = 0;
    for (; j + 4 <= k; j += 4) {
      const int64_t o = j * n_rows + r;
      const double v0 = ld_stream(val + o), v1 = ld_stream(val + o + n_rows);
      const double v2 = ld_stream(val + o + 2 * n_rows), v3 = ld_stream(val + o + 3 * n_rows);
      const int32_t c0 = ld_stream(idx + o), c1 = ld_stream(idx + o + n_rows);
      const int32_t c2 = ld_stream(idx + o + 2 * n_rows), c3 = ld_stream(idx + o + 3 * n_rows);
      acc = __dadd_rn(acc, __dmul_rn(v0, ldx(x, c0)));
      acc = __dadd_rn(acc, __dmul_rn(v1, ldx(x, c1)));
      acc = __dadd_rn(acc, __dmul_rn(v2, ldx(x, c2)));
      acc = __dadd_rn(acc, __dmul_rn(v3, ldx(x, c3)));
    }
    for (; j < k; ++j) {
      const int64_t o = j * n_rows + r;
      acc = __dadd_rn(acc, __dmul_rn(ld_stream(val + o), ldx(x, ld_stream(idx + o))));
    }
    y[r] = scale_p ? s * acc : acc;
  }
}

// =============================================================== SELL ====
__global__ void k_spmv_sell(int64_t n_rows, int64_t c, const int64_t* __restrict__ widths,
                            const int64_t* __restrict__ slice_off, const int32_t* __restrict__ perm,
                            const int32_t* __restrict__ idx, const double* __restrict__ val,
                            const double* __restrict__ x, double* __restrict__ y, const double* __restrict__ scale_p) {
  const double s = load_scale(scale_p);
  for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < n_rows;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t sl = p / c, local = p - sl * c;
    const int64_t rows_s = (sl + 1) * c <= n_rows ? c : n_rows - sl * c;
    const int64_t w = widths[sl];
    const int64_t o0 = slice_off[sl] + local;
    double acc = 0.0;
    int64_t j = 0;
    for (; j + 4 <= w; j += 4) {
      const int64_t o = o0 + j * rows_s;
      const double v0 = ld_stream(val + o), v1 = ld_stream(val + o + rows_s);
      const double v2 = ld_stream(val + o + 2 * rows_s), v3 = ld_stream(val + o + 3 * rows_s);
      const int32_t c0 = ld_stream(idx + o), c1 = ld_stream(idx + o + rows_s);
      const int32_t c2 = ld_stream(idx + o + 2 * rows_s), c3 = ld_stream(idx + o + 3 * rows_s);
      acc = __dadd_rn(acc, __dmul_rn(v0, ldx(x, c0)));
      acc = __dadd_rn(acc, __dmul_rn(v1, ldx(x, c1)));
      acc = __dadd_rn(acc, __dmul_rn(v2, ldx(x, c2)));
      acc = __dadd_rn(acc, __dmul_rn(v3, ldx(x, c3)));
    }
    for (; j < w; ++j) {
      const int64_t o = o0 + j * rows_s;
      acc = __dadd_rn(acc, __dmul_rn(ld_stream(val + o), ldx(x, ld_stream(idx + o))));
    }
    const int64_t r = perm ? static_cast<int64_t>(perm[p]) : p;
    y[r] = scale_p ? s * acc : acc;
  }
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

extern "C" int spmvb_spmv_csr5(int64_t n_rows, int64_t nnz, int omega, int sigma, const int32_t* tile_ptr,
                               const uint8_t* bit_flag, const int32_t* col, const double* val, const uint32_t* tile_aux,
                               const int32_t* nonempty_rows, int64_t n_nonempty, double* carry, const double* x,
                               double* y, const double* scale, void* stream) {
  return guard([&] {
    cudaStream_t s = as_stream(stream);
    if (n_rows <= 0) return;
    if (nnz == 0) {
      SPMVB_CUDA(cudaMemsetAsync(y, 0, n_rows * sizeof(double), s));
      return;
    }
    if (omega < 1 || sigma < 1) fail(SPMVB_INVALID_ARG, "omega and sigma must be >= 1");
    Csr5Ctx C{n_rows, nnz, n_nonempty, omega, sigma, tile_ptr, bit_flag, col, val, tile_aux,
              nonempty_rows, carry, x, y, scale};
    const int64_t tile = static_cast<int64_t>(omega) * sigma;
    const int64_t num_tiles = (nnz + tile - 1) / tile;
    const int64_t full = nnz / tile;
    int64_t generic_begin = 0;
    auto warp_launch = [&](auto kern, int W) {
      int64_t threads = full * W;
      kern<<<grid_for(threads, 256), 256, 0, s>>>(C, full);
      SPMVB_LAUNCHED("k_csr5_warp");
      generic_begin = full;
    };
    const bool tma_ok = omega == 32 && sigma <= 16 && aligned16(val) && aligned16(col) && aligned16(bit_flag);
    // Kernel variant (experiments): SPMVB_CSR5_KERNEL=tma selects the
    // TMA-staged kernel; the default is the register-unrolled warp kernel.
    const char* variant = getenv("SPMVB_CSR5_KERNEL");
    const bool want_tma = variant && variant[0] == 't';
    auto warp_s_launch = [&](auto kern, auto kern_partial, int W) {  // full tiles, then the partial one
      if (full > 0) {
        kern<<<grid_for(full * W, 256), 256, 0, s>>>(C, 0, full);
        SPMVB_LAUNCHED("k_csr5_warp_s");
      }
      if (num_tiles > full) {
        kern_partial<<<1, 32, 0, s>>>(C, full, num_tiles);
        SPMVB_LAUNCHED("k_csr5_warp_s_partial");
      }
      generic_begin = num_tiles;
    };
    if (!want_tma && (sigma == 16 || sigma == 8) &&
        (omega == 32 || omega == 16 || omega == 8 || omega == 4)) {
      if (sigma == 16) {
        switch (omega) {
          case 32: warp_s_launch(k_csr5_warp_s<32, 16, false>, k_csr5_warp_s<32, 16, true>, 32); break;
          case 16: warp_s_launch(k_csr5_warp_s<16, 16, false>, k_csr5_warp_s<16, 16, true>, 16); break;
          case 8: warp_s_launch(k_csr5_warp_s<8, 16, false>, k_csr5_warp_s<8, 16, true>, 8); break;
          default: warp_s_launch(k_csr5_warp_s<4, 16, false>, k_csr5_warp_s<4, 16, true>, 4); break;
        }
      } else {
        switch (omega) {
          case 32: warp_s_launch(k_csr5_warp_s<32, 8, false>, k_csr5_warp_s<32, 8, true>, 32); break;
          case 16: warp_s_launch(k_csr5_warp_s<16, 8, false>, k_csr5_warp_s<16, 8, true>, 16); break;
          case 8: warp_s_launch(k_csr5_warp_s<8, 8, false>, k_csr5_warp_s<8, 8, true>, 8); break;
          default: warp_s_launch(k_csr5_warp_s<4, 8, false>, k_csr5_warp_s<4, 8, true>, 4); break;
        }
      }
    } else if (want_tma && tma_ok && full > 0) {
      const size_t smem = sizeof(Csr5TmaSmem);
      SPMVB_CUDA(cudaFuncSetAttribute(k_csr5_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      k_csr5_tma<<<static_cast<unsigned>((full + C5_TPB - 1) / C5_TPB), 256, smem, s>>>(C, full);
      SPMVB_LAUNCHED("k_csr5_tma");
      generic_begin = full;
    } else if (sigma <= 1024 && full > 0) {
      switch (omega) {
        case 32: warp_launch(k_csr5_warp<32>, 32); break;
        case 16: warp_launch(k_csr5_warp<16>, 16); break;
        case 8: warp_launch(k_csr5_warp<8>, 8); break;
        case 4: warp_launch(k_csr5_warp<4>, 4); break;
        case 2: warp_launch(k_csr5_warp<2>, 2); break;
        default: break;
      }
    }
    if (generic_begin < num_tiles) {
      k_csr5_generic<<<grid_for(num_tiles - generic_begin, 128, 148 * 64), 128, 0, s>>>(C, generic_begin, num_tiles);
      SPMVB_LAUNCHED("k_csr5_generic");
    }
    if (num_tiles > 1) {
      k_csr5_fixup<<<grid_for(num_tiles, 256, 148 * 8), 256, 0, s>>>(num_tiles, tile_ptr, tile_aux, carry, y);
      SPMVB_LAUNCHED("k_csr5_fixup");
    }
  });
}

extern "C" int spmvb_spmv_ell(int64_t n_rows, int64_t k, const int32_t* idx, const double* val, const double* x,
                              double* y, const double* scale, void* stream) {
  return guard([&] {
    cudaStream_t s = as_stream(stream);
    if (n_rows <= 0) return;
    k_spmv_ell<<<grid_for(n_rows, 256), 256, 0, s>>>(n_rows, k, idx, val, x, y, scale);
    SPMVB_LAUNCHED("k_spmv_ell");
  });
}

extern "C" int spmvb_spmv_sell(int64_t n_rows, int64_t c, const int64_t* widths, const int64_t* slice_off,
                               const int32_t* perm, const int32_t* idx, const double* val, const double* x, double* y,
                               const double* scale, void* stream) {
  return guard([&] {
    cudaStream_t s = as_stream(stream);
    if (n_rows <= 0) return;
    k_spmv_sell<<<grid_for(n_rows, 256), 256, 0, s>>>(n_rows, c, widths, slice_off, perm, idx, val, x, y, scale);
    SPMVB_LAUNCHED("k_spmv_sell");
  });
}
