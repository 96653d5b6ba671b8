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
  for (int i = tid; i <= R; i += MP_THREADS) {
    int64_t r = static_cast<int64_t>(r0) + i;
    sm.row_end[i] = r < n_rows ? ptr[r + 1] : INT32_MAX;
  }
  for (int j = tid; j < Z; j += MP_THREADS) {
    int64_t k = static_cast<int64_t>(z0) + j;
    sm.prod[j] = ld_stream(val + k) * ldx(x, ld_stream(col + k));
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

// Adds each chain of tile carry-outs (ascending tile order) to its row.
__global__ void k_merge_fixup(int64_t num_tiles, const int32_t* __restrict__ carry_row,
                              const double* __restrict__ carry_val, double* __restrict__ y,
                              const double* __restrict__ scale_p) {
  for (int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; c < num_tiles;
       c += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int32_t r = carry_row[c];
    if (r < 0) continue;
    if (c > 0 && carry_row[c - 1] == r) continue;  // not the chain start
    double acc = carry_val[c];
    for (int64_t c2 = c + 1; c2 < num_tiles && carry_row[c2] == r; ++c2) acc += carry_val[c2];
    y[r] += load_scale(scale_p) * acc;
  }
}

void launch_merge(int64_t n_rows, int64_t nnz, const int32_t* ptr, const int32_t* col, const double* val,
                  const int32_t* tile_row, const int32_t* tile_nz, int32_t* carry_row, double* carry_val,
                  const double* x, double* y, const double* scale, int64_t ell_k, const int32_t* ell_idx,
                  const double* ell_val, cudaStream_t s) {
  if (n_rows <= 0) return;
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
  if (tiles > 1) {
    k_merge_fixup<<<grid_for(tiles, 256, 148 * 8), 256, 0, s>>>(tiles, carry_row, carry_val, y, scale);
    SPMVB_LAUNCHED("k_merge_fixup");
  }
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

__global__ void k_csr5_fixup(int64_t num_tiles, const int32_t* __restrict__ tile_ptr, const uint32_t* __restrict__ aux,
                             const double* __restrict__ carry, double* __restrict__ y) {
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < num_tiles;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (!(aux[t] & 0x80000000u)) continue;
    const int32_t r = tile_ptr[t];
    if (t > 0 && (aux[t - 1] & 0x80000000u) && tile_ptr[t - 1] == r) continue;  // not the chain start
    double acc = y[r];
    for (int64_t t2 = t; t2 < num_tiles && (aux[t2] & 0x80000000u) && tile_ptr[t2] == r; ++t2) acc += carry[t2];
    y[r] = acc;
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
    if (sigma <= 1024 && full > 0) {
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
