// CSR -> {CSR5, ELL, SELL(-C-sigma), HYB} conversions, bit-exact against the
// reference's integer arrays (/root/reference/pkg/src/spmvkit/formats.py).
//
// Layout contracts:
//  * CSR5 stored position of CSR entry k (tile t, p = k mod w*s, m = entries
//    in the tile, q = m / sigma, rem = m mod sigma, gi = p mod sigma,
//    gj = p / sigma): t*w*s + gi*q + min(gi, rem) + gj   (formats.py:204-209,
//    "row-major over occupied cells" for the trailing partial tile).
//  * ELL grid (r, j) stored column-major at j*n_rows + r (logical (n, k)
//    C-order view exposed by the Python layer).
//  * SELL slice s, local row l, column j at slice_off[s] + j*rows_s + l, i.e.
//    the concatenation of each slice's Fortran-order ravel (formats.py:326-341).
#include "prims.cuh"

using namespace spmvb;

namespace {

// ------------------------------------------------------------------ CSR5 --
__device__ __forceinline__ int64_t csr5_stored(int64_t k, int64_t tile, int64_t sigma, int64_t nnz) {
  int64_t t = k / tile;
  int64_t base = t * tile;
  int64_t p = k - base;
  int64_t m = nnz - base < tile ? nnz - base : tile;
  int64_t q = m / sigma, rem = m % sigma;
  int64_t gi = p % sigma, gj = p / sigma;
  return base + gi * q + (gi < rem ? gi : rem) + gj;
}

__global__ void k_mark_row_starts(const int32_t* __restrict__ ptr, int64_t n_rows, uint8_t* __restrict__ flags) {
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < n_rows;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int32_t a = ptr[r], b = ptr[r + 1];
    if (b > a) flags[a] = 1;
  }
}

__global__ void k_csr5_scatter(int64_t k0, int64_t nnz, int64_t tile, int64_t sigma,
                               const uint8_t* __restrict__ flags_csr, const int32_t* __restrict__ col,
                               const double* __restrict__ val, uint8_t* __restrict__ bit_flag,
                               int32_t* __restrict__ col_out, double* __restrict__ val_out) {
  for (int64_t k = k0 + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < nnz;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t s = csr5_stored(k, tile, sigma, nnz);
    bool head = (k % tile) == 0;
    bit_flag[s] = (flags_csr[k] || head) ? 1 : 0;
    col_out[s] = col[k];
    val_out[s] = val[k];
  }
}

// Full tiles (tile = omega*sigma <= CSR5_SMEM_TILE entries): `group`
// consecutive tiles (contiguous in memory) per block iteration, read in CSR
// order (coalesced), transposed to the stored order (sigma x omega grid,
// row-major; formats.py:204-209) in shared memory and written out
// coalesced.  32-bit in-tile arithmetic.
constexpr int CSR5_SMEM_TILE = 4096;
__global__ void __launch_bounds__(256) k_csr5_scatter_tiles(int64_t full_tiles, int tile, int group, int omega,
                                                            int sigma, const uint8_t* __restrict__ flags_csr,
                                                            const int32_t* __restrict__ col,
                                                            const double* __restrict__ val,
                                                            uint8_t* __restrict__ bit_flag,
                                                            int32_t* __restrict__ col_out,
                                                            double* __restrict__ val_out) {
  // stored slot st lives at st + st/32 (one pad word per 32: the transposed
  // writes of a warp then fall in distinct banks)
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int chunk = tile * group;
  const int padded = chunk + chunk / 32 + 1;
  double* sv = reinterpret_cast<double*>(smem_raw);
  int32_t* sc = reinterpret_cast<int32_t*>(sv + padded);
  uint8_t* sf = reinterpret_cast<uint8_t*>(sc + padded);
  const int64_t chunks = (full_tiles + group - 1) / group;
  for (int64_t ch = blockIdx.x; ch < chunks; ch += gridDim.x) {
    const int64_t base = ch * chunk;
    const int64_t tiles_here = full_tiles - ch * group < group ? full_tiles - ch * group : group;
    const int m = static_cast<int>(tiles_here) * tile;
    for (int q = threadIdx.x; q < m; q += blockDim.x) {
      const int tl = group > 1 ? q / tile : 0, p = q - tl * tile;
      const int gi = p % sigma, gj = p / sigma;
      const int st = tl * tile + gi * omega + gj;
      const int sp = st + (st >> 5);
      sv[sp] = val[base + q];
      sc[sp] = col[base + q];
      sf[sp] = (p == 0 || flags_csr[base + q]) ? 1 : 0;
    }
    __syncthreads();
    for (int q = threadIdx.x; q < m; q += blockDim.x) {
      const int sp = q + (q >> 5);
      val_out[base + q] = sv[sp];
      col_out[base + q] = sc[sp];
      bit_flag[base + q] = sf[sp];
    }
    __syncthreads();
  }
}

__global__ void k_csr5_tile_ptr(const int32_t* __restrict__ ptr, int64_t n_rows, int64_t num_tiles, int64_t tile,
                                int32_t* __restrict__ tile_ptr) {
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t <= num_tiles;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (t == num_tiles) {
      tile_ptr[t] = static_cast<int32_t>(n_rows);
      continue;
    }
    // upper_bound(ptr[0..n_rows], t*tile) - 1  (formats.py:191-193)
    int64_t v = t * tile;
    int64_t lo = 0, hi = n_rows + 1;
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (ptr[mid] <= v) lo = mid + 1; else hi = mid;
    }
    tile_ptr[t] = static_cast<int32_t>(lo - 1);
  }
}

// One thread per tile: y_off (flags in columns < j), seg_off (run of columns
// > j with an existing unflagged top), and the kernel's aux word.
__global__ void k_csr5_descriptor(int64_t nnz, int64_t num_tiles, int omega, int sigma,
                                  const uint8_t* __restrict__ flags_csr, const int32_t* __restrict__ ptr,
                                  const int32_t* __restrict__ tile_ptr, const int32_t* __restrict__ nz_rank,
                                  int32_t* __restrict__ y_off, int32_t* __restrict__ seg_off,
                                  uint32_t* __restrict__ tile_aux) {
  const int64_t tile = static_cast<int64_t>(omega) * sigma;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < num_tiles;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t base = t * tile;
    const int64_t m = nnz - base < tile ? nnz - base : tile;
    int32_t run = 0;
    for (int j = 0; j < omega; ++j) {
      y_off[t * omega + j] = run;
      int64_t lo = static_cast<int64_t>(j) * sigma;
      int64_t hi = lo + sigma < m ? lo + sigma : m;
      for (int64_t q = lo; q < hi; ++q) run += (flags_csr[base + q] || q == 0) ? 1 : 0;
    }
    int32_t spill = 0;
    for (int j = omega - 1; j >= 0; --j) {
      seg_off[t * omega + j] = spill;
      int64_t top = static_cast<int64_t>(j) * sigma;
      bool unflagged_top = top < m && !(flags_csr[base + top] || top == 0);
      spill = unflagged_top ? spill + 1 : 0;
    }
    int32_t r = tile_ptr[t];
    bool cont = ptr[r] < base;  // head entry continues a row that began earlier
    uint32_t rank = nz_rank ? static_cast<uint32_t>(nz_rank[r]) : static_cast<uint32_t>(r);
    tile_aux[t] = rank | (cont ? 0x80000000u : 0u);
  }
}

// omega <= 32: one warp per tile, lane j = tile column j (coalesced flag
// reads and descriptor writes; seg_off from a ballot of the unflagged tops).
__global__ void k_csr5_descriptor_warp(int64_t nnz, int64_t num_tiles, int omega, int sigma,
                                       const uint8_t* __restrict__ flags_csr, const int32_t* __restrict__ ptr,
                                       const int32_t* __restrict__ tile_ptr, const int32_t* __restrict__ nz_rank,
                                       int32_t* __restrict__ y_off, int32_t* __restrict__ seg_off,
                                       uint32_t* __restrict__ tile_aux) {
  const int lane = threadIdx.x & 31;
  const int64_t tile = static_cast<int64_t>(omega) * sigma;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t t = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5; t < num_tiles; t += nwarps) {
    const int64_t base = t * tile;
    const int64_t m = nnz - base < tile ? nnz - base : tile;
    const bool active = lane < omega;
    const int64_t lo = static_cast<int64_t>(lane) * sigma;
    const int64_t hi = lo + sigma < m ? lo + sigma : m;
    int32_t cnt = 0;
    if (active)
      for (int64_t q = lo; q < hi; ++q) cnt += (flags_csr[base + q] || q == 0) ? 1 : 0;
    int32_t incl = cnt;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int32_t o = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += o;
    }
    const bool unflagged_top = active && lo < m && !(flags_csr[base + lo] || lo == 0);
    const unsigned tops = __ballot_sync(0xffffffffu, unflagged_top);
    // columns lane+1, lane+2, ... with an unflagged top, up to the first one without
    const unsigned above = lane == 31 ? 0u : tops >> (lane + 1);
    const int32_t spill = (~above == 0u) ? 31 - lane : __ffs(~above) - 1;
    if (active) {
      y_off[t * omega + lane] = incl - cnt;
      seg_off[t * omega + lane] = spill;
    }
    if (lane == 0) {
      const int32_t r = tile_ptr[t];
      const bool cont = ptr[r] < base;  // head entry continues a row that began earlier
      const uint32_t rank = nz_rank ? static_cast<uint32_t>(nz_rank[r]) : static_cast<uint32_t>(r);
      tile_aux[t] = rank | (cont ? 0x80000000u : 0u);
    }
  }
}

// ------------------------------------------------------------------- ELL --
__global__ void k_ell_fill(int64_t n_rows, int64_t k, const int32_t* __restrict__ ptr,
                           const int32_t* __restrict__ col, const double* __restrict__ val, int32_t* __restrict__ idx_out,
                           double* __restrict__ val_out, int64_t* __restrict__ row_nnz) {
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < n_rows;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t a = ptr[r], b = ptr[r + 1];
    const int64_t cnt = b - a;
    const int32_t last = cnt ? col[b - 1] : 0;
    for (int64_t j = 0; j < k; ++j) {
      bool real = j < cnt;
      idx_out[j * n_rows + r] = real ? col[a + j] : last;
      val_out[j * n_rows + r] = real ? val[a + j] : 0.0;
    }
    if (row_nnz) row_nnz[r] = cnt;
  }
}

// ------------------------------------------------------------------ SELL --
__global__ void k_sell_keys(const int32_t* __restrict__ ptr, int64_t n_rows, int64_t sigma, int cbits,
                            uint64_t maxc, uint64_t* __restrict__ keys) {
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < n_rows;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    uint64_t cnt = static_cast<uint64_t>(ptr[r + 1] - ptr[r]);
    uint64_t w = static_cast<uint64_t>(r / sigma);
    keys[r] = (w << cbits) | (maxc - cnt);  // descending count inside each window
  }
}

__global__ void k_sell_perm(const uint32_t* __restrict__ sorted_rows, const int32_t* __restrict__ ptr, int64_t n_rows,
                            int32_t* __restrict__ perm, int64_t* __restrict__ row_nnz_perm) {
  for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < n_rows;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int32_t r = sorted_rows ? static_cast<int32_t>(sorted_rows[p]) : static_cast<int32_t>(p);
    perm[p] = r;
    row_nnz_perm[p] = ptr[r + 1] - ptr[r];
  }
}

__global__ void k_sell_widths(const int64_t* __restrict__ row_nnz_perm, int64_t n_rows, int64_t c, int64_t n_slices,
                              int64_t* __restrict__ widths) {
  for (int64_t s = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; s < n_slices;
       s += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t lo = s * c, hi = lo + c < n_rows ? lo + c : n_rows;
    int64_t w = 0;
    for (int64_t p = lo; p < hi; ++p) w = row_nnz_perm[p] > w ? row_nnz_perm[p] : w;
    widths[s] = w;
  }
}

// Thread per permuted row over its slice's column-major grid; rows of wide
// slices (the plan's wide list) are left to k_sell_fill_wide.
__global__ void k_sell_fill(int64_t n_rows, int64_t c, const int32_t* __restrict__ ptr, const int32_t* __restrict__ col,
                            const double* __restrict__ val, const int32_t* __restrict__ perm,
                            const int64_t* __restrict__ widths, const int64_t* __restrict__ slice_off,
                            int32_t* __restrict__ idx_out, double* __restrict__ val_out, bool skip_wide) {
  for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < n_rows;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t s = p / c, local = p - s * c;
    const int64_t rows_s = (s + 1) * c <= n_rows ? c : n_rows - s * c;
    const int64_t w = widths[s], base = slice_off[s];
    if (skip_wide && w > SPMVB_SELL_WIDE_COLS && rows_s <= 128) continue;
    const int32_t r = perm[p];
    const int32_t a = ptr[r], b = ptr[r + 1];
    const int64_t cnt = b - a;
    const int32_t last = cnt ? col[b - 1] : 0;
    for (int64_t j = 0; j < w; ++j) {
      bool real = j < cnt;
      idx_out[base + j * rows_s + local] = real ? col[a + j] : last;
      val_out[base + j * rows_s + local] = real ? val[a + j] : 0.0;
    }
  }
}

// Wide slices (power-law rows: one thread per row would walk up to ~4e5
// columns serially): one CTA per piece of ~32K cells, cells in storage order
// (coalesced writes), the slice's rows staged in shared memory.
__global__ void __launch_bounds__(256) k_sell_fill_wide(int64_t n_rows, int64_t c, const int32_t* __restrict__ ptr,
                                                        const int32_t* __restrict__ col,
                                                        const double* __restrict__ val,
                                                        const int32_t* __restrict__ perm,
                                                        const int64_t* __restrict__ widths,
                                                        const int64_t* __restrict__ slice_off,
                                                        const int32_t* __restrict__ wide, int64_t n_wide,
                                                        const int32_t* __restrict__ first_piece, int64_t n_pieces,
                                                        int32_t* __restrict__ idx_out, double* __restrict__ val_out) {
  __shared__ int32_t ra[128], rc[128], rl[128];  // row start, count, last column
  for (int64_t item = blockIdx.x; item < n_pieces; item += gridDim.x) {
    int64_t lo = 0, hi = n_wide - 1;  // wide slice of this piece: last i with first_piece[i] <= item
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) >> 1;
      if (first_piece[mid] <= item) lo = mid;
      else hi = mid - 1;
    }
    const int64_t sl = wide[lo];
    const int rows_s = sell_rows(sl, c, n_rows);
    const int64_t pc = sell_piece_cols(rows_s);
    const int64_t w = widths[sl];
    const int64_t j0 = (item - first_piece[lo]) * pc;
    const int64_t j1 = j0 + pc < w ? j0 + pc : w;
    __syncthreads();  // previous piece done with the row table
    if (threadIdx.x < rows_s) {
      const int32_t r = perm[sl * c + threadIdx.x];
      const int32_t a = ptr[r], b = ptr[r + 1];
      ra[threadIdx.x] = a;
      rc[threadIdx.x] = b - a;
      rl[threadIdx.x] = b > a ? col[b - 1] : 0;
    }
    __syncthreads();
    const int64_t base = slice_off[sl];
    for (int64_t e = j0 * rows_s + threadIdx.x; e < j1 * rows_s; e += blockDim.x) {
      const int64_t j = e / rows_s;
      const int l = static_cast<int>(e - j * rows_s);
      const bool real = j < rc[l];
      idx_out[base + e] = real ? col[ra[l] + j] : rl[l];
      val_out[base + e] = real ? val[ra[l] + j] : 0.0;
    }
  }
}

// ------------------------------------------------------------------- HYB --
constexpr int HYB_BINS = 4096;

template <typename Count>
__global__ void k_count_hist(Count cnt_of, int64_t n_rows, unsigned int* __restrict__ hist) {
  __shared__ unsigned int h[HYB_BINS];
  for (int i = threadIdx.x; i < HYB_BINS; i += blockDim.x) h[i] = 0;
  __syncthreads();
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < n_rows;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t cnt = cnt_of(r);
    atomicAdd(&h[cnt < HYB_BINS - 1 ? (cnt < 0 ? 0 : cnt) : HYB_BINS - 1], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < HYB_BINS; i += blockDim.x)
    if (h[i]) atomicAdd(&hist[i], h[i]);
}

struct PtrCount {
  const int32_t* ptr;
  __device__ int64_t operator()(int64_t r) const { return static_cast<int64_t>(ptr[r + 1] - ptr[r]); }
};
struct ArrCount {
  const int64_t* c;
  __device__ int64_t operator()(int64_t r) const { return c[r]; }
};

// ELL part: thread per row, column-major slots (coalesced).
__global__ void k_hyb_ell(int64_t n_rows, int64_t k, const int32_t* __restrict__ ptr, const int32_t* __restrict__ col,
                          const double* __restrict__ val, int32_t* __restrict__ ell_idx, double* __restrict__ ell_val,
                          int64_t* __restrict__ ell_row_nnz) {
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < n_rows;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t a = ptr[r], b = ptr[r + 1];
    const int64_t cnt = b - a;
    const int64_t kept = cnt < k ? cnt : k;
    const int32_t last = kept ? col[a + kept - 1] : 0;
    for (int64_t j = 0; j < k; ++j) {
      bool real = j < kept;
      ell_idx[j * n_rows + r] = real ? col[a + j] : last;
      ell_val[j * n_rows + r] = real ? val[a + j] : 0.0;
    }
    ell_row_nnz[r] = kept;
  }
}

// COO tail: one warp per 32 consecutive rows, their tail entries copied as
// one lane-strided stream (coalesced reads and writes even for short rows);
// output position -> row by a 5-step shuffle search over the warp's rows.
// Rows longer than LONG_ROW are left to a CTA each (spmvb_hyb_fill).
__global__ void k_hyb_tail(int64_t n_rows, int64_t k, const int32_t* __restrict__ ptr, const int32_t* __restrict__ col,
                           const double* __restrict__ val, const int32_t* __restrict__ tail_ptr,
                           int32_t* __restrict__ tail_row, int32_t* __restrict__ tail_col,
                           double* __restrict__ tail_val) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r0 = ((blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5) * 32; r0 < n_rows;
       r0 += nwarps * 32) {
    const int64_t r = r0 + lane;
    int32_t len = 0, src = 0, dst = 0;
    if (r < n_rows) {
      const int32_t a = ptr[r], cnt = ptr[r + 1] - a;
      len = (cnt > k && cnt <= LONG_ROW) ? static_cast<int32_t>(cnt - k) : 0;
      src = a + static_cast<int32_t>(k);
      dst = tail_ptr[r];
    }
    int32_t incl = len;  // inclusive prefix of the warp's stream lengths
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int32_t o = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += o;
    }
    const int32_t total = __shfl_sync(0xffffffffu, incl, 31);
    for (int32_t q0 = 0; q0 < total; q0 += 32) {
      const int32_t q = q0 + lane;
      // row of stream position q: the first lane whose inclusive prefix exceeds q
      int l = 0;
#pragma unroll
      for (int step = 16; step >= 1; step >>= 1) {
        const int32_t v = __shfl_sync(0xffffffffu, incl, l + step - 1);
        if (v <= q) l += step;
      }
      const int32_t start = __shfl_sync(0xffffffffu, incl - len, l);
      const int32_t s_l = __shfl_sync(0xffffffffu, src, l), d_l = __shfl_sync(0xffffffffu, dst, l);
      if (q < total) {
        const int32_t off = q - start;
        tail_row[d_l + off] = static_cast<int32_t>(r0 + l);
        tail_col[d_l + off] = col[s_l + off];
        tail_val[d_l + off] = val[s_l + off];
      }
    }
  }
}

template <typename Count>
int64_t count_rows_at_least(Count cnt_of, int64_t n_rows, int64_t kk, cudaStream_t s) {
  DevBuf<int64_t> d(1, s);
  device_reduce<int64_t>(
      n_rows, [=] __device__(int64_t i) { return static_cast<int64_t>(cnt_of(i) >= kk ? 1 : 0); }, OpSum{},
      (int64_t)0, d.get(), s);
  int64_t h = 0;
  copy_to_host(&h, d.get(), 1, s);
  return h;
}

// Largest K with 3 * #{rows with count >= K} > n_rows (formats.py:347-358;
// equivalent to the (n//3+1)-th largest count), floored at 1.
template <typename Count>
int64_t typical_k(Count cnt_of, int64_t n_rows, cudaStream_t s) {
  if (n_rows <= 0) fail(SPMVB_INVALID_ARG, "typical width is undefined for a matrix with no rows");
  DevBuf<unsigned int> hist(HYB_BINS, s);
  SPMVB_CUDA(cudaMemsetAsync(hist.get(), 0, HYB_BINS * sizeof(unsigned int), s));
  k_count_hist<<<grid_for(n_rows, 256, 148 * 4), 256, 0, s>>>(cnt_of, n_rows, hist.get());
  SPMVB_LAUNCHED("k_count_hist");
  static thread_local unsigned int h[HYB_BINS];
  copy_to_host(h, hist.get(), HYB_BINS, s);
  int64_t ge = 0, k = 0;
  for (int b = HYB_BINS - 1; b >= 1; --b) {
    ge += h[b];
    if (k == 0 && 3 * ge > n_rows) k = b;
  }
  if (k == HYB_BINS - 1) {
    // The answer may exceed the histogram range: binary search on counts.
    int64_t lo = HYB_BINS - 1, hi = INT32_MAX;  // invariant: lo qualifies
    while (lo < hi) {
      int64_t mid = lo + (hi - lo + 1) / 2;
      if (3 * count_rows_at_least(cnt_of, n_rows, mid, s) > n_rows) lo = mid; else hi = mid - 1;
    }
    k = lo;
  }
  return k < 1 ? 1 : k;
}

void csr5_build(int64_t n_rows, int64_t nnz, const int32_t* ptr, const int32_t* col, const double* val, int omega,
                int sigma, int32_t* tile_ptr, uint8_t* bit_flag, int32_t* y_off, int32_t* seg_off, int32_t* col_out,
                double* val_out, uint32_t* tile_aux, cudaStream_t s) {
  if (omega < 1 || sigma < 1) fail(SPMVB_INVALID_ARG, "omega and sigma must be >= 1, got %d, %d", omega, sigma);
  const int64_t tile = static_cast<int64_t>(omega) * sigma;
  const int64_t num_tiles = (nnz + tile - 1) / tile;
  k_csr5_tile_ptr<<<grid_for(num_tiles + 1, 256, 148 * 16), 256, 0, s>>>(ptr, n_rows, num_tiles, tile, tile_ptr);
  SPMVB_LAUNCHED("k_csr5_tile_ptr");
  if (nnz == 0) return;
  DevBuf<uint8_t> flags(nnz, s);
  SPMVB_CUDA(cudaMemsetAsync(flags.get(), 0, nnz, s));
  k_mark_row_starts<<<grid_for(n_rows, 256, 148 * 16), 256, 0, s>>>(ptr, n_rows, flags.get());
  SPMVB_LAUNCHED("k_mark_row_starts");
  int64_t scatter_from = 0;  // entries before this went through the shared-memory transpose
  if (tile <= CSR5_SMEM_TILE && nnz / tile > 0) {
    const int64_t full = nnz / tile;
    // small tiles (the reference default omega = 4: 64 entries) go several
    // to a block iteration, ~512 entries each
    const int group = tile >= 512 ? 1 : static_cast<int>(512 / tile);
    const int64_t chunk = tile * group;
    const size_t smem = static_cast<size_t>(chunk + chunk / 32 + 1) * (sizeof(double) + sizeof(int32_t) + 1);
    SPMVB_CUDA(cudaFuncSetAttribute(k_csr5_scatter_tiles, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_csr5_scatter_tiles<<<grid_for((full + group - 1) / group, 1, 148 * 8), 256, smem, s>>>(
        full, static_cast<int>(tile), group, omega, sigma, flags.get(), col, val, bit_flag, col_out, val_out);
    SPMVB_LAUNCHED("k_csr5_scatter_tiles");
    scatter_from = full * tile;
  }
  if (scatter_from < nnz) {
    k_csr5_scatter<<<grid_for(nnz - scatter_from, 256, 148 * 16), 256, 0, s>>>(
        scatter_from, nnz, tile, sigma, flags.get(), col, val, bit_flag, col_out, val_out);
    SPMVB_LAUNCHED("k_csr5_scatter");
  }
  // nz_rank[r] = number of non-empty rows before r
  DevBuf<int32_t> nz_rank(n_rows > 0 ? n_rows : 1, s);
  int32_t* nr = nz_rank.get();
  exclusive_scan<int32_t>(
      n_rows, [=] __device__(int64_t i) { return ptr[i + 1] > ptr[i] ? 1 : 0; }, ArrayStore<int32_t>{nr}, OpSum{},
      0, static_cast<int32_t*>(nullptr), s);
  if (omega <= 32) {
    k_csr5_descriptor_warp<<<grid_for(num_tiles * 32, 256, 148 * 16), 256, 0, s>>>(
        nnz, num_tiles, omega, sigma, flags.get(), ptr, tile_ptr, nr, y_off, seg_off, tile_aux);
    SPMVB_LAUNCHED("k_csr5_descriptor_warp");
  } else {
    k_csr5_descriptor<<<grid_for(num_tiles, 128, 148 * 64), 128, 0, s>>>(nnz, num_tiles, omega, sigma, flags.get(),
                                                                        ptr, tile_ptr, nr, y_off, seg_off, tile_aux);
    SPMVB_LAUNCHED("k_csr5_descriptor");
  }
}

}  // namespace

extern "C" int spmvb_csr_to_csr5(int64_t n_rows, int64_t nnz, const int32_t* ptr, const int32_t* col,
                                 const double* val, int omega, int sigma, int32_t* tile_ptr, uint8_t* bit_flag,
                                 int32_t* y_off, int32_t* seg_off, int32_t* col_out, double* val_out,
                                 uint32_t* tile_aux, void* stream) {
  return guard([&] {
    csr5_build(n_rows, nnz, ptr, col, val, omega, sigma, tile_ptr, bit_flag, y_off, seg_off, col_out, val_out,
               tile_aux, as_stream(stream));
  });
}

extern "C" int spmvb_csr_to_ell(int64_t n_rows, const int32_t* ptr, const int32_t* col, const double* val,
                                int64_t k, int64_t max_cells, int32_t* idx_out, double* val_out,
                                int64_t* row_nnz_out, void* stream) {
  return guard([&] {
    cudaStream_t s = as_stream(stream);
    if (n_rows * k > max_cells)
      fail(SPMVB_GRID_TOO_LARGE, "padded grid of %lldx%lld = %lld cells exceeds the %lld-cell limit",
           (long long)n_rows, (long long)k, (long long)(n_rows * k), (long long)max_cells);
    if (n_rows <= 0) return;
    k_ell_fill<<<grid_for(n_rows, 256, 148 * 64), 256, 0, s>>>(n_rows, k, ptr, col, val, idx_out, val_out,
                                                               row_nnz_out);
    SPMVB_LAUNCHED("k_ell_fill");
  });
}

extern "C" int spmvb_sell_plan(int64_t n_rows, const int32_t* ptr, int64_t c, int64_t sigma, int64_t max_cells,
                               int32_t* perm, int64_t* widths, int64_t* slice_off, int64_t* row_nnz_perm,
                               int64_t* total_cells, void* stream) {
  return guard([&] {
    cudaStream_t s = as_stream(stream);
    if (c < 1) fail(SPMVB_INVALID_ARG, "slice height c must be >= 1, got %lld", (long long)c);
    if (sigma < 0 || (sigma > 0 && sigma % c != 0))
      fail(SPMVB_INVALID_ARG, "sorting window sigma must be 0 or a positive multiple of c, got sigma=%lld, c=%lld",
           (long long)sigma, (long long)c);
    const int64_t n_slices = (n_rows + c - 1) / c;
    *total_cells = 0;
    if (n_rows <= 0) {
      int64_t zero = 0;
      SPMVB_CUDA(cudaMemcpyAsync(slice_off, &zero, sizeof(zero), cudaMemcpyHostToDevice, s));
      SPMVB_CUDA(cudaStreamSynchronize(s));
      return;
    }
    if (sigma > 0) {
      int64_t stats[3];
      {
        DevBuf<int64_t> d(1, s);
        device_reduce<int64_t>(
            n_rows, [=] __device__(int64_t i) { return static_cast<int64_t>(ptr[i + 1] - ptr[i]); }, OpMax{},
            (int64_t)0, d.get(), s);
        copy_to_host(&stats[0], d.get(), 1, s);
      }
      const uint64_t maxc = static_cast<uint64_t>(stats[0]);
      const int cbits = bits_for(maxc);
      const int wbits = bits_for(static_cast<uint64_t>((n_rows - 1) / sigma));
      DevBuf<uint64_t> ka(n_rows, s), kb(n_rows, s);
      DevBuf<uint32_t> vb(n_rows, s), vs(n_rows, s);
      k_sell_keys<<<grid_for(n_rows, 256, 148 * 16), 256, 0, s>>>(ptr, n_rows, sigma, cbits, maxc, ka.get());
      SPMVB_LAUNCHED("k_sell_keys");
      RadixSortResult rs = radix_sort_pairs(ka.get(), nullptr, kb.get(), vb.get(), vs.get(), n_rows, wbits + cbits, s);
      k_sell_perm<<<grid_for(n_rows, 256, 148 * 16), 256, 0, s>>>(rs.vals, ptr, n_rows, perm, row_nnz_perm);
      SPMVB_LAUNCHED("k_sell_perm");
    } else {
      k_sell_perm<<<grid_for(n_rows, 256, 148 * 16), 256, 0, s>>>(nullptr, ptr, n_rows, perm, row_nnz_perm);
      SPMVB_LAUNCHED("k_sell_perm");
    }
    k_sell_widths<<<grid_for(n_slices, 256, 148 * 16), 256, 0, s>>>(row_nnz_perm, n_rows, c, n_slices, widths);
    SPMVB_LAUNCHED("k_sell_widths");
    DevBuf<int64_t> d_total(1, s);
    exclusive_scan<int64_t>(
        n_slices + 1,
        [=] __device__(int64_t sl) -> int64_t {
          if (sl >= n_slices) return 0;
          int64_t rows = (sl + 1) * c <= n_rows ? c : n_rows - sl * c;
          return rows * widths[sl];
        },
        ArrayStore<int64_t>{slice_off}, OpSum{}, (int64_t)0, d_total.get(), s);
    copy_to_host(total_cells, d_total.get(), 1, s);
    if (*total_cells > max_cells)
      fail(SPMVB_GRID_TOO_LARGE, "sliced grids of %lld cells exceed the %lld-cell limit", (long long)*total_cells,
           (long long)max_cells);
  });
}

extern "C" int spmvb_sell_fill(int64_t n_rows, const int32_t* ptr, const int32_t* col, const double* val, int64_t c,
                               const int32_t* perm, const int64_t* widths, const int64_t* slice_off,
                               int32_t* idx_out, double* val_out, void* stream) {
  return guard([&] {
    cudaStream_t s = as_stream(stream);
    if (n_rows <= 0) return;
    const int64_t n_slices = (n_rows + c - 1) / c;
    DevBuf<int32_t> wide(n_slices, s), first_piece(n_slices, s);
    int64_t n_wide = 0, n_pieces = 0;
    // the fill's own split (default width): independent of the SpMV's wide_cols
    if (const int st = spmvb_sell_wide_plan(n_rows, c, widths, SPMVB_SELL_WIDE_COLS, wide.get(), &n_wide, nullptr,
                                            first_piece.get(), &n_pieces, s)) {
      const std::string msg = spmvb_last_error();
      fail(st, "%s", msg.c_str());
    }
    k_sell_fill<<<grid_for(n_rows, 256, 148 * 64), 256, 0, s>>>(n_rows, c, ptr, col, val, perm, widths, slice_off,
                                                                idx_out, val_out, n_wide > 0);
    SPMVB_LAUNCHED("k_sell_fill");
    if (n_wide > 0 && n_pieces > 0) {
      k_sell_fill_wide<<<grid_for(n_pieces, 1, 148 * 8), 256, 0, s>>>(n_rows, c, ptr, col, val, perm, widths,
                                                                        slice_off, wide.get(), n_wide,
                                                                        first_piece.get(), n_pieces, idx_out, val_out);
      SPMVB_LAUNCHED("k_sell_fill_wide");
    }
  });
}

extern "C" int spmvb_hyb_typical_k(const int32_t* ptr, int64_t n_rows, int64_t* k_out, void* stream) {
  return guard([&] { *k_out = typical_k(PtrCount{ptr}, n_rows, as_stream(stream)); });
}

extern "C" int spmvb_typical_k_counts(const int64_t* counts, int64_t n, int64_t* k_out, void* stream) {
  return guard([&] { *k_out = typical_k(ArrCount{counts}, n, as_stream(stream)); });
}

extern "C" int spmvb_hyb_plan(int64_t n_rows, const int32_t* ptr, int64_t k, int64_t max_cells, int32_t* tail_ptr,
                              int64_t* tail_nnz, void* stream) {
  return guard([&] {
    cudaStream_t s = as_stream(stream);
    if (n_rows * k > max_cells)
      fail(SPMVB_GRID_TOO_LARGE, "padded grid of %lldx%lld = %lld cells exceeds the %lld-cell limit",
           (long long)n_rows, (long long)k, (long long)(n_rows * k), (long long)max_cells);
    DevBuf<int32_t> d_total(1, s);
    exclusive_scan<int32_t>(
        n_rows + 1,
        [=] __device__(int64_t i) -> int32_t {
          if (i >= n_rows) return 0;
          int64_t extra = static_cast<int64_t>(ptr[i + 1] - ptr[i]) - k;
          return extra > 0 ? static_cast<int32_t>(extra) : 0;
        },
        ArrayStore<int32_t>{tail_ptr}, OpSum{}, 0, d_total.get(), s);
    int32_t h = 0;
    copy_to_host(&h, d_total.get(), 1, s);
    *tail_nnz = h;
  });
}

extern "C" int spmvb_hyb_fill(int64_t n_rows, const int32_t* ptr, const int32_t* col, const double* val, int64_t k,
                              const int32_t* tail_ptr, int32_t* ell_idx, double* ell_val, int64_t* ell_row_nnz,
                              int32_t* tail_row, int32_t* tail_col, double* tail_val, void* stream) {
  return guard([&] {
    cudaStream_t s = as_stream(stream);
    if (n_rows <= 0) return;
    k_hyb_ell<<<grid_for(n_rows, 256, 148 * 64), 256, 0, s>>>(n_rows, k, ptr, col, val, ell_idx, ell_val,
                                                              ell_row_nnz);
    SPMVB_LAUNCHED("k_hyb_ell");
    k_hyb_tail<<<grid_for((n_rows + 31) / 32 * 32, 256, 148 * 64), 256, 0, s>>>(n_rows, k, ptr, col, val, tail_ptr,
                                                                                 tail_row, tail_col, tail_val);
    SPMVB_LAUNCHED("k_hyb_tail");
    for_long_rows(
        [=] __device__(int64_t r) { return static_cast<int64_t>(ptr[r + 1] - ptr[r]); }, n_rows,
        [=] __device__(int64_t r, int64_t first, int64_t stride) {
          const int64_t a = ptr[r], cnt = ptr[r + 1] - a, t0 = tail_ptr[r] - k;
          for (int64_t j = k + first; j < cnt; j += stride) {
            tail_row[t0 + j] = static_cast<int32_t>(r);
            tail_col[t0 + j] = col[a + j];
            tail_val[t0 + j] = val[a + j];
          }
        },
        s);
  });
}
