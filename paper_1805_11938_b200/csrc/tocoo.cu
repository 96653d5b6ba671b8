// Format -> COO triplet extraction on the GPU (reference formats.py:400-453,
// `to_coo`).  Each function emits triplets that the caller passes through
// spmvb_canonicalize_*, exactly as the reference routes every format
// through `canonicalize`; every format's triplets come out in canonical
// order already (SELL through row-order offsets, HYB by merging each row's
// ELL part and tail), so canonicalize takes its copy-only fast path.
#include "prims.cuh"

using namespace spmvb;

namespace {

// A warp's 32 segments (lane l: length len, per-lane words a, b) copied as
// ONE lane-strided stream: f(off, a_l, b_l) for every off < len_l of every
// lane l, consecutive lanes taking consecutive stream positions (stream
// position -> segment by a 5-step shuffle search over the lanes' inclusive
// prefix).  Short segments then cost no more than long ones per lane.
template <typename F>
__device__ __forceinline__ void warp_segments(int32_t len, int64_t a, int64_t b, F f) {
  const int lane = threadIdx.x & 31;
  int32_t incl = len;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int32_t o = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += o;
  }
  const int32_t total = __shfl_sync(0xffffffffu, incl, 31);
  for (int32_t q0 = 0; q0 < total; q0 += 32) {
    const int32_t q = q0 + lane;
    int l = 0;
#pragma unroll
    for (int step = 16; step >= 1; step >>= 1)
      if (__shfl_sync(0xffffffffu, incl, l + step - 1) <= q) l += step;
    l &= 31;
    const int32_t start = __shfl_sync(0xffffffffu, incl - len, l);
    const int64_t al = __shfl_sync(0xffffffffu, a, l), bl = __shfl_sync(0xffffffffu, b, l);
    if (q < total) f(static_cast<int64_t>(q - start), al, bl);
  }
}

// rows[k] = r for k in [ptr[r], ptr[r+1]): a warp per 32 rows as one stream
// (coalesced stores); rows longer than LONG_ROW get a CTA each.
__global__ void k_expand_rows(const int32_t* __restrict__ ptr, int64_t n_rows, int32_t* __restrict__ rows) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r0 = ((blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5) * 32; r0 < n_rows;
       r0 += nwarps * 32) {
    const int64_t r = r0 + lane;
    int32_t len = 0;
    int64_t a = 0;
    if (r < n_rows) {
      a = ptr[r];
      const int32_t cnt = ptr[r + 1] - static_cast<int32_t>(a);
      len = cnt <= LONG_ROW ? cnt : 0;
    }
    warp_segments(len, a, r, [&](int64_t off, int64_t al, int64_t rl) { rows[al + off] = static_cast<int32_t>(rl); });
  }
}

// Stored CSR5 entry s -> CSR position k (inverse of csr5_stored in formats.cu).
__global__ void k_csr5_unstore(int64_t nnz, int64_t tile, int64_t sigma, const int32_t* __restrict__ col,
                               const double* __restrict__ val, int32_t* __restrict__ col_out,
                               double* __restrict__ val_out) {
  for (int64_t s = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; s < nnz;
       s += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t t = s / tile, base = t * tile, off = s - base;
    const int64_t m = nnz - base < tile ? nnz - base : tile;
    const int64_t q = m / sigma, rem = m % sigma;
    // grid row gi holds q+1 cells for gi < rem, q cells otherwise
    const int64_t big = rem * (q + 1);
    int64_t gi, gj;
    if (off < big) { gi = off / (q + 1); gj = off - gi * (q + 1); }
    else { gi = rem + (off - big) / q; gj = (off - big) - (gi - rem) * q; }
    const int64_t k = base + gj * sigma + gi;
    col_out[k] = col[s];
    val_out[k] = val[s];
  }
}

__global__ void k_grid_to_coo(int64_t n_rows, int64_t k, const int32_t* __restrict__ idx,
                              const double* __restrict__ val, const int64_t* __restrict__ row_nnz,
                              const int32_t* __restrict__ out_ptr, int32_t* __restrict__ rows,
                              int32_t* __restrict__ cols, double* __restrict__ vals) {
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < n_rows;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t cnt = row_nnz[r];
    const int64_t o = out_ptr[r];
    for (int64_t j = 0; j < cnt; ++j) {
      rows[o + j] = static_cast<int32_t>(r);
      cols[o + j] = idx[j * n_rows + r];
      vals[o + j] = val[j * n_rows + r];
    }
  }
}

// SELL -> triplets in canonical (row) order: permuted position p (row
// perm[p]) writes at out_ptr[perm[p]], its cells read down its slice column
// (stride rows_s).  A warp per 32 permuted positions as one stream; rows
// longer than LONG_ROW get a CTA each (spmvb_sell_to_coo).
__global__ void k_sell_to_coo(int64_t n_rows, int64_t c, const int32_t* __restrict__ perm,
                              const int64_t* __restrict__ slice_off, const int64_t* __restrict__ row_nnz_perm,
                              const int32_t* __restrict__ idx, const double* __restrict__ val,
                              const int32_t* __restrict__ out_ptr, int32_t* __restrict__ rows,
                              int32_t* __restrict__ cols, double* __restrict__ vals) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  if (c >= (1ll << 23)) {  // slice heights past the packed stride field: plain thread per row
    for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < n_rows;
         p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
      const int64_t sl = p / c, local = p - sl * c;
      const int64_t rows_s = (sl + 1) * c <= n_rows ? c : n_rows - sl * c;
      const int64_t cnt = row_nnz_perm[p];
      if (cnt > LONG_ROW) continue;
      const int32_t r = perm[p];
      for (int64_t j = 0; j < cnt; ++j) {
        const int64_t g = slice_off[sl] + local + j * rows_s;
        rows[out_ptr[r] + j] = r;
        cols[out_ptr[r] + j] = idx[g];
        vals[out_ptr[r] + j] = val[g];
      }
    }
    return;
  }
  for (int64_t p0 = ((blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5) * 32; p0 < n_rows;
       p0 += nwarps * 32) {
    const int64_t p = p0 + lane;
    int32_t len = 0;
    int64_t src = 0, dst_row = 0;  // src: first cell | rows_s << 40; dst_row: out offset | row << 32
    if (p < n_rows) {
      const int64_t sl = p / c, local = p - sl * c;
      const int64_t rows_s = (sl + 1) * c <= n_rows ? c : n_rows - sl * c;
      const int64_t cnt = row_nnz_perm[p];
      const int32_t r = perm[p];
      len = cnt <= LONG_ROW ? static_cast<int32_t>(cnt) : 0;
      src = (slice_off[sl] + local) | (rows_s << 40);
      dst_row = static_cast<int64_t>(out_ptr[r]) | (static_cast<int64_t>(r) << 32);
    }
    warp_segments(len, src, dst_row, [&](int64_t off, int64_t sv, int64_t dv) {
      const int64_t g = (sv & ((1ll << 40) - 1)) + off * (sv >> 40);
      const int64_t o = (dv & 0xffffffffll) + off;
      rows[o] = static_cast<int32_t>(dv >> 32);
      cols[o] = idx[g];
      vals[o] = val[g];
    });
  }
}

// HYB -> triplets in canonical order: row r's ELL entries at
// ell_excl[r] + tail_ptr[r] + j, tail entry t (row r) at t + ell_incl[r].
__global__ void k_hyb_ell_to_coo(int64_t n_rows, int64_t k, const int32_t* __restrict__ idx,
                                 const double* __restrict__ val, const int64_t* __restrict__ row_nnz,
                                 const int32_t* __restrict__ ell_excl, const int32_t* __restrict__ tail_ptr,
                                 int32_t* __restrict__ rows, int32_t* __restrict__ cols, double* __restrict__ vals) {
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < n_rows;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t cnt = row_nnz[r];
    const int64_t o = static_cast<int64_t>(ell_excl[r]) + tail_ptr[r];
    for (int64_t j = 0; j < cnt; ++j) {
      rows[o + j] = static_cast<int32_t>(r);
      cols[o + j] = idx[j * n_rows + r];
      vals[o + j] = val[j * n_rows + r];
    }
  }
}

__global__ void k_hyb_tail_to_coo(int64_t tail_nnz, const int32_t* __restrict__ trow, const int32_t* __restrict__ tcol,
                                  const double* __restrict__ tval, const int32_t* __restrict__ ell_excl,
                                  const int64_t* __restrict__ row_nnz, int32_t* __restrict__ rows,
                                  int32_t* __restrict__ cols, double* __restrict__ vals) {
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < tail_nnz;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t r = trow[t];
    const int64_t o = t + ell_excl[r] + row_nnz[r];
    rows[o] = r;
    cols[o] = tcol[t];
    vals[o] = tval[t];
  }
}

__global__ void k_scatter_counts(int64_t n, const int32_t* __restrict__ perm, const int64_t* __restrict__ cnt_perm,
                                 int64_t* __restrict__ cnt) {
  for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < n;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x)
    cnt[perm[p]] = cnt_perm[p];
}

void offsets_from_counts(const int64_t* counts, int64_t n, int32_t* out_ptr, cudaStream_t s) {
  exclusive_scan<int32_t>(
      n + 1, [=] __device__(int64_t i) -> int32_t { return i < n ? static_cast<int32_t>(counts[i]) : 0; },
      ArrayStore<int32_t>{out_ptr}, OpSum{}, 0, static_cast<int32_t*>(nullptr), s);
}

}  // namespace

extern "C" int spmvb_csr_expand_rows(const int32_t* ptr, int64_t n_rows, int32_t* rows_out, void* stream) {
  return guard([&] {
    cudaStream_t s = as_stream(stream);
    if (n_rows <= 0) return;
    k_expand_rows<<<grid_for((n_rows + 31) / 32 * 32, 256, 148 * 32), 256, 0, s>>>(ptr, n_rows, rows_out);
    SPMVB_LAUNCHED("k_expand_rows");
    for_long_rows(
        [=] __device__(int64_t r) { return static_cast<int64_t>(ptr[r + 1] - ptr[r]); }, n_rows,
        [=] __device__(int64_t r, int64_t first, int64_t stride) {
          for (int64_t k = ptr[r] + first; k < ptr[r + 1]; k += stride) rows_out[k] = static_cast<int32_t>(r);
        },
        s);
  });
}

extern "C" int spmvb_csr5_unstore(int64_t nnz, int omega, int sigma, const int32_t* col, const double* val,
                                  int32_t* col_out, double* val_out, void* stream) {
  return guard([&] {
    cudaStream_t s = as_stream(stream);
    if (omega < 1 || sigma < 1) fail(SPMVB_INVALID_ARG, "omega and sigma must be >= 1");
    if (nnz <= 0) return;
    k_csr5_unstore<<<grid_for(nnz, 256, 148 * 32), 256, 0, s>>>(nnz, static_cast<int64_t>(omega) * sigma, sigma, col,
                                                                val, col_out, val_out);
    SPMVB_LAUNCHED("k_csr5_unstore");
  });
}

extern "C" int spmvb_ell_to_coo(int64_t n_rows, int64_t k, const int32_t* idx, const double* val,
                                const int64_t* row_nnz, int32_t* rows_out, int32_t* cols_out, double* vals_out,
                                void* stream) {
  return guard([&] {
    cudaStream_t s = as_stream(stream);
    if (n_rows <= 0) return;
    DevBuf<int32_t> off(n_rows + 1, s);
    offsets_from_counts(row_nnz, n_rows, off.get(), s);
    k_grid_to_coo<<<grid_for(n_rows, 256, 148 * 32), 256, 0, s>>>(n_rows, k, idx, val, row_nnz, off.get(), rows_out,
                                                                  cols_out, vals_out);
    SPMVB_LAUNCHED("k_grid_to_coo");
  });
}

extern "C" int spmvb_sell_to_coo(int64_t n_rows, int64_t c, const int32_t* perm, const int64_t* slice_off,
                                 const int64_t* row_nnz_perm, const int32_t* idx, const double* val,
                                 int32_t* rows_out, int32_t* cols_out, double* vals_out, void* stream) {
  return guard([&] {
    cudaStream_t s = as_stream(stream);
    if (n_rows <= 0) return;
    // row-order counts -> row-order offsets (the output is canonical)
    DevBuf<int64_t> cnt(n_rows, s);
    DevBuf<int32_t> off(n_rows + 1, s);
    int64_t* cp = cnt.get();
    k_scatter_counts<<<grid_for(n_rows, 256, 148 * 32), 256, 0, s>>>(n_rows, perm, row_nnz_perm, cp);
    SPMVB_LAUNCHED("k_scatter_counts");
    offsets_from_counts(cp, n_rows, off.get(), s);
    k_sell_to_coo<<<grid_for((n_rows + 31) / 32 * 32, 256, 148 * 32), 256, 0, s>>>(
        n_rows, c, perm, slice_off, row_nnz_perm, idx, val, off.get(), rows_out, cols_out, vals_out);
    SPMVB_LAUNCHED("k_sell_to_coo");
    const int32_t* op = off.get();
    for_long_rows(
        [=] __device__(int64_t p) { return row_nnz_perm[p]; }, n_rows,
        [=] __device__(int64_t p, int64_t first, int64_t stride) {
          const int64_t sl = p / c, local = p - sl * c;
          const int64_t rows_s = (sl + 1) * c <= n_rows ? c : n_rows - sl * c;
          const int32_t r = perm[p];
          const int64_t o = op[r], base = slice_off[sl] + local;
          for (int64_t j = first; j < row_nnz_perm[p]; j += stride) {
            rows_out[o + j] = r;
            cols_out[o + j] = idx[base + j * rows_s];
            vals_out[o + j] = val[base + j * rows_s];
          }
        },
        s);
  });
}

extern "C" int spmvb_hyb_to_coo(int64_t n_rows, int64_t k, const int32_t* ell_idx, const double* ell_val,
                                const int64_t* ell_row_nnz, int64_t tail_nnz, const int32_t* tail_row,
                                const int32_t* tail_col, const double* tail_val, const int32_t* tail_ptr,
                                int32_t* rows_out, int32_t* cols_out, double* vals_out, void* stream) {
  return guard([&] {
    cudaStream_t s = as_stream(stream);
    if (n_rows <= 0) return;
    DevBuf<int32_t> excl(n_rows + 1, s);
    offsets_from_counts(ell_row_nnz, n_rows, excl.get(), s);
    k_hyb_ell_to_coo<<<grid_for(n_rows, 256, 148 * 32), 256, 0, s>>>(n_rows, k, ell_idx, ell_val, ell_row_nnz,
                                                                     excl.get(), tail_ptr, rows_out, cols_out,
                                                                     vals_out);
    SPMVB_LAUNCHED("k_hyb_ell_to_coo");
    if (tail_nnz > 0) {
      k_hyb_tail_to_coo<<<grid_for(tail_nnz, 256, 148 * 32), 256, 0, s>>>(tail_nnz, tail_row, tail_col, tail_val,
                                                                         excl.get(), ell_row_nnz, rows_out,
                                                                         cols_out, vals_out);
      SPMVB_LAUNCHED("k_hyb_tail_to_coo");
    }
  });
}
