// Format -> COO triplet extraction on the GPU (reference formats.py:400-453,
// `to_coo`).  Each function emits triplets that the caller passes through
// spmvb_canonicalize_*, exactly as the reference routes every format
// through `canonicalize`; for CSR, CSR5 and ELL the triplets come out in
// canonical order already, so canonicalize takes its copy-only fast path.
#include "prims.cuh"

using namespace spmvb;

namespace {

__global__ void k_expand_rows(const int32_t* __restrict__ ptr, int64_t n_rows, int32_t* __restrict__ rows) {
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < n_rows;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x)
    for (int32_t k = ptr[r]; k < ptr[r + 1]; ++k) rows[k] = static_cast<int32_t>(r);
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

__global__ void k_sell_to_coo(int64_t n_rows, int64_t c, const int32_t* __restrict__ perm,
                              const int64_t* __restrict__ slice_off, const int64_t* __restrict__ row_nnz_perm,
                              const int32_t* __restrict__ idx, const double* __restrict__ val,
                              const int32_t* __restrict__ out_ptr, int32_t* __restrict__ rows,
                              int32_t* __restrict__ cols, double* __restrict__ vals) {
  for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < n_rows;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t s = p / c, local = p - s * c;
    const int64_t rows_s = (s + 1) * c <= n_rows ? c : n_rows - s * c;
    const int64_t cnt = row_nnz_perm[p];
    const int64_t o = out_ptr[p];
    const int32_t r = perm[p];
    for (int64_t j = 0; j < cnt; ++j) {
      const int64_t g = slice_off[s] + j * rows_s + local;
      rows[o + j] = r;
      cols[o + j] = idx[g];
      vals[o + j] = val[g];
    }
  }
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
    k_expand_rows<<<grid_for(n_rows, 256, 148 * 32), 256, 0, s>>>(ptr, n_rows, rows_out);
    SPMVB_LAUNCHED("k_expand_rows");
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
    DevBuf<int32_t> off(n_rows + 1, s);
    offsets_from_counts(row_nnz_perm, n_rows, off.get(), s);
    k_sell_to_coo<<<grid_for(n_rows, 256, 148 * 32), 256, 0, s>>>(n_rows, c, perm, slice_off, row_nnz_perm, idx, val,
                                                                  off.get(), rows_out, cols_out, vals_out);
    SPMVB_LAUNCHED("k_sell_to_coo");
  });
}
