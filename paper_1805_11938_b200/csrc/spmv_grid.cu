// ELL and SELL(-C-sigma) SpMV (reference kernels.py:98-136): one thread per
// (permuted) row, sequential accumulation over all slots with separately
// rounded products, which is bit-identical to the reference kernels.
#include "spmv_common.cuh"

using namespace spmvb;

namespace {

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

