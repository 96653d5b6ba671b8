// Reference-order ("bit-parity") SpMV for the three formats whose fast
// kernels sum in a different order than spmvkit: CSR, CSR5 and HYB.  Each
// kernel here reproduces the reference's own floating-point order, so y
// equals spmvkit's output (workers = 1) bit for bit:
//
//   CSR  (kernels.py:76-95)   products rounded separately, then
//        np.add.reduceat over the row starts: y_r = p_first + pairwise(rest)
//        with numpy's pairwise tree (np_pairwise, common.cuh).
//   CSR5 (kernels.py:139-174) per tile, reduceat over the flag segments -- a
//        row's entries inside one tile -- then y[rows] += sums in ascending
//        tile order: y_r = ((0 + s_1) + s_2) + ..., s_i = first + pairwise(rest)
//        over the row's piece in tile i.
//   HYB  (kernels.py:177-199) the ELL recurrence ((0 + p_0) + p_1) + ... over
//        the K slots (pads included), then y += bincount(tail rows, weights):
//        y_r = ell_r + ((0 + t_1) + t_2 + ...) when the tail is non-empty.
//
// ELL and SELL need no such mode: their fast kernels already are the
// reference recurrence (SELL with every slice on the thread-per-row path).
// These kernels are a verification mode, written for exactness first: a
// thread per row, and a CTA per row longer than EXACT_LONG entries.
#include <algorithm>

#include "spmv_common.cuh"

using namespace spmvb;

namespace {

constexpr int EXACT_LONG = 256;      // rows above this go to the CTA-per-row kernel
constexpr int EXACT_THREADS = 256;   // CTA size of the long-row kernel
constexpr int EXACT_BATCH = 1024;    // items (products / piece sums) per shared-memory batch
constexpr int EXACT_MAX_L = 12;      // long CSR rows: 2^L subtrees combined in shared memory (32 KB)

// products in CSR order
struct ProdCsr {
  const int32_t* idx;
  const double* val;
  const double* x;
  __device__ double operator()(int64_t i) const { return __dmul_rn(val[i], x[idx[i]]); }
};

// products in CSR order of a CSR5 matrix, whose indices/data are in stored
// order: CSR-order position k of a tile filled with m entries sits at
// base + gi*q + min(gi, rem) + gj (formats.py:204-209)
struct ProdCsr5 {
  const int32_t* idx;
  const double* val;
  const double* x;
  int64_t nnz;
  int32_t tile, sigma;
  __device__ double operator()(int64_t k) const {
    const int64_t base = k / tile * tile;
    const int32_t p = static_cast<int32_t>(k - base);
    const int64_t m = nnz - base < tile ? nnz - base : tile;
    const int32_t q = static_cast<int32_t>(m / sigma), rem = static_cast<int32_t>(m % sigma);
    const int32_t gi = p % sigma, gj = p / sigma;
    const int64_t s = base + static_cast<int64_t>(gi) * q + (gi < rem ? gi : rem) + gj;
    return __dmul_rn(val[s], x[idx[s]]);
  }
};

// np.add.reduceat over one segment [a, b), b > a
template <typename At>
__device__ __forceinline__ double reduceat_segment(const At& at, int64_t a, int64_t b) {
  return at(a) + np_pairwise(at, a + 1, b - a - 1);
}

__device__ __forceinline__ void append_long(int32_t* list, unsigned int* n_long, int64_t r) {
  list[atomicAdd(n_long, 1u)] = static_cast<int32_t>(r);
}

__device__ __forceinline__ void store_row(double* y, int64_t r, double acc, const double* scale_p, double s) {
  y[r] = scale_p ? s * acc : acc;
}

// ------------------------------------------------------------------ CSR ----
__global__ void k_exact_csr(int64_t n_rows, const int32_t* __restrict__ ptr, ProdCsr at, double* __restrict__ y,
                            const double* __restrict__ scale_p, int32_t* __restrict__ list,
                            unsigned int* __restrict__ n_long) {
  const double s = load_scale(scale_p);
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < n_rows;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t a = ptr[r], b = ptr[r + 1];
    if (b - a > EXACT_LONG) {
      append_long(list, n_long, r);
      continue;
    }
    store_row(y, r, b > a ? reduceat_segment(at, a, b) : 0.0, scale_p, s);
  }
}

// numpy's split: a block of len > 128 splits at n2 = len/2 rounded down to a
// multiple of 8.  Descends `d` levels from the block [off, off+len) following
// the bits of idx (MSB first); a block that becomes a leaf (<= 128) above
// depth d is represented by its leftmost virtual descendant only.
__device__ bool exact_descend(int d, int64_t idx, int64_t& off, int64_t& len) {
  for (int l = 0; l < d; ++l) {
    if (len <= 128) return (idx & ((1ll << (d - l)) - 1)) == 0;
    int64_t n2 = len / 2;
    n2 -= n2 % 8;
    if ((idx >> (d - 1 - l)) & 1) {
      off += n2;
      len -= n2;
    } else {
      len = n2;
    }
  }
  return true;
}

// One CTA per long row: the pairwise tree over rest = [a+1, b) is cut at
// depth L; every thread sums whole depth-L subtrees (np_pairwise: the same
// order as numpy's recursion below that depth), then the top L levels are
// combined in shared memory, left + right as numpy does.
__global__ void __launch_bounds__(EXACT_THREADS) k_exact_csr_long(const int32_t* __restrict__ list,
                                                                  const unsigned int* __restrict__ n_long,
                                                                  const int32_t* __restrict__ ptr, ProdCsr at,
                                                                  double* __restrict__ y,
                                                                  const double* __restrict__ scale_p) {
  __shared__ double v[1 << EXACT_MAX_L];
  const double s = load_scale(scale_p);
  const unsigned int count = *n_long;
  for (unsigned int i = blockIdx.x; i < count; i += gridDim.x) {
    const int64_t r = list[i];
    const int64_t a = ptr[r], b = ptr[r + 1];
    const int64_t off0 = a + 1, n = b - a - 1;
    int L = 0;
    while (L < EXACT_MAX_L && (n >> L) > 128) ++L;
    const int64_t nodes = 1ll << L;
    for (int64_t k = threadIdx.x; k < nodes; k += EXACT_THREADS) {
      int64_t off = off0, len = n;
      v[k] = exact_descend(L, k, off, len) ? np_pairwise(at, off, len) : 0.0;
    }
    __syncthreads();
    for (int d = L - 1; d >= 0; --d) {
      for (int64_t k = threadIdx.x; k < (1ll << d); k += EXACT_THREADS) {
        int64_t off = off0, len = n;
        if (exact_descend(d, k, off, len) && len > 128) {  // internal node: left + right
          const int64_t base = k << (L - d);
          v[base] = v[base] + v[base + (1ll << (L - d - 1))];
        }
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) store_row(y, r, at(a) + v[0], scale_p, s);
    __syncthreads();
  }
}

// ----------------------------------------------------------------- CSR5 ----
// piece i of the row [a, b): its entries inside tile (a / tile + i)
__device__ __forceinline__ double csr5_piece(const ProdCsr5& at, int64_t a, int64_t b, int64_t t0, int64_t i) {
  const int64_t lo = (t0 + i) * at.tile, hi = lo + at.tile;
  return reduceat_segment(at, lo > a ? lo : a, hi < b ? hi : b);
}

__global__ void k_exact_csr5(int64_t n_rows, const int32_t* __restrict__ ptr, ProdCsr5 at, double* __restrict__ y,
                             const double* __restrict__ scale_p, int32_t* __restrict__ list,
                             unsigned int* __restrict__ n_long) {
  const double s = load_scale(scale_p);
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < n_rows;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t a = ptr[r], b = ptr[r + 1];
    if (b - a > EXACT_LONG) {
      append_long(list, n_long, r);
      continue;
    }
    double acc = 0.0;
    if (b > a) {
      const int64_t t0 = a / at.tile, t1 = (b - 1) / at.tile;
      for (int64_t i = 0; i <= t1 - t0; ++i) acc = acc + csr5_piece(at, a, b, t0, i);
    }
    store_row(y, r, acc, scale_p, s);
  }
}

// One CTA per long row: batches of piece sums computed in parallel, added in
// tile order by one thread.
__global__ void __launch_bounds__(EXACT_THREADS) k_exact_csr5_long(const int32_t* __restrict__ list,
                                                                   const unsigned int* __restrict__ n_long,
                                                                   const int32_t* __restrict__ ptr, ProdCsr5 at,
                                                                   double* __restrict__ y,
                                                                   const double* __restrict__ scale_p) {
  __shared__ double v[EXACT_BATCH];
  const double s = load_scale(scale_p);
  const unsigned int count = *n_long;
  for (unsigned int i = blockIdx.x; i < count; i += gridDim.x) {
    const int64_t r = list[i];
    const int64_t a = ptr[r], b = ptr[r + 1];
    const int64_t t0 = a / at.tile, pieces = (b - 1) / at.tile - t0 + 1;
    double acc = 0.0;
    for (int64_t p0 = 0; p0 < pieces; p0 += EXACT_BATCH) {
      const int64_t m = pieces - p0 < EXACT_BATCH ? pieces - p0 : EXACT_BATCH;
      for (int64_t k = threadIdx.x; k < m; k += EXACT_THREADS) v[k] = csr5_piece(at, a, b, t0, p0 + k);
      __syncthreads();
      if (threadIdx.x == 0)
        for (int64_t k = 0; k < m; ++k) acc = acc + v[k];
      __syncthreads();
    }
    if (threadIdx.x == 0) store_row(y, r, acc, scale_p, s);
  }
}

// ------------------------------------------------------------------ HYB ----
__device__ __forceinline__ double ell_row_exact(int64_t n_rows, int64_t k, int64_t r, const int32_t* __restrict__ gi,
                                                const double* __restrict__ gd, const double* __restrict__ x) {
  double acc = 0.0;
  for (int64_t j = 0; j < k; ++j) acc = __dadd_rn(acc, __dmul_rn(gd[j * n_rows + r], x[gi[j * n_rows + r]]));
  return acc;
}

__global__ void k_exact_hyb(int64_t n_rows, int64_t k, const int32_t* __restrict__ gi, const double* __restrict__ gd,
                            int64_t tail_nnz, const int32_t* __restrict__ tail_ptr, ProdCsr tail,
                            const double* __restrict__ x, double* __restrict__ y, const double* __restrict__ scale_p,
                            int32_t* __restrict__ list, unsigned int* __restrict__ n_long) {
  const double s = load_scale(scale_p);
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < n_rows;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t a = tail_nnz > 0 ? tail_ptr[r] : 0, b = tail_nnz > 0 ? tail_ptr[r + 1] : 0;
    if (b - a > EXACT_LONG) {
      append_long(list, n_long, r);
      continue;
    }
    double acc = ell_row_exact(n_rows, k, r, gi, gd, x);
    if (tail_nnz > 0) {  // y += bincount(...): every row, also those without tail entries
      double t = 0.0;
      for (int64_t i = a; i < b; ++i) t = t + tail(i);
      acc = acc + t;
    }
    store_row(y, r, acc, scale_p, s);
  }
}

// One CTA per row with a long tail: batches of products formed in parallel,
// added in order by one thread (bincount's sequential sum).
__global__ void __launch_bounds__(EXACT_THREADS) k_exact_hyb_long(const int32_t* __restrict__ list,
                                                                  const unsigned int* __restrict__ n_long,
                                                                  int64_t n_rows, int64_t k,
                                                                  const int32_t* __restrict__ gi,
                                                                  const double* __restrict__ gd,
                                                                  const int32_t* __restrict__ tail_ptr, ProdCsr tail,
                                                                  const double* __restrict__ x,
                                                                  double* __restrict__ y,
                                                                  const double* __restrict__ scale_p) {
  __shared__ double v[EXACT_BATCH];
  const double s = load_scale(scale_p);
  const unsigned int count = *n_long;
  for (unsigned int i = blockIdx.x; i < count; i += gridDim.x) {
    const int64_t r = list[i];
    const int64_t a = tail_ptr[r], b = tail_ptr[r + 1];
    double t = 0.0;
    for (int64_t p0 = a; p0 < b; p0 += EXACT_BATCH) {
      const int64_t m = b - p0 < EXACT_BATCH ? b - p0 : EXACT_BATCH;
      for (int64_t q = threadIdx.x; q < m; q += EXACT_THREADS) v[q] = tail(p0 + q);
      __syncthreads();
      if (threadIdx.x == 0)
        for (int64_t q = 0; q < m; ++q) t = t + v[q];
      __syncthreads();
    }
    if (threadIdx.x == 0) store_row(y, r, ell_row_exact(n_rows, k, r, gi, gd, x) + t, scale_p, s);
  }
}

struct LongRows {
  DevBuf<int32_t> list;
  DevBuf<unsigned int> count;
  LongRows(int64_t n_rows, int64_t nnz, cudaStream_t s)
      : list(static_cast<size_t>(std::min<int64_t>(n_rows, nnz / EXACT_LONG) + 1), s), count(1, s) {
    SPMVB_CUDA(cudaMemsetAsync(count.get(), 0, sizeof(unsigned int), s));
  }
};

constexpr unsigned LONG_GRID = 148 * 4;

}  // namespace

extern "C" int spmvb_spmv_csr_exact(int64_t n_rows, int64_t nnz, const int32_t* ptr, const int32_t* indices,
                                    const double* data, const double* x, double* y, const double* scale,
                                    void* stream) {
  return guard([&] {
    cudaStream_t s = as_stream(stream);
    if (n_rows <= 0) return;
    LongRows lr(n_rows, nnz, s);
    const ProdCsr at{indices, data, x};
    k_exact_csr<<<grid_for(n_rows, 128, 148 * 64), 128, 0, s>>>(n_rows, ptr, at, y, scale, lr.list.get(),
                                                               lr.count.get());
    SPMVB_LAUNCHED("k_exact_csr");
    if (nnz > EXACT_LONG) {
      k_exact_csr_long<<<LONG_GRID, EXACT_THREADS, 0, s>>>(lr.list.get(), lr.count.get(), ptr, at, y, scale);
      SPMVB_LAUNCHED("k_exact_csr_long");
    }
  });
}

extern "C" int spmvb_spmv_csr5_exact(int64_t n_rows, int64_t nnz, const int32_t* ptr, int omega, int sigma,
                                     const int32_t* indices, const double* data, const double* x, double* y,
                                     const double* scale, void* stream) {
  return guard([&] {
    cudaStream_t s = as_stream(stream);
    if (omega < 1 || sigma < 1) fail(SPMVB_INVALID_ARG, "omega and sigma must be >= 1, got %d, %d", omega, sigma);
    if (static_cast<int64_t>(omega) * sigma > INT32_MAX) fail(SPMVB_INVALID_ARG, "omega * sigma exceeds 2^31 - 1");
    if (n_rows <= 0) return;
    LongRows lr(n_rows, nnz, s);
    const ProdCsr5 at{indices, data, x, nnz, omega * sigma, sigma};
    k_exact_csr5<<<grid_for(n_rows, 128, 148 * 64), 128, 0, s>>>(n_rows, ptr, at, y, scale, lr.list.get(),
                                                                lr.count.get());
    SPMVB_LAUNCHED("k_exact_csr5");
    if (nnz > EXACT_LONG) {
      k_exact_csr5_long<<<LONG_GRID, EXACT_THREADS, 0, s>>>(lr.list.get(), lr.count.get(), ptr, at, y, scale);
      SPMVB_LAUNCHED("k_exact_csr5_long");
    }
  });
}

extern "C" int spmvb_spmv_hyb_exact(int64_t n_rows, int64_t k, const int32_t* ell_idx, const double* ell_val,
                                    int64_t tail_nnz, const int32_t* tail_ptr, const int32_t* tail_col,
                                    const double* tail_val, const double* x, double* y, const double* scale,
                                    void* stream) {
  return guard([&] {
    cudaStream_t s = as_stream(stream);
    if (n_rows <= 0) return;
    if (tail_nnz > 0 && !tail_ptr) fail(SPMVB_INVALID_ARG, "tail_ptr is required for a non-empty tail");
    LongRows lr(n_rows, tail_nnz, s);
    const ProdCsr tail{tail_col, tail_val, x};
    k_exact_hyb<<<grid_for(n_rows, 128, 148 * 64), 128, 0, s>>>(n_rows, k, ell_idx, ell_val, tail_nnz, tail_ptr, tail,
                                                               x, y, scale, lr.list.get(), lr.count.get());
    SPMVB_LAUNCHED("k_exact_hyb");
    if (tail_nnz > EXACT_LONG) {
      k_exact_hyb_long<<<LONG_GRID, EXACT_THREADS, 0, s>>>(lr.list.get(), lr.count.get(), n_rows, k, ell_idx, ell_val,
                                                           tail_ptr, tail, x, y, scale);
      SPMVB_LAUNCHED("k_exact_hyb_long");
    }
  });
}
