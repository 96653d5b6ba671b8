// Degree-ordered symmetric relabelling (an internal shadow layout for
// iterative SpMV on square matrices; the reference's arrays are untouched).
//
// New ids sort rows/columns by (row is empty, -(row degree + column degree)),
// stable by old id: every empty row goes last (the CSR5 tile kernel then
// needs no non-empty-row indirection and zeroes the tail with plain stores),
// and the hot columns of a power-law matrix are packed into the first x
// lines (more L1/L2 hits per gathered line).  The power iteration runs on
// P A P^T with x' = P x and maps back with x = P^T x' (spmvb_gather_f64).
// R-MAT scale 25: CSR5 SpMV 2.84 -> 2.45 ms; scale 21: 107.5 -> 97.3 us
// (scripts/relabel_probe.py, profiles/r02_relabel_probe_c{4,5}.txt).
#include "common.cuh"
#include "prims.cuh"

using namespace spmvb;

namespace {

__global__ void k_col_degree(const int32_t* __restrict__ col, int64_t nnz, int32_t* __restrict__ deg) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < nnz; k += stride)
    atomicAdd(deg + ld_stream(col + k), 1);
}

// mode 0: key(i) = empty(i) << dbits | (max_sum - (rowdeg(i) + coldeg(i)))
// mode 1: key(i) = empty(i) << dbits | (max_rd - rowdeg(i)) << cbits | (max_cd - coldeg(i))
//         (rows in exact descending length: SELL slices need no sigma window)
__global__ void k_degree_keys(const int32_t* __restrict__ ptr, const int32_t* __restrict__ coldeg, int64_t n,
                              int mode, uint64_t max_a, uint64_t max_b, int cbits, int dbits,
                              uint64_t* __restrict__ keys) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n; i += stride) {
    const uint64_t rd = static_cast<uint64_t>(ptr[i + 1] - ptr[i]);
    const uint64_t cd = static_cast<uint64_t>(coldeg[i]);
    const uint64_t low = mode == 0 ? max_a - (rd + cd) : ((max_a - rd) << cbits) | (max_b - cd);
    keys[i] = (static_cast<uint64_t>(rd == 0) << dbits) | low;
  }
}

__global__ void k_invert_perm(const uint32_t* __restrict__ order, int64_t n, int32_t* __restrict__ perm,
                              int32_t* __restrict__ new_id) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n; i += stride) {
    const int32_t old = static_cast<int32_t>(order ? order[i] : static_cast<uint32_t>(i));
    perm[i] = old;
    new_id[old] = static_cast<int32_t>(i);
  }
}

__global__ void k_relabel_entries(int64_t nnz, const int32_t* __restrict__ new_id, const int32_t* __restrict__ col,
                                  const double* __restrict__ val, int32_t* __restrict__ row_io,
                                  int32_t* __restrict__ col_out, double* __restrict__ val_out) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < nnz; k += stride) {
    row_io[k] = __ldg(new_id + row_io[k]);
    col_out[k] = __ldg(new_id + ld_stream(col + k));
    val_out[k] = ld_stream(val + k);
  }
}

}  // namespace

extern "C" int spmvb_degree_order(int64_t n, const int32_t* ptr, const int32_t* col, int64_t nnz, int mode,
                                  int32_t* perm, int32_t* new_id, int64_t* n_nonempty, void* stream) {
  return guard([&] {
    cudaStream_t s = as_stream(stream);
    if (n < 0 || nnz < 0) fail(SPMVB_INVALID_ARG, "negative size");
    if (mode != 0 && mode != 1) fail(SPMVB_INVALID_ARG, "mode must be 0 (row + column degree) or 1 (row degree)");
    if (!n_nonempty) fail(SPMVB_INVALID_ARG, "n_nonempty is required");
    *n_nonempty = 0;
    if (n == 0) return;
    DevBuf<int32_t> deg(n, s);
    SPMVB_CUDA(cudaMemsetAsync(deg.get(), 0, n * sizeof(int32_t), s));
    if (nnz > 0) {
      k_col_degree<<<grid_for(nnz, 256, 148 * 16), 256, 0, s>>>(col, nnz, deg.get());
      SPMVB_LAUNCHED("k_col_degree");
    }
    const int32_t* dg = deg.get();
    DevBuf<int64_t> stats(4, s);
    device_reduce<int64_t>(
        n, [=] __device__(int64_t i) { return static_cast<int64_t>(ptr[i + 1] - ptr[i]) + dg[i]; }, OpMax{},
        (int64_t)0, stats.get(), s);
    device_reduce<int64_t>(
        n, [=] __device__(int64_t i) { return static_cast<int64_t>(ptr[i + 1] > ptr[i]); }, OpSum{}, (int64_t)0,
        stats.get() + 1, s);
    device_reduce<int64_t>(
        n, [=] __device__(int64_t i) { return static_cast<int64_t>(ptr[i + 1] - ptr[i]); }, OpMax{}, (int64_t)0,
        stats.get() + 2, s);
    device_reduce<int64_t>(
        n, [=] __device__(int64_t i) { return static_cast<int64_t>(dg[i]); }, OpMax{}, (int64_t)0, stats.get() + 3, s);
    int64_t h[4];
    copy_to_host(h, stats.get(), 4, s);
    *n_nonempty = h[1];
    const uint64_t max_a = static_cast<uint64_t>(mode == 0 ? h[0] : h[2]);
    const uint64_t max_b = static_cast<uint64_t>(h[3]);
    const int cbits = bits_for(max_b);
    const int dbits = mode == 0 ? bits_for(max_a) : bits_for(max_a) + cbits;
    DevBuf<uint64_t> ka(n, s), kb(n, s);
    DevBuf<uint32_t> vb(n, s), vs(n, s);
    k_degree_keys<<<grid_for(n, 256, 148 * 16), 256, 0, s>>>(ptr, dg, n, mode, max_a, max_b, cbits, dbits, ka.get());
    SPMVB_LAUNCHED("k_degree_keys");
    RadixSortResult rs = radix_sort_pairs(ka.get(), nullptr, kb.get(), vb.get(), vs.get(), n, dbits + 1, s);
    k_invert_perm<<<grid_for(n, 256, 148 * 16), 256, 0, s>>>(rs.vals, n, perm, new_id);
    SPMVB_LAUNCHED("k_invert_perm");
  });
}

extern "C" int spmvb_relabel_csr(int64_t n, const int32_t* ptr, const int32_t* col, const double* val, int64_t nnz,
                                 const int32_t* new_id, int32_t* row_out, int32_t* col_out, double* val_out,
                                 void* stream) {
  return guard([&] {
    cudaStream_t s = as_stream(stream);
    if (n < 0 || nnz < 0) fail(SPMVB_INVALID_ARG, "negative size");
    if (nnz == 0 || n == 0) return;
    if (const int st = spmvb_csr_expand_rows(ptr, n, row_out, stream)) {
      const std::string msg = spmvb_last_error();
      fail(st, "%s", msg.c_str());
    }
    k_relabel_entries<<<grid_for(nnz, 256, 148 * 16), 256, 0, s>>>(nnz, new_id, col, val, row_out, col_out, val_out);
    SPMVB_LAUNCHED("k_relabel_entries");
  });
}
