// GPU feature extraction for the format selector
// (reference features.py:69-84, FEATURE_NAMES :33-42).
//
// The standard deviation reproduces numpy bit for bit: counts.std() computes
// mean = sum/n (exact integer sum, correctly rounded division), squared
// deviations d_i*d_i rounded separately, then add.reduce = 0 + pairwise(s)
// over all n values, divided by n, then sqrt.  The pairwise tree is
// evaluated exactly: kernel 1 computes every subtree rooted at depth L
// (2^L virtual nodes; subtrees that become leaves higher up are computed by
// their leftmost virtual descendant), kernel 2 combines the top L levels in
// shared memory in the same left+right order as numpy's recursion.
#include "prims.cuh"

using namespace spmvb;

namespace {

constexpr int FEAT_LEAF_TARGET = 4096;  // max elements per depth-L subtree
constexpr int FEAT_MAX_L = 13;          // 2^13 virtual nodes (64 KB of doubles)

struct SqDev {
  const int32_t* ptr;
  double mean;
  __device__ double operator()(int64_t i) const {
    double c = static_cast<double>(ptr[i + 1] - ptr[i]);
    double d = __dsub_rn(c, mean);
    return __dmul_rn(d, d);
  }
};

// Descend `d` levels from the root following the bits of `idx` (MSB first);
// returns false if a leaf (len <= 128) is met before depth d and idx is not
// that leaf's leftmost virtual descendant.
__device__ bool pw_descend(int64_t n, int d, int64_t idx, int64_t& off, int64_t& len, int& leaf_depth) {
  off = 0;
  len = n;
  leaf_depth = -1;
  for (int l = 0; l < d; ++l) {
    if (len <= 128) {
      leaf_depth = l;
      int64_t rest = idx & ((1ll << (d - l)) - 1);
      return rest == 0;
    }
    int64_t n2 = len / 2;
    n2 -= n2 % 8;
    if ((idx >> (d - 1 - l)) & 1) {
      off += n2;
      len -= n2;
    } else {
      len = n2;
    }
  }
  if (len <= 128) leaf_depth = d;
  return true;
}

__global__ void k_pw_subtrees(int64_t n, int L, SqDev at, double* __restrict__ out) {
  int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (idx >= (1ll << L)) return;
  int64_t off, len;
  int leaf_depth;
  bool rep = pw_descend(n, L, idx, off, len, leaf_depth);
  out[idx] = rep ? np_pairwise(at, off, len) : 0.0;
}

__global__ void k_pw_combine(int64_t n, int L, const double* __restrict__ sub, double* __restrict__ total) {
  extern __shared__ double v[];
  const int64_t m = 1ll << L;
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x) v[i] = sub[i];
  __syncthreads();
  for (int d = L - 1; d >= 0; --d) {
    for (int64_t i = threadIdx.x; i < (1ll << d); i += blockDim.x) {
      int64_t off, len;
      int leaf_depth;
      bool rep = pw_descend(n, d, i, off, len, leaf_depth);
      if (rep && len > 128) {  // internal node: left + right
        int64_t b = i << (L - d);
        v[b] = v[b] + v[b + (1ll << (L - d - 1))];
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = 0.0 + v[0];
}

__global__ void k_extra_features(int64_t n_rows, int64_t n_cols, const int32_t* __restrict__ ptr,
                                 const int32_t* __restrict__ col, unsigned long long* __restrict__ out2) {
  unsigned long long bw = 0, diag = 0;
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < n_rows;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int32_t a = ptr[r], b = ptr[r + 1];
    if (b <= a) continue;
    int64_t c0 = col[a], c1 = col[b - 1];  // columns ascend within a row
    int64_t d0 = r > c0 ? r - c0 : c0 - r, d1 = r > c1 ? r - c1 : c1 - r;
    unsigned long long m = static_cast<unsigned long long>(d0 > d1 ? d0 : d1);
    bw = m > bw ? m : bw;
    if (r < n_cols && c0 <= r && r <= c1) {
      int32_t lo = a, hi = b;
      while (lo < hi) {
        int32_t mid = (lo + hi) >> 1;
        if (col[mid] < r) lo = mid + 1; else hi = mid;
      }
      if (lo < b && col[lo] == r) ++diag;
    }
  }
  for (int d = 16; d >= 1; d >>= 1) {
    unsigned long long ob = __shfl_down_sync(0xffffffffu, bw, d);
    bw = ob > bw ? ob : bw;
    diag += __shfl_down_sync(0xffffffffu, diag, d);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(&out2[0], bw);
    atomicAdd(&out2[1], diag);
  }
}

}  // namespace

extern "C" int spmvb_csr_features(int64_t n_rows, int64_t n_cols, int64_t nnz, const int32_t* ptr, double* out8,
                                  void* stream) {
  return guard([&] {
    cudaStream_t s = as_stream(stream);
    if (n_rows == 0 || n_cols == 0)
      fail(SPMVB_INVALID_ARG, "features are undefined for a %lldx%lld matrix", (long long)n_rows, (long long)n_cols);
    int64_t st[3];
    {
      DevBuf<int64_t> d(2, s);
      int64_t* dp = d.get();
      auto cnt = [=] __device__(int64_t i) { return static_cast<int64_t>(ptr[i + 1] - ptr[i]); };
      device_reduce<int64_t>(n_rows, cnt, OpMin{}, INT64_MAX, dp + 0, s);
      device_reduce<int64_t>(n_rows, cnt, OpMax{}, (int64_t)0, dp + 1, s);
      copy_to_host(st, dp, 2, s);
    }
    const double mean = static_cast<double>(nnz) / static_cast<double>(n_rows);
    int L = 0;
    while (L < FEAT_MAX_L && (n_rows >> L) > FEAT_LEAF_TARGET) ++L;
    DevBuf<double> sub(1ll << L, s), total(1, s);
    SqDev at{ptr, mean};
    k_pw_subtrees<<<grid_for(1ll << L, 128), 128, 0, s>>>(n_rows, L, at, sub.get());
    SPMVB_LAUNCHED("k_pw_subtrees");
    const size_t smem = (1ll << L) * sizeof(double);  // up to 64 KB: above the default 48 KB
    SPMVB_CUDA(cudaFuncSetAttribute(k_pw_combine, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_pw_combine<<<1, 1024, smem, s>>>(n_rows, L, sub.get(), total.get());
    SPMVB_LAUNCHED("k_pw_combine");
    double sumsq = 0.0;
    copy_to_host(&sumsq, total.get(), 1, s);
    const double var = sumsq / static_cast<double>(n_rows);
    const double sd = sqrt(var);
    // nnz / (n_rows * n_cols) is exact when the product fits in 53 bits; the
    // Python layer recomputes it with exact integer division in any case.
    long double prod = static_cast<long double>(n_rows) * static_cast<long double>(n_cols);
    out8[0] = static_cast<double>(n_rows);
    out8[1] = static_cast<double>(n_cols);
    out8[2] = static_cast<double>(static_cast<long double>(nnz) / prod);
    out8[3] = static_cast<double>(st[0]);
    out8[4] = static_cast<double>(st[1]);
    out8[5] = mean;
    out8[6] = sd;
    out8[7] = mean > 0.0 ? sd / mean : 0.0;
  });
}

extern "C" int spmvb_csr_extra_features(int64_t n_rows, int64_t n_cols, const int32_t* ptr, const int32_t* col,
                                        double* out2, void* stream) {
  return guard([&] {
    cudaStream_t s = as_stream(stream);
    DevBuf<unsigned long long> d(2, s);
    SPMVB_CUDA(cudaMemsetAsync(d.get(), 0, 2 * sizeof(unsigned long long), s));
    if (n_rows > 0) {
      k_extra_features<<<grid_for(n_rows, 256, 148 * 8), 256, 0, s>>>(n_rows, n_cols, ptr, col, d.get());
      SPMVB_LAUNCHED("k_extra_features");
    }
    unsigned long long h[2];
    copy_to_host(h, d.get(), 2, s);
    int64_t mn = n_rows < n_cols ? n_rows : n_cols;
    out2[0] = static_cast<double>(h[0]);
    out2[1] = mn > 0 ? static_cast<double>(h[1]) / static_cast<double>(mn) : 0.0;
  });
}
