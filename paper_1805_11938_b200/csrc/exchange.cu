// Exchange kernels of the row-block power iteration.
// Sparse x exchange: each rank receives only the x entries its shard's
// columns touch, not the whole all-gathered vector; setup finds the shard's
// column set, every step the owner gathers the requested entries of its y
// block into one send buffer and the receiver scatters them into its x.
// Peer-memory exchange: rows pushed straight into the peers' buffers
// (spmvb_push_rows) and the norm slots folded in rank order.  Also the
// gather-rate probe behind bench.py's roofline.gather_bound.
#include "spmv_common.cuh"

using namespace spmvb;

namespace {

__global__ void k_mark_columns(const int32_t* __restrict__ col, int64_t nnz, uint8_t* __restrict__ flags) {
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < nnz;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x)
    flags[col[k]] = 1;
}

// Eight independent gathers in flight per thread (the L1TEX-bound regime:
// one distinct line per SM cycle needs thousands of loads outstanding).
constexpr int GU = 8;

__global__ void k_gather_f64(const double* __restrict__ src, int64_t base, const int32_t* __restrict__ idx, int64_t n,
                             double* __restrict__ dst) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  for (; i + (GU - 1) * stride < n; i += GU * stride) {
    int32_t c[GU];
#pragma unroll
    for (int u = 0; u < GU; ++u) c[u] = ld_stream(idx + i + u * stride);
    double v[GU];
#pragma unroll
    for (int u = 0; u < GU; ++u) v[u] = __ldg(src + (c[u] - base));
#pragma unroll
    for (int u = 0; u < GU; ++u) dst[i + u * stride] = v[u];
  }
  for (; i < n; i += stride) dst[i] = __ldg(src + (idx[i] - base));
}

__global__ void k_scatter_f64(const double* __restrict__ src, const int32_t* __restrict__ idx, int64_t n,
                              double* __restrict__ dst) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  for (; i + (GU - 1) * stride < n; i += GU * stride) {
    int32_t c[GU];
    double v[GU];
#pragma unroll
    for (int u = 0; u < GU; ++u) {
      c[u] = ld_stream(idx + i + u * stride);
      v[u] = ld_stream(src + i + u * stride);
    }
#pragma unroll
    for (int u = 0; u < GU; ++u) dst[c[u]] = v[u];
  }
  for (; i < n; i += stride) dst[idx[i]] = src[i];
}

// Gather-rate probe: sum of src[idx[i]] per thread (no per-element stores),
// sixteen gathers in flight per thread.  The SpMV of the same columns can
// only be slower: it is the roofline's L1TEX gather ceiling.
__global__ void k_gather_sum(const double* __restrict__ src, const int32_t* __restrict__ idx, int64_t n,
                             double* __restrict__ partial) {
  constexpr int U = 16;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t tid = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  double acc = 0.0;
  int64_t i = tid;
  for (; i + (U - 1) * stride < n; i += U * stride) {
    int32_t c[U];
#pragma unroll
    for (int u = 0; u < U; ++u) c[u] = ld_stream(idx + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) acc += __ldg(src + c[u]);
  }
  for (; i < n; i += stride) acc += __ldg(src + idx[i]);
  partial[tid] = acc;
}

// Stream + gather probe: the flat dot product sum val[i] * src[idx[i]] -- an
// SpMV's own traffic (12 streamed bytes and one x gather per entry) with no
// row structure at all (no pointers, permutation, y stores or carries,
// perfectly balanced).  An SpMV over the same entries cannot be faster.
__global__ void k_dot_sum(const double* __restrict__ src, const int32_t* __restrict__ idx,
                          const double* __restrict__ val, int64_t n, double* __restrict__ partial) {
  constexpr int U = 8;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t tid = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  double acc = 0.0;
  int64_t i = tid;
  for (; i + (U - 1) * stride < n; i += U * stride) {
    int32_t c[U];
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      c[u] = ld_stream(idx + i + u * stride);
      v[u] = ld_stream(val + i + u * stride);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u] * __ldg(src + c[u]);
  }
  for (; i < n; i += stride) acc += val[i] * __ldg(src + idx[i]);
  partial[tid] = acc;
}

// Rows [0, n) of src written into every peer buffer dst[p] + offset (peer
// addresses mapped over NVLink, e.g. symmetric-memory buffers): 16-byte
// vector stores where the alignment allows, one pass over src per launch.
__global__ void k_push_rows(const double* __restrict__ src, int64_t n, const uint64_t* __restrict__ dst, int n_peers,
                            int64_t offset) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t tid = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  // head element when offset is odd (peer buffers are 16-byte aligned)
  const int64_t head = (offset & 1) ? 1 : 0;
  if (head && tid == 0 && n > 0)
    for (int p = 0; p < n_peers; ++p) reinterpret_cast<double*>(dst[p])[offset] = src[0];
  const int64_t pairs = (n - head) / 2;
  for (int64_t i = tid; i < pairs; i += stride) {
    const int64_t e = head + 2 * i;
    const double a = src[e], b = src[e + 1];
    for (int p = 0; p < n_peers; ++p) {
      double2* d = reinterpret_cast<double2*>(reinterpret_cast<double*>(dst[p]) + offset + e);
      *d = make_double2(a, b);
    }
  }
  const int64_t last = head + 2 * pairs;
  if (last < n && tid == 0)
    for (int p = 0; p < n_peers; ++p) reinterpret_cast<double*>(dst[p])[offset + last] = src[last];
}

// sumsq = vals[0] + vals[1] + ... (rank order), scale = 1/sqrt(sumsq).
__global__ void k_sum_inv_sqrt(const double* __restrict__ vals, int n, double* __restrict__ sumsq,
                               double* __restrict__ scale) {
  double s = 0.0;
  for (int i = 0; i < n; ++i) s += vals[i];
  *sumsq = s;
  *scale = (s > 0.0) ? 1.0 / sqrt(s) : 1.0;  // as spmvb_inv_sqrt
}

}  // namespace

extern "C" int spmvb_column_set(const int32_t* col, int64_t nnz, int64_t n_cols, int32_t* cols_out, int64_t* n_out,
                                void* stream) {
  return guard([&] {
    cudaStream_t s = as_stream(stream);
    if (!n_out) fail(SPMVB_INVALID_ARG, "n_out is required");
    *n_out = 0;
    if (n_cols <= 0 || nnz <= 0) return;
    DevBuf<uint8_t> flags(n_cols, s);
    const uint8_t* f = flags.get();
    SPMVB_CUDA(cudaMemsetAsync(flags.get(), 0, n_cols, s));
    k_mark_columns<<<grid_for(nnz, 256, 148 * 16), 256, 0, s>>>(col, nnz, flags.get());
    SPMVB_LAUNCHED("k_mark_columns");
    DevBuf<int64_t> total(1, s);
    exclusive_scan<int64_t>(
        n_cols, [=] __device__(int64_t i) -> int64_t { return f[i]; },
        [=] __device__(int64_t i, int64_t v) {
          if (cols_out && f[i]) cols_out[v] = static_cast<int32_t>(i);
        },
        OpSum{}, int64_t{0}, total.get(), s);
    SPMVB_CUDA(cudaMemcpyAsync(n_out, total.get(), sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    SPMVB_CUDA(cudaStreamSynchronize(s));
  });
}

extern "C" int spmvb_gather_f64(const double* src, int64_t base, const int32_t* idx, int64_t n, double* dst,
                                void* stream) {
  return guard([&] {
    cudaStream_t s = as_stream(stream);
    if (n <= 0) return;
    k_gather_f64<<<grid_for(n, 256 * GU, 148 * 8), 256, 0, s>>>(src, base, idx, n, dst);
    SPMVB_LAUNCHED("k_gather_f64");
  });
}

extern "C" int spmvb_scatter_f64(const double* src, const int32_t* idx, int64_t n, double* dst, void* stream) {
  return guard([&] {
    cudaStream_t s = as_stream(stream);
    if (n <= 0) return;
    k_scatter_f64<<<grid_for(n, 256 * GU, 148 * 8), 256, 0, s>>>(src, idx, n, dst);
    SPMVB_LAUNCHED("k_scatter_f64");
  });
}

extern "C" int64_t spmvb_gather_probe_threads(void) { return 148 * 8 * 256; }

extern "C" int spmvb_gather_probe(const double* src, const int32_t* idx, int64_t n, double* partial, void* stream) {
  return guard([&] {
    cudaStream_t s = as_stream(stream);
    k_gather_sum<<<148 * 8, 256, 0, s>>>(src, idx, n, partial);
    SPMVB_LAUNCHED("k_gather_sum");
  });
}

extern "C" int spmvb_dot_probe(const double* src, const int32_t* idx, const double* val, int64_t n, double* partial,
                               void* stream) {
  return guard([&] {
    cudaStream_t s = as_stream(stream);
    k_dot_sum<<<148 * 8, 256, 0, s>>>(src, idx, val, n, partial);
    SPMVB_LAUNCHED("k_dot_sum");
  });
}

extern "C" int spmvb_push_rows(const double* src, int64_t n, const uint64_t* dst_ptrs, int n_peers, int64_t offset,
                               void* stream) {
  return guard([&] {
    cudaStream_t s = as_stream(stream);
    if (n <= 0 || n_peers <= 0) return;
    if (!dst_ptrs) fail(SPMVB_INVALID_ARG, "dst_ptrs is required");
    k_push_rows<<<grid_for((n + 1) / 2, 256, 148 * 8), 256, 0, s>>>(src, n, dst_ptrs, n_peers, offset);
    SPMVB_LAUNCHED("k_push_rows");
  });
}

extern "C" int spmvb_sum_inv_sqrt(const double* vals, int n, double* sumsq, double* scale, void* stream) {
  return guard([&] {
    cudaStream_t s = as_stream(stream);
    if (n < 1) fail(SPMVB_INVALID_ARG, "n must be >= 1");
    k_sum_inv_sqrt<<<1, 1, 0, s>>>(vals, n, sumsq, scale);
    SPMVB_LAUNCHED("k_sum_inv_sqrt");
  });
}
