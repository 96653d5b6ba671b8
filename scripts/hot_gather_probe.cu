// Probe: does staging the hot head x[0, hot) of a degree-ordered x in shared
// memory raise the gather rate?  One persistent CTA per SM, `threads` threads,
// x[0, hot) copied into shared memory once, then the thread-strided sum of
// x[idx[i]] with U gathers in flight: LDS for idx < hot, LDG for the rest.
//   mode 0: per-lane select (predicated LDS / LDG)
//   mode 1: warp-uniform fast paths (all hot / none hot), per-lane otherwise
//   mode 2: no shared memory at all (the same persistent shape, LDG only)
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC
//        -o scripts/libhotprobe.so scripts/hot_gather_probe.cu
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

__device__ __forceinline__ int32_t ld_stream_i32(const int32_t* p) {
  int32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

template <int U, int MODE>
__global__ void __launch_bounds__(1024, 1) k_hot_sum(const double* __restrict__ src, const int32_t* __restrict__ idx,
                                                     int64_t n, int32_t hot, double* __restrict__ partial) {
  extern __shared__ double sx[];
  if (MODE != 2) {
    for (int i = threadIdx.x; i < hot; i += blockDim.x) sx[i] = src[i];
    __syncthreads();
  }
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t tid = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  double acc = 0.0;
  int64_t i = tid;
  for (; i + (U - 1) * stride < n; i += U * stride) {
    int32_t c[U];
#pragma unroll
    for (int u = 0; u < U; ++u) c[u] = ld_stream_i32(idx + i + u * stride);
    if (MODE == 2) {
#pragma unroll
      for (int u = 0; u < U; ++u) acc += __ldg(src + c[u]);
    } else if (MODE == 0) {
#pragma unroll
      for (int u = 0; u < U; ++u) acc += c[u] < hot ? sx[c[u]] : __ldg(src + c[u]);
    } else {
      bool allh = true, anyh = false;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        allh = allh && c[u] < hot;
        anyh = anyh || c[u] < hot;
      }
      if (__all_sync(0xffffffffu, allh)) {
#pragma unroll
        for (int u = 0; u < U; ++u) acc += sx[c[u]];
      } else if (!__any_sync(0xffffffffu, anyh)) {
#pragma unroll
        for (int u = 0; u < U; ++u) acc += __ldg(src + c[u]);
      } else {
#pragma unroll
        for (int u = 0; u < U; ++u) acc += c[u] < hot ? sx[c[u]] : __ldg(src + c[u]);
      }
    }
  }
  for (; i < n; i += stride) {
    const int32_t c = idx[i];
    acc += (MODE != 2 && c < hot) ? sx[c] : __ldg(src + c);
  }
  partial[tid] = acc;
}

// mode 3: the SpMV's own traffic without its row structure: the flat dot
// product sum val[i] * x[idx[i]] (12 streamed bytes + one gather per entry)
__device__ __forceinline__ double ld_stream_f64(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
template <int U>
__global__ void __launch_bounds__(1024, 1) k_dot(const double* __restrict__ src, const int32_t* __restrict__ idx,
                                                 const double* __restrict__ val, int64_t n,
                                                 double* __restrict__ partial) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t tid = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  double acc = 0.0;
  int64_t i = tid;
  for (; i + (U - 1) * stride < n; i += U * stride) {
    int32_t c[U];
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      c[u] = ld_stream_i32(idx + i + u * stride);
      v[u] = ld_stream_f64(val + i + u * stride);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u] * __ldg(src + c[u]);
  }
  for (; i < n; i += stride) acc += val[i] * __ldg(src + idx[i]);
  partial[tid] = acc;
}

template <int U, int MODE>
int launch(const double* src, const int32_t* idx, int64_t n, int32_t hot, int threads, int blocks, double* partial,
           cudaStream_t s) {
  const size_t smem = MODE == 2 ? 0 : static_cast<size_t>(hot) * 8;
  cudaError_t e = cudaFuncSetAttribute(k_hot_sum<U, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return static_cast<int>(e);
  k_hot_sum<U, MODE><<<blocks, threads, smem, s>>>(src, idx, n, hot, partial);
  return static_cast<int>(cudaGetLastError());
}

}  // namespace

extern "C" int dot_probe(const double* src, const int32_t* idx, const double* val, int64_t n, int threads, int blocks,
                         int u, double* partial, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (u == 4) k_dot<4><<<blocks, threads, 0, s>>>(src, idx, val, n, partial);
  else if (u == 8) k_dot<8><<<blocks, threads, 0, s>>>(src, idx, val, n, partial);
  else return -1;
  return static_cast<int>(cudaGetLastError());
}

extern "C" int hot_probe(const double* src, const int32_t* idx, int64_t n, int32_t hot, int threads, int blocks,
                         int mode, int u, double* partial, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
#define GO(U, M) \
  if (u == U && mode == M) return launch<U, M>(src, idx, n, hot, threads, blocks, partial, s);
  GO(4, 0) GO(4, 1) GO(4, 2) GO(8, 0) GO(8, 1) GO(8, 2) GO(16, 0) GO(16, 1) GO(16, 2)
#undef GO
  return -1;
}
