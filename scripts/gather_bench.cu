// Micro-benchmark: random fp64 gathers x[idx[i]] on B200 through the LSU
// (LDG, L1TEX wavefront-limited) versus the TMA unit (cp.async.bulk.tensor
// .2d .tile::gather4: four 16-byte rows per instruction into shared memory).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_bench scripts/gather_bench.cu -lcuda
//   ./gather_bench [log2_n=25] [log2_m=26] [mode=rmat|uniform]
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__global__ void k_ldg(const double* __restrict__ x, const int* __restrict__ idx, int64_t m, double* out) {
  double acc = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 15 * stride < m; i += 16 * stride) {
    int c[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) c[u] = __ldg(idx + i + u * stride);
#pragma unroll
    for (int u = 0; u < 16; ++u) acc += __ldg(x + c[u]);
  }
  for (; i < m; i += stride) acc += __ldg(x + __ldg(idx + i));
  out[(int64_t)blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

constexpr int CH = 512;  // gathers per chunk per CTA
constexpr int TPB = 128;

__global__ void __launch_bounds__(TPB) k_tma(const __grid_constant__ CUtensorMap tm, const int* __restrict__ idx,
                                             int64_t m, double* out) {
  __shared__ __align__(128) double buf[2][CH * 4];  // one 32-byte row (sector) per gathered index
  __shared__ uint64_t bar[2];
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < 2; ++s) {
      uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar[s]);
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  double acc = 0.0;
  const int64_t nchunks = m / CH;
  int phase[2] = {0, 0};
  auto issue = [&](int64_t ch, int s) {
    // warp 0 issues CH/4 gather4 instructions (8 per lane)
    if (tid < 32) {
      uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar[s]);
      if (tid == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(CH * 32) : "memory");
      __syncwarp();
      for (int g = tid; g < CH / 4; g += 32) {
        const int4 c4 = *reinterpret_cast<const int4*>(idx + ch * CH + g * 4);
        uint32_t d = (uint32_t)__cvta_generic_to_shared(&buf[s][g * 16]);
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, "
            "{%2, %3, %4, %5, %6}], [%7];" ::"r"(d),
            "l"(&tm), "r"(0), "r"(c4.x >> 2), "r"(c4.y >> 2), "r"(c4.z >> 2), "r"(c4.w >> 2), "r"(b)
            : "memory");
      }
    }
  };
  int64_t ch = blockIdx.x;
  if (ch < nchunks) issue(ch, 0);
  int s = 0;
  for (; ch < nchunks; ch += gridDim.x) {
    const int64_t nxt = ch + gridDim.x;
    if (nxt < nchunks) issue(nxt, s ^ 1);
    uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar[s]);
    asm volatile(
        "{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(b),
        "r"(phase[s])
        : "memory");
    phase[s] ^= 1;
    for (int j = tid; j < CH; j += TPB) {
      const int c = __ldg(idx + ch * CH + j);
      acc += buf[s][j * 4 + (c & 3)];
    }
    __syncthreads();
    s ^= 1;
  }
  out[(int64_t)blockIdx.x * blockDim.x + tid] = acc;
}

static uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

int main(int argc, char** argv) {
  const int ln = argc > 1 ? atoi(argv[1]) : 25, lm = argc > 2 ? atoi(argv[2]) : 26;
  const bool rmat = !(argc > 3 && argv[3][0] == 'u');
  const int64_t n = 1ll << ln, m = 1ll << lm;
  std::vector<int> hidx(m);
  for (int64_t i = 0; i < m; ++i) {
    uint64_t h = mix64(i * 977 + 13);
    int c = 0;
    if (rmat) {
      for (int l = 0; l < ln; ++l) {
        double u = (double)(mix64(h ^ (l * 0x1234567ull)) >> 11) * 0x1.0p-53;
        c = (c << 1) | ((u >= 0.57 && u < 0.76) || u >= 0.95 ? 1 : 0);
      }
    } else {
      c = (int)(h % n);
    }
    hidx[i] = c;
  }
  double *x, *out;
  int* idx;
  CK(cudaMalloc(&x, n * 8));
  CK(cudaMalloc(&idx, m * 4));
  CK(cudaMalloc(&out, 148 * 64 * 1024 * 8));
  CK(cudaMemset(x, 0, n * 8));
  CK(cudaMemcpy(idx, hidx.data(), m * 4, cudaMemcpyHostToDevice));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms;
  for (int blocks : {148 * 8, 148 * 16}) {
    k_ldg<<<blocks, 256>>>(x, idx, m, out);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) k_ldg<<<blocks, 256>>>(x, idx, m, out);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    cudaEventElapsedTime(&ms, a, b);
    printf("LDG  blocks=%d: %.3f ms/pass, %.1f Ggathers/s\n", blocks, ms / 5, m / (ms / 5 * 1e-3) / 1e9);
  }
  // tensor map: x as (n/2 rows) x (2 cols) of f64, box 2 x 1
  typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                               const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                               CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  CUtensorMap tm;
  cuuint64_t dims[2] = {4, (cuuint64_t)(n / 4)};
  cuuint64_t strides[1] = {32};
  cuuint32_t box[2] = {4, 1};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, x, dims, strides, box, estr,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                      CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    printf("cuTensorMapEncodeTiled failed: %d\n", (int)r);
    return 1;
  }
  for (int blocks : {148 * 4, 148 * 8, 148 * 16}) {
    k_tma<<<blocks, TPB>>>(tm, idx, m, out);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    cudaEventRecord(a);
    for (int rr = 0; rr < 5; ++rr) k_tma<<<blocks, TPB>>>(tm, idx, m, out);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    cudaEventElapsedTime(&ms, a, b);
    printf("TMA  blocks=%d: %.3f ms/pass, %.1f Ggathers/s\n", blocks, ms / 5, m / (ms / 5 * 1e-3) / 1e9);
  }
  return 0;
}
