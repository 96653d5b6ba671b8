// Micro-benchmark: random fp64 gathers x[idx[i]] on B200 through the LSU
// (LDG, L1TEX wavefront-limited) versus the TMA unit (cp.async.bulk.tensor
// .2d .tile::gather4: four 16-byte rows per instruction into shared memory).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_bench scripts/gather_bench.cu -lcuda
//   ./gather_bench [log2_n=25] [log2_m=26] [mode=rmat|uniform|sorted] [hot_cols=0]
// sorted = R-MAT columns relabelled by descending probability (popcount, then colex rank), i.e. the
// hot columns packed at the front of x; hot_cols > 0 additionally serves x[0..hot_cols) from shared memory.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__global__ void k_ldg_hot(const double* __restrict__ x, const int* __restrict__ idx, int64_t m, double* out,
                          int hot) {
  extern __shared__ double xs[];
  for (int i = threadIdx.x; i < hot; i += blockDim.x) xs[i] = x[i];
  __syncthreads();
  double acc = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 15 * stride < m; i += 16 * stride) {
    int c[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) c[u] = __ldg(idx + i + u * stride);
#pragma unroll
    for (int u = 0; u < 16; ++u) acc += c[u] < hot ? xs[c[u]] : __ldg(x + c[u]);
  }
  for (; i < m; i += stride) {
    const int c = __ldg(idx + i);
    acc += c < hot ? xs[c] : __ldg(x + c);
  }
  out[(int64_t)blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

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

// LDG and TMA gathers side by side: each CTA chunk = MIX_L LSU gathers (8 warps) + MIX_T TMA gather4 rows
// (issued by warp 8 one chunk ahead, double-buffered); tests whether the TMA unit adds gather throughput
// on top of the LSU's ~1 line/clk.
constexpr int MIX_L = 4096;
template <int MIX_T>
__global__ void __launch_bounds__(288) k_mix(const __grid_constant__ CUtensorMap tm, const double* __restrict__ x,
                                             const int* __restrict__ idx, int64_t nchunks, double* out) {
  __shared__ __align__(128) double buf[2][MIX_T * 4];
  __shared__ uint64_t bar[2];
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  constexpr int CH = MIX_L + MIX_T;
  if (tid == 0) {
    for (int s = 0; s < 2; ++s) {
      uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar[s]);
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int64_t ch, int s) {
    uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar[s]);
    if (lane == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(MIX_T * 32) : "memory");
    __syncwarp();
    for (int g = lane; g < MIX_T / 4; g += 32) {
      const int4 c4 = *reinterpret_cast<const int4*>(idx + ch * CH + MIX_L + g * 4);
      uint32_t d = (uint32_t)__cvta_generic_to_shared(&buf[s][g * 16]);
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, "
          "{%2, %3, %4, %5, %6}], [%7];" ::"r"(d),
          "l"(&tm), "r"(0), "r"(c4.x >> 2), "r"(c4.y >> 2), "r"(c4.z >> 2), "r"(c4.w >> 2), "r"(b)
          : "memory");
    }
  };
  double acc = 0.0;
  int64_t ch = blockIdx.x;
  if (warp == 8 && ch < nchunks) issue(ch, 0);
  int s = 0, phase[2] = {0, 0};
  for (; ch < nchunks; ch += gridDim.x) {
    const int64_t nxt = ch + gridDim.x;
    if (warp == 8) {
      if (nxt < nchunks) issue(nxt, s ^ 1);
    } else {
      const int* ci = idx + ch * CH;
      int c[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) c[u] = __ldg(ci + tid + u * 256);
#pragma unroll
      for (int u = 0; u < 16; ++u) acc += __ldg(x + c[u]);
    }
    uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar[s]);
    asm volatile(
        "{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(b),
        "r"(phase[s])
        : "memory");
    phase[s] ^= 1;
    if (warp < 8)
      for (int j = tid; j < MIX_T; j += 256) acc += buf[s][j * 4 + (__ldg(idx + ch * CH + MIX_L + j) & 3)];
    __syncthreads();
    s ^= 1;
  }
  out[(int64_t)blockIdx.x * blockDim.x + tid] = acc;
}

// Texture-path gathers (tex1Dfetch<int2> over linear memory), optionally mixed with LSU gathers: every
// `every`-th unrolled gather goes through TEX, the rest through LDG (every = 1: all TEX).
__global__ void k_tex(cudaTextureObject_t tx, const double* __restrict__ x, const int* __restrict__ idx, int64_t m,
                      double* out, int every) {
  double acc = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 15 * stride < m; i += 16 * stride) {
    int c[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) c[u] = __ldg(idx + i + u * stride);
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      if (u % every == 0) {
        const int2 t = tex1Dfetch<int2>(tx, c[u]);
        acc += __hiloint2double(t.y, t.x);
      } else {
        acc += __ldg(x + c[u]);
      }
    }
  }
  out[(int64_t)blockIdx.x * blockDim.x + threadIdx.x] = acc;
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
  const bool sorted = argc > 3 && argv[3][0] == 's';
  const int hot = argc > 4 ? atoi(argv[4]) : 0;
  std::vector<std::vector<int64_t>> binom(ln + 1, std::vector<int64_t>(ln + 2, 0));
  for (int a = 0; a <= ln; ++a) {
    binom[a][0] = 1;
    for (int b = 1; b <= a; ++b) binom[a][b] = binom[a - 1][b - 1] + (b <= a - 1 ? binom[a - 1][b] : 0);
  }
  auto relabel = [&](int c) {  // rank by (popcount, colex)
    int pc = __builtin_popcount(c);
    int64_t r = 0;
    for (int k = 0; k < pc; ++k) r += binom[ln][k];
    int i = 0;
    for (int b = 0; b < ln; ++b)
      if (c >> b & 1) r += (++i <= b) ? binom[b][i] : 0;
    return (int)r;
  };
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
    hidx[i] = sorted ? relabel(c) : c;
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
  {
    cudaResourceDesc rd = {};
    rd.resType = cudaResourceTypeLinear;
    rd.res.linear.devPtr = x;
    rd.res.linear.desc = cudaCreateChannelDesc<int2>();
    rd.res.linear.sizeInBytes = n * 8;
    cudaTextureDesc td = {};
    td.readMode = cudaReadModeElementType;
    cudaTextureObject_t tx;
    CK(cudaCreateTextureObject(&tx, &rd, &td, nullptr));
    for (int every : {1, 2, 4, 8}) {
      for (int blocks : {148 * 8, 148 * 16}) {
        k_tex<<<blocks, 256>>>(tx, x, idx, m, out, every);
        CK(cudaGetLastError());
        cudaEventRecord(a);
        for (int r = 0; r < 5; ++r) k_tex<<<blocks, 256>>>(tx, x, idx, m, out, every);
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        cudaEventElapsedTime(&ms, a, b);
        printf("TEX 1/%d blocks=%d: %.3f ms/pass, %.1f Ggathers/s\n", every, blocks, ms / 5, m / (ms / 5 * 1e-3) / 1e9);
      }
    }
  }
  if (hot > 0) {
    CK(cudaFuncSetAttribute(k_ldg_hot, cudaFuncAttributeMaxDynamicSharedMemorySize, hot * 8));
    for (int blocks : {148, 148 * 2}) {
      int tpb = blocks == 148 ? 1024 : 512;
      if (hot * 8 * (blocks / 148) > 220 * 1024) continue;
      k_ldg_hot<<<blocks, tpb, hot * 8>>>(x, idx, m, out, hot);
      CK(cudaGetLastError());
      cudaEventRecord(a);
      for (int r = 0; r < 5; ++r) k_ldg_hot<<<blocks, tpb, hot * 8>>>(x, idx, m, out, hot);
      cudaEventRecord(b);
      CK(cudaEventSynchronize(b));
      cudaEventElapsedTime(&ms, a, b);
      printf("HOT%d blocks=%d: %.3f ms/pass, %.1f Ggathers/s\n", hot, blocks, ms / 5, m / (ms / 5 * 1e-3) / 1e9);
    }
    for (int blocks : {148, 148 * 2}) {
      int tpb = blocks == 148 ? 1024 : 512;
      k_ldg<<<blocks, tpb>>>(x, idx, m, out);
      cudaEventRecord(a);
      for (int r = 0; r < 5; ++r) k_ldg<<<blocks, tpb>>>(x, idx, m, out);
      cudaEventRecord(b);
      CK(cudaEventSynchronize(b));
      cudaEventElapsedTime(&ms, a, b);
      printf("LDG  blocks=%d tpb=%d: %.3f ms/pass, %.1f Ggathers/s\n", blocks, tpb, ms / 5, m / (ms / 5 * 1e-3) / 1e9);
    }
    return 0;
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
  auto mix = [&](auto kern, int mt) {
    const int64_t nch = m / (MIX_L + mt);
    for (int blocks : {148 * 4, 148 * 7}) {
      kern<<<blocks, 288>>>(tm, x, idx, nch, out);
      CK(cudaGetLastError());
      CK(cudaDeviceSynchronize());
      cudaEventRecord(a);
      for (int rr = 0; rr < 5; ++rr) kern<<<blocks, 288>>>(tm, x, idx, nch, out);
      cudaEventRecord(b);
      CK(cudaEventSynchronize(b));
      cudaEventElapsedTime(&ms, a, b);
      printf("MIX T=%d blocks=%d: %.3f ms/pass, %.1f Ggathers/s\n", mt, blocks, ms / 5,
             nch * (MIX_L + mt) / (ms / 5 * 1e-3) / 1e9);
    }
  };
  mix(k_mix<256>, 256);
  mix(k_mix<512>, 512);

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
