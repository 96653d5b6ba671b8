// Shared infrastructure for the spmvb C-ABI library (B200 / sm_100a only).
//
// Error model: internal code throws spmvb::Failure; every extern "C" entry
// point is wrapped by spmvb::guard(), which converts the exception into an
// integer status and a thread-local message (spmvb_last_error()).  Status
// values are declared in include/spmvb.h.
#pragma once

#include <cuda_runtime.h>
#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstdarg>
#include <cstdlib>
#include <mutex>
#include <string>
#include <utility>

#include "../../include/spmvb.h"

namespace spmvb {

struct Failure {
  int status;
};

void set_error_message(const char* fmt, ...);

[[noreturn]] inline void fail(int status, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  set_error_message("%s", buf);
  throw Failure{status};
}

[[noreturn]] inline void fail_cuda(cudaError_t e, const char* what, const char* file, int line) {
  int status = (e == cudaErrorMemoryAllocation) ? SPMVB_OUT_OF_MEMORY : SPMVB_CUDA_ERROR;
  fail(status, "CUDA error %s (%s) in %s at %s:%d", cudaGetErrorName(e), cudaGetErrorString(e),
       what, file, line);
}

#define SPMVB_CUDA(call)                                            \
  do {                                                              \
    cudaError_t e__ = (call);                                       \
    if (e__ != cudaSuccess) ::spmvb::fail_cuda(e__, #call, __FILE__, __LINE__); \
  } while (0)

extern std::atomic<unsigned long long> g_launches;  // kernels launched by this library

#define SPMVB_LAUNCHED(name)                                        \
  do {                                                              \
    ::spmvb::g_launches.fetch_add(1, std::memory_order_relaxed);    \
    cudaError_t e__ = cudaGetLastError();                           \
    if (e__ != cudaSuccess) ::spmvb::fail_cuda(e__, name, __FILE__, __LINE__); \
  } while (0)

template <typename F>
int guard(F&& f) {
  try {
    f();
    return SPMVB_OK;
  } catch (const Failure& e) {
    return e.status;
  } catch (...) {
    set_error_message("unexpected C++ exception");
    return SPMVB_INTERNAL;
  }
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// The stream-ordered pool returns freed memory to the driver at every
// synchronization by default (release threshold 0), so a conversion that
// syncs between phases re-maps its multi-GB temporaries each call.  Keep up
// to 32 GB cached per device (cheap against 180 GB of HBM; canonicalize of
// the 5.3e8-entry C5 holds ~21 GB of temporaries at its peak).
inline void pool_keep_memory() {
  static std::atomic<uint64_t> done_mask{0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return;
  const uint64_t bit = 1ull << dev;
  if (done_mask.load(std::memory_order_relaxed) & bit) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = 32ull << 30;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done_mask.fetch_or(bit);
}

// Stream-ordered temporary device buffer (cudaMallocAsync / cudaFreeAsync).
template <typename T>
struct DevBuf {
  T* ptr = nullptr;
  size_t count = 0;
  cudaStream_t stream = nullptr;
  DevBuf() = default;
  DevBuf(size_t n, cudaStream_t s) : count(n), stream(s) {
    if (n) {
      pool_keep_memory();
      SPMVB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&ptr), n * sizeof(T), s));
    }
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : ptr(o.ptr), count(o.count), stream(o.stream) {
    o.ptr = nullptr;
    o.count = 0;
  }
  DevBuf& operator=(DevBuf&& o) noexcept {
    release();
    ptr = o.ptr; count = o.count; stream = o.stream;
    o.ptr = nullptr; o.count = 0;
    return *this;
  }
  ~DevBuf() { release(); }
  void release() {
    if (ptr) cudaFreeAsync(ptr, stream);
    ptr = nullptr;
    count = 0;
  }
  T* get() const { return ptr; }
};

inline int num_sms() {
  static int sms = [] {
    int dev = 0, n = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
  }();
  return sms;
}

// Programmatic dependent launch: a kernel launched with launch_pdl may start
// while its predecessor in the stream is still draining; it must call
// pdl_wait() before touching anything the predecessor writes (or writing
// anything the predecessor reads).  In a kernel launched normally the wait
// returns at once.  Chained SpMV -> fix-up -> norm -> scale kernels thereby
// overlap each launch with the previous kernel's tail.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  SPMVB_CUDA(cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...));
}

inline unsigned grid_for(int64_t n, int block, int64_t cap = (1ll << 30)) {
  int64_t g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return static_cast<unsigned>(g);
}

// SELL wide slices (width > SPMVB_SELL_WIDE_COLS, at most 128 rows) are
// processed in pieces of about SELL_PIECE_CELLS cells (whole columns), one
// CTA per piece, by the SpMV and by the fill (spmvb_sell_wide_plan).
#ifndef SPMVB_SELL_PIECE_MIN_COLS
#define SPMVB_SELL_PIECE_MIN_COLS 256
#endif
#ifndef SPMVB_SELL_PIECE_CELLS
#define SPMVB_SELL_PIECE_CELLS 32768
#endif
constexpr int64_t SELL_PIECE_CELLS = SPMVB_SELL_PIECE_CELLS;
__host__ __device__ __forceinline__ int64_t sell_piece_cols(int rows_s) {
  const int64_t pc = SELL_PIECE_CELLS / rows_s;
  return pc < SPMVB_SELL_PIECE_MIN_COLS ? SPMVB_SELL_PIECE_MIN_COLS : pc;
}
__host__ __device__ __forceinline__ int sell_rows(int64_t sl, int64_t c, int64_t n_rows) {
  return static_cast<int>((sl + 1) * c <= n_rows ? c : n_rows - sl * c);
}

inline int bits_for(uint64_t maxval) {  // bits needed to represent 0..maxval
  int b = 0;
  while (b < 64 && (maxval >> b) != 0) ++b;
  return b;
}

template <typename T>
void copy_to_host(T* host, const T* dev, size_t n, cudaStream_t s) {
  if (!n) return;
  SPMVB_CUDA(cudaMemcpyAsync(host, dev, n * sizeof(T), cudaMemcpyDeviceToHost, s));
  SPMVB_CUDA(cudaStreamSynchronize(s));
}

// ---------------------------------------------------------------------------
// Device helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Streaming loads that do not pollute L1 (format arrays are read exactly once).
__device__ __forceinline__ double ld_stream(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ int ld_stream(const int* p) {
  int v;
  asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ unsigned char ld_stream(const unsigned char* p) {
  unsigned short v;
  asm volatile("ld.global.nc.L1::no_allocate.u8 %0, [%1];" : "=h"(v) : "l"(p));
  return static_cast<unsigned char>(v);
}

// numpy's pairwise summation (numpy/_core/src/umath/loops_utils.h.src,
// pairwise_sum for float64): blocks < 8 summed sequentially from -0.0,
// blocks <= 128 with eight strided accumulators, larger blocks split at
// n/2 rounded down to a multiple of 8.  `at(i)` yields element i.
template <typename At>
__host__ __device__ inline double np_pairwise_leaf(const At& at, int64_t off, int64_t n) {
  if (n < 8) {
    double r = -0.0;
    for (int64_t i = 0; i < n; ++i) r = r + at(off + i);
    return r;
  }
  double r0 = at(off + 0), r1 = at(off + 1), r2 = at(off + 2), r3 = at(off + 3);
  double r4 = at(off + 4), r5 = at(off + 5), r6 = at(off + 6), r7 = at(off + 7);
  int64_t i = 8;
  for (; i < n - (n % 8); i += 8) {
    r0 = r0 + at(off + i + 0); r1 = r1 + at(off + i + 1);
    r2 = r2 + at(off + i + 2); r3 = r3 + at(off + i + 3);
    r4 = r4 + at(off + i + 4); r5 = r5 + at(off + i + 5);
    r6 = r6 + at(off + i + 6); r7 = r7 + at(off + i + 7);
  }
  double res = ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7));
  for (; i < n; ++i) res = res + at(off + i);
  return res;
}

template <typename At>
__host__ __device__ inline double np_pairwise(const At& at, int64_t off, int64_t n) {
  // Iterative form of the recursion (explicit stack, depth <= 64).
  if (n <= 128) return np_pairwise_leaf(at, off, n);
  struct Frame { int64_t off, n; int state; double left; };
  Frame st[64];
  int sp = 0;
  st[0] = {off, n, 0, 0.0};
  double ret = 0.0;
  while (sp >= 0) {
    Frame& f = st[sp];
    if (f.n <= 128) {
      ret = np_pairwise_leaf(at, f.off, f.n);
      --sp;
      continue;
    }
    int64_t n2 = f.n / 2;
    n2 -= n2 % 8;
    if (f.state == 0) {
      f.state = 1;
      st[sp + 1] = {f.off, n2, 0, 0.0};
      ++sp;
    } else if (f.state == 1) {
      f.left = ret;
      f.state = 2;
      st[sp + 1] = {f.off + n2, f.n - n2, 0, 0.0};
      ++sp;
    } else {
      ret = f.left + ret;
      --sp;
    }
  }
  return ret;
}

}  // namespace spmvb
