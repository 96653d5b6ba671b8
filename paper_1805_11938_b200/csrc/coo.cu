// COO core on the GPU: canonicalize, row histogram, COO->CSR, row stats,
// the sequential-order SpMV used as the on-device oracle, and small
// reductions used by power iteration.
//
// Reference: /root/reference/pkg/src/spmvkit/coo.py:86-146, formats.py:183-188.
#include "prims.cuh"

using namespace spmvb;

struct spmvb_canon {
  int64_t n_in = 0, n_out = 0, n_rows = 0, n_cols = 0;
  int colbits = 0;
  int index_width = 4;
  bool fast = false;  // input already canonical: finish is a narrowing copy
  const void* row = nullptr;
  const void* col = nullptr;
  const double* val = nullptr;
  DevBuf<uint64_t> keys_a, keys_b;
  DevBuf<uint64_t> vals_a, vals_b;  // the values (bit patterns) carried through the sort
  uint64_t* skeys = nullptr;
  const double* svals = nullptr;
  DevBuf<uint32_t> tile_off;  // kept runs before each compaction tile
  DevBuf<uint32_t> hist;      // radix digit counts taken by the key build
};

namespace {

#ifndef SPMVB_PREP_U
#define SPMVB_PREP_U 4
#endif
constexpr int CANON_HIST_COPIES = 4;  // shared-memory digit-count copies per block (warp & 3)
constexpr int CANON_MAX_PASSES = 8;

template <typename I>
__global__ void k_canon_prepare(const I* __restrict__ row, const I* __restrict__ col, const double* __restrict__ val,
                                int64_t n, int64_t n_rows, int64_t n_cols, int colbits, uint64_t* __restrict__ keys,
                                unsigned long long* bad, int* noncanonical, int passes, int key_bits,
                                uint32_t* __restrict__ hist) {
  // the radix sort's digit counts of every pass, taken while the keys are
  // in registers (passes == 0: not wanted)
  __shared__ uint32_t cnt[CANON_HIST_COPIES][CANON_MAX_PASSES * 256];
  for (int i = threadIdx.x; i < CANON_HIST_COPIES * passes * 256; i += blockDim.x)
    cnt[i / (passes * 256)][i % (passes * 256)] = 0;
  __syncthreads();
  uint32_t* mine = cnt[(threadIdx.x >> 5) & (CANON_HIST_COPIES - 1)];
  // flags are reduced per block before touching global memory: unsorted
  // input would otherwise put one atomic per entry on a single address.
  // U warp-contiguous groups per thread are loaded before any is used; the
  // previous entry comes from the neighbouring lane (lane 0 loads it).
  constexpr int U = SPMVB_PREP_U;
  const int lane = threadIdx.x & 31;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  int nc_any = 0;
  for (int64_t wb = blockIdx.x * static_cast<int64_t>(blockDim.x) + (threadIdx.x & ~31); wb < n; wb += U * stride) {
    int64_t r[U], c[U], pr[U], pc[U];
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = wb + u * stride + lane;
      const bool ok = i < n;
      r[u] = ok ? static_cast<int64_t>(row[i]) : 0;
      c[u] = ok ? static_cast<int64_t>(col[i]) : 0;
      v[u] = ok ? val[i] : 1.0;
      const bool first = lane == 0 && ok && i > 0;
      pr[u] = first ? static_cast<int64_t>(row[i - 1]) : 0;
      pc[u] = first ? static_cast<int64_t>(col[i - 1]) : 0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = wb + u * stride + lane;
      const int64_t ur = __shfl_up_sync(0xffffffffu, r[u], 1), uc = __shfl_up_sync(0xffffffffu, c[u], 1);
      if (lane > 0) {
        pr[u] = ur;
        pc[u] = uc;
      }
      if (i >= n) continue;
      const bool oob = r[u] < 0 || r[u] >= n_rows || c[u] < 0 || c[u] >= n_cols;
      const uint64_t key = oob ? 0ull : ((static_cast<uint64_t>(r[u]) << colbits) | static_cast<uint64_t>(c[u]));
      keys[i] = key;
      for (int p = 0, sh = 0; p < passes; ++p, sh += 8) {
        const int nb = key_bits - sh < 8 ? key_bits - sh : 8;
        atomicAdd(&mine[p * 256 + static_cast<unsigned>((key >> sh) & ((1u << nb) - 1u))], 1u);
      }
      if (oob) atomicMin(bad, static_cast<unsigned long long>(i));  // rare: any out-of-range entry aborts
      bool nc = (v[u] == 0.0);
      if (i > 0 && !oob && (pr[u] > r[u] || (pr[u] == r[u] && pc[u] >= c[u]))) nc = true;
      nc_any |= nc ? 1 : 0;
    }
  }
  if (__syncthreads_or(nc_any) && threadIdx.x == 0) atomicOr(noncanonical, 1);
  for (int i = threadIdx.x; i < passes * 256; i += blockDim.x) {
    uint32_t t = 0;
#pragma unroll
    for (int c = 0; c < CANON_HIST_COPIES; ++c) t += cnt[c][i];
    if (t) atomicAdd(&hist[i], t);
  }
}

// Runs of equal keys in the sorted stream; the values were carried through
// the (stable) sort, so each run holds its duplicates in input order.  A run
// is reduced by the item at its head: numpy add.reduceat = first element +
// pairwise(rest) (coo.py:123); the run is kept iff that sum != 0.0 (NaN
// kept, coo.py:124).  Rare (duplicates), so out of line.
__device__ __noinline__ double canon_run_sum(const uint64_t* __restrict__ skeys, const double* __restrict__ sval,
                                             int64_t i, int64_t n) {
  const uint64_t k = skeys[i];
  int64_t e = i + 2;
  while (e < n && skeys[e] == k) ++e;
  auto at = [&](int64_t j) { return sval[j]; };
  return sval[i] + np_pairwise(at, i + 1, e - i - 1);
}

// One tile of CANON_TILE sorted items per block; warp w owns the contiguous
// items [w*32*CANON_STEPS, (w+1)*32*CANON_STEPS) of the tile, 32 per step.  COUNT: the tile's
// number of kept runs -> tile_cnt[b].  !COUNT: the kept runs are written at
// tile_off[b] + (their rank among the tile's kept runs) -- a compaction whose
// offsets come from the scan of the counts (so canonicalize needs no
// per-item sums/flags/positions arrays).
constexpr int CANON_THREADS = 256;
constexpr int CANON_STEPS = 8;
constexpr int64_t CANON_TILE = CANON_THREADS * CANON_STEPS;

template <bool COUNT>
__global__ void __launch_bounds__(CANON_THREADS, 4) k_canon_compact(const uint64_t* __restrict__ skeys,
                                                                  const double* __restrict__ sval, int64_t n,
                                                                  uint32_t* __restrict__ tile_cnt,
                                                                  const uint32_t* __restrict__ tile_off, int colbits,
                                                                  int32_t* __restrict__ row_out,
                                                                  int32_t* __restrict__ col_out,
                                                                  double* __restrict__ val_out) {
  __shared__ uint32_t wsum[CANON_THREADS / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t base = blockIdx.x * CANON_TILE + static_cast<int64_t>(warp) * (32 * CANON_STEPS);
  uint64_t key[CANON_STEPS];
  double sum[CANON_STEPS];
  uint32_t keep = 0;  // bit r: item of step r starts a kept run
#pragma unroll
  for (int r = 0; r < CANON_STEPS; ++r) {
    const int64_t i = base + r * 32 + lane;
    key[r] = i < n ? skeys[i] : 0;
    sum[r] = i < n ? sval[i] : 0.0;
  }
  // keys just before and just after this warp's items
  const int64_t after = base + 32 * CANON_STEPS;
  uint64_t before_key = 0, after_key = ~0ull;
  if (lane == 0 && base > 0 && base - 1 < n) before_key = skeys[base - 1];
  if (lane == 31 && after < n) after_key = skeys[after];
#pragma unroll
  for (int r = 0; r < CANON_STEPS; ++r) {
    const int64_t i = base + r * 32 + lane;
    uint64_t prev = __shfl_up_sync(0xffffffffu, key[r], 1);
    const uint64_t first_next = __shfl_sync(0xffffffffu, r + 1 < CANON_STEPS ? key[r + 1 < CANON_STEPS ? r + 1 : r] : 0, 0);
    uint64_t next = __shfl_down_sync(0xffffffffu, key[r], 1);
    if (lane == 0) prev = before_key;
    if (lane == 31) next = r + 1 < CANON_STEPS ? first_next : after_key;
    before_key = __shfl_sync(0xffffffffu, key[r], 31);  // lane 0's prev in the next step
    if (i < n && (i == 0 || prev != key[r])) {
      if (i + 1 < n && next == key[r]) sum[r] = canon_run_sum(skeys, sval, i, n);
      if (sum[r] != 0.0) keep |= 1u << r;
    }
  }
  // kept runs of this warp, of the warps before it, of the tiles before
  uint32_t wcount = 0;
#pragma unroll
  for (int r = 0; r < CANON_STEPS; ++r) wcount += __popc(__ballot_sync(0xffffffffu, (keep >> r) & 1u));
  if (lane == 0) wsum[warp] = wcount;
  __syncthreads();
  if (COUNT) {
    if (threadIdx.x == 0) {
      uint32_t t = 0;
#pragma unroll
      for (int w = 0; w < CANON_THREADS / 32; ++w) t += wsum[w];
      tile_cnt[blockIdx.x] = t;
    }
    return;
  }
  uint32_t pos = tile_off[blockIdx.x];
  for (int w = 0; w < warp; ++w) pos += wsum[w];
  const uint64_t cmask = (colbits >= 64) ? ~0ull : ((1ull << colbits) - 1ull);
#pragma unroll
  for (int r = 0; r < CANON_STEPS; ++r) {
    const bool kp = (keep >> r) & 1u;
    const unsigned bal = __ballot_sync(0xffffffffu, kp);
    if (kp) {
      const uint32_t p = pos + __popc(bal & lanemask_lt());
      row_out[p] = static_cast<int32_t>(key[r] >> colbits);
      col_out[p] = static_cast<int32_t>(key[r] & cmask);
      val_out[p] = sum[r];
    }
    pos += __popc(bal);
  }
}

template <typename I>
__global__ void k_narrow_copy(const I* __restrict__ row, const I* __restrict__ col, const double* __restrict__ val,
                              int64_t n, int32_t* __restrict__ row_out, int32_t* __restrict__ col_out,
                              double* __restrict__ val_out) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    row_out[i] = static_cast<int32_t>(row[i]);
    col_out[i] = static_cast<int32_t>(col[i]);
    val_out[i] = val[i];
  }
}

__global__ void k_row_counts(const int32_t* __restrict__ row, int64_t nnz, unsigned int* __restrict__ counts) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i - threadIdx.x < nnz;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    bool valid = i < nnz;
    int r = valid ? row[i] : -1;
    unsigned peers = __match_any_sync(0xffffffffu, r);
    if (valid && (threadIdx.x & 31) == static_cast<unsigned>(__ffs(peers) - 1))
      atomicAdd(&counts[r], static_cast<unsigned>(__popc(peers)));
  }
}

__global__ void k_counts_to_i64(const unsigned int* __restrict__ c, int64_t n, int64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = static_cast<int64_t>(c[i]);
}

// The reference's oracle order (coo.py:128-141): y_r = ((0 + p_0) + p_1) + ...
// with separately rounded products.  Thread per row; rows longer than
// SEQ_LONG are left to k_spmv_sequential_long.
constexpr int32_t SEQ_LONG = 48;
__global__ void k_spmv_sequential(int64_t n_rows, const int32_t* __restrict__ ptr, const int32_t* __restrict__ col,
                                  const double* __restrict__ val, const double* __restrict__ x,
                                  double* __restrict__ y) {
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < n_rows;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t a = ptr[r], b = ptr[r + 1];
    if (b - a > SEQ_LONG) continue;
    double acc = 0.0;
    for (int k = a; k < b; ++k) acc = __dadd_rn(acc, __dmul_rn(val[k], x[col[k]]));
    y[r] = acc;
  }
}

// One warp per long row: the lanes form 32 products at a time (the next
// 32 already in flight), then every lane adds them in order -- the same
// sequential recurrence, without one thread walking ~4e5 dependent loads.
__global__ void k_spmv_sequential_long(const int32_t* __restrict__ list, int64_t n_long,
                                       const int32_t* __restrict__ ptr, const int32_t* __restrict__ col,
                                       const double* __restrict__ val, const double* __restrict__ x,
                                       double* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t i = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5; i < n_long; i += nwarps) {
    const int32_t r = list[i];
    const int64_t a = ptr[r], b = ptr[r + 1];
    // software pipeline over 32-entry chunks, D deep, slot u = chunk mod D
    // and no register moved while its load is pending: while chunk c is
    // summed, the x gather and value of chunk c+D (whose column index was
    // loaded during chunk c-D) and the column index of chunk c+2D are issued
    constexpr int D = 4;
    int32_t rc[D];
    double rv[D], rx[D];
    auto ld_col = [&](int64_t k) { return k < b ? col[k] : 0; };
#pragma unroll
    for (int u = 0; u < D; ++u) rc[u] = ld_col(a + 32 * u + lane);  // chunks 0..D-1: columns
#pragma unroll
    for (int u = 0; u < D; ++u) {  // chunks 0..D-1: gathers and values; chunks D..2D-1: columns
      const int64_t k = a + 32 * u + lane;
      rx[u] = k < b ? x[rc[u]] : 0.0;
      rv[u] = k < b ? val[k] : 0.0;
      rc[u] = ld_col(k + 32 * D);
    }
    double acc = 0.0;
    for (int64_t k0 = a; k0 < b; k0 += 32 * D) {
#pragma unroll
      for (int u = 0; u < D; ++u) {
        const int64_t kc = k0 + 32 * u;  // this chunk (warp-uniform)
        if (kc >= b) break;
        const double p = __dmul_rn(rv[u], rx[u]);
        const int64_t kn = kc + 32 * D + lane;  // chunk c+D: its column is in rc[u]
        rx[u] = kn < b ? x[rc[u]] : 0.0;
        rv[u] = kn < b ? val[kn] : 0.0;
        rc[u] = ld_col(kn + 32 * D);
        const int m = b - kc < 32 ? static_cast<int>(b - kc) : 32;
        double q[32];  // all 32 broadcasts issued before the dependent adds
#pragma unroll
        for (int t = 0; t < 32; ++t) q[t] = __shfl_sync(0xffffffffu, p, t);
#pragma unroll
        for (int t = 0; t < 32; ++t)
          if (t < m) acc = __dadd_rn(acc, q[t]);
      }
    }
    if (lane == 0) y[r] = acc;
  }
}

__global__ void k_inv_sqrt(const double* sumsq, double* scale) {
  pdl_wait();
  double s = *sumsq;
  *scale = (s > 0.0) ? 1.0 / sqrt(s) : 1.0;
}

// ||y||^2 and 1/||y|| in ONE launch (the normalisation of a single-process
// power-iteration step): each block writes its partial sum, the last block
// to take a ticket folds the partials in block order and resets the ticket.
// The grid depends on n only, so the result is the same on every call.
constexpr int NORM_THREADS = 256;
constexpr int NORM_MAX_BLOCKS = 148 * 8;
struct NormWs {
  double part[NORM_MAX_BLOCKS];
  unsigned ticket;
};

__global__ void __launch_bounds__(NORM_THREADS) k_norm_scale(const double* __restrict__ y, int64_t n, NormWs* ws,
                                                             double* __restrict__ sumsq, double* __restrict__ scale) {
  __shared__ double tmp[NORM_THREADS / 32];
  __shared__ bool last;
  pdl_wait();
  double acc = 0.0;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * NORM_THREADS;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(NORM_THREADS) + threadIdx.x; i < n; i += stride) {
    const double v = y[i];
    acc = fma(v, v, acc);
  }
  acc = block_reduce<double, NORM_THREADS>(acc, OpSum{}, 0.0, tmp);
  if (threadIdx.x == 0) {
    ws->part[blockIdx.x] = acc;
    __threadfence();
    last = atomicAdd(&ws->ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double s = 0.0;
  for (int b = threadIdx.x; b < static_cast<int>(gridDim.x); b += NORM_THREADS) s += __ldcg(ws->part + b);
  s = block_reduce<double, NORM_THREADS>(s, OpSum{}, 0.0, tmp);
  if (threadIdx.x == 0) {
    *sumsq = s;
    *scale = (s > 0.0) ? 1.0 / sqrt(s) : 1.0;
    ws->ticket = 0;
  }
}

void check_shape(int64_t n_rows, int64_t n_cols) {
  if (n_rows < 0 || n_cols < 0) fail(SPMVB_INVALID_ARG, "negative matrix shape %lldx%lld", (long long)n_rows, (long long)n_cols);
  if (n_rows > INT32_MAX || n_cols > INT32_MAX)
    fail(SPMVB_INVALID_ARG, "matrix shape %lldx%lld exceeds the 32-bit index range of the GPU layout (int32)",
         (long long)n_rows, (long long)n_cols);
}

}  // namespace

extern "C" int spmvb_canonicalize_begin(const void* row, const void* col, int index_width, const double* val,
                                        int64_t nnz_in, int64_t n_rows, int64_t n_cols, spmvb_canon** plan,
                                        int64_t* nnz_out, int64_t* bad, void* stream) {
  return guard([&] {
    cudaStream_t s = as_stream(stream);
    check_shape(n_rows, n_cols);
    if (index_width != 4 && index_width != 8) fail(SPMVB_INVALID_ARG, "index_width must be 4 or 8");
    if (nnz_in < 0) fail(SPMVB_INVALID_ARG, "negative nnz");
    if (nnz_in > INT32_MAX) fail(SPMVB_INVALID_ARG, "nnz %lld exceeds the int32 row-pointer range", (long long)nnz_in);
    auto* p = new spmvb_canon();
    p->n_in = nnz_in; p->n_rows = n_rows; p->n_cols = n_cols; p->index_width = index_width;
    p->row = row; p->col = col; p->val = val;
    p->colbits = bits_for(n_cols > 0 ? static_cast<uint64_t>(n_cols - 1) : 0);
    const int rowbits = bits_for(n_rows > 0 ? static_cast<uint64_t>(n_rows - 1) : 0);
    try {
      if (nnz_in == 0) {
        p->fast = true;
        p->n_out = 0;
      } else {
        p->keys_a = DevBuf<uint64_t>(nnz_in, s);
        DevBuf<unsigned long long> d_bad(1, s);
        DevBuf<int> d_flag(1, s);
        unsigned long long init_bad = ~0ull;
        int init_flag = 0;
        SPMVB_CUDA(cudaMemcpyAsync(d_bad.get(), &init_bad, sizeof(init_bad), cudaMemcpyHostToDevice, s));
        SPMVB_CUDA(cudaMemcpyAsync(d_flag.get(), &init_flag, sizeof(init_flag), cudaMemcpyHostToDevice, s));
        unsigned g = grid_for(nnz_in, 256, 148 * 16);
        // digit counts for the single-pass radix sort (below 2^30 items)
        const int key_bits = rowbits + p->colbits;
        const int passes = (nnz_in < (1ll << 30) && key_bits > 0) ? (key_bits + 7) / 8 : 0;
        if (passes > CANON_MAX_PASSES) fail(SPMVB_INTERNAL, "key of %d bits", key_bits);
        p->hist = DevBuf<uint32_t>(passes > 0 ? passes * 256 : 1, s);
        if (passes > 0) SPMVB_CUDA(cudaMemsetAsync(p->hist.get(), 0, passes * 256 * sizeof(uint32_t), s));
        if (index_width == 4)
          k_canon_prepare<int32_t><<<g, 256, 0, s>>>(static_cast<const int32_t*>(row), static_cast<const int32_t*>(col),
                                                     val, nnz_in, n_rows, n_cols, p->colbits, p->keys_a.get(),
                                                     d_bad.get(), d_flag.get(), passes, key_bits, p->hist.get());
        else
          k_canon_prepare<int64_t><<<g, 256, 0, s>>>(static_cast<const int64_t*>(row), static_cast<const int64_t*>(col),
                                                     val, nnz_in, n_rows, n_cols, p->colbits, p->keys_a.get(),
                                                     d_bad.get(), d_flag.get(), passes, key_bits, p->hist.get());
        SPMVB_LAUNCHED("k_canon_prepare");
        unsigned long long h_bad = 0;
        int h_flag = 0;
        SPMVB_CUDA(cudaMemcpyAsync(&h_bad, d_bad.get(), sizeof(h_bad), cudaMemcpyDeviceToHost, s));
        SPMVB_CUDA(cudaMemcpyAsync(&h_flag, d_flag.get(), sizeof(h_flag), cudaMemcpyDeviceToHost, s));
        SPMVB_CUDA(cudaStreamSynchronize(s));
        if (h_bad != ~0ull) {
          int64_t br = 0, bc = 0;
          if (index_width == 4) {
            int32_t t[2];
            SPMVB_CUDA(cudaMemcpyAsync(&t[0], static_cast<const int32_t*>(row) + h_bad, 4, cudaMemcpyDeviceToHost, s));
            SPMVB_CUDA(cudaMemcpyAsync(&t[1], static_cast<const int32_t*>(col) + h_bad, 4, cudaMemcpyDeviceToHost, s));
            SPMVB_CUDA(cudaStreamSynchronize(s));
            br = t[0]; bc = t[1];
          } else {
            SPMVB_CUDA(cudaMemcpyAsync(&br, static_cast<const int64_t*>(row) + h_bad, 8, cudaMemcpyDeviceToHost, s));
            SPMVB_CUDA(cudaMemcpyAsync(&bc, static_cast<const int64_t*>(col) + h_bad, 8, cudaMemcpyDeviceToHost, s));
            SPMVB_CUDA(cudaStreamSynchronize(s));
          }
          if (bad) { bad[0] = (int64_t)h_bad; bad[1] = br; bad[2] = bc; }
          fail(SPMVB_OUT_OF_RANGE, "entry %lld at (%lld, %lld) is outside %lldx%lld", (long long)h_bad,
               (long long)br, (long long)bc, (long long)n_rows, (long long)n_cols);
        }
        if (!h_flag) {
          p->fast = true;
          p->n_out = nnz_in;
          p->keys_a.release();
        } else {
          p->keys_b = DevBuf<uint64_t>(nnz_in, s);
          p->vals_a = DevBuf<uint64_t>(nnz_in, s);
          p->vals_b = DevBuf<uint64_t>(nnz_in, s);
          uint32_t h_total = 0;
          RadixSortResult64 rs =
              radix_sort_pairs64(p->keys_a.get(), p->keys_b.get(), reinterpret_cast<const uint64_t*>(val),
                                 p->vals_a.get(), p->vals_b.get(), nnz_in, rowbits + p->colbits, s,
                                 passes > 0 ? p->hist.get() : nullptr);
          p->skeys = rs.keys;
          p->svals = reinterpret_cast<const double*>(rs.vals);
          const int64_t tiles = (nnz_in + CANON_TILE - 1) / CANON_TILE;
          p->tile_off = DevBuf<uint32_t>(tiles, s);
          {
            DevBuf<uint32_t> cnt(tiles, s), d_total(1, s);
            k_canon_compact<true><<<static_cast<unsigned>(tiles), CANON_THREADS, 0, s>>>(
                p->skeys, p->svals, nnz_in, cnt.get(), nullptr, 0, nullptr, nullptr, nullptr);
            SPMVB_LAUNCHED("k_canon_compact");
            exclusive_scan<uint32_t>(tiles, ArrayLoad<uint32_t>{cnt.get()}, ArrayStore<uint32_t>{p->tile_off.get()},
                                     OpSum{}, 0u, d_total.get(), s);
            copy_to_host(&h_total, d_total.get(), 1, s);
          }
          p->n_out = h_total;
          // buffers not holding the sorted keys/values are no longer needed
          if (p->skeys != p->keys_a.get()) p->keys_a.release(); else p->keys_b.release();
          if (p->svals != reinterpret_cast<const double*>(p->vals_a.get())) p->vals_a.release(); else p->vals_b.release();
        }
      }
    } catch (...) {
      delete p;
      throw;
    }
    *plan = p;
    *nnz_out = p->n_out;
  });
}

extern "C" int spmvb_canonicalize_finish(spmvb_canon* p, int32_t* row_out, int32_t* col_out, double* val_out,
                                         void* stream) {
  return guard([&] {
    cudaStream_t s = as_stream(stream);
    if (!p) fail(SPMVB_INVALID_ARG, "null plan");
    if (p->n_out > 0) {
      unsigned g = grid_for(p->n_in, 256, 148 * 16);
      if (p->fast) {
        if (p->index_width == 4)
          k_narrow_copy<int32_t><<<g, 256, 0, s>>>(static_cast<const int32_t*>(p->row),
                                                   static_cast<const int32_t*>(p->col), p->val, p->n_in, row_out,
                                                   col_out, val_out);
        else
          k_narrow_copy<int64_t><<<g, 256, 0, s>>>(static_cast<const int64_t*>(p->row),
                                                   static_cast<const int64_t*>(p->col), p->val, p->n_in, row_out,
                                                   col_out, val_out);
        SPMVB_LAUNCHED("k_narrow_copy");
      } else {
        const int64_t tiles = (p->n_in + CANON_TILE - 1) / CANON_TILE;
        k_canon_compact<false><<<static_cast<unsigned>(tiles), CANON_THREADS, 0, s>>>(
            p->skeys, p->svals, p->n_in, nullptr, p->tile_off.get(), p->colbits, row_out, col_out, val_out);
        SPMVB_LAUNCHED("k_canon_compact");
      }
    }
    delete p;
  });
}

extern "C" void spmvb_canonicalize_free(spmvb_canon* p) { delete p; }

namespace spmvb {
// ptr[0..n_rows] from row-sorted COO rows (histogram + exclusive scan).
void build_row_ptr(const int32_t* row, int64_t nnz, int64_t n_rows, int32_t* ptr, cudaStream_t s) {
  DevBuf<unsigned int> counts(n_rows > 0 ? n_rows : 1, s);
  if (n_rows > 0) SPMVB_CUDA(cudaMemsetAsync(counts.get(), 0, n_rows * sizeof(unsigned int), s));
  if (nnz > 0) {
    k_row_counts<<<grid_for(nnz, 256, 148 * 16), 256, 0, s>>>(row, nnz, counts.get());
    SPMVB_LAUNCHED("k_row_counts");
  }
  const unsigned int* c = counts.get();
  const int64_t n = n_rows;
  exclusive_scan<int32_t>(
      n_rows + 1, [=] __device__(int64_t i) { return i < n ? static_cast<int32_t>(c[i]) : 0; },
      ArrayStore<int32_t>{ptr}, OpSum{}, 0, static_cast<int32_t*>(nullptr), s);
}
}  // namespace spmvb

extern "C" int spmvb_row_nnz_histogram(const int32_t* row, int64_t nnz, int64_t n_rows, int64_t* counts_out,
                                       void* stream) {
  return guard([&] {
    cudaStream_t s = as_stream(stream);
    if (n_rows <= 0) return;
    DevBuf<unsigned int> counts(n_rows, s);
    SPMVB_CUDA(cudaMemsetAsync(counts.get(), 0, n_rows * sizeof(unsigned int), s));
    if (nnz > 0) {
      k_row_counts<<<grid_for(nnz, 256, 148 * 16), 256, 0, s>>>(row, nnz, counts.get());
      SPMVB_LAUNCHED("k_row_counts");
    }
    k_counts_to_i64<<<grid_for(n_rows, 256, 148 * 16), 256, 0, s>>>(counts.get(), n_rows, counts_out);
    SPMVB_LAUNCHED("k_counts_to_i64");
  });
}

extern "C" int spmvb_coo_to_csr(const int32_t* row, const int32_t* col, const double* val, int64_t nnz,
                                int64_t n_rows, int32_t* ptr_out, int32_t* col_out, double* val_out,
                                void* stream) {
  return guard([&] {
    cudaStream_t s = as_stream(stream);
    if (nnz > INT32_MAX) fail(SPMVB_INVALID_ARG, "nnz exceeds the int32 row-pointer range");
    build_row_ptr(row, nnz, n_rows, ptr_out, s);
    if (nnz > 0) {
      SPMVB_CUDA(cudaMemcpyAsync(col_out, col, nnz * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
      SPMVB_CUDA(cudaMemcpyAsync(val_out, val, nnz * sizeof(double), cudaMemcpyDeviceToDevice, s));
    }
  });
}

extern "C" int spmvb_csr_row_stats(const int32_t* ptr, int64_t n_rows, int64_t* out3, void* stream) {
  return guard([&] {
    cudaStream_t s = as_stream(stream);
    if (n_rows <= 0) {
      out3[0] = out3[1] = out3[2] = 0;
      return;
    }
    DevBuf<int64_t> d(3, s);
    int64_t* dp = d.get();
    auto cnt = [=] __device__(int64_t i) { return static_cast<int64_t>(ptr[i + 1] - ptr[i]); };
    device_reduce<int64_t>(n_rows, cnt, OpMin{}, INT64_MAX, dp + 0, s);
    device_reduce<int64_t>(n_rows, cnt, OpMax{}, (int64_t)0, dp + 1, s);
    device_reduce<int64_t>(
        n_rows, [=] __device__(int64_t i) { return static_cast<int64_t>(ptr[i + 1] > ptr[i] ? 1 : 0); }, OpSum{},
        (int64_t)0, dp + 2, s);
    copy_to_host(out3, dp, 3, s);
  });
}

extern "C" int spmvb_csr_nonempty_rows(const int32_t* ptr, int64_t n_rows, int32_t* rows_out, void* stream) {
  return guard([&] {
    cudaStream_t s = as_stream(stream);
    if (n_rows <= 0) return;
    exclusive_scan<int32_t>(
        n_rows, [=] __device__(int64_t i) { return ptr[i + 1] > ptr[i] ? 1 : 0; },
        [=] __device__(int64_t i, int32_t v) {
          if (ptr[i + 1] > ptr[i]) rows_out[v] = static_cast<int32_t>(i);
        },
        OpSum{}, 0, static_cast<int32_t*>(nullptr), s);
  });
}

extern "C" int spmvb_spmv_sequential(int64_t n_rows, const int32_t* ptr, const int32_t* col, const double* val,
                                     const double* x, double* y, void* stream) {
  return guard([&] {
    cudaStream_t s = as_stream(stream);
    if (n_rows <= 0) return;
    k_spmv_sequential<<<grid_for(n_rows, 128, 148 * 64), 128, 0, s>>>(n_rows, ptr, col, val, x, y);
    SPMVB_LAUNCHED("k_spmv_sequential");
    DevBuf<int32_t> list(n_rows, s), total(1, s);
    int32_t* lp = list.get();
    exclusive_scan<int32_t>(
        n_rows, [=] __device__(int64_t i) { return ptr[i + 1] - ptr[i] > SEQ_LONG ? 1 : 0; },
        [=] __device__(int64_t i, int32_t v) {
          if (ptr[i + 1] - ptr[i] > SEQ_LONG) lp[v] = static_cast<int32_t>(i);
        },
        OpSum{}, 0, total.get(), s);
    int32_t n_long = 0;
    copy_to_host(&n_long, total.get(), 1, s);
    if (n_long > 0) {
      k_spmv_sequential_long<<<grid_for(static_cast<int64_t>(n_long) * 32, 256, 148 * 8), 256, 0, s>>>(
          lp, n_long, ptr, col, val, x, y);
      SPMVB_LAUNCHED("k_spmv_sequential_long");
    }
  });
}

extern "C" int spmvb_sumsq(const double* y, int64_t n, double* out, void* stream) {
  return guard([&] {
    cudaStream_t s = as_stream(stream);
    device_reduce<double>(
        n, [=] __device__(int64_t i) { double v = y[i]; return v * v; }, OpSum{}, 0.0, out, s, /*pdl=*/true);
  });
}

extern "C" int64_t spmvb_norm_ws_bytes(void) { return static_cast<int64_t>(sizeof(NormWs)); }

extern "C" int spmvb_norm_scale(const double* y, int64_t n, void* ws, double* sumsq, double* scale_out,
                                void* stream) {
  return guard([&] {
    cudaStream_t s = as_stream(stream);
    if (!ws || !sumsq || !scale_out) fail(SPMVB_INVALID_ARG, "ws, sumsq and scale_out are required");
    if (n < 0) fail(SPMVB_INVALID_ARG, "negative length %lld", (long long)n);
    const unsigned blocks = grid_for(n, NORM_THREADS * 8, NORM_MAX_BLOCKS);
    launch_pdl(k_norm_scale, dim3(blocks), dim3(NORM_THREADS), 0, s, y, n, static_cast<NormWs*>(ws), sumsq,
               scale_out);
    SPMVB_LAUNCHED("k_norm_scale");
  });
}

extern "C" int spmvb_inv_sqrt(const double* sumsq, double* scale_out, void* stream) {
  return guard([&] {
    cudaStream_t s = as_stream(stream);
    launch_pdl(k_inv_sqrt, dim3(1), dim3(1), 0, s, sumsq, scale_out);
    SPMVB_LAUNCHED("k_inv_sqrt");
  });
}
