// CSR SpMV by nnz chunks with on-the-fly segment flags (reference
// kernels.py:76-95 spmv_csr), and the HYB kernel built on it
// (kernels.py:177-199 spmv_hyb: ELL part + COO tail reduced through the
// tail's row pointer).
//
// A warp owns a chunk of CH = 32*S (S = 8) consecutive nonzeros:
//  1. lane l loads its S consecutive entries with 256-bit loads (one for the
//     column indices, two for the values: whole sectors, no transposition —
//     on sm_100 the LDG.256 path makes CSR5's stored reordering unnecessary)
//     and keeps S independent x gathers in flight;
//  2. the non-empty rows whose first entry lies in the chunk (a contiguous
//     range of the non-empty row list, from the analysis step) mark their
//     start positions (bit mask + row id in shared memory);
//  3. each lane sums its segments; a warp-shuffle suffix scan joins segments
//     that cross lanes; segment sums are written to y.
// Entries before the chunk's first row start continue the previous
// non-empty row: their sum is the chunk's carry, folded by k_chunk_fixup in
// ascending chunk order (deterministic, no floating-point atomics).  Empty
// rows are written by one coalesced grid-stride pass (0, or for HYB the
// row's ELL part), so a long run of empty rows never serialises one warp.
#include "spmv_common.cuh"

using namespace spmvb;

namespace {

constexpr int CK_WARPS = 8;

// chunk_row[c] = first index i of the non-empty row list (the identity when
// nz_rows is null) whose row starts at or after c*CH; chunk_row[nchunks] = n_nz.
__global__ void k_chunk_plan(int64_t n_nz, int64_t ch, const int32_t* __restrict__ ptr,
                             const int32_t* __restrict__ nz_rows, int64_t nchunks, int32_t* __restrict__ chunk_row) {
  for (int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; c <= nchunks;
       c += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (c == nchunks) {
      chunk_row[c] = static_cast<int32_t>(n_nz);
      continue;
    }
    const int64_t v = c * ch;
    int64_t lo = 0, hi = n_nz;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      const int64_t r = nz_rows ? nz_rows[mid] : mid;
      if (ptr[r] < v) lo = mid + 1; else hi = mid;
    }
    chunk_row[c] = static_cast<int32_t>(lo);
  }
}

template <int S>
struct ChunkSmem {
  static constexpr int CH = 32 * S;
  int32_t seg[CK_WARPS][CH];          // row id of the row starting at position e (valid where flagged)
  uint32_t flag[CK_WARPS][CH / 32];   // bit e: a row starts at chunk position e
};

template <bool HAS_ELL>
__device__ __forceinline__ double ell_row(int64_t n_rows, int64_t r, int64_t ell_k, const int32_t* __restrict__ ell_idx,
                                          const double* __restrict__ ell_val, const double* __restrict__ x) {
  // sequential over the K slots with separately rounded products, as the
  // reference's spmv_ell (kernels.py:101-104)
  return HAS_ELL ? seq_slots4(ell_k, n_rows, r, ell_idx, ell_val, x) : 0.0;
}

template <int S, bool HAS_ELL, bool VEC>
__global__ void __launch_bounds__(CK_WARPS * 32) k_spmv_chunk(
    int64_t n_rows, int64_t nnz, const int32_t* __restrict__ ptr, const int32_t* __restrict__ col,
    const double* __restrict__ val, const int32_t* __restrict__ nz_rows, const int32_t* __restrict__ chunk_row,
    int64_t nchunks, int32_t* __restrict__ carry_row, double* __restrict__ carry_val, const double* __restrict__ x,
    double* __restrict__ y, const double* __restrict__ scale_p, int64_t ell_k, const int32_t* __restrict__ ell_idx,
    const double* __restrict__ ell_val, int64_t rows_per_block) {
  static_assert(S == 8, "lane-contiguous loads assume 8 entries (32 B of indices) per lane");
  constexpr int CH = 32 * S;
  pdl_wait();
  if (rows_per_block > 0) {
    // this block's slice of the empty rows (HYB: rows whose tail is empty get
    // their ELL part), riding along with the gather-bound chunk work
    const double sc = load_scale(scale_p);
    const int64_t r0 = blockIdx.x * rows_per_block;
    const int64_t r1 = r0 + rows_per_block < n_rows ? r0 + rows_per_block : n_rows;
    for (int64_t r = r0 + threadIdx.x; r < r1; r += blockDim.x)
      if (ld_stream(ptr + r) == ld_stream(ptr + r + 1)) y[r] = 0.0;
  }
  extern __shared__ __align__(16) unsigned char smem_raw[];
  ChunkSmem<S>& sm = *reinterpret_cast<ChunkSmem<S>*>(smem_raw);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t c = static_cast<int64_t>(blockIdx.x) * CK_WARPS + w;
  if (c >= nchunks) return;  // whole warps only
  const int64_t k0 = c * CH;
  const int cnt = static_cast<int>(nnz - k0 < CH ? nnz - k0 : CH);
  int32_t* seg = sm.seg[w];
  uint32_t* flag = sm.flag[w];

  // The chunk's row table first: its loads (chunk_row -> nz_rows -> ptr) are
  // a dependent chain, issued so that they overlap the value/column loads
  // and the x gathers instead of following them.
  const int32_t ia = chunk_row[c], ib = chunk_row[c + 1];
  // 1. lane l owns entries [8l, 8l+8): one 256-bit load of its column
  //    indices and two of its values (full sectors; with the lanes' rows
  //    consecutive, the x gathers of one instruction fall in few lines on
  //    banded/stencil matrices), then 8 independent gathers in flight.
  double v[S];
  int32_t ci[S];
  const int e0 = lane * S;
  if (VEC && e0 + S <= cnt) {
    ld_stream8(col + k0 + e0, ci);
    ld_stream4(val + k0 + e0, v);
    ld_stream4(val + k0 + e0 + 4, v + 4);
  } else {
#pragma unroll
    for (int i = 0; i < S; ++i) {
      const bool ok = e0 + i < cnt;
      ci[i] = ok ? ld_stream(col + k0 + e0 + i) : 0;
      v[i] = ok ? ld_stream(val + k0 + e0 + i) : 0.0;
    }
  }
  // first batch of row starts (most chunks have at most 32)
  const int32_t i0 = ia + lane;
  const int32_t r0 = i0 < ib ? (nz_rows ? nz_rows[i0] : i0) : 0;
#pragma unroll
  for (int i = 0; i < S; ++i) v[i] = e0 + i < cnt ? v[i] * ldx(x, ci[i]) : 0.0;
  const int32_t p0 = i0 < ib ? ptr[r0] : 0;
  if (lane < CH / 32) flag[lane] = 0u;
  __syncwarp();
  // 2. non-empty rows starting in this chunk (at most CH of them)
  const double sc = load_scale(scale_p);
  for (int32_t i = i0; i < ib; i += 32) {
    const int32_t r = i == i0 ? r0 : (nz_rows ? nz_rows[i] : i);
    const int p = static_cast<int>((i == i0 ? p0 : ptr[r]) - k0);
    seg[p] = r;
    atomicOr(&flag[p >> 5], 1u << (p & 31));
  }
  __syncwarp();  // also orders the parked y[r] stores before the reads below
  // 3. lane-contiguous segments
  const uint32_t fmask = (flag[lane >> 2] >> ((lane & 3) * S)) & 0xffu;
  double head = 0.0, sum = 0.0;
  int open_row = -1;
#pragma unroll
  for (int i = 0; i < S; ++i) {
    if ((fmask >> i) & 1u) {
      if (open_row < 0) head = sum;
      else y[open_row] = sc * (HAS_ELL ? y[open_row] + sum : sum);
      open_row = seg[lane * S + i];
      sum = 0.0;
    }
    sum += v[i];
  }
  const bool F = open_row >= 0;
  if (!F) head = sum;
  // R_l = H_l + (F_l ? 0 : R_{l+1}): segmented suffix sum of lane heads
  double rv = head;
  bool stop = F;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const double ov = __shfl_down_sync(0xffffffffu, rv, d);
    const bool ostop = __shfl_down_sync(0xffffffffu, stop ? 1 : 0, d) != 0;
    if (!stop && lane + d < 32) {
      rv += ov;
      stop = ostop;
    }
  }
  double right = __shfl_down_sync(0xffffffffu, rv, 1);
  if (lane == 31) right = 0.0;
  if (F) y[open_row] = sc * (HAS_ELL ? y[open_row] + (sum + right) : sum + right);
  if (lane == 0) {
    // leading entries continue the previous non-empty row unless a row
    // starts at position 0
    const bool cont = !(fmask & 1u);
    carry_row[c] = cont ? (nz_rows ? nz_rows[ia - 1] : ia - 1) : -1;
    carry_val[c] = cont ? rv : 0.0;
  }
}

// Empty rows: y = 0, or for HYB the ELL part (rows with an empty tail).
template <bool HAS_ELL>
__global__ void k_empty_rows(int64_t n_rows, const int32_t* __restrict__ ptr, int64_t ell_k,
                             const int32_t* __restrict__ ell_idx, const double* __restrict__ ell_val,
                             const double* __restrict__ x, double* __restrict__ y, const double* __restrict__ scale_p) {
  const double sc = load_scale(scale_p);
  auto write = [&](int64_t r) { y[r] = HAS_ELL ? sc * ell_row<HAS_ELL>(n_rows, r, ell_k, ell_idx, ell_val, x) : 0.0; };
  if (ptr) {
    for_each_empty_row(n_rows, ptr, write);
  } else {  // every row is empty (e.g. a HYB whose tail is empty)
    for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < n_rows;
         r += static_cast<int64_t>(gridDim.x) * blockDim.x)
      write(r);
  }
}

// Folds every chain of chunk carry-outs (consecutive chunks whose carry row is
// the same) into its row, chain by chain in chunk order (fold_chains).
__global__ void k_chunk_fixup(int64_t num, const int32_t* __restrict__ carry_row, const double* __restrict__ carry_val,
                              double* __restrict__ y, const double* __restrict__ scale_p) {
  pdl_wait();
  const double sc = load_scale(scale_p);
  fold_chains(
      0, num, [&](int64_t c) { return carry_row[c]; }, [&](int64_t c) { return carry_val[c]; },
      [&](int32_t r, double acc) { y[r] += sc * acc; });
}

constexpr int CHUNK_S = 8;  // entries per lane: one 256-bit load of indices
inline int chunk_s() { return CHUNK_S; }

struct ChunkArgs {
  int64_t n_rows, nnz;
  const int32_t *ptr, *col;
  const double* val;
  const int32_t *nz_rows, *chunk_row;
  int64_t n_nz;
  int32_t* carry_row;
  double* carry_val;
  const double* x;
  double* y;
  const double* scale;
  int64_t ell_k;
  const int32_t* ell_idx;
  const double* ell_val;
};

// HYB ELL part for every row, one coalesced thread-per-row pass: rows whose
// tail is empty get their final value sc * ell; rows with a tail get ell
// unscaled, parked in y for the chunk kernel, whose closing lane writes
// sc * (ell + tail sum) -- the order the per-row fused version used.
template <bool PF>
__global__ void k_hyb_ell_prepass(int64_t n_rows, const int32_t* __restrict__ tail_ptr, int64_t k,
                                  const int32_t* __restrict__ idx, const double* __restrict__ val,
                                  const double* __restrict__ x, double* __restrict__ y,
                                  const double* __restrict__ scale_p) {
  pdl_wait();
  const double sc = load_scale(scale_p);
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < n_rows;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double e = PF ? seq_slots(k, n_rows, r, idx, val, x) : seq_slots4(k, n_rows, r, idx, val, x);
    y[r] = ld_stream(tail_ptr + r) == ld_stream(tail_ptr + r + 1) ? sc * e : e;
  }
}

template <int S, bool HAS_ELL, bool VEC>
void launch_main(const ChunkArgs& a, int64_t nchunks, bool empties, cudaStream_t s) {
  const size_t smem = sizeof(ChunkSmem<S>);
  const int64_t blocks = (nchunks + CK_WARPS - 1) / CK_WARPS;
  const int64_t rpb = (empties && !HAS_ELL) ? (a.n_rows + blocks - 1) / blocks : 0;
  launch_pdl(k_spmv_chunk<S, HAS_ELL, VEC>, dim3(static_cast<unsigned>(blocks)), dim3(CK_WARPS * 32), smem, s,
             a.n_rows, a.nnz, a.ptr, a.col, a.val, a.nz_rows, a.chunk_row, nchunks, a.carry_row, a.carry_val, a.x,
             a.y, a.scale, a.ell_k, a.ell_idx, a.ell_val, rpb);
  SPMVB_LAUNCHED("k_spmv_chunk");
}

template <int S, bool HAS_ELL>
void launch_chunk_t(const ChunkArgs& a, cudaStream_t s) {
  constexpr int CH = 32 * S;
  const int64_t nchunks = (a.nnz + CH - 1) / CH;
  const bool empties = a.n_nz < a.n_rows;  // empty rows (and, for HYB, rows whose tail is empty)
  if (nchunks == 0) {
    if (empties) {
      k_empty_rows<HAS_ELL><<<grid_for(a.n_rows, 256, 148 * 32), 256, 0, s>>>(a.n_rows, nullptr, a.ell_k, a.ell_idx,
                                                                              a.ell_val, a.x, a.y, a.scale);
      SPMVB_LAUNCHED("k_empty_rows");
    }
    return;
  }
  if (HAS_ELL) {
    const dim3 g(grid_for(a.n_rows, 256)), b(256);
    if (a.ell_k >= 8)
      launch_pdl(k_hyb_ell_prepass<true>, g, b, 0, s, a.n_rows, a.ptr, a.ell_k, a.ell_idx, a.ell_val, a.x, a.y,
                 a.scale);
    else
      launch_pdl(k_hyb_ell_prepass<false>, g, b, 0, s, a.n_rows, a.ptr, a.ell_k, a.ell_idx, a.ell_val, a.x, a.y,
                 a.scale);
    SPMVB_LAUNCHED("k_hyb_ell_prepass");
  }
  // 256-bit loads need 32-byte aligned index/value arrays (torch allocations are)
  if (aligned32(a.col) && aligned32(a.val)) launch_main<S, HAS_ELL, true>(a, nchunks, empties, s);
  else launch_main<S, HAS_ELL, false>(a, nchunks, empties, s);
  if (nchunks > 1) {
    launch_pdl(k_chunk_fixup, dim3(grid_for(nchunks, 256)), dim3(256), 0, s, nchunks, a.carry_row, a.carry_val, a.y,
               a.scale);
    SPMVB_LAUNCHED("k_chunk_fixup");
  }
}

void launch_chunk(const ChunkArgs& a, cudaStream_t s) {
  if (a.n_rows <= 0) return;
  if (a.ell_k > 0) launch_chunk_t<CHUNK_S, true>(a, s);
  else launch_chunk_t<CHUNK_S, false>(a, s);
}

}  // namespace

extern "C" int64_t spmvb_csr_chunk_size(void) { return 32 * chunk_s(); }

extern "C" int64_t spmvb_csr_chunks(int64_t nnz) {
  const int64_t ch = 32 * chunk_s();
  return nnz > 0 ? (nnz + ch - 1) / ch : 0;
}

extern "C" int spmvb_csr_chunk_plan(int64_t n_rows, int64_t nnz, const int32_t* ptr, const int32_t* nz_rows,
                                    int64_t n_nz, int32_t* chunk_row, void* stream) {
  return guard([&] {
    cudaStream_t s = as_stream(stream);
    if (n_rows <= 0) return;
    const int64_t ch = 32 * chunk_s();
    const int64_t nchunks = nnz > 0 ? (nnz + ch - 1) / ch : 0;
    k_chunk_plan<<<grid_for(nchunks + 1, 256, 148 * 16), 256, 0, s>>>(n_nz, ch, ptr, nz_rows, nchunks, chunk_row);
    SPMVB_LAUNCHED("k_chunk_plan");
  });
}

extern "C" int spmvb_spmv_csr(int64_t n_rows, int64_t nnz, const int32_t* ptr, const int32_t* col, const double* val,
                              const int32_t* nz_rows, int64_t n_nz, const int32_t* chunk_row, int32_t* carry_row,
                              double* carry_val, const double* x, double* y, const double* scale, void* stream) {
  return guard([&] {
    launch_chunk(ChunkArgs{n_rows, nnz, ptr, col, val, nz_rows, chunk_row, n_nz, carry_row, carry_val, x, y, scale,
                           0, nullptr, nullptr},
                 as_stream(stream));
  });
}

extern "C" int spmvb_spmv_hyb(int64_t n_rows, int64_t k, const int32_t* ell_idx, const double* ell_val,
                              int64_t tail_nnz, const int32_t* tail_ptr, const int32_t* tail_col,
                              const double* tail_val, const int32_t* nz_rows, int64_t n_nz, const int32_t* chunk_row,
                              int32_t* carry_row, double* carry_val, const double* x, double* y, const double* scale,
                              void* stream) {
  return guard([&] {
    if (tail_nnz == 0 && k > 0) {  // empty tail: the ELL part is the whole result
      const int rc = spmvb_spmv_ell(n_rows, 0, k, ell_idx, ell_val, x, y, scale, stream);  // (no x length: no prefetch)
      if (rc != SPMVB_OK) fail(rc, "%s", spmvb_last_error());
      return;
    }
    launch_chunk(ChunkArgs{n_rows, tail_nnz, tail_ptr, tail_col, tail_val, nz_rows, chunk_row, n_nz, carry_row,
                           carry_val, x, y, scale, k, ell_idx, ell_val},
                 as_stream(stream));
  });
}
