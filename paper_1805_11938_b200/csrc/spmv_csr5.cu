// CSR5 SpMV (reference kernels.py:139-174 spmv_csr5): per-tile segmented
// sums over the reference's descriptor layout, warp shuffles across tile
// columns, and an ordered carry fix-up for rows spanning tiles; plus the
// row-range and host-buffer entry points and the variant fused with the
// multi-GPU exchange (rows stored into peer buffers by the same kernel).
#include <mutex>
#include <vector>

#include "spmv_common.cuh"

#ifndef SPMVB_CSR5_MINB
#define SPMVB_CSR5_MINB 4  // resident blocks per SM the tile kernel is compiled for (64 registers)
#endif
#ifndef SPMVB_CSR5_MINB8
#define SPMVB_CSR5_MINB8 5  // sigma = 8 (half the per-lane tile registers): 5 blocks, C4 89.1 -> 85.0 us
#endif

using namespace spmvb;

namespace {

// =========================================================================
// CSR5.  Segment ordinal s inside tile t maps to the g-th non-empty row with
// g = rank(tile_ptr[t]) + s (tile_aux bits 0-30); bit 31 marks a tile whose
// head continues a row begun earlier: that first segment is a carry.  Empty
// rows receive no segment; the tile kernel's blocks zero them, each a
// contiguous slice of the row range.  Row lookup: nonempty[g] (the list of
// non-empty rows), or g itself when nonempty is null -- either no row is
// empty, or (n_nonempty < n_rows) the non-empty rows are exactly the prefix
// [0, n_nonempty) and the empty tail is zeroed without any ptr test (the
// degree-ordered layout of relabel.cu puts every empty row last).
// =========================================================================
struct Csr5Ctx {
  int64_t n_rows, nnz, n_nonempty;
  int omega, sigma;
  const int32_t* ptr;
  const int32_t* tile_ptr;
  const uint8_t* bit_flag;
  const uint32_t* fbits;  // bit_flag packed one bit per entry, or null
  const int32_t* col;
  const double* val;
  const uint32_t* aux;
  const int32_t* nonempty;
  double* carry;
  const double* x;
  double* y;
  const double* scale_p;
};

// Fused exchange (PUSH kernels): every finished row r of y is also stored at
// peers[p][push_off + r] (peer buffers mapped over NVLink).
struct Csr5Push {
  const uint64_t* peers = nullptr;
  int n_peers = 0;
  int64_t push_off = 0;
};

__device__ __forceinline__ int64_t csr5_row_of(const Csr5Ctx& C, int64_t g) {
  return C.nonempty ? static_cast<int64_t>(C.nonempty[g]) : g;
}

__device__ __forceinline__ void csr5_emit(const Csr5Ctx& C, double sc, int64_t t, uint32_t aux, int64_t s, double v) {
  const bool cont = (aux & 0x80000000u) != 0;
  if (s == 0 && cont) {
    C.carry[t] = sc * v;
    return;
  }
  const int64_t g = static_cast<int64_t>(aux & 0x7fffffffu) + s;
  C.y[csr5_row_of(C, g)] = sc * v;
}


// Empty rows never receive a segment: one coalesced pass writes their zeros.
__global__ void k_csr5_empty_rows(int64_t n_rows, const int32_t* __restrict__ ptr, double* __restrict__ y) {
  for_each_empty_row(n_rows, ptr, [&](int64_t r) { y[r] = 0.0; });
}

// Generic: one thread per tile, CSR order recovered from the stored layout.
__global__ void k_csr5_generic(Csr5Ctx C, int64_t t_begin, int64_t t_end) {
  const int64_t tile = static_cast<int64_t>(C.omega) * C.sigma;
  const double sc = load_scale(C.scale_p);
  for (int64_t t = t_begin + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < t_end;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t base = t * tile;
    const int64_t m = C.nnz - base < tile ? C.nnz - base : tile;
    const int64_t q = m / C.sigma, rem = m % C.sigma;
    const uint32_t aux = C.aux[t];
    int64_t seg = -1;
    double sum = 0.0;
    for (int64_t p = 0; p < m; ++p) {
      const int64_t gi = p % C.sigma, gj = p / C.sigma;
      const int64_t pos = base + gi * q + (gi < rem ? gi : rem) + gj;
      if (C.bit_flag[pos]) {
        if (seg >= 0) csr5_emit(C, sc, t, aux, seg, sum);
        ++seg;
        sum = 0.0;
      }
      sum += C.val[pos] * ldx(C.x, C.col[pos]);
    }
    if (seg >= 0) csr5_emit(C, sc, t, aux, seg, sum);
  }
}

// Fast path: W lanes per full tile (omega == W), lane j owns tile column j
// (sigma consecutive CSR-order entries stored at base + i*W + j).
template <int W>
__global__ void __launch_bounds__(256) k_csr5_warp(Csr5Ctx C, int64_t t_begin, int64_t t_end) {
  const int lane = threadIdx.x & 31;
  const int j = lane % W;
  const int64_t group = t_begin + (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) / W;
  const bool active = group < t_end;
  const int64_t t = active ? group : t_begin;
  const int sigma = C.sigma;
  const int64_t base = t * static_cast<int64_t>(W) * sigma;
  const uint32_t aux = active ? C.aux[t] : 0u;
  const double sc = load_scale(C.scale_p);

  double head = 0.0, sum = 0.0;
  int nflags = 0;
  // First pass: count this lane's flags so segment ordinals are known while
  // streaming; flags are 1 byte/entry and re-read from L1.
  for (int i = 0; i < sigma && active; ++i) nflags += C.bit_flag[base + static_cast<int64_t>(i) * W + j] ? 1 : 0;
  // Exclusive prefix of flag counts across the group's lanes.
  int incl = nflags;
#pragma unroll
  for (int d = 1; d < W; d <<= 1) {
    int o = __shfl_up_sync(0xffffffffu, incl, d, W);
    if (j >= d) incl += o;
  }
  const int seg_base = incl - nflags;
  int seen = 0;
  if (active) {
    for (int i = 0; i < sigma; ++i) {
      const int64_t pos = base + static_cast<int64_t>(i) * W + j;
      const bool f = C.bit_flag[pos] != 0;
      const double v = ld_stream(C.val + pos) * ldx(C.x, ld_stream(C.col + pos));
      if (f) {
        if (seen == 0) head = sum;
        else csr5_emit(C, sc, t, aux, seg_base + seen - 1, sum);
        ++seen;
        sum = 0.0;
      }
      sum += v;
    }
  }
  const bool F = seen > 0;
  if (!F) head = sum;
  // R_j = H_j + (F_j ? 0 : R_{j+1}): segmented suffix sum of heads.
  double rv = head;
  bool stop = F;
#pragma unroll
  for (int d = 1; d < W; d <<= 1) {
    double ov = __shfl_down_sync(0xffffffffu, rv, d, W);
    bool ostop = __shfl_down_sync(0xffffffffu, stop ? 1 : 0, d, W) != 0;
    if (!stop && j + d < W) {
      rv += ov;
      stop = ostop;
    }
  }
  double right = __shfl_down_sync(0xffffffffu, rv, 1, W);
  if (j == W - 1) right = 0.0;
  if (active && F) csr5_emit(C, sc, t, aux, seg_base + seen - 1, sum + right);
}

// The tile's segmented sums once the products v[] and the lane's flag mask
// are in registers: segment ordinals by a shuffle scan of the flag counts,
// in-lane segment sums emitted as they close, the heads of the lanes joined
// by a segmented suffix scan (shared by the tile kernels below).
template <int W, int S>
__device__ __forceinline__ void csr5_tile_sums(const Csr5Ctx& C, int64_t t, int j, bool active, uint32_t fmask,
                                               const double (&v)[S], double sc) {
  const uint32_t aux = active ? C.aux[t] : 0u;
  const int nflags = __popc(fmask);
  int incl = nflags;
#pragma unroll
  for (int d = 1; d < W; d <<= 1) {
    int o = __shfl_up_sync(0xffffffffu, incl, d, W);
    if (j >= d) incl += o;
  }
  const int seg_base = incl - nflags;
  double head = 0.0, sum = 0.0;
  int seen = 0;
  if (active) {
#pragma unroll
    for (int i = 0; i < S; ++i) {
      if ((fmask >> i) & 1u) {
        if (seen == 0) head = sum;
        else csr5_emit(C, sc, t, aux, seg_base + seen - 1, sum);
        ++seen;
        sum = 0.0;
      }
      sum += v[i];
    }
  }
  const bool F = seen > 0;
  if (!F) head = sum;
  double rv = head;
  bool stop = F;
#pragma unroll
  for (int d = 1; d < W; d <<= 1) {
    double ov = __shfl_down_sync(0xffffffffu, rv, d, W);
    bool ostop = __shfl_down_sync(0xffffffffu, stop ? 1 : 0, d, W) != 0;
    if (!stop && j + d < W) {
      rv += ov;
      stop = ostop;
    }
  }
  double right = __shfl_down_sync(0xffffffffu, rv, 1, W);
  if (j == W - 1) right = 0.0;
  if (active && F) csr5_emit(C, sc, t, aux, seg_base + seen - 1, sum + right);
}

// Fused exchange epilogue of a PUSH tile kernel: the block owns the rows
// [B(t0), B(t1)) of its tiles [t0, t1), B(t) = tile_ptr[t] (row_begin /
// row_end at the range ends).  Once all its warps have emitted, it zeroes the
// empty ones and stores every one of them into each peer buffer with 16-byte
// stores (contiguous per block: a per-emit 8-byte store to the peers was
// 2.4x costlier at C5).  A row that continues across a tile boundary is
// stored here with its partial (or not yet written) value and again, final,
// by the fix-up (k_csr5_fixup<true>), which runs after this grid completes.
template <int W>
__device__ __forceinline__ void csr5_push_block(const Csr5Ctx& C, const Csr5Push& P, int64_t t_begin, int64_t t_end,
                                                int64_t row_begin, int64_t row_end) {
  __syncthreads();  // the block's emits are done
  constexpr int64_t TPB = 256 / W;
  const int64_t t0 = t_begin + blockIdx.x * TPB;
  const int64_t t1 = t0 + TPB < t_end ? t0 + TPB : t_end;
  const int64_t r0 = t0 <= t_begin ? row_begin : static_cast<int64_t>(C.tile_ptr[t0]);
  const int64_t r1 = t1 >= t_end ? row_end : static_cast<int64_t>(C.tile_ptr[t1]);
  if (C.nonempty) {
    for (int64_t r = r0 + threadIdx.x; r < r1; r += blockDim.x)
      if (ld_stream(C.ptr + r) == ld_stream(C.ptr + r + 1)) C.y[r] = 0.0;
  } else if (C.n_nonempty < C.n_rows) {  // prefix layout: the empty tail
    for (int64_t r = (r0 > C.n_nonempty ? r0 : C.n_nonempty) + threadIdx.x; r < r1; r += blockDim.x) C.y[r] = 0.0;
  }
  __syncthreads();
  const int64_t off = P.push_off;
  // pairs (r, r+1) with off + r even: 16-byte aligned in the peer buffers
  const int64_t first = ((off + r0) & 1) ? r0 + 1 : r0;
  if (first > r0 && threadIdx.x == 0 && r0 < r1)
    for (int p = 0; p < P.n_peers; ++p) reinterpret_cast<double*>(P.peers[p])[off + r0] = C.y[r0];
  const int64_t pairs = r1 > first ? (r1 - first) / 2 : 0;
  for (int64_t i = threadIdx.x; i < pairs; i += blockDim.x) {
    const int64_t r = first + 2 * i;
    const double a = C.y[r], b = C.y[r + 1];
    for (int p = 0; p < P.n_peers; ++p)
      *reinterpret_cast<double2*>(reinterpret_cast<double*>(P.peers[p]) + off + r) = make_double2(a, b);
  }
  const int64_t last = first + 2 * pairs;
  if (last < r1 && last >= r0 && threadIdx.x == 0)
    for (int p = 0; p < P.n_peers; ++p) reinterpret_cast<double*>(P.peers[p])[off + last] = C.y[last];
}

// Same algorithm with a compile-time sigma: each lane issues its S flag,
// column and value loads back to back, then S independent x gathers, so a
// warp keeps 32*S gathers in flight (random-column matrices are bound by the
// L1TEX rate of these gathers, ~1 distinct line per SM cycle).  The trailing
// partial tile (row-major over its occupied cells, formats.py:24-25) takes a
// different load path in the same kernel.  Every block also zeroes its share
// of the empty rows of [row_begin, row_end) (a coalesced slice of ptr/y per
// block), so that streaming pass rides along with the gather-bound tiles
// instead of costing its own launch.
// MODE: 0 no empty row in the range, 1 empty rows found by ptr tests (the
// non-empty row list is in use), 2 empty tail [row_begin, row_end) zeroed by
// plain stores (prefix layout; row_begin is then the first tail row).
template <int W, int S, int MODE, bool PUSH>
__device__ __forceinline__ void csr5_tiles(const Csr5Ctx& C, const Csr5Push& P, int64_t t_begin, int64_t t_end,
                                           int64_t rows_per_block, int64_t row_begin, int64_t row_end) {
  constexpr bool EMPTIES = MODE == 1;
  const int lane = threadIdx.x & 31;
  const int j = lane % W;
  const int64_t group = t_begin + (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) / W;
  const int64_t zr0 = MODE != 0 ? row_begin + blockIdx.x * rows_per_block : 0;
  const int64_t zr1 = MODE != 0 ? (zr0 + rows_per_block < row_end ? zr0 + rows_per_block : row_end) : 0;
  // This block's slice of the empty rows: the ptr pairs of its first ZP
  // rows per thread are loaded up front with the tile's streams (ptr is not
  // written by the predecessor kernel) and tested/zeroed after the tile's
  // emits, so the slice adds no dependent DRAM round trip in front of the x
  // gathers (C4 SpMV 102.8 -> 97.3 us; zeroing first, or after the emits
  // without the early loads, was slower).
  // EMPTIES == false (no empty rows in the range, rows_per_block == 0) is
  // instantiated without the early loads and keeps the plain zeroing loop
  // after pdl_wait: a no-op there, but without it ptxas schedules the tile
  // code differently and matrices without empty rows lose ~9 % (C3).
  constexpr int ZP = EMPTIES ? 2 : 0;
  int32_t zp0[ZP > 0 ? ZP : 1], zp1[ZP > 0 ? ZP : 1];
#pragma unroll
  for (int k = 0; k < ZP; ++k) {
    const int64_t r = zr0 + threadIdx.x + k * 256;
    zp0[k] = r < zr1 ? ld_stream(C.ptr + r) : 0;
    zp1[k] = r < zr1 ? ld_stream(C.ptr + r + 1) : 0;
  }
  auto zero_empty_rows_first = [&] {  // MODE 0 only (see above)
    if (MODE == 0 && rows_per_block > 0) {
      const int64_t r0 = row_begin + blockIdx.x * rows_per_block;
      const int64_t r1 = r0 + rows_per_block < row_end ? r0 + rows_per_block : row_end;
      for (int64_t r = r0 + threadIdx.x; r < r1; r += blockDim.x)
        if (ld_stream(C.ptr + r) == ld_stream(C.ptr + r + 1)) C.y[r] = 0.0;
    }
  };
  auto zero_row = [&](int64_t r) { C.y[r] = 0.0; };
  auto zero_empty_rows = [&] {
    if (MODE == 2) {  // the block's slice of the empty tail
      for (int64_t r = zr0 + threadIdx.x; r < zr1; r += blockDim.x) zero_row(r);
    }
    if (EMPTIES && rows_per_block > 0) {
      int64_t r = zr0 + threadIdx.x;
#pragma unroll
      for (int k = 0; k < ZP; ++k, r += 256)
        if (r < zr1 && zp0[k] == zp1[k]) zero_row(r);
      for (; r < zr1; r += blockDim.x)
        if (ld_stream(C.ptr + r) == ld_stream(C.ptr + r + 1)) zero_row(r);
    }
  };
  const bool active = group < t_end;
  const int64_t t = active ? group : t_begin;
  const int64_t tile0 = t * static_cast<int64_t>(W) * S;
  uint32_t fmask = 0;
  int32_t cidx[S];
  double v[S];
  if (active && tile0 + W * S <= C.nnz) {
    const int64_t base = tile0 + j;
    if (C.fbits) {
      // the tile's W*S flag bits: NW words, the same for every lane of the
      // group (broadcast); entry i of lane j is bit (i*W + j) of the tile
      constexpr int NW = W * S / 32;
      int32_t fw[NW];
      const int32_t* tw = reinterpret_cast<const int32_t*>(C.fbits) + (tile0 >> 5);
      if constexpr (NW % 8 == 0) {
#pragma unroll
        for (int q = 0; q < NW / 8; ++q) {
          int32_t tmp[8];
          ld_stream8(tw + 8 * q, tmp);
#pragma unroll
          for (int u = 0; u < 8; ++u) fw[8 * q + u] = tmp[u];
        }
      } else {
#pragma unroll
        for (int q = 0; q < NW; ++q) fw[q] = ld_stream(tw + q);
      }
#pragma unroll
      for (int i = 0; i < S; ++i) {
        fmask |= ((static_cast<uint32_t>(fw[(i * W) >> 5]) >> (((i * W) & 31) + j)) & 1u) << i;
        cidx[i] = ld_stream(C.col + base + i * W);
        v[i] = ld_stream(C.val + base + i * W);
      }
    } else {
#pragma unroll
      for (int i = 0; i < S; ++i) {
        fmask |= (C.bit_flag[base + i * W] ? 1u : 0u) << i;
        cidx[i] = ld_stream(C.col + base + i * W);
        v[i] = ld_stream(C.val + base + i * W);
      }
    }
    // the matrix loads above may overlap the previous kernel's tail (PDL);
    // x, scale and y only after it has finished
    pdl_wait();
    if constexpr (!EMPTIES) zero_empty_rows_first();
#pragma unroll
    for (int i = 0; i < S; ++i) v[i] *= ldx(C.x, cidx[i]);
  } else {
    pdl_wait();
    if constexpr (!EMPTIES) zero_empty_rows_first();
  }
  if (active && tile0 + W * S > C.nnz) {
    // partial tile: every load is issued (clamped to the tile start when the
    // cell is unoccupied) before any is used
    const int64_t m = C.nnz - tile0;
    const int q = static_cast<int>(m / S), rem = static_cast<int>(m % S);
    uint32_t okm = 0;
    uint8_t fl[S];
#pragma unroll
    for (int i = 0; i < S; ++i) {
      const bool ok = static_cast<int64_t>(j) * S + i < m;
      okm |= (ok ? 1u : 0u) << i;
      const int64_t pos = ok ? tile0 + static_cast<int64_t>(i) * q + (i < rem ? i : rem) + j : tile0;
      fl[i] = C.bit_flag[pos];
      cidx[i] = C.col[pos];
      v[i] = C.val[pos];
    }
#pragma unroll
    for (int i = 0; i < S; ++i) {
      const bool ok = (okm >> i) & 1u;
      fmask |= (ok && fl[i] ? 1u : 0u) << i;
      v[i] = ok ? v[i] * ldx(C.x, cidx[i]) : 0.0;
    }
  }
  csr5_tile_sums<W, S>(C, t, j, active, fmask, v, load_scale(C.scale_p));
  zero_empty_rows();
  if constexpr (PUSH) csr5_push_block<W>(C, P, t_begin, t_end, row_begin, row_end);
}

template <int W, int S, int MODE>
__global__ void __launch_bounds__(256, S <= 8 ? SPMVB_CSR5_MINB8 : SPMVB_CSR5_MINB) k_csr5_warp_s(Csr5Ctx C, int64_t t_begin, int64_t t_end,
                                                     int64_t rows_per_block, int64_t row_begin, int64_t row_end) {
  csr5_tiles<W, S, MODE, false>(C, Csr5Push{}, t_begin, t_end, rows_per_block, row_begin, row_end);
}

// The same tiles fused with the exchange (csr5_push_block epilogue).
template <int W, int S>
__global__ void __launch_bounds__(256, SPMVB_CSR5_MINB) k_csr5_warp_s_push(Csr5Ctx C, Csr5Push P, int64_t t_begin,
                                                                          int64_t t_end, int64_t row_begin,
                                                                          int64_t row_end) {
  csr5_tiles<W, S, 0, true>(C, P, t_begin, t_end, 0, row_begin, row_end);
}

// Carry fix-up of the continuation chains (consecutive tiles whose head
// continues the same row) inside [t_begin, t_end), chain by chain in tile
// order (fold_chains); the carries are already scaled.
template <bool PUSH = false>
__global__ void k_csr5_fixup(int64_t t_begin, int64_t t_end, const int32_t* __restrict__ tile_ptr,
                             const uint32_t* __restrict__ aux, const double* __restrict__ carry,
                             double* __restrict__ y, const uint64_t* __restrict__ peers, int n_peers,
                             int64_t push_off) {
  pdl_wait();  // launched as a programmatic dependent of the tile kernel
  // chain key = the continued row, tile_ptr[t] (coalesced, loaded alongside
  // aux[t] rather than after it)
  fold_chains(
      t_begin, t_end,
      [&](int64_t t) -> int32_t {
        const uint32_t a = aux[t];
        const int32_t r = tile_ptr[t];
        return (a & 0x80000000u) ? r : -1;
      },
      [&](int64_t t) { return carry[t]; },
      [&](int32_t r, double acc) {
        const double v = y[r] + acc;
        y[r] = v;
        if constexpr (PUSH)
          for (int p = 0; p < n_peers; ++p) reinterpret_cast<double*>(peers[p])[push_off + r] = v;
      });
}

// One range of tiles, [t_begin, t_end), with the empty rows of [row_begin,
// row_end): the per-tile kernel(s), then the carry fix-up of the chains
// inside the range.  Ranges that start at row-start tiles (the range plan)
// fold exactly like the whole matrix, in any order.
void launch_range(const Csr5Ctx& C, int64_t t_begin, int64_t t_end, int64_t row_begin, int64_t row_end,
                  cudaStream_t s, const Csr5Push& P = Csr5Push{}) {
  const bool empties = C.nonempty && row_end > row_begin;
  // prefix layout: rows [tail0, row_end) of the range are empty
  const int64_t tail0 = C.n_nonempty > row_begin ? C.n_nonempty : row_begin;
  const bool tail = !C.nonempty && C.n_nonempty < C.n_rows && row_end > tail0;
  auto empty_pass = [&] {
    if (empties || tail) {
      const int64_t z0 = empties ? row_begin : tail0;
      k_csr5_empty_rows<<<grid_for(row_end - z0, 256, 148 * 32), 256, 0, s>>>(row_end - z0, C.ptr + z0, C.y + z0);
      SPMVB_LAUNCHED("k_csr5_empty_rows");
    }
  };
  if (t_end <= t_begin) {
    empty_pass();
    return;
  }
  const int64_t tile = static_cast<int64_t>(C.omega) * C.sigma;
  const int64_t full = C.nnz / tile;
  const int64_t fe = t_end < full ? t_end : full;  // full tiles in range: [t_begin, fe)
  int64_t generic_begin = t_begin;
  auto warp_launch = [&](auto kern, int W) {
    empty_pass();
    if (fe > t_begin) {
      kern<<<grid_for((fe - t_begin) * W, 256), 256, 0, s>>>(C, t_begin, fe);
      SPMVB_LAUNCHED("k_csr5_warp");
      generic_begin = fe;
    }
  };
  auto warp_s_launch = [&](auto kern_e, auto kern_t, auto kern, int W) {  // every tile incl. the partial one, plus the empty rows
    const int64_t blocks = ((t_end - t_begin) * W + 255) / 256;
    int64_t rpb = 0, z0 = row_begin;
    if (empties) {
      rpb = (row_end - row_begin + blocks - 1) / blocks;
      kern = kern_e;
    } else if (tail) {
      z0 = tail0;
      rpb = (row_end - tail0 + blocks - 1) / blocks;
      kern = kern_t;
    }
    launch_pdl(kern, dim3(static_cast<unsigned>(blocks)), dim3(256), 0, s, C, t_begin, t_end, rpb, z0, row_end);
    SPMVB_LAUNCHED("k_csr5_warp_s");
    generic_begin = t_end;
  };
  const int omega = C.omega, sigma = C.sigma;
  if (P.n_peers > 0) {  // fused exchange: each block also stores its rows into the peers
    if (omega != 32 || (sigma != 16 && sigma != 8))
      fail(SPMVB_INVALID_ARG, "the fused exchange needs omega = 32 and sigma = 16 or 8, got %d, %d", omega, sigma);
    const int64_t blocks = ((t_end - t_begin) * 32 + 255) / 256;
    auto kern = sigma == 16 ? k_csr5_warp_s_push<32, 16> : k_csr5_warp_s_push<32, 8>;
    launch_pdl(kern, dim3(static_cast<unsigned>(blocks)), dim3(256), 0, s, C, P, t_begin, t_end, row_begin, row_end);
    SPMVB_LAUNCHED("k_csr5_warp_s_push");
    generic_begin = t_end;
  } else if ((sigma == 16 || sigma == 8) && (omega == 32 || omega == 16 || omega == 8 || omega == 4)) {
    if (sigma == 16) {
      switch (omega) {
        case 32: warp_s_launch(k_csr5_warp_s<32, 16, 1>, k_csr5_warp_s<32, 16, 2>, k_csr5_warp_s<32, 16, 0>, 32); break;
        case 16: warp_s_launch(k_csr5_warp_s<16, 16, 1>, k_csr5_warp_s<16, 16, 2>, k_csr5_warp_s<16, 16, 0>, 16); break;
        case 8: warp_s_launch(k_csr5_warp_s<8, 16, 1>, k_csr5_warp_s<8, 16, 2>, k_csr5_warp_s<8, 16, 0>, 8); break;
        default: warp_s_launch(k_csr5_warp_s<4, 16, 1>, k_csr5_warp_s<4, 16, 2>, k_csr5_warp_s<4, 16, 0>, 4); break;
      }
    } else {
      switch (omega) {
        case 32: warp_s_launch(k_csr5_warp_s<32, 8, 1>, k_csr5_warp_s<32, 8, 2>, k_csr5_warp_s<32, 8, 0>, 32); break;
        case 16: warp_s_launch(k_csr5_warp_s<16, 8, 1>, k_csr5_warp_s<16, 8, 2>, k_csr5_warp_s<16, 8, 0>, 16); break;
        case 8: warp_s_launch(k_csr5_warp_s<8, 8, 1>, k_csr5_warp_s<8, 8, 2>, k_csr5_warp_s<8, 8, 0>, 8); break;
        default: warp_s_launch(k_csr5_warp_s<4, 8, 1>, k_csr5_warp_s<4, 8, 2>, k_csr5_warp_s<4, 8, 0>, 4); break;
      }
    }
  } else if (sigma <= 1024 && (omega == 32 || omega == 16 || omega == 8 || omega == 4 || omega == 2)) {
    switch (omega) {
      case 32: warp_launch(k_csr5_warp<32>, 32); break;
      case 16: warp_launch(k_csr5_warp<16>, 16); break;
      case 8: warp_launch(k_csr5_warp<8>, 8); break;
      case 4: warp_launch(k_csr5_warp<4>, 4); break;
      default: warp_launch(k_csr5_warp<2>, 2); break;
    }
  } else {
    empty_pass();
  }
  if (generic_begin < t_end) {
    k_csr5_generic<<<grid_for(t_end - generic_begin, 128, 148 * 64), 128, 0, s>>>(C, generic_begin, t_end);
    SPMVB_LAUNCHED("k_csr5_generic");
  }
  if (t_end - t_begin > 1 || t_begin > 0) {
    // one 32-tile window per warp: every window's loads are in flight at once
    if (P.n_peers > 0)
      launch_pdl(k_csr5_fixup<true>, dim3(grid_for(t_end - t_begin, 256)), dim3(256), 0, s, t_begin, t_end,
                 C.tile_ptr, C.aux, C.carry, C.y, P.peers, P.n_peers, P.push_off);
    else
      launch_pdl(k_csr5_fixup<false>, dim3(grid_for(t_end - t_begin, 256)), dim3(256), 0, s, t_begin, t_end,
                 C.tile_ptr, C.aux, C.carry, C.y, static_cast<const uint64_t*>(nullptr), 0, int64_t(0));
    SPMVB_LAUNCHED("k_csr5_fixup");
  }
}

// bit_flag (one byte per stored entry) -> one bit per entry: word w holds
// entries 32w .. 32w+31 (a warp ballot per word).
__global__ void k_csr5_pack_flags(int64_t nnz, const uint8_t* __restrict__ flag, uint32_t* __restrict__ bits) {
  const int lane = threadIdx.x & 31;
  const int64_t words = (nnz + 31) / 32;
  for (int64_t w = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5; w < words;
       w += (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5) {
    const int64_t e = w * 32 + lane;
    const unsigned b = __ballot_sync(0xffffffffu, e < nnz && flag[e] != 0);
    if (lane == 0) bits[w] = b;
  }
}

// First tile at or after `target` whose head starts a row (not a continuation).
__global__ void k_csr5_range_starts(int64_t num_tiles, const uint32_t* __restrict__ aux, int n_ranges,
                                    int64_t* __restrict__ bounds) {
  const int k = blockIdx.x + 1;  // interior bounds 1 .. n_ranges-1
  const int lane = threadIdx.x;
  const int64_t target = num_tiles * k / n_ranges;
  int64_t found = num_tiles;
  for (int64_t b = target; b < num_tiles; b += 32) {
    const int64_t t = b + lane;
    const unsigned m = __ballot_sync(0xffffffffu, t < num_tiles && !(aux[t] & 0x80000000u));
    if (m) {
      found = b + __ffs(m) - 1;
      break;
    }
  }
  if (lane == 0) bounds[k] = found;
}

cudaStream_t copy_stream(int dev) {
  static std::mutex mu;
  static cudaStream_t streams[64] = {};
  std::lock_guard<std::mutex> lock(mu);
  if (dev < 0 || dev >= 64) fail(SPMVB_INVALID_ARG, "device ordinal out of range");
  if (!streams[dev]) SPMVB_CUDA(cudaStreamCreateWithFlags(&streams[dev], cudaStreamNonBlocking));
  return streams[dev];
}

}  // namespace

extern "C" int spmvb_spmv_csr5(int64_t n_rows, int64_t nnz, const int32_t* ptr, int omega, int sigma,
                               const int32_t* tile_ptr, const uint8_t* bit_flag, const uint32_t* flag_bits,
                               const int32_t* col, const double* val,
                               const uint32_t* tile_aux, const int32_t* nonempty_rows, int64_t n_nonempty,
                               double* carry, const double* x, double* y, const double* scale, void* stream) {
  return guard([&] {
    cudaStream_t s = as_stream(stream);
    if (n_rows <= 0) return;
    if (nnz == 0) {
      SPMVB_CUDA(cudaMemsetAsync(y, 0, n_rows * sizeof(double), s));
      return;
    }
    if (omega < 1 || sigma < 1) fail(SPMVB_INVALID_ARG, "omega and sigma must be >= 1");
    Csr5Ctx C{n_rows, nnz, n_nonempty, omega, sigma, ptr, tile_ptr, bit_flag, flag_bits, col, val, tile_aux,
              nonempty_rows, carry, x, y, scale};
    const int64_t tile = static_cast<int64_t>(omega) * sigma;
    launch_range(C, 0, (nnz + tile - 1) / tile, 0, n_rows, s);
  });
}


extern "C" int spmvb_csr5_range_bounds(int64_t nnz, int omega, int sigma, const int32_t* tile_ptr,
                                       const uint32_t* tile_aux, int n_ranges, int64_t* tile_bounds,
                                       int64_t* row_bounds, void* stream) {
  return guard([&] {
    cudaStream_t s = as_stream(stream);
    if (omega < 1 || sigma < 1) fail(SPMVB_INVALID_ARG, "omega and sigma must be >= 1");
    if (n_ranges < 1) fail(SPMVB_INVALID_ARG, "n_ranges must be >= 1");
    const int64_t tile = static_cast<int64_t>(omega) * sigma;
    const int64_t num_tiles = (nnz + tile - 1) / tile;
    DevBuf<int64_t> d(n_ranges + 1, s);
    if (n_ranges > 1 && num_tiles > 0) {
      k_csr5_range_starts<<<n_ranges - 1, 32, 0, s>>>(num_tiles, tile_aux, n_ranges, d.ptr);
      SPMVB_LAUNCHED("k_csr5_range_starts");
      SPMVB_CUDA(cudaMemcpyAsync(tile_bounds + 1, d.ptr + 1, (n_ranges - 1) * sizeof(int64_t),
                                 cudaMemcpyDeviceToHost, s));
    }
    std::vector<int32_t> tp(num_tiles + 1);
    SPMVB_CUDA(cudaMemcpyAsync(tp.data(), tile_ptr, (num_tiles + 1) * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    SPMVB_CUDA(cudaStreamSynchronize(s));
    tile_bounds[0] = 0;
    tile_bounds[n_ranges] = num_tiles;
    if (num_tiles == 0)
      for (int k = 1; k < n_ranges; ++k) tile_bounds[k] = 0;
    for (int k = 1; k <= n_ranges; ++k)
      if (tile_bounds[k] < tile_bounds[k - 1]) tile_bounds[k] = tile_bounds[k - 1];
    for (int k = 0; k <= n_ranges; ++k) row_bounds[k] = tp[tile_bounds[k]];
    row_bounds[0] = 0;
  });
}

extern "C" int spmvb_spmv_csr5_host(int64_t n_rows, int64_t n_cols, int64_t nnz, const int32_t* ptr, int omega,
                                    int sigma, const int32_t* tile_ptr, const uint8_t* bit_flag,
                                    const uint32_t* flag_bits, const int32_t* col,
                                    const double* val, const uint32_t* tile_aux, const int32_t* nonempty_rows,
                                    int64_t n_nonempty, double* carry, const double* x_host, double* x_dev,
                                    double* y_dev, double* y_host, const double* scale, int n_ranges,
                                    const int64_t* tile_bounds, const int64_t* row_bounds, void* stream) {
  return guard([&] {
    cudaStream_t s = as_stream(stream);
    if (omega < 1 || sigma < 1) fail(SPMVB_INVALID_ARG, "omega and sigma must be >= 1");
    if (n_ranges < 1 || !tile_bounds || !row_bounds) fail(SPMVB_INVALID_ARG, "range plan missing");
    if (n_cols > 0) SPMVB_CUDA(cudaMemcpyAsync(x_dev, x_host, n_cols * sizeof(double), cudaMemcpyHostToDevice, s));
    if (n_rows <= 0) {
      SPMVB_CUDA(cudaStreamSynchronize(s));
      return;
    }
    if (nnz == 0) {
      SPMVB_CUDA(cudaMemsetAsync(y_dev, 0, n_rows * sizeof(double), s));
      SPMVB_CUDA(cudaMemcpyAsync(y_host, y_dev, n_rows * sizeof(double), cudaMemcpyDeviceToHost, s));
      SPMVB_CUDA(cudaStreamSynchronize(s));
      return;
    }
    const int64_t tile = static_cast<int64_t>(omega) * sigma;
    const int64_t num_tiles = (nnz + tile - 1) / tile;
    if (tile_bounds[0] != 0 || tile_bounds[n_ranges] != num_tiles || row_bounds[0] != 0)
      fail(SPMVB_INVALID_ARG, "range plan does not cover the tiles");
    int dev = 0;
    SPMVB_CUDA(cudaGetDevice(&dev));
    cudaStream_t cs = copy_stream(dev);
    Csr5Ctx C{n_rows, nnz, n_nonempty, omega, sigma, ptr, tile_ptr, bit_flag, flag_bits, col, val, tile_aux,
              nonempty_rows, carry, x_dev, y_dev, scale};
    std::vector<cudaEvent_t> evs;
    auto event_on = [&](cudaStream_t st) {
      cudaEvent_t e;
      SPMVB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      evs.push_back(e);
      SPMVB_CUDA(cudaEventRecord(e, st));
      return e;
    };
    // Ranges run last-to-first: R-MAT-like matrices put their light rows at
    // the end, so the first ranges finish many rows and the copy-back starts
    // early.  No carry chain crosses a range (each starts at a row-start
    // tile), so the rows of a range are final after its own fix-up.
    for (int k = n_ranges - 1; k >= 0; --k) {
      const int64_t tb = tile_bounds[k], te = tile_bounds[k + 1];
      if (te < tb || te > num_tiles) fail(SPMVB_INVALID_ARG, "range plan is not monotone");
      const int64_t lo = row_bounds[k], hi = k + 1 == n_ranges ? n_rows : row_bounds[k + 1];
      if (lo < 0 || hi < lo || hi > n_rows) fail(SPMVB_INVALID_ARG, "range plan rows out of bounds");
      launch_range(C, tb, te, lo, hi, s);
      if (hi > lo) {
        SPMVB_CUDA(cudaStreamWaitEvent(cs, event_on(s), 0));
        SPMVB_CUDA(cudaMemcpyAsync(y_host + lo, y_dev + lo, (hi - lo) * sizeof(double), cudaMemcpyDeviceToHost, cs));
      }
    }
    SPMVB_CUDA(cudaStreamWaitEvent(s, event_on(cs), 0));
    SPMVB_CUDA(cudaStreamSynchronize(s));
    for (cudaEvent_t e : evs) cudaEventDestroy(e);
  });
}

extern "C" int spmvb_spmv_csr5_tiles(int64_t n_rows, int64_t nnz, const int32_t* ptr, int omega, int sigma,
                                     const int32_t* tile_ptr, const uint8_t* bit_flag, const uint32_t* flag_bits,
                                     const int32_t* col,
                                     const double* val, const uint32_t* tile_aux, const int32_t* nonempty_rows,
                                     int64_t n_nonempty, double* carry, const double* x, double* y,
                                     const double* scale, int64_t t_begin, int64_t t_end, int64_t row_begin,
                                     int64_t row_end, void* stream) {
  return guard([&] {
    cudaStream_t s = as_stream(stream);
    if (omega < 1 || sigma < 1) fail(SPMVB_INVALID_ARG, "omega and sigma must be >= 1");
    const int64_t tile = static_cast<int64_t>(omega) * sigma;
    const int64_t num_tiles = (nnz + tile - 1) / tile;
    if (t_begin < 0 || t_end < t_begin || t_end > num_tiles || row_begin < 0 || row_end < row_begin ||
        row_end > n_rows)
      fail(SPMVB_INVALID_ARG, "tile/row range out of bounds");
    if (nnz == 0) {
      if (row_end > row_begin)
        SPMVB_CUDA(cudaMemsetAsync(y + row_begin, 0, (row_end - row_begin) * sizeof(double), s));
      return;
    }
    Csr5Ctx C{n_rows, nnz, n_nonempty, omega, sigma, ptr, tile_ptr, bit_flag, flag_bits, col, val, tile_aux,
              nonempty_rows, carry, x, y, scale};
    launch_range(C, t_begin, t_end, row_begin, row_end, s);
  });
}

extern "C" int spmvb_csr5_pack_flags(int64_t nnz, const uint8_t* bit_flag, uint32_t* flag_bits, void* stream) {
  return guard([&] {
    cudaStream_t s = as_stream(stream);
    if (nnz <= 0) return;
    k_csr5_pack_flags<<<grid_for((nnz + 31) / 32 * 32, 256, 148 * 16), 256, 0, s>>>(nnz, bit_flag, flag_bits);
    SPMVB_LAUNCHED("k_csr5_pack_flags");
  });
}

extern "C" int spmvb_spmv_csr5_push(int64_t n_rows, int64_t nnz, const int32_t* ptr, int omega, int sigma,
                                    const int32_t* tile_ptr, const uint8_t* bit_flag, const uint32_t* flag_bits,
                                    const int32_t* col, const double* val, const uint32_t* tile_aux,
                                    const int32_t* nonempty_rows, int64_t n_nonempty, double* carry, const double* x,
                                    double* y, const double* scale, const uint64_t* peers, int n_peers,
                                    int64_t push_off, void* stream) {
  return guard([&] {
    cudaStream_t s = as_stream(stream);
    if (n_peers < 0 || (n_peers > 0 && !peers)) fail(SPMVB_INVALID_ARG, "peer buffer list missing");
    if (push_off < 0) fail(SPMVB_INVALID_ARG, "negative push offset");
    if (n_rows <= 0) return;
    if (omega < 1 || sigma < 1) fail(SPMVB_INVALID_ARG, "omega and sigma must be >= 1");
    if (nnz == 0 || n_peers == 0) {  // nothing to fuse with: plain SpMV, then the rows (if any peers) pushed
      if (nnz == 0) SPMVB_CUDA(cudaMemsetAsync(y, 0, n_rows * sizeof(double), s));
      else {
        Csr5Ctx C{n_rows, nnz, n_nonempty, omega, sigma, ptr, tile_ptr, bit_flag, flag_bits, col, val, tile_aux,
                  nonempty_rows, carry, x, y, scale};
        const int64_t tile = static_cast<int64_t>(omega) * sigma;
        launch_range(C, 0, (nnz + tile - 1) / tile, 0, n_rows, s);
      }
      if (n_peers > 0)
        if (const int st = spmvb_push_rows(y, n_rows, peers, n_peers, push_off, stream)) {
          const std::string msg = spmvb_last_error();
          fail(st, "%s", msg.c_str());
        }
      return;
    }
    Csr5Ctx C{n_rows, nnz, n_nonempty, omega, sigma, ptr, tile_ptr, bit_flag, flag_bits, col, val, tile_aux,
              nonempty_rows, carry, x, y, scale};
    const int64_t tile = static_cast<int64_t>(omega) * sigma;
    launch_range(C, 0, (nnz + tile - 1) / tile, 0, n_rows, s, Csr5Push{peers, n_peers, push_off});
  });
}
