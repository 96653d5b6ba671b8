// ELL and SELL(-C-sigma) SpMV (reference kernels.py:98-136): one thread per
// (permuted) row, sequential accumulation over all slots with separately
// rounded products, which is bit-identical to the reference kernels.
#include "spmv_common.cuh"

using namespace spmvb;

namespace {

// ================================================================ ELL ====
// Thread per row over the column-major grid (coalesced slot loads), the
// reference's sequential slot recurrence (bit-identical).  PF: the next four
// slots' loads are in flight while the current four are summed (k >= 8);
// without it more threads fit per SM (short rows).
#ifndef SPMVB_ELL_PREFETCH_X
#define SPMVB_ELL_PREFETCH_X 1
#endif
template <bool PF>
__global__ void k_spmv_ell(int64_t n_rows, int64_t k, const int32_t* __restrict__ idx, const double* __restrict__ val,
                           const double* __restrict__ x, double* __restrict__ y, const double* __restrict__ scale_p,
                           int64_t n_cols) {
  pdl_wait();
#if SPMVB_ELL_PREFETCH_X
  // x into L2 alongside the first slot loads: the gathers that follow them
  // then wait for L2, not for a second DRAM round trip (a one-wave kernel
  // such as C1 is two dependent DRAM latencies long)
  {
    const int64_t line = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (line * 16 < n_cols) asm volatile("prefetch.global.L2 [%0];" ::"l"(x + line * 16));
  }
#endif
  const double s = load_scale(scale_p);
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < n_rows;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double acc = PF ? seq_slots(k, n_rows, r, idx, val, x) : seq_slots4(k, n_rows, r, idx, val, x);
    y[r] = scale_p ? s * acc : acc;
  }
}

// =============================================================== SELL ====
#ifndef SPMVB_SELL_PF
#define SPMVB_SELL_PF 4  // slots per prefetch step of the narrow SELL loop (MODE 2/3)
#endif
#ifndef SPMVB_SELL_WIDE_U
#define SPMVB_SELL_WIDE_U 8  // column cells in flight per thread in k_sell_wide_part
#endif
// MODE 0: four slots per step; 1: the same through L1 (c < 8); 2: with the
// next four slots prefetched (rows of 8 slots or more); 3: prefetched and
// through L1 (c < 8, rows of 8 slots or more).
template <int MODE>
#ifndef SPMVB_SELL_MINB2
#define SPMVB_SELL_MINB2 5  // resident blocks of the prefetching (MODE 2/3) loop
#endif
__global__ void __launch_bounds__(256, MODE == 0 ? 8 : (MODE >= 2 ? (SPMVB_SELL_PF > 4 ? 4 : SPMVB_SELL_MINB2) : 4)) k_spmv_sell(int64_t n_rows, int64_t c, const int64_t* __restrict__ widths,
                            const int64_t* __restrict__ slice_off, const int32_t* __restrict__ perm,
                            const int32_t* __restrict__ idx, const double* __restrict__ val,
                            const double* __restrict__ x, double* __restrict__ y, const double* __restrict__ scale_p,
                            int64_t wide_cols, int64_t tail_from, int64_t p_begin, int64_t p_end) {
  pdl_wait();
  const double s = load_scale(scale_p);
  const double zero = scale_p ? s * 0.0 : 0.0;  // an empty row's result
  const int32_t c32 = static_cast<int32_t>(c);  // n_rows < 2^31: 32-bit slice arithmetic
  for (int64_t p = p_begin + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < p_end;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (p >= tail_from) {  // the empty tail (perm is the identity there): plain coalesced stores
      y[p] = zero;
      continue;
    }
    const int32_t p32 = static_cast<int32_t>(p);
    const int32_t sl = p32 / c32, local = p32 - sl * c32;
    const int64_t rows_s = (static_cast<int64_t>(sl) + 1) * c <= n_rows ? c : n_rows - static_cast<int64_t>(sl) * c;
    const int64_t w = widths[sl];
    if (w > wide_cols && rows_s <= 128) continue;  // k_sell_wide_part's slice
    const int64_t base = slice_off[sl] + local;
    const double acc = MODE >= 2 ? seq_slots<MODE == 3, SPMVB_SELL_PF>(w, rows_s, base, idx, val, x)
                                 : seq_slots4<MODE == 1>(w, rows_s, base, idx, val, x);
    const int64_t r = perm ? static_cast<int64_t>(perm[p]) : p;
    y[r] = scale_p ? s * acc : acc;
  }
}

// Wide slices (width > SPMVB_SELL_WIDE_COLS, power-law rows; up to 128
// rows): split into pieces of about SELL_PIECE_CELLS cells (whole columns),
// one CTA per piece.  256/rows threads per row each sum every (256/rows)-th
// column of the piece (coalesced: consecutive threads read consecutive
// column-major cells), a fixed-order per-row sum of the thread partials goes
// to the piece's slot, and a second kernel adds each row's pieces in order.
// Deterministic; not the reference's sequential order, so within tolerance
// rather than bit-exact.  (One CTA per whole slice serialised the widest
// R-MAT slices: 33 ms of a C5 SELL SpMV.)
constexpr int SELL_PART_STRIDE = 128;  // partial slots per piece (max rows of a wide slice)

// pieces per wide slice
__global__ void k_sell_wide_pieces(int64_t n_rows, int64_t c, const int32_t* __restrict__ wide, int64_t n_wide,
                                   const int64_t* __restrict__ widths, int32_t* __restrict__ pieces) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n_wide;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t sl = wide[i];
    const int64_t pc = sell_piece_cols(sell_rows(sl, c, n_rows));
    pieces[i] = static_cast<int32_t>((widths[sl] + pc - 1) / pc);
  }
}

// One CTA per piece (grid-stride over the device-side piece count).
__global__ void __launch_bounds__(256) k_sell_wide_part(int64_t n_rows, int64_t c, const int32_t* __restrict__ wide,
                                                        int64_t n_wide, const int32_t* __restrict__ first_piece,
                                                        int64_t n_pieces,
                                                        const int64_t* __restrict__ widths,
                                                        const int64_t* __restrict__ slice_off,
                                                        const int32_t* __restrict__ idx, const double* __restrict__ val,
                                                        const double* __restrict__ x, double* __restrict__ part,
                                                        int32_t pc_begin, int32_t pc_end) {
  pdl_wait();
  __shared__ double red[256];
  const int t = threadIdx.x;
  for (int32_t item = pc_begin + blockIdx.x; item < pc_end; item += gridDim.x) {
    // wide slice holding this piece: last i with first_piece[i] <= item
    int64_t lo = 0, hi = n_wide - 1;
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) >> 1;
      if (first_piece[mid] <= item) lo = mid;
      else hi = mid - 1;
    }
    const int64_t sl = wide[lo];
    const int rows_s = sell_rows(sl, c, n_rows);
    const int64_t pc = sell_piece_cols(rows_s);
    const int64_t j0 = static_cast<int64_t>(item - first_piece[lo]) * pc;
    const int64_t w = widths[sl];
    const int64_t j1 = j0 + pc < w ? j0 + pc : w;
    const int nsub = 256 / rows_s;
    const int sub = t / rows_s, l = t - sub * rows_s;
    const int64_t base = slice_off[sl];
    double acc = 0.0;
    if (sub < nsub) {
      const int64_t st = static_cast<int64_t>(nsub) * rows_s;
      int64_t j = j0 + sub;
      constexpr int WU = SPMVB_SELL_WIDE_U;
      for (; j + (WU - 1) * nsub < j1; j += WU * nsub) {
        const int64_t o = base + j * rows_s + l;
        double v[WU];
        int32_t cc[WU];
#pragma unroll
        for (int u = 0; u < WU; ++u) {
          v[u] = ld_stream(val + o + u * st);
          cc[u] = ld_stream(idx + o + u * st);
        }
#pragma unroll
        for (int u = 0; u < WU; ++u) acc += v[u] * ldx(x, cc[u]);
      }
      for (; j < j1; j += nsub) {
        const int64_t o = base + j * rows_s + l;
        acc += ld_stream(val + o) * ldx(x, ld_stream(idx + o));
      }
    }
    red[t] = acc;
    __syncthreads();
    if (t < rows_s) {
      double sum = 0.0;
      for (int k = 0; k < nsub; ++k) sum += red[t + k * rows_s];
      part[static_cast<int64_t>(item) * SELL_PART_STRIDE + t] = sum;
    }
    __syncthreads();
  }
}

// The rows of the wide slices, summed from their pieces in a fixed order:
// deterministic.  A slice of at most SPMVB_SELL_HUB_PIECES pieces (the
// common case; a reference-layout power-law matrix has ~1e5 of them) is a
// thread per row adding its pieces in order.  Slices with more pieces (a
// degree-ordered matrix's hub rows, ~400 pieces at C5) are listed in `hub`
// and summed by k_sell_wide_hub instead: one thread walking ~400 dependent
// loads took 41 us.
__global__ void k_sell_wide_final(int64_t n_rows, int64_t c, const int32_t* __restrict__ wide, int64_t n_wide,
                                  const int32_t* __restrict__ first_piece, int64_t n_pieces,
                                  const double* __restrict__ part, const int32_t* __restrict__ perm,
                                  double* __restrict__ y, const double* __restrict__ scale_p, int64_t i_begin,
                                  int64_t i_end) {
  pdl_wait();
  const double sc = load_scale(scale_p);
  for (int64_t q = i_begin * c + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < i_end * c;
       q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = q / c;
    const int l = static_cast<int>(q - i * c);
    const int64_t sl = wide[i];
    if (l >= sell_rows(sl, c, n_rows)) continue;
    const int32_t p0 = first_piece[i], p1 = i + 1 < n_wide ? first_piece[i + 1] : static_cast<int32_t>(n_pieces);
    if (p1 - p0 > SPMVB_SELL_HUB_PIECES) continue;  // k_sell_wide_hub's slice
    double sum = 0.0;
    for (int32_t pc = p0; pc < p1; ++pc) sum += part[static_cast<int64_t>(pc) * SELL_PART_STRIDE + l];
    const int64_t p = sl * c + l;
    const int64_t r = perm ? static_cast<int64_t>(perm[p]) : p;
    y[r] = scale_p ? sc * sum : sum;
  }
}

// Warp per (hub slice, row): lane k adds pieces k, k+32, ... in order, then
// the xor butterfly.  hub[h] = index into the wide list.
__global__ void k_sell_wide_hub(int64_t n_rows, int64_t c, const int32_t* __restrict__ wide, int64_t n_wide,
                                const int32_t* __restrict__ first_piece, int64_t n_pieces,
                                const int32_t* __restrict__ hub, const double* __restrict__ part,
                                const int32_t* __restrict__ perm, double* __restrict__ y,
                                const double* __restrict__ scale_p, int64_t h_begin, int64_t h_end) {
  pdl_wait();
  const double sc = load_scale(scale_p);
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t q = h_begin * c + warp; q < h_end * c; q += nwarps) {
    const int64_t h = q / c;
    const int l = static_cast<int>(q - h * c);
    const int64_t i = hub[h];
    const int64_t sl = wide[i];
    if (l >= sell_rows(sl, c, n_rows)) continue;
    const int32_t p0 = first_piece[i], p1 = i + 1 < n_wide ? first_piece[i + 1] : static_cast<int32_t>(n_pieces);
    double sum = 0.0;
    for (int32_t pc = p0 + lane; pc < p1; pc += 32) sum += part[static_cast<int64_t>(pc) * SELL_PART_STRIDE + l];
    sum = warp_sum(sum);
    if (lane == 0) {
      const int64_t p = sl * c + l;
      const int64_t r = perm ? static_cast<int64_t>(perm[p]) : p;
      y[r] = scale_p ? sc * sum : sum;
    }
  }
}

__global__ void k_sell_mark_wide(const int64_t* __restrict__ widths, int64_t n_rows, int64_t c, int64_t n_slices,
                                 int64_t wide_cols, uint8_t* __restrict__ flag) {
  for (int64_t s = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; s < n_slices;
       s += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t rows_s = (s + 1) * c <= n_rows ? c : n_rows - s * c;
    flag[s] = (widths[s] > wide_cols && rows_s <= 128) ? 1 : 0;
  }
}

}  // namespace

extern "C" int spmvb_sell_wide_plan(int64_t n_rows, int64_t c, const int64_t* widths, int64_t wide_cols,
                                    int32_t* wide_out, int64_t* n_wide, int64_t* max_narrow_width,
                                    int32_t* first_piece_out, int64_t* n_pieces, void* stream) {
  return guard([&] {
    cudaStream_t s = as_stream(stream);
    if (wide_cols <= 0) wide_cols = SPMVB_SELL_WIDE_COLS;
    if (wide_cols < SPMVB_SELL_WIDE_COLS) fail(SPMVB_INVALID_ARG, "wide_cols must be >= %d", SPMVB_SELL_WIDE_COLS);
    *n_wide = 0;
    if (max_narrow_width) *max_narrow_width = 0;
    if (n_pieces) *n_pieces = 0;
    if (n_rows <= 0 || c < 1) return;
    const int64_t n_slices = (n_rows + c - 1) / c;
    DevBuf<uint8_t> flag(n_slices, s);
    k_sell_mark_wide<<<grid_for(n_slices, 256, 148 * 16), 256, 0, s>>>(widths, n_rows, c, n_slices, wide_cols,
                                                                      flag.get());
    SPMVB_LAUNCHED("k_sell_mark_wide");
    const uint8_t* f = flag.get();
    DevBuf<int32_t> total(1, s);
    exclusive_scan<int32_t>(
        n_slices, [=] __device__(int64_t i) { return static_cast<int32_t>(f[i]); },
        [=] __device__(int64_t i, int32_t v) {
          if (f[i]) wide_out[v] = static_cast<int32_t>(i);
        },
        OpSum{}, 0, total.get(), s);
    int32_t h = 0;
    copy_to_host(&h, total.get(), 1, s);
    *n_wide = h;
    if (max_narrow_width) {
      DevBuf<int64_t> mx(1, s);
      device_reduce<int64_t>(
          n_slices, [=] __device__(int64_t i) -> int64_t { return f[i] ? 0 : widths[i]; }, OpMax{}, int64_t{0},
          mx.get(), s);
      copy_to_host(max_narrow_width, mx.get(), 1, s);
    }
    if (h > 0 && first_piece_out && n_pieces) {
      // pieces of ~SELL_PIECE_CELLS cells per wide slice, as a prefix
      DevBuf<int32_t> np(h, s), tp(1, s);
      k_sell_wide_pieces<<<grid_for(h, 256), 256, 0, s>>>(n_rows, c, wide_out, h, widths, np.get());
      SPMVB_LAUNCHED("k_sell_wide_pieces");
      exclusive_scan<int32_t>(h, ArrayLoad<int32_t>{np.get()}, ArrayStore<int32_t>{first_piece_out}, OpSum{}, 0,
                              tp.get(), s);
      int32_t hp = 0;
      copy_to_host(&hp, tp.get(), 1, s);
      *n_pieces = hp;
    }
  });
}

extern "C" int spmvb_spmv_ell(int64_t n_rows, int64_t n_cols, int64_t k, const int32_t* idx, const double* val,
                              const double* x, double* y, const double* scale, void* stream) {
  return guard([&] {
    cudaStream_t s = as_stream(stream);
    if (n_rows <= 0) return;
    const dim3 g(grid_for(n_rows, 256)), b(256);
    // the prefetching slot loop from two full 4-slot steps on (C2, k = 8:
    // 24.6 -> 22.7 us L2-flushed); shorter rows keep the lighter loop
    if (k >= 8) launch_pdl(k_spmv_ell<true>, g, b, 0, s, n_rows, k, idx, val, x, y, scale, n_cols);
    else launch_pdl(k_spmv_ell<false>, g, b, 0, s, n_rows, k, idx, val, x, y, scale, n_cols);
    SPMVB_LAUNCHED("k_spmv_ell");
  });
}

namespace {

// Slices [s_begin, s_end) of a SELL SpMV: the per-row kernel over their rows,
// the pieces [pc_begin, pc_end) of the wide slices [i_begin, i_end) among
// them, and those wide rows' sums.
void sell_launch(int64_t n_rows, int64_t c, const int64_t* widths, const int64_t* slice_off, const int32_t* perm,
                 const int32_t* idx, const double* val, const int32_t* wide, int64_t n_wide,
                 const int32_t* first_piece, int64_t n_pieces, const int32_t* hub, int64_t n_hub, int64_t wide_cols,
                 int64_t tail_from, int64_t max_narrow_width, const double* x, double* y, const double* scale,
                 int64_t s_begin, int64_t s_end, int64_t i_begin, int64_t i_end, int64_t pc_begin, int64_t pc_end,
                 int64_t h_begin, int64_t h_end, cudaStream_t s) {
  if (wide_cols <= 0) wide_cols = SPMVB_SELL_WIDE_COLS;
  if (tail_from < 0 || tail_from > n_rows) tail_from = n_rows;
  const int64_t p_begin = s_begin * c, p_end = s_end * c < n_rows ? s_end * c : n_rows;
  if (p_end > p_begin) {
    // c < 8: slot loads through L1 (the other half of each index sector is
    // the next slot's); rows of 8 or more slots: next four slots prefetched
    // (C2 / C3 with the reference default C = 4: mode 3 41.0 / 63.5 ->
    // 36.9 / 50.2 us L2-flushed against mode 1)
    const unsigned g = grid_for(p_end - p_begin, 256);
    const bool wide_rows = max_narrow_width >= 8 || max_narrow_width < 0;
    auto kern = c < 8 ? (wide_rows ? k_spmv_sell<3> : k_spmv_sell<1>) : (wide_rows ? k_spmv_sell<2> : k_spmv_sell<0>);
    launch_pdl(kern, dim3(g), dim3(256), 0, s, n_rows, c, widths, slice_off, perm, idx, val, x, y, scale, wide_cols,
               tail_from, p_begin, p_end);
    SPMVB_LAUNCHED("k_spmv_sell");
  }
  if (i_end > i_begin) {
    if (!first_piece || n_pieces < n_wide || pc_end <= pc_begin) fail(SPMVB_INVALID_ARG, "wide-slice piece plan missing");
    DevBuf<double> part(static_cast<size_t>(n_pieces) * SELL_PART_STRIDE, s);
    launch_pdl(k_sell_wide_part, dim3(grid_for(pc_end - pc_begin, 1, 148 * 16)), dim3(256), 0, s, n_rows, c, wide,
               n_wide, first_piece, n_pieces, widths, slice_off, idx, val, x, part.get(),
               static_cast<int32_t>(pc_begin), static_cast<int32_t>(pc_end));
    SPMVB_LAUNCHED("k_sell_wide_part");
    launch_pdl(k_sell_wide_final, dim3(grid_for((i_end - i_begin) * c, 256, 148 * 16)), dim3(256), 0, s, n_rows, c,
               wide, n_wide, first_piece, n_pieces, part.get(), perm, y, scale, i_begin, i_end);
    SPMVB_LAUNCHED("k_sell_wide_final");
    if (h_end > h_begin) {
      if (!hub || h_end > n_hub) fail(SPMVB_INVALID_ARG, "hub slice list missing");
      launch_pdl(k_sell_wide_hub, dim3(grid_for((h_end - h_begin) * c * 32, 256, 148 * 16)), dim3(256), 0, s, n_rows,
                 c, wide, n_wide, first_piece, n_pieces, hub, part.get(), perm, y, scale, h_begin, h_end);
      SPMVB_LAUNCHED("k_sell_wide_hub");
    }
  }
}

}  // namespace

extern "C" int spmvb_spmv_sell(int64_t n_rows, int64_t c, const int64_t* widths, const int64_t* slice_off,
                               const int32_t* perm, const int32_t* idx, const double* val, const int32_t* wide,
                               int64_t n_wide, const int32_t* first_piece, int64_t n_pieces, const int32_t* hub,
                               int64_t n_hub, int64_t wide_cols, int64_t tail_from, int64_t max_narrow_width,
                               const double* x, double* y, const double* scale, void* stream) {
  return guard([&] {
    if (n_rows <= 0) return;
    sell_launch(n_rows, c, widths, slice_off, perm, idx, val, wide, n_wide, first_piece, n_pieces, hub, n_hub,
                wide_cols, tail_from, max_narrow_width, x, y, scale, 0, (n_rows + c - 1) / c, 0, n_wide, 0,
                n_pieces, 0, n_hub, as_stream(stream));
  });
}

extern "C" int spmvb_spmv_sell_range(int64_t n_rows, int64_t c, const int64_t* widths, const int64_t* slice_off,
                                     const int32_t* perm, const int32_t* idx, const double* val, const int32_t* wide,
                                     int64_t n_wide, const int32_t* first_piece, int64_t n_pieces,
                                     const int32_t* hub, int64_t n_hub, int64_t wide_cols, int64_t tail_from,
                                     int64_t max_narrow_width, const double* x, double* y, const double* scale,
                                     int64_t s_begin, int64_t s_end, int64_t i_begin, int64_t i_end, int64_t pc_begin,
                                     int64_t pc_end, int64_t h_begin, int64_t h_end, void* stream) {
  return guard([&] {
    if (n_rows <= 0) return;
    const int64_t n_slices = (n_rows + c - 1) / c;
    if (s_begin < 0 || s_end < s_begin || s_end > n_slices || i_begin < 0 || i_end < i_begin || i_end > n_wide ||
        pc_begin < 0 || pc_end < pc_begin || pc_end > n_pieces || h_begin < 0 || h_end < h_begin || h_end > n_hub)
      fail(SPMVB_INVALID_ARG, "slice / wide-slice / piece / hub range out of bounds");
    sell_launch(n_rows, c, widths, slice_off, perm, idx, val, wide, n_wide, first_piece, n_pieces, hub, n_hub,
                wide_cols, tail_from, max_narrow_width, x, y, scale, s_begin, s_end, i_begin, i_end, pc_begin, pc_end,
                h_begin, h_end, as_stream(stream));
  });
}

