/*
 * spmvb.h — C ABI of the B200-native fp64 SpMV library (libspmvb.so).
 *
 * This is the drop-in boundary for the hot path of the reference package
 * `spmvkit` (arXiv 1805.11938 artifact, /root/reference/pkg/src/spmvkit).
 * The reference is pure Python, so its "FFI" is its Python function surface;
 * each entry point below names the reference function it replaces
 * (file:line relative to /root/reference/pkg/src/spmvkit/).  The Python
 * binding that a maintainer would add is shown in INTEGRATION.md and is
 * implemented by paper_1805_11938_b200/_lib.py (ctypes).
 *
 * Conventions
 *  - Every function is extern "C", reentrant, and stream-ordered on the
 *    `stream` argument (a cudaStream_t passed as void*; NULL = legacy
 *    default stream).  Device pointers are caller-allocated unless noted.
 *  - Indices are int32 (the reference stores int64 with a 32-bit range
 *    contract, coo.py:37-38; the byte model assumes 4-byte indices,
 *    bench.py:13-14).  Row pointers are int32, so nnz < 2^31.
 *  - Values are IEEE fp64.
 *  - Return value: SPMVB_OK or an error status; the message for the last
 *    failure on the calling thread is returned by spmvb_last_error().
 *  - Functions whose output size depends on the data are split into a
 *    *_begin / *_plan step that returns the size (synchronizing the stream)
 *    and a *_finish / fill step that writes caller-allocated outputs.
 *  - Temporaries are allocated stream-ordered (cudaMallocAsync).
 *  - No CPU fallback exists: every compute entry point launches CUDA kernels.
 */
#ifndef SPMVB_H_
#define SPMVB_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (mapped to Python exceptions by _lib.py) ------------- */
#define SPMVB_OK 0
#define SPMVB_INVALID_ARG 1     /* ValueError                                  */
#define SPMVB_GRID_TOO_LARGE 2  /* ConversionError (formats.py:61-62)          */
#define SPMVB_OUT_OF_RANGE 3    /* ValueError "... is outside ..." (coo.py:108-115) */
#define SPMVB_CUDA_ERROR 4      /* RuntimeError                                */
#define SPMVB_OUT_OF_MEMORY 5   /* MemoryError                                 */
#define SPMVB_INTERNAL 6        /* RuntimeError                                */

#define SPMVB_ABI_VERSION 1

const char* spmvb_last_error(void);
int spmvb_abi_version(void);
/* Number of CUDA kernels this library has launched in the process. */
unsigned long long spmvb_launch_count(void);

/* ======================================================================== */
/* COO core — replaces coo.py                                               */
/* ======================================================================== */

typedef struct spmvb_canon spmvb_canon;

/* canonicalize (coo.py:86-125), phase 1.  Sorts (row, col) stably, sums
 * duplicates in numpy reduceat order (first + pairwise(rest)) and drops sums
 * equal to 0.0.  row/col are int32 (index_width 4) or int64 (index_width 8)
 * device arrays.  On an out-of-bounds entry returns SPMVB_OUT_OF_RANGE and
 * writes bad[0..2] = {first bad entry index, its row, its col} (host array).
 * On success *nnz_out (host) holds the canonical nnz and *plan must be passed
 * to spmvb_canonicalize_finish (or spmvb_canonicalize_free).  The input
 * arrays must stay alive until finish. */
int spmvb_canonicalize_begin(const void* row, const void* col, int index_width, const double* val,
                             int64_t nnz_in, int64_t n_rows, int64_t n_cols, spmvb_canon** plan,
                             int64_t* nnz_out, int64_t* bad, void* stream);
int spmvb_canonicalize_finish(spmvb_canon* plan, int32_t* row_out, int32_t* col_out, double* val_out,
                              void* stream);
void spmvb_canonicalize_free(spmvb_canon* plan);

/* read_matrix_market entry tokenizer (coo.py:222-262), host code,
 * multithreaded: `text` is everything after the size line.  Writes the
 * expanded 0-based triplets (symmetric off-diagonal entries mirrored,
 * pattern entries 1.0) into host arrays of capacity `cap` and *n_out.
 * Returns 0 on success; any nonzero value means "not handled here" (an entry
 * error or text outside the fast path's ASCII/"\n" grammar) and the caller
 * re-parses with the reference-semantics parser for the exact error. */
int spmvb_mm_parse(const char* text, int64_t len, int pattern, int symmetric, int64_t n_rows, int64_t n_cols,
                   int64_t declared, int64_t cap, int64_t* row_out, int64_t* col_out, double* val_out, int64_t* n_out,
                   int64_t* err_line, int64_t* err_ij, int n_threads);

/* write_matrix_market entry formatter (coo.py:266-278), host code,
 * multithreaded: one "<row+1> <col+1> <value:.17g>\n" line per entry, the
 * text Python's f"{v:.17g}" produces.  _begin formats into a plan and returns
 * the text length; _finish copies it into `out` (len bytes; NULL = discard)
 * and frees the plan.  The banner and the size line are the caller's. */
typedef struct spmvb_mm_text spmvb_mm_text;
int spmvb_mm_format_begin(const int64_t* row, const int64_t* col, const double* val, int64_t nnz, int n_threads,
                          spmvb_mm_text** plan_out, int64_t* len_out);
int spmvb_mm_format_finish(spmvb_mm_text* plan, char* out);

/* row_nnz_histogram (coo.py:144-146) on canonical (row-sorted) COO. */
int spmvb_row_nnz_histogram(const int32_t* row, int64_t nnz, int64_t n_rows, int64_t* counts_out,
                            void* stream);

/* dense_spmv_oracle (coo.py:128-141): y_i accumulated entry by entry in
 * ascending (row, col) order with separately rounded products (no FMA);
 * bit-identical to the reference oracle. ptr is the CSR row pointer. */
int spmvb_spmv_sequential(int64_t n_rows, const int32_t* ptr, const int32_t* col, const double* val,
                          const double* x, double* y, void* stream);

/* ======================================================================== */
/* Formats — replaces formats.py                                            */
/* ======================================================================== */

/* to_csr (formats.py:183-188): ptr[n_rows+1] from row-sorted COO rows;
 * col/val copied (the reference returns new arrays). */
int spmvb_coo_to_csr(const int32_t* row, const int32_t* col, const double* val, int64_t nnz,
                     int64_t n_rows, int32_t* ptr_out, int32_t* col_out, double* val_out, void* stream);

/* Row-length statistics from a CSR ptr (host output):
 * out[0] = min count, out[1] = max count, out[2] = number of non-empty rows. */
int spmvb_csr_row_stats(const int32_t* ptr, int64_t n_rows, int64_t* out3, void* stream);

/* to_csr5 (formats.py:196-250).  num_tiles = ceil(nnz/(omega*sigma)).
 * Outputs (device): tile_ptr[num_tiles+1], bit_flag[nnz] (uint8, stored
 * order), y_off[num_tiles*omega], seg_off[num_tiles*omega] (int32, row-major
 * (tile, column)), col_out[nnz], val_out[nnz] (stored order).
 * Also writes the kernel's auxiliary per-tile word tile_aux[num_tiles]
 * (bit 31: the tile head continues a row begun in an earlier tile; bits 0-30:
 * rank of tile_ptr[t] among non-empty rows).  SPMVB_INVALID_ARG if omega < 1
 * or sigma < 1 (message names omega/sigma as the reference does). */
int spmvb_csr_to_csr5(int64_t n_rows, int64_t nnz, const int32_t* ptr, const int32_t* col, const double* val,
                      int omega, int sigma, int32_t* tile_ptr, uint8_t* bit_flag, int32_t* y_off,
                      int32_t* seg_off, int32_t* col_out, double* val_out, uint32_t* tile_aux, void* stream);

/* List of non-empty rows (ascending) used by the CSR5 kernel when empty rows
 * exist; rows_out has `nonempty` entries (from spmvb_csr_row_stats). */
int spmvb_csr_nonempty_rows(const int32_t* ptr, int64_t n_rows, int32_t* rows_out, void* stream);

/* to_ell (formats.py:281-288 via _padded_grids :253-278).  Grid stored
 * column-major: element (r, j) at j*n_rows + r.  Pads repeat the row's last
 * valid column (0 for an empty row) with value 0.0.  SPMVB_GRID_TOO_LARGE
 * (checked before any write) if n_rows*k > max_cells. Writes row_nnz. */
int spmvb_csr_to_ell(int64_t n_rows, const int32_t* ptr, const int32_t* col, const double* val, int64_t k,
                     int64_t max_cells, int32_t* idx_out, double* val_out, int64_t* row_nnz_out, void* stream);

/* to_sell (formats.py:291-344), phase 1: permutation, slice widths, slice
 * offsets (in cells) and permuted row counts; *total_cells (host) returned.
 * SPMVB_INVALID_ARG for c < 1 or sigma not in {0} U cN ("multiple");
 * SPMVB_GRID_TOO_LARGE if total cells > max_cells.  Arrays: perm[n_rows],
 * widths[S], slice_off[S+1] (int64), row_nnz_perm[n_rows]; S = ceil(n/c). */
int spmvb_sell_plan(int64_t n_rows, const int32_t* ptr, int64_t c, int64_t sigma, int64_t max_cells,
                    int32_t* perm, int64_t* widths, int64_t* slice_off, int64_t* row_nnz_perm,
                    int64_t* total_cells, void* stream);
/* Phase 2: fill the per-slice column-major grids into flat arrays. */
int spmvb_sell_fill(int64_t n_rows, const int32_t* ptr, const int32_t* col, const double* val, int64_t c,
                    const int32_t* perm, const int64_t* widths, const int64_t* slice_off, int32_t* idx_out,
                    double* val_out, void* stream);

/* hyb_typical_k (formats.py:347-358) on a CSR ptr; *k_out (host). */
int spmvb_hyb_typical_k(const int32_t* ptr, int64_t n_rows, int64_t* k_out, void* stream);
/* hyb_typical_k on an int64 per-row count array (device). */
int spmvb_typical_k_counts(const int64_t* counts, int64_t n, int64_t* k_out, void* stream);
/* to_hyb (formats.py:361-397), phase 1: tail_ptr[n_rows+1] (exclusive scan of
 * max(count-K,0)); *tail_nnz (host). */
int spmvb_hyb_plan(int64_t n_rows, const int32_t* ptr, int64_t k, int64_t max_cells, int32_t* tail_ptr,
                   int64_t* tail_nnz, void* stream);
/* Phase 2: ELL part (column-major, pads = last kept col) with row_nnz =
 * min(count, K), and the canonical-order COO tail. */
int spmvb_hyb_fill(int64_t n_rows, const int32_t* ptr, const int32_t* col, const double* val, int64_t k,
                   const int32_t* tail_ptr, int32_t* ell_idx, double* ell_val, int64_t* ell_row_nnz,
                   int32_t* tail_row, int32_t* tail_col, double* tail_val, void* stream);

/* ---- to_coo (formats.py:400-453): triplet extraction; the Python layer
 *      passes the triplets through spmvb_canonicalize_* as the reference
 *      passes them through canonicalize. ------------------------------------ */
/* rows_out[k] = row of CSR position k. */
int spmvb_csr_expand_rows(const int32_t* ptr, int64_t n_rows, int32_t* rows_out, void* stream);
/* Undo the CSR5 stored order: col/val in stored order -> CSR order. */
int spmvb_csr5_unstore(int64_t nnz, int omega, int sigma, const int32_t* col, const double* val, int32_t* col_out,
                       double* val_out, void* stream);
/* ELL grid (column-major) -> triplets in row-major order, first row_nnz[r]
 * slots per row; outputs sized sum(row_nnz). */
int spmvb_ell_to_coo(int64_t n_rows, int64_t k, const int32_t* idx, const double* val, const int64_t* row_nnz,
                     int32_t* rows_out, int32_t* cols_out, double* vals_out, void* stream);
/* SELL slices -> triplets in canonical (row, col) order. */
int spmvb_sell_to_coo(int64_t n_rows, int64_t c, const int32_t* perm, const int64_t* slice_off,
                      const int64_t* row_nnz_perm, const int32_t* idx, const double* val, int32_t* rows_out,
                      int32_t* cols_out, double* vals_out, void* stream);

/* HYB (ELL part + COO tail with its per-row offsets tail_ptr[n_rows+1]) ->
 * triplets in canonical (row, col) order (formats.py:446-453 to_coo(hyb)). */
int spmvb_hyb_to_coo(int64_t n_rows, int64_t k, const int32_t* ell_idx, const double* ell_val,
                     const int64_t* ell_row_nnz, int64_t tail_nnz, const int32_t* tail_row, const int32_t* tail_col,
                     const double* tail_val, const int32_t* tail_ptr, int32_t* rows_out, int32_t* cols_out,
                     double* vals_out, void* stream);

/* ======================================================================== */
/* SpMV kernels — replaces kernels.py (y = scale * A x).                    */
/* `scale` is an optional device scalar (NULL = 1.0) multiplying each row   */
/* result; power iteration uses it for deferred normalisation.              */
/* Results are deterministic (no floating-point atomics).                   */
/* ======================================================================== */

/* CSR and HYB kernels work on chunks of spmvb_csr_chunk_size() consecutive
 * nonzeros (one warp each).  Analysis step (like a cuSPARSE buffer): the
 * ascending list of non-empty rows nz_rows[n_nz] (spmvb_csr_nonempty_rows;
 * pass NULL and n_nz = n_rows when every row is non-empty) and
 * chunk_row[c] = first index into that list whose row starts at or after
 * chunk c (spmvb_csr_chunks(nnz) + 1 entries, the last = n_nz).
 * carry_row/carry_val: spmvb_csr_chunks(nnz) scratch entries. */
int64_t spmvb_csr_chunk_size(void);
int64_t spmvb_csr_chunks(int64_t nnz);
int spmvb_csr_chunk_plan(int64_t n_rows, int64_t nnz, const int32_t* ptr, const int32_t* nz_rows, int64_t n_nz,
                         int32_t* chunk_row, void* stream);
/* spmv_csr (kernels.py:76-95). */
int spmvb_spmv_csr(int64_t n_rows, int64_t nnz, const int32_t* ptr, const int32_t* col, const double* val,
                   const int32_t* nz_rows, int64_t n_nz, const int32_t* chunk_row, int32_t* carry_row,
                   double* carry_val, const double* x, double* y, const double* scale, void* stream);
/* spmv_hyb (kernels.py:177-199): ELL part plus the COO tail, the tail reduced
 * through its row pointer (tail_ptr from spmvb_hyb_plan; nz_rows/chunk_row
 * from the analysis above over (tail_ptr, tail_nnz)). */
int spmvb_spmv_hyb(int64_t n_rows, int64_t k, const int32_t* ell_idx, const double* ell_val, int64_t tail_nnz,
                   const int32_t* tail_ptr, const int32_t* tail_col, const double* tail_val, const int32_t* nz_rows,
                   int64_t n_nz, const int32_t* chunk_row, int32_t* carry_row, double* carry_val, const double* x,
                   double* y, const double* scale, void* stream);

/* Reference-order ("bit-parity") SpMV (csrc/spmv_exact.cu): the reference's
 * own summation orders, so y equals spmvkit's result (workers = 1) bit for
 * bit, where the fast kernels above meet the 1e-12 (|A||x|) tolerance in a
 * different fixed order.  CSR: y_r = p_first + numpy-pairwise(rest)
 * (np.add.reduceat, kernels.py:84).  CSR5: the same per row piece inside each
 * tile, pieces added in ascending tile order from 0.0 (kernels.py:161-173);
 * indices/data in CSR5 stored order.  HYB: the sequential ELL recurrence, then
 * + the row's tail entries summed sequentially from 0.0 (np.bincount,
 * kernels.py:186-198).  ELL and SELL (every slice on the thread-per-row path)
 * already are the reference recurrence.  A verification mode: a thread per
 * row, a CTA per row longer than 256 entries. */
int spmvb_spmv_csr_exact(int64_t n_rows, int64_t nnz, const int32_t* ptr, const int32_t* col, const double* val,
                         const double* x, double* y, const double* scale, void* stream);
int spmvb_spmv_csr5_exact(int64_t n_rows, int64_t nnz, const int32_t* ptr, int omega, int sigma,
                          const int32_t* indices, const double* data, const double* x, double* y,
                          const double* scale, void* stream);
int spmvb_spmv_hyb_exact(int64_t n_rows, int64_t k, const int32_t* ell_idx, const double* ell_val, int64_t tail_nnz,
                         const int32_t* tail_ptr, const int32_t* tail_col, const double* tail_val, const double* x,
                         double* y, const double* scale, void* stream);

/* spmv_csr5 (kernels.py:139-174). nonempty_rows may be NULL when every row is
 * non-empty, or when the non-empty rows are exactly the prefix
 * [0, n_nonempty) (n_nonempty < n_rows: the empty tail is zeroed by plain
 * stores, no ptr tests; spmvb_degree_order's layout). carry: num_tiles scratch doubles.  flag_bits (may be NULL) is
 * bit_flag packed one bit per entry (spmvb_csr5_pack_flags): the tile kernel
 * then reads 64 bytes of flags per 512-entry tile instead of 512. */
/* CSR5 SpMV fused with the multi-GPU exchange: as
 * spmvb_spmv_csr5, and every row r of y is also stored at
 * peers[p][push_off + r] for p < n_peers (device array of peer buffer
 * addresses, e.g. symmetric memory mapped over NVLink): each block stores its
 * own rows (16-byte stores) right after computing them, the carry fix-up
 * re-stores the rows it completes.  omega = 32, sigma = 16 or 8.  The caller
 * orders the peers' reads of those buffers (one barrier per step). */
int spmvb_spmv_csr5_push(int64_t n_rows, int64_t nnz, const int32_t* ptr, int omega, int sigma,
                         const int32_t* tile_ptr, const uint8_t* bit_flag, const uint32_t* flag_bits,
                         const int32_t* col, const double* val, const uint32_t* tile_aux, const int32_t* nonempty_rows,
                         int64_t n_nonempty, double* carry, const double* x, double* y, const double* scale,
                         const uint64_t* peers, int n_peers, int64_t push_off, void* stream);
int spmvb_csr5_pack_flags(int64_t nnz, const uint8_t* bit_flag, uint32_t* flag_bits, void* stream);
int spmvb_spmv_csr5(int64_t n_rows, int64_t nnz, const int32_t* ptr, int omega, int sigma, const int32_t* tile_ptr,
                    const uint8_t* bit_flag, const uint32_t* flag_bits, const int32_t* col, const double* val,
                    const uint32_t* tile_aux,
                    const int32_t* nonempty_rows, int64_t n_nonempty, double* carry, const double* x, double* y,
                    const double* scale, void* stream);

/* One range of spmvb_spmv_csr5: zero the empty rows of [row_begin, row_end)
 * and run tiles [t_begin, t_end) with their carry fix-up.  With the ranges
 * of spmvb_csr5_range_bounds (each starting at a row-start tile) the ranges
 * may run in any order and rows [row_bounds[k], row_bounds[k+1]) are final
 * after range k -- the multi-GPU power iteration sends them to the peers
 * while the next range computes.  Bit-identical to spmvb_spmv_csr5. */
int spmvb_spmv_csr5_tiles(int64_t n_rows, int64_t nnz, const int32_t* ptr, int omega, int sigma,
                          const int32_t* tile_ptr, const uint8_t* bit_flag, const uint32_t* flag_bits,
                          const int32_t* col, const double* val,
                          const uint32_t* tile_aux, const int32_t* nonempty_rows, int64_t n_nonempty, double* carry,
                          const double* x, double* y, const double* scale, int64_t t_begin, int64_t t_end,
                          int64_t row_begin, int64_t row_end, void* stream);

/* Range plan for spmvb_spmv_csr5_host: n_ranges tile ranges whose first tile
 * starts a row (no carry chain crosses a range), as HOST int64 arrays of
 * n_ranges+1 entries: tile_bounds (0 .. num_tiles) and row_bounds (the first
 * row each range touches; row_bounds[n_ranges] = n_rows).  Synchronizes. */
int spmvb_csr5_range_bounds(int64_t nnz, int omega, int sigma, const int32_t* tile_ptr, const uint32_t* tile_aux,
                            int n_ranges, int64_t* tile_bounds, int64_t* row_bounds, void* stream);

/* spmv(tag="csr5", m, x_host) with HOST buffers -- the reference call shape
 * (kernels.py:139-174, x and y are host numpy arrays there): copies x_host
 * (n_cols doubles) into x_dev, runs the ranges of the plan above (last to
 * first) and streams each range's finished rows of y_dev back into y_host on
 * a second stream while the other ranges compute.  Returns after y_host is complete.
 * Bit-identical to spmvb_spmv_csr5 on the same inputs.  Pinned host buffers
 * make the copies asynchronous; pageable ones are still correct. */
int spmvb_spmv_csr5_host(int64_t n_rows, int64_t n_cols, int64_t nnz, const int32_t* ptr, int omega, int sigma,
                         const int32_t* tile_ptr, const uint8_t* bit_flag, const uint32_t* flag_bits,
                         const int32_t* col, const double* val,
                         const uint32_t* tile_aux, const int32_t* nonempty_rows, int64_t n_nonempty, double* carry,
                         const double* x_host, double* x_dev, double* y_dev, double* y_host, const double* scale,
                         int n_ranges, const int64_t* tile_bounds, const int64_t* row_bounds, void* stream);

/* spmv_ell (kernels.py:98-116): per-row sequential accumulation over all k
 * slots (pads included), separately rounded products: bit-identical to the
 * reference kernel.  n_cols: the length of x (its lines are prefetched into
 * L2 with the first slot loads; 0 = no prefetch). */
int spmvb_spmv_ell(int64_t n_rows, int64_t n_cols, int64_t k, const int32_t* idx, const double* val, const double* x,
                   double* y, const double* scale, void* stream);

/* spmv_sell (kernels.py:119-136); perm may be NULL for sigma == 0.  Slices
 * up to wide_cols (>= SPMVB_SELL_WIDE_COLS; 0 = that default) wide, or taller
 * than 128 rows, are summed one thread per row, sequentially and without
 * FMA: bit-identical to the reference.  Wider slices (power-law rows) are
 * listed by spmvb_sell_wide_plan (same wide_cols) and summed by a CTA each
 * (within tolerance).  A larger wide_cols pays on big matrices, where the
 * long per-thread rows hide behind the rest of the grid (the library picks
 * it from nnz: formats.SellMatrix.wide_plan). */
#ifndef SPMVB_SELL_WIDE_COLS
#define SPMVB_SELL_WIDE_COLS 256
#endif
/* Also reports (host, may be NULL) the widest slice left to the per-row
 * kernel, which spmvb_spmv_sell uses to pick its slot loop (-1 = unknown),
 * and (first_piece_out: device, n_slices entries; n_pieces: host) how the
 * wide slices split into pieces of ~32K cells, one CTA each. */
int spmvb_sell_wide_plan(int64_t n_rows, int64_t c, const int64_t* widths, int64_t wide_cols, int32_t* wide_out,
                         int64_t* n_wide, int64_t* max_narrow_width, int32_t* first_piece_out, int64_t* n_pieces,
                         void* stream);
/* tail_from (n_rows = none): the caller's promise that every permuted row
 * p >= tail_from is empty with perm[p] == p (a degree-ordered matrix's empty
 * tail); those rows get y = 0 without any slice or perm lookups. */
/* hub (device, may be NULL when n_hub == 0): the ascending indices into the
 * wide list of the wide slices with more than SPMVB_SELL_HUB_PIECES pieces;
 * their rows are summed a warp per row, the other wide rows a thread per
 * row. */
#define SPMVB_SELL_HUB_PIECES 32
int spmvb_spmv_sell(int64_t n_rows, int64_t c, const int64_t* widths, const int64_t* slice_off,
                    const int32_t* perm, const int32_t* idx, const double* val, const int32_t* wide, int64_t n_wide,
                    const int32_t* first_piece, int64_t n_pieces, const int32_t* hub, int64_t n_hub,
                    int64_t wide_cols, int64_t tail_from, int64_t max_narrow_width, const double* x, double* y,
                    const double* scale, void* stream);
/* Slices [s_begin, s_end) of spmvb_spmv_sell (e.g. to send finished rows to
 * other GPUs while later slices compute): [i_begin, i_end) = the entries of
 * the wide list whose slices lie in the range, [pc_begin, pc_end) = their
 * pieces (first_piece[i_begin] .. first_piece[i_end], or n_pieces),
 * [h_begin, h_end) = the hub entries among them.  Over a
 * partition of the slices, the same y as one spmvb_spmv_sell, bit for bit;
 * with sigma > 0 a range's rows are perm[s_begin*c .. s_end*c), contiguous
 * when the range is aligned to sorting windows. */
int spmvb_spmv_sell_range(int64_t n_rows, int64_t c, const int64_t* widths, const int64_t* slice_off,
                          const int32_t* perm, const int32_t* idx, const double* val, const int32_t* wide,
                          int64_t n_wide, const int32_t* first_piece, int64_t n_pieces, const int32_t* hub,
                          int64_t n_hub, int64_t wide_cols, int64_t tail_from, int64_t max_narrow_width,
                          const double* x, double* y, const double* scale, int64_t s_begin, int64_t s_end,
                          int64_t i_begin, int64_t i_end, int64_t pc_begin, int64_t pc_end, int64_t h_begin,
                          int64_t h_end, void* stream);

/* ||y||^2 over n entries into *out (device), deterministic two-level sum.
 * Used by power iteration. */
int spmvb_sumsq(const double* y, int64_t n, double* out, void* stream);
/* scale_out = 1/sqrt(*sumsq) (device scalars). */
int spmvb_inv_sqrt(const double* sumsq, double* scale_out, void* stream);
/* Both in one launch: *sumsq = ||y||^2, *scale_out = 1/||y|| (1 if y == 0),
 * deterministic (block partials folded in block order).  ws: a device
 * buffer of spmvb_norm_ws_bytes() bytes, zeroed once when allocated, used by
 * one stream at a time (the kernel leaves it ready for the next call).  The
 * normalisation of a single-process power-iteration step. */
int64_t spmvb_norm_ws_bytes(void);
int spmvb_norm_scale(const double* y, int64_t n, void* ws, double* sumsq, double* scale_out, void* stream);

/* Sparse x exchange of the row-block power iteration (a shard
 * reads only ~20% of the columns at C4/C5, so receiving just those entries
 * cuts the per-step exchange ~4-5x against the full all-gatherv).
 * spmvb_column_set: sorted distinct column ids of col[0..nnz) into cols_out
 * (NULL = count only); *n_out (host) = how many.  Synchronizes.
 * spmvb_gather_f64: dst[i] = src[idx[i] - base] (owner packs requested rows).
 * spmvb_scatter_f64: dst[idx[i]] = src[i] (receiver unpacks into x). */
int spmvb_column_set(const int32_t* col, int64_t nnz, int64_t n_cols, int32_t* cols_out, int64_t* n_out,
                     void* stream);
int spmvb_gather_f64(const double* src, int64_t base, const int32_t* idx, int64_t n, double* dst, void* stream);
int spmvb_scatter_f64(const double* src, const int32_t* idx, int64_t n, double* dst, void* stream);

/* Row-block power iteration over a caller-owned NCCL communicator (SURVEY
 * §8(b) dist_{init,spmv_iter,destroy}; the torch.distributed version is
 * dist.PowerIteration).  spmvb_dist_init: nccl_comm is an ncclComm_t of
 * `world` ranks (this one is `rank`); bounds: world + 1 host row boundaries
 * (e.g. nnz-balanced).  spmvb_dist_step, on `stream`: local_spmv(ctx, x,
 * x_next + bounds[rank], scale, stream) must write this rank's rows
 * scale * A_p x (any spmvb_spmv_* call; return its status); then
 * *sumsq = ||y||^2 over all ranks (NCCL all-reduce), x_next gathered from
 * every rank (grouped NCCL send/recv with per-rank counts) and *scale =
 * 1/||y|| (device scalars), so x_{k+1} = x_next * scale.  NCCL is resolved
 * at run time from the libnccl.so.2 loaded in the process. */
typedef struct spmvb_dist spmvb_dist;
typedef int (*spmvb_local_spmv_fn)(void* ctx, const double* x, double* y_local, const double* scale, void* stream);
int spmvb_dist_init(void* nccl_comm, int rank, int world, const int64_t* bounds, spmvb_dist** out);
int spmvb_dist_step(spmvb_dist* d, spmvb_local_spmv_fn local_spmv, void* ctx, const double* x, double* x_next,
                    double* sumsq, double* scale, void* stream);
int spmvb_dist_destroy(spmvb_dist* d);
/* The version (NCCL_VERSION_CODE) of the libnccl.so.2 the dist entry points
 * resolved: it must be the one that created the caller's communicator. */
int spmvb_dist_nccl_version(int* version);
/* The same step with the exchange overlapped: range_spmv(ctx, k, x,
 * y_local, scale, stream) is called for k = 0 .. n_ranges-1 in order and
 * computes this rank's range k into y_local (the shard's rows; a no-op for
 * a k past its own ranges); after each call the rows spans[rank][k] = local
 * [a, b) are sent to every peer (and each peer's spans[p][k] received) on an
 * internal exchange stream while the next range computes.  spans: world *
 * n_ranges * 2, the same array on every rank; a == b sends nothing (rows
 * known to be zero, e.g. an empty tail, need not travel).
 * Range bounds must not split a row's computation (e.g. CSR5 range_plan,
 * SELL range_plan); then x_next is the same, bit for bit, as spmvb_dist_step. */
typedef int (*spmvb_range_spmv_fn)(void* ctx, int k, const double* x, double* y_local, const double* scale,
                                   void* stream);
int spmvb_dist_init_ranges(void* nccl_comm, int rank, int world, const int64_t* bounds, int n_ranges,
                           const int64_t* spans, spmvb_dist** out);
int spmvb_dist_step_ranges(spmvb_dist* d, spmvb_range_spmv_fn range_spmv, void* ctx, const double* x,
                           double* x_next, double* sumsq, double* scale, void* stream);

/* Degree-ordered symmetric relabelling (relabel.cu): an internal shadow
 * layout P A P^T of a square n x n CSR for iterative SpMV (power iteration
 * on R-MAT: CSR5 SpMV ~13 % faster at scale 25); the reference's arrays are
 * left untouched and the iterate is mapped with spmvb_gather_f64.
 * spmvb_degree_order: new ids sorted by (row empty, -(row degree + column
 * degree)) (mode 0) or by (row empty, -row degree, -column degree) (mode 1:
 * rows in exact descending length), stable by old id, so every empty row is
 * last.  perm[new] = old,
 * new_id[old] = new (n entries each); *n_nonempty (host) = non-empty rows.
 * Synchronizes.
 * spmvb_relabel_csr: the entries of P A P^T as triplets in the old CSR
 * order (row_out[k] = new_id[row(k)], col_out[k] = new_id[col[k]],
 * val_out[k] = val[k]); canonicalize them to get its CSR. */
int spmvb_degree_order(int64_t n, const int32_t* ptr, const int32_t* col, int64_t nnz, int mode, int32_t* perm,
                       int32_t* new_id, int64_t* n_nonempty, void* stream);
int spmvb_relabel_csr(int64_t n, const int32_t* ptr, const int32_t* col, const double* val, int64_t nnz,
                      const int32_t* new_id, int32_t* row_out, int32_t* col_out, double* val_out, void* stream);

/* Peer-memory exchange of the row-block power iteration (dist.py
 * exchange="p2p"): spmvb_push_rows writes src[0..n) into every peer buffer
 * dst_ptrs[p] + offset (a device array of n_peers addresses mapped over
 * NVLink, e.g. symmetric-memory peers; 16-byte stores) -- the all-gather of
 * x done by our own kernel, one launch per finished row range, overlapping
 * the next range's SpMV.  spmvb_sum_inv_sqrt folds the ranks' pushed
 * ||y_p||^2 values in rank order and writes sumsq and 1/sqrt(sumsq). */
int spmvb_push_rows(const double* src, int64_t n, const uint64_t* dst_ptrs, int n_peers, int64_t offset,
                    void* stream);
int spmvb_sum_inv_sqrt(const double* vals, int n, double* sumsq, double* scale, void* stream);

/* Roofline probe (bench.py): partial[t] = sum of src[idx[i]] over thread t's
 * share of [0, n), 16 gathers in flight per thread, no per-element stores --
 * the L1TEX rate of a matrix's x gathers, which its SpMV cannot beat.
 * partial holds spmvb_gather_probe_threads() doubles. */
int64_t spmvb_gather_probe_threads(void);
int spmvb_gather_probe(const double* src, const int32_t* idx, int64_t n, double* partial, void* stream);
/* The same with the values: partial[t] = sum of val[i] * src[idx[i]] -- the
 * flat dot product over a matrix's entries, i.e. an SpMV's own traffic (12
 * streamed bytes + one gather per entry) without any row structure.  The
 * stream + gather ceiling of that matrix on this GPU (bench.py reports the
 * SpMV against it). */
int spmvb_dot_probe(const double* src, const int32_t* idx, const double* val, int64_t n, double* partial,
                    void* stream);

/* ======================================================================== */
/* Features — replaces features.py:69-84 (extract_features)                 */
/* ======================================================================== */

/* out8 (host): n_rows, n_cols, nnz_frac, nnz_min, nnz_max, nnz_avg, nnz_std,
 * variation — bit-identical to numpy (mean = nnz/n_rows, population std via
 * numpy's pairwise summation of squared deviations).  Zero-dimension input
 * returns SPMVB_INVALID_ARG ("undefined"). */
int spmvb_csr_features(int64_t n_rows, int64_t n_cols, int64_t nnz, const int32_t* ptr, double* out8,
                       void* stream);
/* Extra structure features kept outside FeatureVector (north star): out2
 * (host) = {bandwidth = max |i-j| over stored entries (0 if nnz == 0),
 * diagonal density = #{i : (i,i) stored} / min(n_rows, n_cols)}. */
int spmvb_csr_extra_features(int64_t n_rows, int64_t n_cols, const int32_t* ptr, const int32_t* col,
                             double* out2, void* stream);

/* ======================================================================== */
/* Synthetic inputs; not part of the reference API.          */
/* ======================================================================== */

/* R-MAT edge list: `draws` edges over a 2^scale square, quadrant
 * probabilities (a, b, c, 1-a-b-c) per bit from a counter-based hash of
 * (seed, draw, level); value 1 - U[0,1).  Duplicates removed keeping the first
 * draw; survivors emitted in draw order (unsorted).  Phase 1 returns the
 * survivor count and a plan; phase 2 writes them. */
typedef struct spmvb_rmat spmvb_rmat;
int spmvb_rmat_begin(int scale, int64_t draws, double a, double b, double c, uint64_t seed, spmvb_rmat** plan,
                     int64_t* nnz_out, void* stream);
int spmvb_rmat_finish(spmvb_rmat* plan, int32_t* row_out, int32_t* col_out, double* val_out, void* stream);
void spmvb_rmat_free(spmvb_rmat* plan);

/* Fill a device vector with U[lo, hi) from the same hash (x for benchmarks). */
int spmvb_fill_uniform(double* x, int64_t n, double lo, double hi, uint64_t seed, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* SPMVB_H_ */
