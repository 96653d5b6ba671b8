/*
 * Host R-MAT row sampler for the CPU baseline (TEST/BENCH INFRASTRUCTURE,
 * see oracle/port.py).  Regenerates the GPU generator's draws
 * (paper_1805_11938_b200/csrc/gen.cu) with the same counter hash and keeps
 * only draws whose row r satisfies mix64(r ^ 0xA5A5A5A5) % keep_mod == 0,
 * i.e. an unbiased 1/keep_mod sample of the rows of the full R-MAT matrix.
 * rmat_sample_ranges() additionally keeps every row inside any of a list of
 * half-open row ranges (the contiguous row windows behind a CSR5 tile
 * window, tests/test_gpu_c5_oracle.py).
 * Output: draws in ascending draw order (deduplication is done by the
 * caller, keeping the first draw as the GPU generator does).
 *
 * Built by oracle/Makefile into oracle/_build/librmat_sample.so (pthreads).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

static inline uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static inline double u01(uint64_t sm, uint64_t e, unsigned l) {
  return (double)(mix64(sm ^ (e * 64ull + l)) >> 11) * 0x1.0p-53;
}

int rmat_row_keep(int32_t row, uint32_t keep_mod) { return (mix64((uint64_t)row ^ 0xA5A5A5A5ull) % keep_mod) == 0; }

typedef struct {
  int scale;
  int64_t lo, hi, n, cap, off, max_out;
  uint64_t sm;
  double a, ab, abc;
  uint32_t keep_mod;
  const int32_t* ranges; /* n_ranges pairs [lo, hi) */
  int n_ranges;
  int64_t* buf;
  int64_t* e_out;
  int32_t *row_out, *col_out;
  double* val_out;
} Job;

static void* scan_rows(void* p) {
  Job* j = (Job*)p;
  j->cap = 1 << 16;
  j->n = 0;
  j->buf = (int64_t*)malloc((size_t)j->cap * sizeof(int64_t));
  for (int64_t e = j->lo; e < j->hi; ++e) {
    uint32_t row = 0;
    for (int l = 0; l < j->scale; ++l) row = (row << 1) | (u01(j->sm, (uint64_t)e, l) >= j->ab ? 1u : 0u);
    int keep = j->keep_mod > 0 && rmat_row_keep((int32_t)row, j->keep_mod);
    for (int q = 0; q < j->n_ranges && !keep; ++q)
      keep = (int32_t)row >= j->ranges[2 * q] && (int32_t)row < j->ranges[2 * q + 1];
    if (!keep) continue;
    if (j->n == j->cap) {
      j->cap *= 2;
      j->buf = (int64_t*)realloc(j->buf, (size_t)j->cap * sizeof(int64_t));
    }
    j->buf[j->n++] = e;
  }
  return NULL;
}

static void* emit(void* p) {
  Job* j = (Job*)p;
  for (int64_t i = 0; i < j->n; ++i) {
    const int64_t o = j->off + i;
    if (o >= j->max_out) break;
    const int64_t e = j->buf[i];
    uint32_t row = 0, col = 0;
    for (int l = 0; l < j->scale; ++l) {
      const double u = u01(j->sm, (uint64_t)e, l);
      const uint32_t rb = u >= j->ab, cb = (u >= j->a && u < j->ab) || u >= j->abc;
      row = (row << 1) | rb;
      col = (col << 1) | cb;
    }
    j->e_out[o] = e;
    j->row_out[o] = (int32_t)row;
    j->col_out[o] = (int32_t)col;
    j->val_out[o] = 1.0 - u01(j->sm, (uint64_t)e, 63);
  }
  return NULL;
}

/* Returns the number of sampled draws; writes at most max_out of them.
 * keep_mod == 0 keeps no hashed rows (ranges only). */
int64_t rmat_sample_ranges(int scale, int64_t draws, double a, double b, double c, uint64_t seed,
                           uint32_t keep_mod, const int32_t* ranges, int n_ranges, int64_t max_out,
                           int64_t* e_out, int32_t* row_out, int32_t* col_out, double* val_out, int nthreads) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  Job jobs[256];
  pthread_t th[256];
  for (int t = 0; t < nthreads; ++t) {
    Job* j = &jobs[t];
    memset(j, 0, sizeof(*j));
    j->scale = scale;
    j->lo = draws * t / nthreads;
    j->hi = draws * (t + 1) / nthreads;
    j->sm = mix64(seed);
    j->a = a;
    j->ab = a + b;
    j->abc = a + b + c;
    j->keep_mod = keep_mod;
    j->ranges = ranges;
    j->n_ranges = n_ranges;
    j->max_out = max_out;
    j->e_out = e_out;
    j->row_out = row_out;
    j->col_out = col_out;
    j->val_out = val_out;
    pthread_create(&th[t], NULL, scan_rows, j);
  }
  for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
  int64_t total = 0;
  for (int t = 0; t < nthreads; ++t) {
    jobs[t].off = total;
    total += jobs[t].n;
  }
  if (e_out) {
    for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, emit, &jobs[t]);
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
  }
  for (int t = 0; t < nthreads; ++t) free(jobs[t].buf);
  return total;
}

int64_t rmat_sample(int scale, int64_t draws, double a, double b, double c, uint64_t seed, uint32_t keep_mod,
                    int64_t max_out, int64_t* e_out, int32_t* row_out, int32_t* col_out, double* val_out,
                    int nthreads) {
  return rmat_sample_ranges(scale, draws, a, b, c, seed, keep_mod, NULL, 0, max_out, e_out, row_out, col_out,
                            val_out, nthreads);
}
