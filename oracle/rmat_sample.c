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

/* ------------------------------------------------------------------------
 * The whole R-MAT matrix as canonical CSR on the host (the CPU reference arm
 * of bench.py times the reference's CSR algorithm on it).  Same draws and
 * dedup rule as the GPU generator: the first draw of every (row, col) wins.
 * Pass 1 counts draws per row, pass 2 buckets (col, draw index) by row,
 * then every row is sorted by (col, draw) and deduplicated in place; the
 * value of a kept entry is a function of its draw index.  ~12 B per draw of
 * scratch (6.4 GB at scale 25, edge factor 16).
 * ------------------------------------------------------------------------ */
#include <stdatomic.h>

typedef struct {
  int scale;
  int64_t lo, hi;
  uint64_t sm;
  double ab, a, abc;
  _Atomic int64_t* fill; /* per-row cursor (pass 1: counts) */
  int32_t* col;
  int64_t* ev;
  int pass;
} CsrJob;

static void* csr_pass(void* p) {
  CsrJob* j = (CsrJob*)p;
  for (int64_t e = j->lo; e < j->hi; ++e) {
    uint32_t row = 0, col = 0;
    for (int l = 0; l < j->scale; ++l) {
      const double u = u01(j->sm, (uint64_t)e, l);
      row = (row << 1) | (u >= j->ab ? 1u : 0u);
      col = (col << 1) | (((u >= j->a && u < j->ab) || u >= j->abc) ? 1u : 0u);
    }
    const int64_t slot = atomic_fetch_add_explicit(&j->fill[row], 1, memory_order_relaxed);
    if (j->pass == 2) {
      j->col[slot] = (int32_t)col;
      j->ev[slot] = e;
    }
  }
  return NULL;
}

typedef struct {
  int64_t n;
  _Atomic int64_t* next;
  const int64_t* start; /* n + 1 bucket offsets */
  int32_t* col;
  int64_t* ev;
  int64_t* kept; /* per row: entries kept after dedup */
} RowJob;

static int cmp_entry(const void* x, const void* y) {
  const int64_t a = *(const int64_t*)x, b = *(const int64_t*)y;
  return (a > b) - (a < b);
}

static void* csr_rows(void* p) {
  RowJob* j = (RowJob*)p;
  int64_t cap = 0;
  int64_t* key = NULL;
  for (;;) {
    const int64_t r0 = atomic_fetch_add_explicit(j->next, 4096, memory_order_relaxed);
    if (r0 >= j->n) break;
    const int64_t r1 = r0 + 4096 < j->n ? r0 + 4096 : j->n;
    for (int64_t r = r0; r < r1; ++r) {
      const int64_t b = j->start[r], m = j->start[r + 1] - b;
      if (m > cap) {
        cap = m * 2;
        key = (int64_t*)realloc(key, (size_t)cap * sizeof(int64_t));
      }
      /* (col, draw) packed: col < 2^31, draw < 2^32 for every config here */
      for (int64_t i = 0; i < m; ++i) key[i] = ((int64_t)j->col[b + i] << 32) | j->ev[b + i];
      qsort(key, (size_t)m, sizeof(int64_t), cmp_entry);
      int64_t k = 0;
      for (int64_t i = 0; i < m; ++i) {
        if (k > 0 && (key[i] >> 32) == (int64_t)j->col[b + k - 1]) continue;
        j->col[b + k] = (int32_t)(key[i] >> 32);
        j->ev[b + k] = key[i] & 0xffffffffll;
        ++k;
      }
      j->kept[r] = k;
    }
  }
  free(key);
  return NULL;
}

typedef struct {
  int64_t r0, r1;
  uint64_t sm;
  const int64_t *ptr, *start, *kept;
  const int32_t* col;
  const int64_t* ev;
  int32_t* oc;
  double* ov;
} OutJob;

static void* csr_out(void* p) {
  OutJob* j = (OutJob*)p;
  for (int64_t r = j->r0; r < j->r1; ++r)
    for (int64_t k = 0; k < j->kept[r]; ++k) {
      j->oc[j->ptr[r] + k] = j->col[j->start[r] + k];
      j->ov[j->ptr[r] + k] = 1.0 - u01(j->sm, (uint64_t)j->ev[j->start[r] + k], 63);
    }
  return NULL;
}

/* Builds the canonical CSR of the whole matrix.  Outputs (malloc'd, freed
 * with rmat_csr_free): *ptr_out int64[n+1], *col_out int32[nnz], *val_out
 * double[nnz]; returns nnz, or -1 on allocation failure / draws >= 2^32. */
int64_t rmat_csr(int scale, int64_t draws, double a, double b, double c, uint64_t seed, int nthreads,
                 int64_t** ptr_out, int32_t** col_out, double** val_out) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  if (draws >= (1ll << 32)) return -1;
  const int64_t n = 1ll << scale;
  _Atomic int64_t* fill = (_Atomic int64_t*)calloc((size_t)n, sizeof(int64_t));
  int64_t* start = (int64_t*)malloc((size_t)(n + 1) * sizeof(int64_t));
  int32_t* col = (int32_t*)malloc((size_t)(draws > 0 ? draws : 1) * sizeof(int32_t));
  int64_t* ev = (int64_t*)malloc((size_t)(draws > 0 ? draws : 1) * sizeof(int64_t));
  int64_t* kept = (int64_t*)calloc((size_t)n, sizeof(int64_t));
  if (!fill || !start || !col || !ev || !kept) {
    free((void*)fill), free(start), free(col), free(ev), free(kept);
    return -1;
  }
  CsrJob jobs[256];
  pthread_t th[256];
  for (int pass = 1; pass <= 2; ++pass) {
    if (pass == 2) {
      start[0] = 0;
      for (int64_t r = 0; r < n; ++r) start[r + 1] = start[r] + atomic_load(&fill[r]);
      for (int64_t r = 0; r < n; ++r) atomic_store(&fill[r], start[r]);
    }
    for (int t = 0; t < nthreads; ++t) {
      CsrJob* j = &jobs[t];
      j->scale = scale;
      j->lo = draws * t / nthreads;
      j->hi = draws * (t + 1) / nthreads;
      j->sm = mix64(seed);
      j->a = a;
      j->ab = a + b;
      j->abc = a + b + c;
      j->fill = fill;
      j->col = col;
      j->ev = ev;
      j->pass = pass;
      pthread_create(&th[t], NULL, csr_pass, j);
    }
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
  }
  free((void*)fill);
  _Atomic int64_t next = 0;
  RowJob rj[256];
  for (int t = 0; t < nthreads; ++t) {
    rj[t] = (RowJob){n, &next, start, col, ev, kept};
    pthread_create(&th[t], NULL, csr_rows, &rj[t]);
  }
  for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
  int64_t* ptr = (int64_t*)malloc((size_t)(n + 1) * sizeof(int64_t));
  ptr[0] = 0;
  for (int64_t r = 0; r < n; ++r) ptr[r + 1] = ptr[r] + kept[r];
  const int64_t nnz = ptr[n];
  int32_t* oc = (int32_t*)malloc((size_t)(nnz > 0 ? nnz : 1) * sizeof(int32_t));
  double* ov = (double*)malloc((size_t)(nnz > 0 ? nnz : 1) * sizeof(double));
  OutJob oj[256];
  for (int t = 0; t < nthreads; ++t) {
    oj[t] = (OutJob){n * t / nthreads, n * (t + 1) / nthreads, mix64(seed), ptr, start, kept, col, ev, oc, ov};
    pthread_create(&th[t], NULL, csr_out, &oj[t]);
  }
  for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
  free(start), free(col), free(ev), free(kept);
  *ptr_out = ptr;
  *col_out = oc;
  *val_out = ov;
  return nnz;
}

void rmat_csr_free(int64_t* ptr, int32_t* col, double* val) { free(ptr), free(col), free(val); }
