// Synthetic inputs for the benchmark configurations:
// R-MAT edge lists and uniform vectors from a counter-based hash, so the
// same matrix can be regenerated bit-identically on the host
// (oracle/synth_ref.py, oracle/rmat_sample.c) for parity checks and the CPU
// baseline sample.
//
// hash(seed, e, l) = mix64(mix64(seed) ^ (e * 64 + l)), mix64 = splitmix64
// finaliser; U = (hash >> 11) * 2^-53.  R-MAT level l (0 = most significant
// bit) picks quadrant (0,0) if U < a, (0,1) if U < a+b, (1,0) if U < a+b+c,
// else (1,1); the value is 1 - U(seed, e, 63) in (0, 1].
#include "prims.cuh"

using namespace spmvb;

struct spmvb_rmat {
  int scale = 0;
  int64_t draws = 0, nnz = 0;
  double a = 0, ab = 0, abc = 0;
  uint64_t seed_mixed = 0;
  DevBuf<uint8_t> keep;
  DevBuf<uint32_t> pos;
};

namespace {

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ double hash_u01(uint64_t seed_mixed, uint64_t e, unsigned l) {
  uint64_t h = mix64(seed_mixed ^ (e * 64ull + l));
  return static_cast<double>(h >> 11) * 0x1.0p-53;
}

__device__ __forceinline__ void rmat_edge(uint64_t sm, int64_t e, int scale, double a, double ab, double abc,
                                          uint32_t& r, uint32_t& c) {
  uint32_t row = 0, col = 0;
  for (int l = 0; l < scale; ++l) {
    double u = hash_u01(sm, static_cast<uint64_t>(e), l);
    uint32_t rb, cb;
    if (u < a) { rb = 0; cb = 0; }
    else if (u < ab) { rb = 0; cb = 1; }
    else if (u < abc) { rb = 1; cb = 0; }
    else { rb = 1; cb = 1; }
    row = (row << 1) | rb;
    col = (col << 1) | cb;
  }
  r = row;
  c = col;
}

__global__ void k_rmat_keys(int64_t draws, int scale, double a, double ab, double abc, uint64_t sm,
                            uint64_t* __restrict__ keys) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < draws;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    uint32_t r, c;
    rmat_edge(sm, e, scale, a, ab, abc, r, c);
    keys[e] = (static_cast<uint64_t>(r) << scale) | c;
  }
}

// keep[draw] = 1 iff the draw is the first occurrence of its (row, col).
__global__ void k_rmat_first(const uint64_t* __restrict__ skeys, const uint32_t* __restrict__ sidx, int64_t n,
                             uint8_t* __restrict__ keep) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    keep[sidx[i]] = (i == 0 || skeys[i - 1] != skeys[i]) ? 1 : 0;
}

__global__ void k_rmat_emit(int64_t draws, int scale, double a, double ab, double abc, uint64_t sm,
                            const uint8_t* __restrict__ keep, const uint32_t* __restrict__ pos,
                            int32_t* __restrict__ row_out, int32_t* __restrict__ col_out,
                            double* __restrict__ val_out) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < draws;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (!keep[e]) continue;
    uint32_t r, c;
    rmat_edge(sm, e, scale, a, ab, abc, r, c);
    uint32_t p = pos[e];
    row_out[p] = static_cast<int32_t>(r);
    col_out[p] = static_cast<int32_t>(c);
    val_out[p] = 1.0 - hash_u01(sm, static_cast<uint64_t>(e), 63);
  }
}

__global__ void k_fill_uniform(double* __restrict__ x, int64_t n, double lo, double span, uint64_t sm) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    x[i] = __dadd_rn(lo, __dmul_rn(span, hash_u01(sm, static_cast<uint64_t>(i), 0)));
}

}  // namespace

extern "C" int spmvb_rmat_begin(int scale, int64_t draws, double a, double b, double c, uint64_t seed,
                                spmvb_rmat** plan, int64_t* nnz_out, void* stream) {
  return guard([&] {
    cudaStream_t s = as_stream(stream);
    if (scale < 1 || scale > 30) fail(SPMVB_INVALID_ARG, "R-MAT scale must be in [1, 30]");
    if (draws < 0 || draws >= (1ll << 32)) fail(SPMVB_INVALID_ARG, "R-MAT draws must be in [0, 2^32)");
    auto* p = new spmvb_rmat();
    try {
      p->scale = scale;
      p->draws = draws;
      p->a = a;
      p->ab = a + b;
      p->abc = a + b + c;
      p->seed_mixed = mix64(seed);
      if (draws > 0) {
        DevBuf<uint64_t> ka(draws, s), kb(draws, s);
        DevBuf<uint32_t> vb(draws, s), vs(draws, s);
        k_rmat_keys<<<grid_for(draws, 256, 148 * 32), 256, 0, s>>>(draws, scale, p->a, p->ab, p->abc, p->seed_mixed,
                                                                   ka.get());
        SPMVB_LAUNCHED("k_rmat_keys");
        RadixSortResult rs = radix_sort_pairs(ka.get(), nullptr, kb.get(), vb.get(), vs.get(), draws, 2 * scale, s);
        p->keep = DevBuf<uint8_t>(draws, s);
        k_rmat_first<<<grid_for(draws, 256, 148 * 32), 256, 0, s>>>(rs.keys, rs.vals, draws, p->keep.get());
        SPMVB_LAUNCHED("k_rmat_first");
        p->pos = DevBuf<uint32_t>(draws, s);
        DevBuf<uint32_t> total(1, s);
        const uint8_t* kp = p->keep.get();
        exclusive_scan<uint32_t>(
            draws, [=] __device__(int64_t i) { return static_cast<uint32_t>(kp[i]); },
            ArrayStore<uint32_t>{p->pos.get()}, OpSum{}, 0u, total.get(), s);
        uint32_t h = 0;
        copy_to_host(&h, total.get(), 1, s);
        p->nnz = h;
      }
    } catch (...) {
      delete p;
      throw;
    }
    *plan = p;
    *nnz_out = p->nnz;
  });
}

extern "C" int spmvb_rmat_finish(spmvb_rmat* p, int32_t* row_out, int32_t* col_out, double* val_out, void* stream) {
  return guard([&] {
    cudaStream_t s = as_stream(stream);
    if (!p) fail(SPMVB_INVALID_ARG, "null plan");
    if (p->nnz > 0) {
      k_rmat_emit<<<grid_for(p->draws, 256, 148 * 32), 256, 0, s>>>(p->draws, p->scale, p->a, p->ab, p->abc,
                                                                    p->seed_mixed, p->keep.get(), p->pos.get(),
                                                                    row_out, col_out, val_out);
      SPMVB_LAUNCHED("k_rmat_emit");
    }
    delete p;
  });
}

extern "C" void spmvb_rmat_free(spmvb_rmat* p) { delete p; }

extern "C" int spmvb_fill_uniform(double* x, int64_t n, double lo, double hi, uint64_t seed, void* stream) {
  return guard([&] {
    cudaStream_t s = as_stream(stream);
    if (n <= 0) return;
    k_fill_uniform<<<grid_for(n, 256, 148 * 32), 256, 0, s>>>(x, n, lo, hi - lo, mix64(seed));
    SPMVB_LAUNCHED("k_fill_uniform");
  });
}
