// Row-block power iteration behind the C ABI (the
// dist_{init,spmv_iter,destroy} entry points around a caller-owned NCCL
// communicator), for callers that do not go through torch.distributed.
//
// One step, all on the caller's stream (the same algorithm as
// dist.PowerIteration's plain all-gatherv path):
//   y_p = scale * A_p x      local SpMV through the caller's callback (any
//                            format of this library; ctx is the caller's)
//   ||y||^2 = sum_p ||y_p||^2  spmvb_sumsq + ncclAllReduce (1 double)
//   x_next <- all-gatherv(y_p) grouped ncclSend/ncclRecv, true per-rank counts
//   scale <- 1 / ||y||          spmvb_inv_sqrt
// NCCL is not linked: its entry points are resolved at first use from the
// libnccl.so.2 already loaded in the process (the one that created the
// communicator, e.g. torch's), else loaded by soname.
#include <dlfcn.h>
#include <nccl.h>

#include <mutex>
#include <vector>

#include "common.cuh"

using namespace spmvb;

struct spmvb_dist {
  ncclComm_t comm;
  int rank, world;
  std::vector<int64_t> bounds;
  int n_ranges = 0;             // K: row ranges per step (0: the whole shard at once)
  std::vector<int64_t> spans;   // world * K * 2: rank p's range k = local rows [a, b)
  cudaStream_t comm_stream = nullptr;
  std::vector<cudaEvent_t> events;
  ~spmvb_dist() {
    for (cudaEvent_t e : events) cudaEventDestroy(e);
    if (comm_stream) cudaStreamDestroy(comm_stream);
  }
};

namespace {

struct Nccl {
  decltype(&ncclAllReduce) all_reduce = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
  decltype(&ncclGetVersion) get_version = nullptr;
  bool ok = false;
};

const Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) return;
    n.all_reduce = reinterpret_cast<decltype(&ncclAllReduce)>(dlsym(h, "ncclAllReduce"));
    n.send = reinterpret_cast<decltype(&ncclSend)>(dlsym(h, "ncclSend"));
    n.recv = reinterpret_cast<decltype(&ncclRecv)>(dlsym(h, "ncclRecv"));
    n.group_start = reinterpret_cast<decltype(&ncclGroupStart)>(dlsym(h, "ncclGroupStart"));
    n.group_end = reinterpret_cast<decltype(&ncclGroupEnd)>(dlsym(h, "ncclGroupEnd"));
    n.error_string = reinterpret_cast<decltype(&ncclGetErrorString)>(dlsym(h, "ncclGetErrorString"));
    n.get_version = reinterpret_cast<decltype(&ncclGetVersion)>(dlsym(h, "ncclGetVersion"));
    n.ok = n.all_reduce && n.send && n.recv && n.group_start && n.group_end && n.error_string && n.get_version;
  });
  if (!n.ok) fail(SPMVB_INTERNAL, "libnccl.so.2 could not be loaded (needed by the spmvb_dist_* entry points)");
  return n;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) fail(SPMVB_CUDA_ERROR, "%s failed: %s", what, nccl().error_string(r));
}

void forward(int st) {  // a nested C-ABI call's failure, message kept
  if (st) {
    const std::string msg = spmvb_last_error();
    fail(st, "%s", msg.c_str());
  }
}

}  // namespace

extern "C" int spmvb_dist_nccl_version(int* version) {
  return guard([&] {
    if (!version) fail(SPMVB_INVALID_ARG, "version is required");
    nccl_check(nccl().get_version(version), "ncclGetVersion");
  });
}

extern "C" int spmvb_dist_init(void* nccl_comm, int rank, int world, const int64_t* bounds, spmvb_dist** out) {
  return guard([&] {
    if (!out) fail(SPMVB_INVALID_ARG, "out is required");
    *out = nullptr;
    if (!nccl_comm) fail(SPMVB_INVALID_ARG, "an NCCL communicator is required");
    if (world < 1 || rank < 0 || rank >= world) fail(SPMVB_INVALID_ARG, "rank %d out of range for world %d", rank, world);
    if (!bounds) fail(SPMVB_INVALID_ARG, "bounds (world + 1 row boundaries) are required");
    if (bounds[0] != 0) fail(SPMVB_INVALID_ARG, "bounds must start at row 0");
    for (int p = 0; p < world; ++p)
      if (bounds[p + 1] < bounds[p]) fail(SPMVB_INVALID_ARG, "bounds must be non-decreasing");
    nccl();  // fail now, not at the first step, if NCCL is missing
    auto* d = new spmvb_dist{static_cast<ncclComm_t>(nccl_comm), rank, world,
                             std::vector<int64_t>(bounds, bounds + world + 1)};
    *out = d;
  });
}

extern "C" int spmvb_dist_step(spmvb_dist* d, spmvb_local_spmv_fn local_spmv, void* ctx, const double* x,
                               double* x_next, double* sumsq, double* scale, void* stream) {
  return guard([&] {
    if (!d || !local_spmv) fail(SPMVB_INVALID_ARG, "handle and local SpMV are required");
    if (!x || !x_next || !sumsq || !scale) fail(SPMVB_INVALID_ARG, "x, x_next, sumsq and scale are required");
    cudaStream_t s = as_stream(stream);
    const int64_t lo = d->bounds[d->rank], hi = d->bounds[d->rank + 1];
    forward(local_spmv(ctx, x, x_next + lo, scale, stream));
    forward(spmvb_sumsq(x_next + lo, hi - lo, sumsq, stream));
    const Nccl& n = nccl();
    if (d->world > 1) {
      nccl_check(n.all_reduce(sumsq, sumsq, 1, ncclFloat64, ncclSum, d->comm, s), "ncclAllReduce");
      nccl_check(n.group_start(), "ncclGroupStart");
      for (int p = 0; p < d->world; ++p) {
        if (p == d->rank) continue;
        const int64_t plo = d->bounds[p], phi = d->bounds[p + 1];
        if (hi > lo) nccl_check(n.send(x_next + lo, hi - lo, ncclFloat64, p, d->comm, s), "ncclSend");
        if (phi > plo) nccl_check(n.recv(x_next + plo, phi - plo, ncclFloat64, p, d->comm, s), "ncclRecv");
      }
      nccl_check(n.group_end(), "ncclGroupEnd");
    }
    forward(spmvb_inv_sqrt(sumsq, scale, stream));
  });
}

extern "C" int spmvb_dist_init_ranges(void* nccl_comm, int rank, int world, const int64_t* bounds, int n_ranges,
                                      const int64_t* spans, spmvb_dist** out) {
  return guard([&] {
    if (const int st = spmvb_dist_init(nccl_comm, rank, world, bounds, out)) forward(st);
    spmvb_dist* d = *out;
    *out = nullptr;
    auto fail_free = [&](const char* msg) {
      delete d;
      fail(SPMVB_INVALID_ARG, "%s", msg);
    };
    if (n_ranges < 1 || !spans) fail_free("n_ranges >= 1 and spans (world * n_ranges * 2) are required");
    for (int p = 0; p < world; ++p)
      for (int k = 0; k < n_ranges; ++k) {
        const int64_t a = spans[(p * n_ranges + k) * 2], b = spans[(p * n_ranges + k) * 2 + 1];
        if (a < 0 || b < a || b > bounds[p + 1] - bounds[p]) fail_free("a range lies outside its rank's rows");
      }
    d->n_ranges = n_ranges;
    d->spans.assign(spans, spans + static_cast<size_t>(world) * n_ranges * 2);
    if (cudaStreamCreateWithFlags(&d->comm_stream, cudaStreamNonBlocking) != cudaSuccess)
      fail_free("could not create the exchange stream");
    d->events.resize(n_ranges + 2, nullptr);
    for (auto& e : d->events)
      if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) fail_free("could not create events");
    *out = d;
  });
}

// Ranges in order k = 0..K-1 on the caller's stream; after each one its rows
// go to every peer (and the peers' range-k rows come in) on the exchange
// stream while range k+1 computes.  Every rank walks the same k, so the k-th
// NCCL groups pair up.  Then ||y||^2 (all-reduce on the exchange stream, in
// the same order on every rank), and the caller's stream waits for the
// exchange before 1/||y||.
extern "C" int spmvb_dist_step_ranges(spmvb_dist* d, spmvb_range_spmv_fn range_spmv, void* ctx, const double* x,
                                      double* x_next, double* sumsq, double* scale, void* stream) {
  return guard([&] {
    if (!d || !range_spmv) fail(SPMVB_INVALID_ARG, "handle and range SpMV are required");
    if (d->n_ranges < 1) fail(SPMVB_INVALID_ARG, "the handle has no range plan (spmvb_dist_init_ranges)");
    if (!x || !x_next || !sumsq || !scale) fail(SPMVB_INVALID_ARG, "x, x_next, sumsq and scale are required");
    cudaStream_t s = as_stream(stream), cs = d->comm_stream;
    const int K = d->n_ranges, me = d->rank;
    const int64_t lo = d->bounds[me], hi = d->bounds[me + 1];
    auto span = [&](int p, int k, int64_t& a, int64_t& b) {
      a = d->spans[(static_cast<size_t>(p) * K + k) * 2];
      b = d->spans[(static_cast<size_t>(p) * K + k) * 2 + 1];
    };
    const Nccl& n = nccl();
    for (int k = 0; k < K; ++k) {
      int64_t a, b;
      span(me, k, a, b);
      // every k is computed (the callback knows its own ranges); the spans
      // only say which rows travel (a range in the empty tail sends none)
      forward(range_spmv(ctx, k, x, x_next + lo, scale, stream));
      if (d->world == 1) continue;
      SPMVB_CUDA(cudaEventRecord(d->events[k], s));
      SPMVB_CUDA(cudaStreamWaitEvent(cs, d->events[k], 0));
      nccl_check(n.group_start(), "ncclGroupStart");
      for (int p = 0; p < d->world; ++p) {
        if (p == me) continue;
        int64_t pa, pb;
        span(p, k, pa, pb);
        if (b > a) nccl_check(n.send(x_next + lo + a, b - a, ncclFloat64, p, d->comm, cs), "ncclSend");
        if (pb > pa) nccl_check(n.recv(x_next + d->bounds[p] + pa, pb - pa, ncclFloat64, p, d->comm, cs), "ncclRecv");
      }
      nccl_check(n.group_end(), "ncclGroupEnd");
    }
    forward(spmvb_sumsq(x_next + lo, hi - lo, sumsq, stream));
    if (d->world > 1) {
      SPMVB_CUDA(cudaEventRecord(d->events[K], s));
      SPMVB_CUDA(cudaStreamWaitEvent(cs, d->events[K], 0));
      nccl_check(n.all_reduce(sumsq, sumsq, 1, ncclFloat64, ncclSum, d->comm, cs), "ncclAllReduce");
      SPMVB_CUDA(cudaEventRecord(d->events[K + 1], cs));
      SPMVB_CUDA(cudaStreamWaitEvent(s, d->events[K + 1], 0));
    }
    forward(spmvb_inv_sqrt(sumsq, scale, stream));
  });
}

extern "C" int spmvb_dist_destroy(spmvb_dist* d) {
  return guard([&] { delete d; });
}
