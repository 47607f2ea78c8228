// extern "C" boundary (include/cprand_b200.h). Exceptions never cross it:
// each entry point maps the internal error taxonomy onto status codes.

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <string>
#include <thread>
#include <vector>

#include "../../include/cprand_b200.h"
#include "session.hpp"

using namespace cpb;

namespace {

thread_local std::string g_err;

void need(const void* h) {
  if (!h) throw InvalidArgument("null (or destroyed) handle");
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return CPRAND_OK;
  } catch (const Error& e) {
    g_err = e.what();
    return e.status;
  } catch (const std::bad_alloc& e) {
    g_err = std::string("host allocation failed: ") + e.what();
    return CPRAND_ERR_INTERNAL;
  } catch (const std::exception& e) {
    g_err = e.what();
    return CPRAND_ERR_INTERNAL;
  }
}

std::vector<i64> dims_of(const int64_t* dims, int32_t order) {
  if (dims == nullptr || order < 1) throw InvalidArgument("tensor order must be >= 1");
  std::vector<i64> d(dims, dims + order);
  for (i64 v : d)
    if (v < 1) throw InvalidArgument("tensor dims must be >= 1");
  return d;
}

}  // namespace

struct cprand_comm_s {
  std::unique_ptr<cpb::Comm> comm;  // NCCL, or a rank of a loopback group
  int rank = 0, nranks = 1, device = 0;
};

struct cprand_loopback_s {
  std::shared_ptr<cpb::LoopbackGroup> g;
};

namespace {

Options opts_of(const cprand_options_t* o) {
  Options r;
  if (!o) return r;
  r.max_iters = o->max_iters;
  r.fit_tolerance = o->fit_tolerance;
  if (o->has_fit_threshold) r.fit_threshold = o->fit_threshold;
  r.rng_seed = o->rng_seed;
  r.init = o->init;
  r.fit_sample_count = o->fit_sample_count;
  r.stall_limit = o->stall_limit;
  r.transform = o->transform;
  r.bench_mode = o->bench_mode != 0;
  r.exhaustive_samples = o->exhaustive_samples != 0;
  r.exact_fit_trace = o->exact_fit_trace != 0;
  r.device = o->device;
  r.x_mutable = o->x_mutable != 0;
  r.replicas = o->replicas;
  r.fused = o->fused;
  r.atomic_gram = o->atomic_gram != 0;
  if (o->comm != nullptr) {
    const auto* c = static_cast<const cprand_comm_s*>(o->comm);
    r.comm = c->comm.get();
    r.nranks = c->nranks;
    r.rank = c->rank;
    r.shard_total = o->shard_total;
  } else if (o->shard_total != 0) {
    throw InvalidArgument("shard_total requires a communicator");
  }
  return r;
}

int pick_device(int requested) {
  int n = 0;
  CPB_CUDA(cudaGetDeviceCount(&n));
  if (n == 0) throw CudaError("no CUDA device");
  if (requested >= 0) {
    if (requested >= n) throw InvalidArgument("device ordinal out of range");
    return requested;
  }
  int d = 0;
  CPB_CUDA(cudaGetDevice(&d));
  return d;
}

void fill_result(Session& s, double* out_lambda, double* const* out_factors,
                 cprand_trace_record_t* trace, int32_t cap, cprand_result_t* res) {
  std::vector<Trace> tr;
  int iters = 0, reason = 0;
  double setup = 0, total = 0, loop = 0;
  s.result(out_lambda, out_factors, tr, &iters, &reason, &setup, &total, &loop);
  if (trace)
    for (size_t i = 0; i < tr.size() && static_cast<int32_t>(i) < cap; ++i)
      trace[i] = {tr[i].iteration, tr[i].elapsed, tr[i].fit, tr[i].is_estimate ? 1 : 0, tr[i].best};
  if (res) {
    res->iterations = iters;
    res->reason = reason;
    res->setup_seconds = setup;
    res->total_seconds = total;
    res->trace_len = static_cast<int32_t>(tr.size());
    res->loop_seconds_device = loop;
  }
}

}  // namespace

struct cprand_tensor_s {
  std::unique_ptr<Tensor> t;
};
struct cprand_session_s {
  std::unique_ptr<Session> s;
};


extern "C" {

void cprand_options_init(cprand_options_t* o) {
  if (!o) return;
  std::memset(o, 0, sizeof(*o));
  o->max_iters = 200;
  o->fit_tolerance = 1e-4;
  o->rng_seed = 0;
  o->init = CPRAND_INIT_RANDOM;
  o->fit_sample_count = int64_t{1} << 14;
  o->stall_limit = 10;
  o->transform = CPRAND_TRANSFORM_UNSET;
  o->device = -1;
  o->replicas = -1;
  o->fused = -1;
}

const char* cprand_last_error(void) { return g_err.c_str(); }

int cprand_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int64_t cprand_default_sample_count(int64_t r) {  // sampling.hpp:18-23
  if (r < 1) {
    g_err = "rank must be >= 1";
    return -1;
  }
  if (r == 1) return 10;
  return static_cast<int64_t>(std::lround(10.0 * static_cast<double>(r) * std::log(static_cast<double>(r))));
}

const char* cprand_build_info(void) {
  return "cprand_b200: sm_100a (compute_100a), fp64 gather/SKR/Gram/RHS fused kernels, "
         "normal-equation pivoted solve, device fit + stop rule, Makhoul DCT mixing";
}

int cprand_solve(int32_t method, const double* x, const int64_t* dims, int32_t order, int64_t r,
                 int64_t s, const cprand_options_t* opts, const double* init_lambda,
                 const double* const* init_factors, double* out_lambda, double* const* out_factors,
                 cprand_trace_record_t* trace, int32_t trace_cap, cprand_result_t* res) {
  return guarded([&] {
    Options o = opts_of(opts);
    const auto d = dims_of(dims, order);
    if (!out_lambda || !out_factors) throw InvalidArgument("output buffers are required");
    if (r < 1) throw InvalidArgument("rank must be >= 1");
    const int dev = pick_device(o.device);
    CPB_CUDA(cudaSetDevice(dev));
    Tensor t(d, dev);
    const size_t bytes = static_cast<size_t>(t.p) * sizeof(double);
    const bool on_device = opts && opts->x_is_device;
    // A pinned host tensor is uploaded in parts along the last mode by an
    // uploader thread (every part queued at once on its own stream) while the
    // session sets up: the host-side setup (sample tables, work buffers, the
    // kernel arguments) and each part's share of the mode-major replicas
    // overlap the copy (Tensor::chunk_ev, Session::launch_replicas).
    // Pageable memory is copied synchronously.
    struct Upload {
      cudaStream_t st = nullptr;
      Tensor* t = nullptr;
      std::thread th;
      std::atomic<int> err{0};
      ~Upload() {
        if (th.joinable()) th.join();
        if (st) cudaStreamSynchronize(st);
        if (t) {
          for (cudaEvent_t e : t->chunk_ev) cudaEventDestroy(e);
          t->chunk_ev.clear();
          t->chunk_end.clear();
        }
        if (st) cudaStreamDestroy(st);
      }
    } up;  // (declared after t: joined and drained before the tensor is freed)
    bool pinned = false;
    if (!on_device && bytes >= (size_t{64} << 20) && !std::getenv("CPRAND_SYNC_UPLOAD")) {
      cudaPointerAttributes at{};
      if (cudaPointerGetAttributes(&at, x) == cudaSuccess) pinned = at.type == cudaMemoryTypeHost;
      (void)cudaGetLastError();
    }
    if (pinned) {
      const i64 ilast = d.back(), slice = t.p / ilast;
      // parts of >= 256 MB, at most 32 (CPRAND_UPLOAD_PARTS: tests)
      const char* pe = std::getenv("CPRAND_UPLOAD_PARTS");
      const i64 want = pe ? std::atoll(pe) : std::min<i64>(32, static_cast<i64>(bytes >> 28));
      const i64 parts = std::min<i64>(ilast, std::max<i64>(1, want));
      CPB_CUDA(cudaStreamCreateWithFlags(&up.st, cudaStreamNonBlocking));
      up.t = &t;
      for (i64 c = 0; c < parts; ++c) {
        cudaEvent_t e = nullptr;
        CPB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        t.chunk_ev.push_back(e);
        t.chunk_end.push_back(ilast * (c + 1) / parts);
      }
      t.chunk_submitted.store(0);
      up.th = std::thread([&up, &t, x, slice, dev] {
        cudaSetDevice(dev);
        const auto t0 = std::chrono::steady_clock::now();
        i64 a = 0;
        for (size_t c = 0; c < t.chunk_ev.size(); ++c) {
          const i64 b = t.chunk_end[c];
          cudaError_t e = cudaMemcpyAsync(t.d + a * slice, x + a * slice, static_cast<size_t>((b - a) * slice) * sizeof(double),
                                          cudaMemcpyHostToDevice, up.st);
          if (e == cudaSuccess) e = cudaEventRecord(t.chunk_ev[c], up.st);
          if (e != cudaSuccess) up.err.store(static_cast<int>(e));
          t.chunk_submitted.store(static_cast<int>(c) + 1, std::memory_order_release);
          a = b;
        }
        if (std::getenv("CPRAND_DEBUG_SETUP")) {
          cudaEventSynchronize(t.chunk_ev.back());
          std::fprintf(stderr, "upload: %zu parts resident %.2f ms after the first was submitted\n", t.chunk_ev.size(),
                       1e3 * std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
        }
      });
    } else {
      CPB_CUDA(cudaMemcpy(t.d, x, bytes, on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice));
    }
    o.x_mutable = true;  // t is our private copy
    Session sess(method, &t, static_cast<int>(r), static_cast<int>(s), o, init_lambda, init_factors);
    if (up.th.joinable()) up.th.join();
    if (up.err.load()) throw CudaError(std::string("tensor upload: ") + cudaGetErrorString(static_cast<cudaError_t>(up.err.load())));
    sess.run(o.max_iters);
    fill_result(sess, out_lambda, out_factors, trace, trace_cap, res);
  });
}

int cprand_tensor_exact_fit(cprand_tensor_t t, const double* lambda, const double* const* factors, int64_t r,
                            double* fit) {
  return guarded([&] {
    need(t);
    if (!lambda || !factors || !fit) throw InvalidArgument("exact_fit: null model or output");
    *fit = device_exact_fit(*t->t, lambda, factors, static_cast<int>(r));
  });
}

int cprand_exact_fit(const double* x, const int64_t* dims, int32_t order, const double* lambda,
                     const double* const* factors, int64_t r, int32_t device, double* fit) {
  return guarded([&] {
    const auto d = dims_of(dims, order);
    if (!x || !lambda || !factors || !fit) throw InvalidArgument("exact_fit: null input");
    const int dev = pick_device(device);
    CPB_CUDA(cudaSetDevice(dev));
    Tensor t(d, dev);
    CPB_CUDA(cudaMemcpy(t.d, x, sizeof(double) * t.p, cudaMemcpyHostToDevice));
    *fit = device_exact_fit(t, lambda, factors, static_cast<int>(r));
  });
}

int cprand_tensor_create(const int64_t* dims, int32_t order, int32_t device, cprand_tensor_t* out) {
  return guarded([&] {
    if (dims == nullptr || order < 1) throw InvalidArgument("tensor order must be >= 1");
    const std::vector<i64> d(dims, dims + order);  // Tensor checks them (an empty slab may have last dim 0)
    auto* h = new cprand_tensor_s;
    h->t = std::make_unique<Tensor>(d, pick_device(device));
    *out = h;
  });
}

int cprand_tensor_upload(cprand_tensor_t t, const double* host) {
  return guarded([&] {
    need(t);
    CPB_CUDA(cudaSetDevice(t->t->device));
    CPB_CUDA(cudaMemcpy(t->t->d, host, sizeof(double) * t->t->p, cudaMemcpyHostToDevice));
  });
}

int cprand_tensor_download(cprand_tensor_t t, double* host) {
  return guarded([&] {
    need(t);
    CPB_CUDA(cudaSetDevice(t->t->device));
    CPB_CUDA(cudaMemcpy(host, t->t->d, sizeof(double) * t->t->p, cudaMemcpyDeviceToHost));
  });
}

int cprand_tensor_synth(cprand_tensor_t t, int64_t r, double c, double eta, uint64_t seed,
                        double* const* out_factors) {
  return guarded([&] {
    need(t);
    if (r < 1) throw InvalidArgument("rank must be >= 1");
    op_synth(t->t.get(), static_cast<int>(r), c, eta, seed, out_factors);
  });
}

int cprand_tensor_synth_slab(cprand_tensor_t t, int64_t r, double c, double eta, uint64_t seed,
                             int64_t shard_total, cprand_comm_t comm, double* const* out_factors) {
  return guarded([&] {
    need(t);
    need(comm);
    if (r < 1) throw InvalidArgument("rank must be >= 1");
    const i64 lmax = (shard_total + comm->nranks - 1) / comm->nranks;
    const i64 off = lmax * comm->rank;
    const i64 len = std::max<i64>(0, std::min<i64>(shard_total, off + lmax) - off);
    if (t->t->dims.back() != len) throw InvalidArgument("slab tensor must hold rows [rank*ceil(I/P), ...)");
    auto reduce = [&](double* sums) { comm->comm->allreduce_sum(sums, 2, nullptr); };
    op_synth(t->t.get(), static_cast<int>(r), c, eta, seed, out_factors, off, shard_total, reduce);
  });
}

int cprand_tensor_mix(cprand_tensor_t t, int32_t transform, uint64_t seed, double* ms_per_mode) {
  return guarded([&] {
    need(t);
    op_tensor_mix(t->t.get(), transform, seed, ms_per_mode);
  });
}

int cprand_tensor_mix_modes(cprand_tensor_t t, int32_t transform, uint64_t seed, int32_t mode_begin,
                            int32_t mode_end, double* ms_per_mode) {
  return guarded([&] {
    need(t);
    op_tensor_mix(t->t.get(), transform, seed, ms_per_mode, mode_begin, mode_end);
  });
}

int cprand_tensor_read_fibers(cprand_tensor_t t, int32_t mode, const int64_t* idxs, int64_t s, double* out) {
  return guarded([&] {
    need(t);
    if (s < 0) throw InvalidArgument("sample count must be >= 0");
    op_read_fibers(t->t.get(), mode, idxs, s, out);
  });
}

double* cprand_tensor_device_ptr(cprand_tensor_t t) { return t ? t->t->d : nullptr; }

void cprand_tensor_destroy(cprand_tensor_t t) { delete t; }

int cprand_session_create(int32_t method, cprand_tensor_t t, int64_t r, int64_t s,
                          const cprand_options_t* opts, const double* init_lambda,
                          const double* const* init_factors, cprand_session_t* out) {
  return guarded([&] {
    Options o = opts_of(opts);
    auto* h = new cprand_session_s;
    try {
      h->s = std::make_unique<Session>(method, t->t.get(), static_cast<int>(r), static_cast<int>(s), o,
                                       init_lambda, init_factors);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

int cprand_session_run(cprand_session_t s, int32_t n, int32_t* ran) {
  return guarded([&] {
    need(s);
    const int k = s->s->run(n);
    if (ran) *ran = k;
  });
}

int cprand_session_enqueue(cprand_session_t s, int32_t n) {
  return guarded([&] { need(s); s->s->enqueue(n); });
}

int cprand_session_sync(cprand_session_t s) {
  return guarded([&] { need(s); s->s->sync(); });
}

int cprand_session_timed_enqueue(cprand_session_t s, int32_t n, double* ms) {
  return guarded([&] { need(s); *ms = s->s->timed_enqueue(n); });
}

void* cprand_host_alloc_pinned(uint64_t bytes) {
  void* p = nullptr;
  if (cudaHostAlloc(&p, bytes, cudaHostAllocDefault) != cudaSuccess) {
    cudaGetLastError();
    g_err = "cudaHostAlloc failed";
    return nullptr;
  }
  return p;
}

void cprand_host_free_pinned(void* p) {
  if (p) cudaFreeHost(p);
}

void cprand_device_cache_release(void) { cpb::big_release_all(); }

void* cprand_session_stream(cprand_session_t s) { return s ? static_cast<void*>(s->s->stream()) : nullptr; }

int cprand_session_set_kernel_timing(cprand_session_t s, int32_t on) {
  return guarded([&] { need(s); s->s->set_timing(on != 0); });
}

int cprand_session_kernel_stats(cprand_session_t s, int32_t mode, int32_t kind, int64_t* launches,
                                double* total_ms, double* work) {
  return guarded([&] {
    need(s);
    i64 l = 0;
    s->s->kernel_stats(mode, kind, &l, total_ms, work);
    *launches = l;
  });
}

int cprand_session_phase_us(cprand_session_t s, double* out, int32_t cap, int32_t* n) {
  return guarded([&] {
    need(s);
    const auto v = s->s->phase_us();
    *n = static_cast<int32_t>(v.size());
    for (size_t i = 0; i < v.size() && static_cast<int32_t>(i) < cap; ++i) out[i] = v[i];
  });
}

int cprand_session_fused(cprand_session_t s, int32_t* out) {
  return guarded([&] {
    need(s);
    *out = s->s->fused() ? 1 : 0;
  });
}

int cprand_session_gram_fallbacks(cprand_session_t s, int64_t* out) {
  return guarded([&] { need(s); *out = s->s->gram_fallbacks(); });
}

int cprand_session_gather_bench(cprand_session_t s, int32_t iters, int32_t replicas, double* ms,
                                double* bytes_useful, double* bytes_min) {
  return guarded([&] {
    need(s);
    *ms = s->s->gather_bench(iters, replicas != 0, bytes_useful, bytes_min);
  });
}

int cprand_session_result(cprand_session_t s, double* out_lambda, double* const* out_factors,
                          cprand_trace_record_t* trace, int32_t trace_cap, cprand_result_t* res) {
  return guarded([&] { need(s); fill_result(*s->s, out_lambda, out_factors, trace, trace_cap, res); });
}

void cprand_session_destroy(cprand_session_t s) { delete s; }

int cprand_gather_fibers(const double* x, const int64_t* dims, int32_t order, int32_t mode,
                         const int64_t* idxs, int64_t s, double* out) {
  return guarded([&] { op_gather(x, dims_of(dims, order), mode, idxs, s, out); });
}

int cprand_skr(const int64_t* idxs, int64_t s, const int64_t* dims, int32_t order, int32_t mode,
               int64_t r, const double* const* factors, double* out) {
  return guarded([&] { op_skr(idxs, s, dims_of(dims, order), mode, static_cast<int>(r), factors, out); });
}

int cprand_mode_update(const double* x, const int64_t* dims, int32_t order, int32_t mode,
                       const int64_t* idxs, int64_t s, int64_t r, const double* const* factors,
                       double* lambda, int32_t first_of_pass, int32_t mixing_transform,
                       uint64_t mixing_seed, double* out_factor, int32_t* rank) {
  return guarded([&] {
    const int k = op_mode_update(x, dims_of(dims, order), mode, idxs, s, static_cast<int>(r), factors,
                                 lambda, first_of_pass, mixing_transform, mixing_seed, out_factor);
    if (rank) *rank = k;
  });
}

int cprand_fit_values(const double* x, const int64_t* dims, int32_t order, const int64_t* offsets,
                      int64_t n, double* out_values, double* out_norm) {
  return guarded([&] {
    const auto d = dims_of(dims, order);
    i64 p = 1;
    for (i64 v : d) p *= v;
    op_fit_values(x, p, offsets, n, out_values, out_norm);
  });
}

int cprand_estimate_fit(const double* lambda, const double* const* factors, const int64_t* dims,
                        int32_t order, int64_t r, const int64_t* idxs, const double* values,
                        int64_t phat, double x_norm, int64_t total, double* out_fit) {
  return guarded([&] {
    *out_fit = op_estimate_fit(lambda, factors, dims_of(dims, order), static_cast<int>(r), idxs, values,
                               phat, x_norm, total);
  });
}

int cprand_mix_tensor(const double* x, const int64_t* dims, int32_t order, int32_t transform,
                      uint64_t seed, double* out) {
  return guarded([&] { op_transform_tensor(x, dims_of(dims, order), transform, seed, out); });
}

int cprand_mix_factor(const double* a, int64_t rows, int64_t r, const int64_t* dims, int32_t order,
                      int32_t transform, uint64_t seed, int32_t mode, double* out) {
  return guarded([&] {
    op_transform_factor(a, rows, static_cast<int>(r), dims_of(dims, order), transform, seed, mode, 1, out);
  });
}

int cprand_unmix_factor(const double* a, int64_t rows, int64_t r, const int64_t* dims,
                        int32_t order, int32_t transform, uint64_t seed, int32_t mode, double* out) {
  return guarded([&] {
    op_transform_factor(a, rows, static_cast<int>(r), dims_of(dims, order), transform, seed, mode, 0, out);
  });
}

int cprand_unmix_rows(const double* g, int64_t s, int64_t in, const int64_t* dims, int32_t order,
                      int32_t transform, uint64_t seed, int32_t mode, double* out) {
  return guarded([&] { op_unmix_rows(g, s, in, dims_of(dims, order), transform, seed, mode, out); });
}

int cprand_debug_normal_stream(uint64_t seed, int32_t n, double* out) {
  return guarded([&] { op_debug_normals(seed, n, out); });
}

int cprand_comm_unique_id(uint8_t out[128]) {
  return guarded([&] { nccl_unique_id(out); });
}

int cprand_comm_create(const uint8_t id[128], int32_t rank, int32_t nranks, int32_t device,
                       cprand_comm_t* out) {
  return guarded([&] {
    if (nranks < 1 || rank < 0 || rank >= nranks) throw InvalidArgument("bad rank / nranks");
    auto c = std::make_unique<cprand_comm_s>();
    c->rank = rank;
    c->nranks = nranks;
    c->device = pick_device(device);
    c->comm = make_nccl_comm(id, rank, nranks, c->device);
    *out = c.release();
  });
}

int cprand_loopback_group_create(int32_t nranks, cprand_loopback_t* out) {
  return guarded([&] {
    auto g = std::make_unique<cprand_loopback_s>();
    g->g = std::make_shared<LoopbackGroup>(nranks);
    *out = g.release();
  });
}

void cprand_loopback_group_destroy(cprand_loopback_t g) { delete g; }

int cprand_comm_create_loopback(cprand_loopback_t g, int32_t rank, int32_t device, cprand_comm_t* out) {
  return guarded([&] {
    if (!g) throw InvalidArgument("null loopback group");
    auto c = std::make_unique<cprand_comm_s>();
    c->rank = rank;
    c->nranks = g->g->nranks;
    c->device = pick_device(device);
    c->comm = make_loopback_comm(g->g, rank, c->device);
    *out = c.release();
  });
}

void cprand_comm_destroy(cprand_comm_t c) { delete c; }

}  // extern "C"
