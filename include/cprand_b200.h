/* cprand_b200.h — C ABI of the B200 (sm_100a) CPRAND / CPRAND-MIX hot path.
 *
 * Drop-in boundary for the reference's C++ entry points (paths relative to
 * /root/reference/proj/include/cprand/):
 *   cprand()          sampling.hpp:257      -> cprand_solve(CPRAND_METHOD_RAND, ...)
 *   cprand_mix()      mixing.hpp:326, :340  -> cprand_solve(CPRAND_METHOD_MIX, ...)
 *   cprand_premix()   mixing.hpp:351, :372  -> cprand_solve(CPRAND_METHOD_PREMIX, ...)
 *   SolveOptions      solver.hpp:40-64      -> cprand_options_t
 *   SolveResult       solver.hpp:83-90      -> cprand_result_t + out buffers
 *   TraceRecord       solver.hpp:75-81      -> cprand_trace_record_t
 *   StopReason        solver.hpp:66-73      -> CPRAND_STOP_*
 * Operator-level entry points mirror the reference's free functions:
 *   gather_fibers     tensor.hpp:188        -> cprand_gather_fibers
 *   skr               sampling.hpp:75       -> cprand_skr
 *   sampled_update +  sampling.hpp:96,      -> cprand_mode_update (one fused
 *   normalize_columns kruskal.hpp:51           mode step, teacher-forced)
 *   make_fit_estimator sampling.hpp:155     -> cprand_fit_values
 *   estimate_fit      sampling.hpp:191      -> cprand_estimate_fit
 *   mix_tensor        mixing.hpp:131        -> cprand_mix_tensor
 *   mix_factor        mixing.hpp:160        -> cprand_mix_factor
 *   unmix_sampled_rhs mixing.hpp:219        -> cprand_unmix_rows
 *   unmix_factor      mixing.hpp:191        -> cprand_unmix_factor
 *   default_sample_count sampling.hpp:18    -> cprand_default_sample_count
 *
 * Conventions: plain pointers and sizes, no C++ or CUDA types. Matrices are
 * column-major (Eigen's default, so an Eigen::Map over the caller's storage
 * is zero-copy); tensors are generalized column-major, mode-1 fastest
 * (tensor.hpp:11-33). Index tables are int64 S x (N-1) column-major
 * (IndexTable, types.hpp:33). Every call blocks the calling thread until its
 * result is on the host, like the reference.
 *
 * Errors (the reference throws; the ABI returns a status, message in
 * cprand_last_error(), thread-local):
 *   0 ok
 *   2 std::invalid_argument / std::out_of_range   (CLI exit 2)
 *   3 numerical_consistency_error                 (CLI exit 3)
 *   4 CUDA / NCCL runtime failure
 *   5 valid for the reference but outside this path (e.g. R > 128, R > 64 with
 *     mixing or sharding, HOSVD init)
 *   1 anything else
 */
#ifndef CPRAND_B200_H
#define CPRAND_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  CPRAND_OK = 0,
  CPRAND_ERR_INTERNAL = 1,
  CPRAND_ERR_INVALID = 2,
  CPRAND_ERR_NUMERICAL = 3,
  CPRAND_ERR_CUDA = 4,
  CPRAND_ERR_UNSUPPORTED = 5
};

enum { CPRAND_METHOD_ALS = 0, CPRAND_METHOD_RAND = 1, CPRAND_METHOD_MIX = 2, CPRAND_METHOD_PREMIX = 3 };
enum {
  CPRAND_TRANSFORM_UNSET = -1,
  CPRAND_TRANSFORM_FFT = 0,
  CPRAND_TRANSFORM_DCT = 1,
  CPRAND_TRANSFORM_WHT = 2,
  CPRAND_TRANSFORM_IDENTITY = 3
};
enum { CPRAND_INIT_RANDOM = 0, CPRAND_INIT_HOSVD = 1, CPRAND_INIT_GIVEN = 2 };
enum {
  CPRAND_STOP_MAX_ITERATIONS = 0,
  CPRAND_STOP_FIT_STAGNATION = 1,
  CPRAND_STOP_FIT_THRESHOLD = 2,
  CPRAND_STOP_BEST_FIT_STALL = 3,
  CPRAND_STOP_ZERO_TENSOR = 4,
  CPRAND_STOP_BENCH_COMPLETE = 5
};

/* SolveOptions (solver.hpp:40-64); first 12 fields mirror it one to one. */
typedef struct cprand_options {
  int32_t max_iters;          /* 200 */
  double fit_tolerance;       /* 1e-4 (ALS only; validated) */
  int32_t has_fit_threshold;  /* std::optional<double> fit_threshold */
  double fit_threshold;
  uint64_t rng_seed;          /* 0 */
  int32_t init;               /* CPRAND_INIT_*; given -> init_lambda/init_factors */
  int64_t fit_sample_count;   /* 1 << 14 */
  int32_t stall_limit;        /* 10 */
  int32_t transform;          /* CPRAND_TRANSFORM_*; -1 = method default */
  int32_t bench_mode;
  int32_t exhaustive_samples; /* test hook */
  int32_t exact_fit_trace;    /* test hook */
  /* B200 extensions */
  int32_t device;             /* CUDA ordinal, -1 = current */
  int32_t x_is_device;        /* cprand_solve: x is a device pointer */
  int32_t x_mutable;          /* device x may be mixed in place (MIX/PREMIX) */
  void* comm;                 /* cprand_comm_t for slab-sharded runs, NULL = 1 GPU */
  int32_t replicas;           /* mode-major copies of strided modes: -1 auto (fit in
                                 free HBM), 0 off (gather ring), 1 on */
  int32_t fused;              /* one persistent cooperative kernel per outer
                                 iteration: -1 auto (when every mode reads its
                                 fibers in place), 0 off (multi-kernel chain) */
  int64_t shard_total;        /* with comm: global length of the last mode; x is
                                 this rank's slab, rows [rank*ceil(I/P), ...) */
  int32_t atomic_gram;        /* 0 (default): bitwise run-to-run reproducible;
                                 1: the fused CPRAND kernel sums the sampled
                                 Gram with L2 fp64 atomic adds (one inter-CTA
                                 round trip fewer per mode; the summation
                                 order, so the last bits, vary run to run) */
} cprand_options_t;

typedef struct cprand_trace_record {
  int32_t iteration;
  double elapsed_seconds;
  double fit;
  int32_t fit_is_estimate;
  double best_fit_so_far;
} cprand_trace_record_t;

typedef struct cprand_result {
  int32_t iterations;
  int32_t reason;             /* CPRAND_STOP_* */
  double setup_seconds;
  double total_seconds;
  int32_t trace_len;          /* records produced (may exceed trace_cap) */
  double loop_seconds_device; /* CUDA-event time of the outer loop */
} cprand_result_t;

void cprand_options_init(cprand_options_t* opts);
const char* cprand_last_error(void);
int cprand_device_count(void);
int64_t cprand_default_sample_count(int64_t r); /* -1 on invalid r */
const char* cprand_build_info(void);

/* One-shot drop-in solve. x: host (or device with x_is_device) tensor in
 * storage order; dims[order]. Outputs: out_lambda[r], out_factors[n] ->
 * dims[n] x r column-major (caller-allocated). trace may be NULL.
 * A page-locked host tensor (cprand_host_alloc_pinned, cudaHostAlloc or
 * cudaHostRegister) of >= 64 MB is uploaded in parts while the session sets
 * up (bench mode also builds the mode-major replicas part by part); pageable
 * memory is copied synchronously. x must stay unchanged until the call
 * returns either way. Results do not depend on the upload path. */
int cprand_solve(int32_t method, const double* x, const int64_t* dims, int32_t order, int64_t r,
                 int64_t s, const cprand_options_t* opts, const double* init_lambda,
                 const double* const* init_factors, double* out_lambda, double* const* out_factors,
                 cprand_trace_record_t* trace, int32_t trace_cap, cprand_result_t* res);

/* ---- device-resident tensors and solver sessions (bench / serving) ---- */
typedef struct cprand_tensor_s* cprand_tensor_t;
typedef struct cprand_session_s* cprand_session_t;

int cprand_tensor_create(const int64_t* dims, int32_t order, int32_t device, cprand_tensor_t* out);
int cprand_tensor_upload(cprand_tensor_t t, const double* host);
/* exact_fit (solver.hpp:161-181): 1 - ||X - M|| / ||X|| of the Kruskal model
 * (lambda[r], column-major factors I_n x r) via the mode-1 MTTKRP on the
 * device and the Gram expansion; 1 for a zero tensor. */
int cprand_tensor_exact_fit(cprand_tensor_t t, const double* lambda, const double* const* factors, int64_t r,
                            double* fit);
int cprand_exact_fit(const double* x, const int64_t* dims, int32_t order, const double* lambda,
                     const double* const* factors, int64_t r, int32_t device, double* fit);
int cprand_tensor_download(cprand_tensor_t t, double* host);
/* BASELINE.json generator in HBM: factors G_n L^T (host RNG, seeded_engine
 * (seed, 5)), lambda = 1, eta-scaled Philox Gaussian noise. out_factors
 * (nullable) receives the truth, column-major. */
int cprand_tensor_synth(cprand_tensor_t t, int64_t r, double collinearity, double eta,
                        uint64_t seed, double* const* out_factors);
double* cprand_tensor_device_ptr(cprand_tensor_t t);
/* mix_tensor (mixing.hpp:130-156) in place on a device tensor (dct): per
 * mode, sign then orthonormal DCT-II; ms_per_mode[order] (nullable) receives
 * the CUDA-event time of each mode's pass. */
int cprand_tensor_mix(cprand_tensor_t t, int32_t transform, uint64_t seed, double* ms_per_mode);
/* The passes of modes [mode_begin, mode_end) of mix_tensor only (signs drawn
 * for every mode, as the whole pass does), ms_per_mode indexed by mode. */
int cprand_tensor_mix_modes(cprand_tensor_t t, int32_t transform, uint64_t seed, int32_t mode_begin,
                            int32_t mode_end, double* ms_per_mode);
/* gather_fibers (tensor.hpp:188-212) read from a device tensor by plain
 * strided copies (no kernel): idxs S x (order-1) column-major, out I_n x S
 * column-major. For checking tensors too large to download. */
int cprand_tensor_read_fibers(cprand_tensor_t t, int32_t mode, const int64_t* idxs, int64_t s, double* out);
/* Slab of the BASELINE.json tensor with last dim shard_total (rank/nranks
 * from comm); noise scaled by the global norms (allreduced). Declared after
 * cprand_comm_t below. */
void cprand_tensor_destroy(cprand_tensor_t t);

/* Setup (init, sample tables, fit estimator, mixing pass). The session keeps
 * a reference to t; MIX/PREMIX mix t in place when opts->x_mutable, else
 * into a private copy. */
int cprand_session_create(int32_t method, cprand_tensor_t t, int64_t r, int64_t s,
                          const cprand_options_t* opts, const double* init_lambda,
                          const double* const* init_factors, cprand_session_t* out);
/* Runs up to n more outer iterations (fewer if the stop rule fires or
 * max_iters is reached) and waits for them. *ran = iterations executed. */
int cprand_session_run(cprand_session_t s, int32_t n, int32_t* ran);
/* Bench mode only: enqueues n iterations on the session stream, no wait. */
int cprand_session_enqueue(cprand_session_t s, int32_t n);
int cprand_session_sync(cprand_session_t s);
/* Bench mode: waits for queued work, then enqueues n iterations between two
 * CUDA events on the session stream and waits; *ms = event time. */
int cprand_session_timed_enqueue(cprand_session_t s, int32_t n, double* ms);
void* cprand_session_stream(cprand_session_t s); /* cudaStream_t */
/* Per-launch CUDA-event timing (on the launching stream) of the sampled-
 * fiber gather (kind 0) and the RHS GEMM (kind 1). Enable before enqueueing. */
int cprand_session_set_kernel_timing(cprand_session_t s, int32_t on);
/* Totals per mode over the timed launches since enabling: count, ms, and the
 * algorithmic work: bytes under B_min accounting (kind 0) or flops (kind 1). */
int cprand_session_kernel_stats(cprand_session_t s, int32_t mode, int32_t kind, int64_t* launches,
                                double* total_ms, double* work);
/* Fused path, timing mode: mean per-mode phase durations in microseconds
 * (z, z-barrier, phase B on CTA 0, B-barrier, apply, apply-barrier,
 * inverse completion after the Z barrier); *n = 0 when unavailable. */
int cprand_session_phase_us(cprand_session_t s, double* out, int32_t cap, int32_t* n);
/* Diagnostics: Gram solves that took the pivoted-Cholesky (min-norm) path. */
int cprand_session_gram_fallbacks(cprand_session_t s, int64_t* out);
/* 1 when the session runs one persistent kernel per outer iteration, 0 for
 * the multi-kernel chain. */
int cprand_session_fused(cprand_session_t s, int32_t* out);
/* Measurement: batched gather_fibers (tensor.hpp:188-212) of the session's
 * sample tables, iterations 1..iters x every mode, from the mode-major
 * replicas (replicas != 0) or the tensor itself; CUDA-event ms and the
 * useful / minimum-traffic bytes moved. */
int cprand_session_gather_bench(cprand_session_t s, int32_t iters, int32_t replicas, double* ms,
                                double* bytes_useful, double* bytes_min);
int cprand_session_result(cprand_session_t s, double* out_lambda, double* const* out_factors,
                          cprand_trace_record_t* trace, int32_t trace_cap, cprand_result_t* res);
void cprand_session_destroy(cprand_session_t s);

/* Page-locked host buffers (cudaHostAlloc) for fast H2D of large tensors. */
void* cprand_host_alloc_pinned(uint64_t bytes);
void cprand_host_free_pinned(void* p);

/* Tensor-sized device blocks (a solve's uploaded tensor, its mixed copy,
 * the mode-major replicas) are cached after release and reused by the next
 * solve of the same shape; this frees the cache (all devices). */
void cprand_device_cache_release(void);

/* ---- operator-level entry points (host buffers in/out) ---- */
int cprand_gather_fibers(const double* x, const int64_t* dims, int32_t order, int32_t mode,
                         const int64_t* idxs, int64_t s, double* out /* I_n x S */);
int cprand_skr(const int64_t* idxs, int64_t s, const int64_t* dims, int32_t order, int32_t mode,
               int64_t r, const double* const* factors, double* out /* S x R */);
/* One fused mode update (gather + SKR + Gram + RHS + solve + normalize)
 * from the given factors: writes the new factor (dims[mode] x r) and lambda
 * (in/out). mixing_transform >= 0 runs the MIX step (x already mixed,
 * factors unmixed; signs from seed). */
int cprand_mode_update(const double* x, const int64_t* dims, int32_t order, int32_t mode,
                       const int64_t* idxs, int64_t s, int64_t r, const double* const* factors,
                       double* lambda, int32_t first_of_pass, int32_t mixing_transform,
                       uint64_t mixing_seed, double* out_factor, int32_t* rank);
int cprand_fit_values(const double* x, const int64_t* dims, int32_t order, const int64_t* offsets,
                      int64_t n, double* out_values, double* out_norm);
int cprand_estimate_fit(const double* lambda, const double* const* factors, const int64_t* dims,
                        int32_t order, int64_t r, const int64_t* idxs /* P_hat x N */,
                        const double* values, int64_t phat, double x_norm, int64_t total,
                        double* out_fit);
int cprand_mix_tensor(const double* x, const int64_t* dims, int32_t order, int32_t transform,
                      uint64_t seed, double* out);
int cprand_mix_factor(const double* a, int64_t rows, int64_t r, const int64_t* dims, int32_t order,
                      int32_t transform, uint64_t seed, int32_t mode, double* out);
int cprand_unmix_factor(const double* a, int64_t rows, int64_t r, const int64_t* dims,
                        int32_t order, int32_t transform, uint64_t seed, int32_t mode, double* out);
/* unmix_sampled_rhs on G (S x I_n column-major) */
int cprand_unmix_rows(const double* g, int64_t s, int64_t in, const int64_t* dims, int32_t order,
                      int32_t transform, uint64_t seed, int32_t mode, double* out);
/* Device normalize-RNG self check: n normals from seeded_engine(seed, 8)
 * drawn by the device mt19937_64 + polar method. */
int cprand_debug_normal_stream(uint64_t seed, int32_t n, double* out);

/* ---- slab sharding over NCCL (one process per GPU) ----
 * The tensor is split along its last mode: rank p holds rows
 * [p*ceil(I/P), min(I, (p+1)*ceil(I/P))). Sample tables, factors and the fit
 * estimator are replicated; modes n < N-1 contract each rank's fibers and
 * allreduce the R x I_n right-hand sides, mode N-1 forms each rank's factor
 * rows, allreduces the column sums of squares and allgathers the slabs
 * (SURVEY.md §8e). Methods rand and mix with a real transform (dct, wht);
 * the DCT/WHT mixing pass exchanges slab blocks across the ranks. */
typedef struct cprand_comm_s* cprand_comm_t;
int cprand_comm_unique_id(uint8_t out[128]);
int cprand_comm_create(const uint8_t id[128], int32_t rank, int32_t nranks, int32_t device,
                       cprand_comm_t* out);
void cprand_comm_destroy(cprand_comm_t c);
/* Loopback communicators: P ranks of ONE process on one device, one host
 * thread per rank (each creates its slab tensor and session and drives it).
 * Collectives meet at host barriers and read each other's device buffers in
 * rank order. For running the sharded path where only one GPU exists (tests);
 * not a performance path. */
typedef struct cprand_loopback_s* cprand_loopback_t;
int cprand_loopback_group_create(int32_t nranks, cprand_loopback_t* out);
void cprand_loopback_group_destroy(cprand_loopback_t g);  /* after its communicators */
int cprand_comm_create_loopback(cprand_loopback_t g, int32_t rank, int32_t device, cprand_comm_t* out);
int cprand_tensor_synth_slab(cprand_tensor_t t, int64_t r, double collinearity, double eta, uint64_t seed,
                             int64_t shard_total, cprand_comm_t comm, double* const* out_factors);

#ifdef __cplusplus
}
#endif

#endif /* CPRAND_B200_H */
