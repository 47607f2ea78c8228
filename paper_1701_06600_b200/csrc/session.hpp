// Host runtime of the B200 CPRAND path: device tensors, solver sessions.
#pragma once

#include <atomic>
#include <future>
#include <chrono>
#include <functional>
#include <memory>
#include <thread>
#include <cstdint>
#include <optional>
#include <random>
#include <vector>

#include "comm.hpp"
#include "kernels.cuh"

namespace cpb {

// rng.hpp:11-34 stream ids and seeding (identical libstdc++ engine).
constexpr std::uint64_t kInitStream = 1, kSamplingStream = 2, kFitStream = 3, kMixingStream = 4,
                        kSynthStream = 5;
std::mt19937_64 seeded_engine(std::uint64_t seed, std::uint64_t stream);
std::uint64_t seeded_engine_seed_value(std::uint64_t seed, std::uint64_t stream);

struct Options {  // SolveOptions (solver.hpp:40-64) + device extensions
  int max_iters = 200;
  double fit_tolerance = 1e-4;
  std::optional<double> fit_threshold;
  std::uint64_t rng_seed = 0;
  int init = 0;  // 0 random, 1 hosvd, 2 given
  i64 fit_sample_count = i64{1} << 14;
  int stall_limit = 10;
  int transform = -1;
  bool bench_mode = false;
  bool exhaustive_samples = false;
  bool exact_fit_trace = false;
  int device = -1;
  bool x_mutable = false;
  int replicas = -1;  // mode-major replicas for strided modes: -1 auto, 0 off, 1 on
  int fused = -1;     // persistent per-iteration kernel: -1 auto, 0 off (multi-kernel chain)
  // slab sharding: the session's tensor is this rank's slab of the last
  // mode, rows [rank * ceil(I/P), ...) of a tensor with last dim shard_total
  Comm* comm = nullptr;  // NCCL (one process per GPU) or loopback (tests)
  int nranks = 1, rank = 0;
  i64 shard_total = 0;
  bool atomic_gram = false;  // fused CPRAND kernel: Gram summed with L2 fp64 atomics (not reproducible)
  void validate() const;
};

struct Trace {
  int iteration;
  double elapsed;
  double fit;
  bool is_estimate;
  double best;
};

// Cache of tensor-sized device blocks (bigalloc.cu).
void* big_alloc(size_t bytes);
void big_free(void* p, size_t bytes);
// small pinned device-mapped host blocks, kept for reuse after release
void* pinned_mapped_alloc(size_t bytes);
void pinned_mapped_free(void* p, size_t bytes);
size_t big_cached_bytes();
void big_release_all();

struct Tensor;
// exact_fit (solver.hpp:161-181) of the model (lambda, column-major factors)
// to a device tensor: mode-1 MTTKRP on the device + the Gram expansion
double device_exact_fit(const Tensor& t, const double* lambda, const double* const* factors, int r);

struct Tensor {
  std::vector<i64> dims, strides;
  i64 p = 0;
  int device = 0;
  double* d = nullptr;
  bool owned = true;
  // a host tensor still arriving (cprand_solve uploads it in parts along the
  // last mode while the session sets up): part c covers last-mode indices
  // [chunk_end[c-1], chunk_end[c]); chunk_ev[c] is recorded behind its copy.
  // Owned by whoever filled them; empty when the tensor is resident.
  std::vector<cudaEvent_t> chunk_ev;
  std::vector<i64> chunk_end;
  // events [0, chunk_submitted) have been recorded by the uploader thread;
  // waiting on an unrecorded event would be a no-op, so consumers wait for
  // the count first
  std::atomic<int> chunk_submitted{0};
  explicit Tensor(const std::vector<i64>& dims, int device);
  ~Tensor();
};

// Host-side model in the reference layout (column-major factors).
struct HostModel {
  std::vector<double> lambda;
  std::vector<std::vector<double>> factors;  // dims[n] x R column-major
};

HostModel init_random(const std::vector<i64>& dims, int r, std::uint64_t seed);  // solver.hpp:104-123
void normalize_columns_host(HostModel& m, const std::vector<i64>& dims, int mode, bool first,
                            std::mt19937_64& rng);                                 // kruskal.hpp:51-67
std::vector<i64> sample_offsets_without_replacement(i64 total, i64 want, std::mt19937_64& rng);
std::vector<std::vector<double>> mixing_signs(const std::vector<i64>& dims, int kind,
                                              std::uint64_t seed);                // mixing.hpp:25-49
void baseline_factors_host(const std::vector<i64>& dims, int r, double c, std::uint64_t seed,
                           std::vector<std::vector<double>>& out);

// A session's small device buffers (work arrays, sample tables, kernel
// arguments: ~45 allocations) come out of 256 MB blocks that big_alloc keeps
// across sessions, so a session costs no cudaMalloc / cudaFree of its own
// (each cudaFree waits for the device: ~3 ms of a one-shot call's teardown;
// C4 one-shot call 166.1 -> 163.9 ms). Requests above 64 MB and sharded
// sessions (whose buffers are exported through CUDA IPC) use cudaMalloc;
// CPRAND_ARENA=0 turns it off. CPRAND_ARENA_POISON=1 fills every block with
// 0xFF first (a read of memory the session has not written then shows).
struct DevArena {
  struct Blk {
    char* p;
    size_t cap, used;
  };
  std::vector<Blk> blks;
  void* take(size_t bytes);
  bool owns(const void* q) const;
  void release();
  ~DevArena() { release(); }
};

class Session {
 public:
  Session(int method, Tensor* x, int r, int s, const Options& o, const double* init_lambda,
          const double* const* init_factors);
  ~Session();
  int run(int n);  // returns iterations executed
  void enqueue(int n);
  double timed_enqueue(int n);  // ms between events around n enqueued iterations
  void sync();
  cudaStream_t stream() const { return stream_; }
  void set_timing(bool on) { timing_ = on; }
  // kind 0: sampled-fiber gather (work = B_min bytes); 1: RHS GEMM (flops);
  // 2: Z_S; 3: Gram; 4: Gram inverse; 5: apply (+ MIX unmix); 6: MIX factor;
  // 7: whole fused iteration (reported under mode 0)
  void kernel_stats(int mode, int kind, i64* launches, double* ms, double* work);
  static constexpr int kKinds = 8;
  bool fused() const { return fused_; }
  void result(double* out_lambda, double* const* out_factors, std::vector<Trace>& trace,
              int* iterations, int* reason, double* setup_s, double* total_s, double* loop_dev_s);

 private:
  void setup(const double* init_lambda, const double* const* init_factors);
  void build_tables();
  // sample tables beyond the first chunk are drawn by a host thread while
  // the device iterates (sampling is data independent; one RNG stream)
  void wait_tables(int it, cudaStream_t st, int& synced);
  void stop_table_thread();
  void build_fit_estimator(const double* xsrc);
  std::vector<i64> draw_fit_offsets() const;
  std::future<std::vector<i64>> fit_offsets_;  // drawn by a host thread from setup entry
  void mix_setup();
  void cmix_setup();                          // FFT-kind MIX: complex X_hat, mixed factors
  void enqueue_mode_cmix(int it, int n, const int* stop);
  void alloc_ring();
  void enqueue_gather(int git);
  void enqueue_iteration();
  void finish_zero_tensor();
  ModeView view(int it, int n) const;
  ModeWork work(int n) const;
  const i64* base_ptr(int it, int n) const;
  const i64* dbase_ptr(int it, int n) const;
  void download_model(HostModel& m);
  void allreduce_sum(double* buf, i64 n);
  void allgather(double* buf, i64 per_rank);
  void enqueue_mode_sharded(int it, int n, const int* stop);
  void mix_last_mode_sharded();  // mode N-1 of mix_tensor across the slabs (two all-to-alls)
  void collect_kernel_times();
  cudaEvent_t timing_event();

  int method_;
  Tensor* x_;
  int order_, r_, s_;
  int rt_ = 16;
  Options o_;
  int transform_ = -1;
  bool mix_ = false, premix_ = false;
  bool cmix_ = false;
  double* rhs_gather_ = nullptr;    // sharded MIX: P * lmax rows of the last mode's RHS  // cprand_mix with the FFT kind (complex mixing, cfft.cu)
  double* xc_ = nullptr;            // complex X_hat (interleaved), P pairs
  std::vector<double*> mixedc_;     // complex mixed factors, I_n x R row-major pairs
  double* zc_ = nullptr;            // complex Z_S as stacked real [Re Z; Im Z], 2S x RT
  double* cbuf_ = nullptr;          // C = Z^H X_hat_S, I_n x R pairs
  double* cpart_ = nullptr;         // split-K partials of C
  std::vector<i64> dims_, strides_;  // global (model) shape
  i64 p_ = 0;
  std::vector<i64> tdims_, tstrides_;  // the tensor this session reads (a slab when sharded)
  i64 tp_ = 0;
  // slab sharding
  bool shard_ = false;
  Comm* comm_ = nullptr;
  int nranks_ = 1, rank_ = 0;
  i64 slab_off_ = 0, slab_len_ = 0, lmax_ = 0;
  std::vector<i64> loc_off_;   // [iter][mode] offset into loc_idx_ / loc_dbase_
  std::vector<int> loc_cnt_;   // [iter][mode] samples whose fiber lies in this slab
  int* loc_idx_ = nullptr;     // their sample indices
  i64* loc_dbase_ = nullptr;   // their row offsets in the (slab) replica
  double* zloc_ = nullptr;     // Z rows of the local samples
  double* sh_part_ = nullptr;  // mode N-1: per-CTA column sums of squares, then [R] totals
  int sms_ = 148;
  cudaStream_t stream_ = nullptr;   // s1: solve chain
  cudaStream_t stream2_ = nullptr;  // s2: Gram pseudo-inverse
  cudaStream_t gstream_ = nullptr;  // gather ring producer
  double* xsolve_ = nullptr;  // tensor the iterations gather from (mixed for MIX/PREMIX)
  double* xcopy_ = nullptr;   // private mixed copy when x is not mutable
  // model
  std::vector<double*> fac_, mixed_;
  double* lambda_ = nullptr;
  double* norms_ = nullptr;  // [N][R]
  // tables
  std::vector<int> s_mode_;         // samples per mode (S, or P/I_n when exhaustive)
  int table_iters_ = 0;
  std::thread table_thread_;
  std::atomic<int> tables_ready_{0};  // iterations whose tables are uploaded (chunk events recorded)
  std::atomic<bool> tables_stop_{false};
  int table_chunk_ = 16;
  int synced_main_ = 0, synced_g_ = 0;  // iterations each stream already waits for
  std::vector<cudaEvent_t> table_ev_;   // one per chunk
  cudaStream_t tstream_ = nullptr;
  std::unique_ptr<int[]> rows_hv_;      // host tables (async drawing)
  std::unique_ptr<i64[]> base_hv_, dbase_hv_;
  int* rows_ = nullptr;             // [iter][mode] blocks of (N-1) x S_n
  i64* base_ = nullptr;             // [iter][mode] blocks of S_n
  i64* dbase_ = nullptr;            // same layout: row offsets the GEMM reads in place
  std::vector<double*> rep_;        // per mode: mode-major replica X_(n) (or null)
  std::vector<char> direct_;        // per mode: GEMM reads fibers in place
  std::vector<char> vec16_;         // per mode: in-place rows are 16 B aligned
  void plan_replicas();
  void build_replicas();
  void wait_upload();  // stream_ waits for a tensor still arriving (Tensor::chunk_ev)
  void wait_part(size_t c);
  void launch_replicas();
  bool upload_waited_ = false;
  bool replicas_pending_ = false;
  // setup-time host -> device copies. While a tensor upload is in flight the
  // source is first copied into pinned staging memory (kept until the session
  // ends), so the call returns at once instead of blocking behind the upload
  // parts queued on the copy engine; otherwise a plain cudaMemcpyAsync.
  void h2d(void* dst, const void* src, size_t bytes, cudaStream_t st, bool always_stage = false);
  bool staging() const { return !x_->chunk_ev.empty(); }
  std::vector<std::pair<void*, size_t>> stage_blocks_;
  size_t stage_used_ = 0;
  DevArena arena_;
  std::vector<void*> trash_;  // setup-time device buffers freed with the session (cudaFree waits for the device)
  void setup_fused();
  bool fused_ = false;
  int fgrid_ = 0;
  size_t fsmem_ = 0;
  FusedIter* fargs_ = nullptr;     // [table iterations] device copies
  unsigned* fsync_ = nullptr;      // gram_done, barrier, tickets
  unsigned* lbar_ = nullptr;       // MIX kernel: per-launch grid-barrier counters [table_iters][kCS]
  unsigned* fcnt_ = nullptr;       // CPRAND kernel counters [order][tm_max + 64 + 2 + tk_max]
  int tk_max_ = 1;
  unsigned long long* cta_t_ = nullptr;  // debug per-CTA stamps (CPRAND_DEBUG_CTA)
  double* gpart_ = nullptr;        // CPRAND kernel Gram block partials
  double* gsum_ = nullptr;         // CPRAND kernel reduced Gram [RT][RT]
  // peer path (sharded CPRAND kernel exchanging through peer memory)
  bool peer_ = false;              // this session launches the peer kernel
  bool lazy_ = false;              // CPRAND kernel, bench mode: last-mode norms formed at the next launch
  int* npend_ = nullptr;           // device flag: the last launch's last-mode norms are pending
  char* parena_ = nullptr;         // receive buffer, counters, last-mode ssq partials
  std::vector<void*> parena_all_, pfac_all_;  // every rank's arena / last-mode factor
  int* perr_host_ = nullptr;       // pinned mapped: a peer wait timed out
  int* perr_dev_ = nullptr;
  std::vector<int> ploff_, plcnt_; // [iter][mode] this rank's range of the owner-ordered samples
  void check_peer_error();
  unsigned long long* phase_t_ = nullptr;  // fused phase timestamps [order][8] (timing mode)
 public:
  // fused path: mean per-mode phase durations (us) over the timed launches:
  // z, z-barrier, phaseB(gemm CTA 0), B-barrier, apply, apply-barrier, inverse-done
  std::vector<double> phase_us() const {
    std::vector<double> v = phase_acc_;
    for (auto& x : v) x /= (phase_acc_n_ ? phase_acc_n_ : 1);
    return v;
  }
  // Gram inverses that took the pivoted-Cholesky fallback so far (waits)
  long long gram_fallbacks();
  // Batched sampled-fiber gather (gather_fibers, tensor.hpp:188-212) of the
  // tables of iterations 1..iters, every mode, into scratch: from the
  // mode-major replicas (replicas = true, contiguous rows) or from the tensor
  // itself (strided modes: one 32-byte sector per element). Returns the
  // CUDA-event time (ms); bytes: useful (8 B / element) and B_min (8 B mode 1
  // or replica rows, 32 B strided).
  double gather_bench(int iters, bool replicas, double* bytes_useful, double* bytes_min);
 private:
  std::vector<double> phase_acc_;
  int phase_acc_n_ = 0;
  std::vector<i64> row_off_, base_off_;  // block offsets per (iter, mode)
  // gather ring: depth_ iterations x N modes of X_S rows
  int depth_ = 2;
  std::vector<i64> ld_;             // X_S row stride per mode
  std::vector<double*> ring_;       // [slot] = [S_n][ld_n]
  std::vector<cudaEvent_t> ev_gathered_, ev_consumed_;
  std::vector<char> slot_used_;
  int gathered_ = 0;                // last iteration whose gathers are enqueued
  int horizon_ = 0;                 // do not gather beyond this iteration
  cudaEvent_t ev_z_ = nullptr, ev_inv_ = nullptr;
  // work
  std::vector<int> ks_, ks_len_;
  double* z_ = nullptr;
  double* part_rhs_ = nullptr;
  double* part_gram_ = nullptr;
  double* ginv_ = nullptr;
  double* gfull_ = nullptr;
  double* qrws_ = nullptr;   // QR path workspace (qr.cuh)
  int* info_ = nullptr;
  unsigned* tickets_ = nullptr;
  double* ssq_ = nullptr;
  double* rhs_full_ = nullptr;
  unsigned long long* rng_state_ = nullptr;
  // fit
  bool has_fit_ = false;
  i64 phat_ = 0;
  std::vector<int*> fit_idx_;
  double* fit_vals_ = nullptr;
  double* fit_part_ = nullptr;
  FitState* state_ = nullptr;
  TraceRec* trace_dev_ = nullptr;
  int* stop_host_ = nullptr;  // pinned mapped
  int* stop_dev_ = nullptr;
  double x_norm_ = 0.0;
  // mixing
  std::vector<DctPlan> plans_;
  std::vector<double*> signs_;
  std::vector<std::vector<double>> signs_host_;
  // progress
  int it_ = 0;  // iterations enqueued
  bool finished_ = false;
  int final_reason_ = 0;
  bool zero_tensor_ = false;
  HostModel zero_model_;
  double setup_seconds_ = 0.0, mix_seconds_ = 0.0;
  std::chrono::steady_clock::time_point t0_;
  cudaEvent_t ev_loop0_ = nullptr, ev_loop1_ = nullptr;
  bool loop_started_ = false;
  std::vector<cudaEvent_t> it_events_;
  // kernel timing
  bool timing_ = false;
  struct Pending {
    int mode, kind;
    cudaEvent_t a, b;
  };
  std::vector<Pending> pending_;
  std::vector<cudaEvent_t> ev_pool_;
  std::vector<i64> k_launches_[kKinds];
  std::vector<double> k_ms_[kKinds], k_work_[kKinds];
  template <class F>
  void timed(int mode, int kind, cudaStream_t st, F&& launch);
};

// operator-level helpers (capi.cu)
void op_gather(const double* x, const std::vector<i64>& dims, int mode, const i64* idxs, i64 s,
               double* out);
void op_skr(const i64* idxs, i64 s, const std::vector<i64>& dims, int mode, int r,
            const double* const* factors, double* out);
int op_mode_update(const double* x, const std::vector<i64>& dims, int mode, const i64* idxs, i64 s,
                   int r, const double* const* factors, double* lambda, int first, int transform,
                   std::uint64_t mix_seed, double* out_factor);
void op_fit_values(const double* x, i64 p, const i64* offsets, i64 n, double* out, double* norm);
double op_estimate_fit(const double* lambda, const double* const* factors,
                       const std::vector<i64>& dims, int r, const i64* idxs, const double* values,
                       i64 phat, double x_norm, i64 total);
void op_transform_tensor(const double* x, const std::vector<i64>& dims, int transform,
                         std::uint64_t seed, double* out);
void op_transform_factor(const double* a, i64 rows, int r, const std::vector<i64>& dims,
                         int transform, std::uint64_t seed, int mode, int forward, double* out);
void op_unmix_rows(const double* g, i64 s, i64 in, const std::vector<i64>& dims, int transform,
                   std::uint64_t seed, int mode, double* out);
void op_debug_normals(std::uint64_t seed, int n, double* out);
void op_tensor_mix(Tensor* t, int transform, std::uint64_t seed, double* ms, int mode_begin = 0,
                   int mode_end = -1);
void op_read_fibers(const Tensor* t, int mode, const i64* idxs, i64 s, double* out);
void op_synth(Tensor* t, int r, double c, double eta, std::uint64_t seed, double* const* out_factors,
              i64 last_off = 0, i64 global_last = 0, const std::function<void(double*)>& reduce_sums = nullptr);

}  // namespace cpb
