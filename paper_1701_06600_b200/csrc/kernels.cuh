// Launch wrappers for the sm_100a kernels (kernels.cu, mix.cu, synth.cu).
#pragma once

#include <functional>

#include "common.cuh"

namespace cpb {

// ---- plain operators (parity / operator-level C ABI) -----------------------
// X_S (I_n x S, column-major) = fibers named by base offsets (tensor.hpp:188).
void launch_gather_fibers(const double* x, i64 in, i64 stride, const i64* base, int s,
                          double* out, cudaStream_t st);
// Z_S (S x R, column-major), ascending-mode Hadamard fold (sampling.hpp:74-92).
void launch_skr(const ModeView& v, double* out, cudaStream_t st);
// base[s] = sum_c rows[c][s] * kstride[c]  (int32 rows -> int64 offsets)
void launch_base_offsets(const int* rows, int kept, int s, const i64* kstride_host, i64* base,
                         cudaStream_t st);

// ---- per-mode update --------------------------------------------------------
// Chain per mode (stream s1 unless noted):
//   gather_rows (side stream, ahead)  X_S rows from the tensor       tensor.hpp:188
//   z                                 Z_S [S][RT]                    sampling.hpp:74
//   gram, gram_inverse (stream s2)    pinv(Z_S^T Z_S)                kr_linalg.hpp:105
//   rhs_gemm                          split-K Z_S^T X_S^T partials
//   mode_apply                        A_un = RHS * Ginv, norms, lambda kruskal.hpp:51
// Fiber source of the QR path's rows (qr.cuh): X_S(i, s) = x[(row_off ?
// row_off[s] : s * ld) + i * est].
struct QrSrc {
  const double* x;
  const i64* row_off;
  i64 ld, est;
  int s;
};

struct ModeWork {
  double* z;           // [S][RT] sampled Khatri-Rao rows (zero padded)
  double* part_gram;   // [gram_parts][RT][RT]
  int gram_parts;      // split-K partials of the Gram
  double* part_rhs;    // [ks][I_n][R]
  double* ginv;        // [R][R]
  double* gfull;       // [R][R] reduced Gram (fallback input)
  int* info;           // [0] = numerical rank of the Gram
  unsigned* ticket;    // [1] norm ticket (self-resetting)
  double* ssq;         // [grid][R] column sum-of-squares partials
  double* norms;       // [R]
  double* lambda;      // [R]
  double* a;           // I_n x R row-major factor, unnormalized (A_un; factor = A_un / norms)
  const int* stop;     // device stop flag (kernels return early when set), may be null
  int ks;              // sample splits of the RHS GEMM
  int ks_len;          // samples per split (multiple of the K tile)
  double tol;          // Gram pivot threshold (relative to the largest diagonal)
  // QR path (qr.cuh, kr_linalg.hpp:105-118): used when a Gram pivot is <= tol
  // * d_max and qrws is set; otherwise the pivoted-Cholesky min-norm fallback
  double* qrws;         // workspace (qr_ws_doubles), or null
  double qtol;          // the reference's rank threshold max(S, R) * eps
  QrSrc q;              // the sampled fibers (set per iteration)
};
// doubles of QR workspace for S samples at rank bucket rt
inline i64 qr_ws_doubles(int s, int rt) { return 2 * static_cast<i64>(s) * rt + 4 * static_cast<i64>(rt) * rt + 64; }
// Gauss-Jordan pivot ratio below which the normal equations give way to the
// QR path (normal-equation error grows like cond(Z_S)^2 eps)
constexpr double kNeTol = 1e-6;

int rank_bucket(int r);  // 16 / 32 / 64
void mode_splits(i64 in, int s, int rt, int* ks, int* ks_len, int sms);
void gram_splits(int s, int* parts, int* klen);
int apply_grid(i64 in, int r);  // CTAs of mode_apply (sizes the ssq partials)
i64 gram_scratch_doubles(int r);

void launch_gather_rows(const double* x, i64 in, i64 stride, const i64* base, int s, double* xs,
                        i64 ld, cudaStream_t st);
void launch_z(const ModeView& v, double* z, const int* stop, cudaStream_t st);
void launch_gram(const double* z, int s, int r, double* part, const int* stop, cudaStream_t st);
// gfull: gram_scratch_doubles(r) of global scratch (the reduced Gram + fallback work)
// w.qrws set: a failed pivot test runs the QR factorization of w.z (qr.cuh),
// else the pivoted-Cholesky pseudo-inverse of the Gram.
void launch_gram_inverse(const double* part_gram, int nparts, int r, double tol, double* ginv,
                         double* gfull, int* info, const int* stop, cudaStream_t st,
                         const double* z = nullptr, int s = 0, double qtol = 0.0, double* qrws = nullptr);
// A rows at xs + row_off[s] (fibers read in place) or xs + s * ld (gathered
// X_S, zero padded to ld); vec16 requires 16 B aligned row starts.
void launch_rhs_gemm(const double* xs, i64 ld, const i64* row_off, bool vec16, const double* z, i64 in,
                     int s, int r, int ks, int ks_len, double* part, const int* stop, cudaStream_t st);
// Mode-major replica y = X_(n) (column-major I_n x P/I_n) of a tensor whose
// mode n has length in and stride st.
void launch_replica(const double* x, i64 in, i64 st, i64 p, double* y, cudaStream_t stream);
// dst (16-byte aligned device memory) <- bytes of mapped pinned host memory, by a kernel (no copy engine)
void launch_stage_copy(void* dst, const void* src_mapped_dev, size_t bytes, cudaStream_t stream);
// rows [i0, i1) of the mode only (a part of the last mode's replica, whose single hi-slab is the whole tensor)
void launch_replica_rows(const double* x, i64 in, i64 st, i64 p, double* y, i64 i0, i64 i1, cudaStream_t stream);
// rhs_override != null: use it (I_n x R row-major, already reduced) instead of
// summing part_rhs (the MIX path unmixes the RHS first). Writes A_un, norms,
// lambda; zero columns refilled from the device normalize RNG.
void launch_mode_apply(i64 in, int r, const ModeWork& w, const double* rhs_override,
                       int first_of_pass, unsigned long long* rng_state, cudaStream_t st);

// ---- fit estimator ----------------------------------------------------------
void launch_gather_values(const double* x, const i64* offsets, i64 n, double* out,
                          cudaStream_t st);
// sum of squares, deterministic two-level reduction into *out
void launch_sumsq(const double* x, i64 n, double* partials, int nparts, double* out,
                  cudaStream_t st);
struct FitState {
  double best_fit;
  int stall_count;
  int stopped;
  int reason;
  int iterations;
  long long t_start_ns;
};
struct TraceRec {
  int iteration;
  int pad;
  long long t_ns;
  double fit;
  double best_fit;
};
struct FitArgs {
  int order;
  int r;
  i64 phat;
  const int* idx[kMaxOrder];     // per mode: P_hat row indices
  const double* fac[kMaxOrder];  // row-major factors (A_un)
  const double* nrm[kMaxOrder];  // column norms (factor = A_un / nrm), or null
  const double* lambda;
  const double* values;          // x at the sampled entries
  double x_norm;
  double total;                  // P as double
  double* partials;              // [blocks]
  unsigned* ticket;
  FitState* state;
  TraceRec* trace;
  int* stop_host_mapped;         // zero-copy stop marks, [iteration] = 1 where the run stopped (may be null)
  int iteration;
  int max_iters;
  int has_threshold;
  double threshold;
  int stall_limit;
  int exact;                     // 1 when values cover every entry (fit_is_estimate = 0 not implied)
};
void launch_estimate_fit(const FitArgs& a, cudaStream_t st);
void launch_stamp_start(FitState* s, cudaStream_t st);

// ---- normalize RNG (device mt19937_64 + libstdc++ polar normal) ----------
void launch_rng_seed(unsigned long long* state, unsigned long long seed_value, cudaStream_t st);
// test hook: n normals from a fresh distribution object
void launch_rng_normals(unsigned long long* state, int n, double* out, cudaStream_t st);

// ---- mixing (mix.cu, dct.cuh) -------------------------------------------
// Device-side view of a DctPlan (by value in kernel arguments).
struct DctArgs {
  int n;
  int nrad;
  int radix[24];
  const double2* tw;
  const double2* phase;
  double s0, sk;
};
struct DctPlan {
  int kind = 1;  // 1: DCT-II (tables below), 2: Walsh-Hadamard (n a power of two, no tables)
  int n = 0;
  int nrad = 0;
  int radix[24];
  double2* tw = nullptr;     // n-th roots exp(-2 pi i t / n), t < n
  double2* phase = nullptr;  // exp(-i pi k / (2n)), k < n
  double s0 = 0, sk = 0;     // orthonormal scales sqrt(1/n), sqrt(2/n)
};
DctPlan make_dct_plan(int n);  // allocates device tables
// the real orthogonal mixing transform of a kind (1 DCT-II, 2 WHT) along length n
DctPlan make_mix_plan(int kind, int n);
void free_dct_plan(DctPlan& p);
DctArgs dct_args(const DctPlan& p);
// fibers per CTA for a length-n transform within smem_budget bytes (even, >= 2)
int dct_fibers_per_cta(int n, size_t smem_budget);
// Applies sign-then-DCT-II (forward) or DCT-III-then-sign (adjoint) along a
// mode: fiber f = (hi, lo) with element i at hi*st*n + lo + i*st, f < nfib.
// in and out may alias (in place).
// col_div (nullable): fiber f's elements are divided by col_div[f] on load
// (lazily normalized factor columns).
// loads the kernel launch_mode_transform(p, x, x, st, nfib, ., forward, nullptr, .)
// would use (lazy module loading stays out of a timed region)
void prepare_mode_transform(const DctPlan& p, i64 st, i64 nfib, int forward);
void launch_mode_transform(const DctPlan& p, const double* in, double* out, i64 st, i64 nfib,
                           const double* sign, int forward, const double* col_div,
                           cudaStream_t st_);
// Whole-tensor mixing pass (mixpass.cu): persistent, pipelined, radices 2-8.
bool mix_pass_supported(const DctPlan& p);
// FFT-kind CPRAND-MIX (cfft.cu): unitary complex FFT along a mode (complex
// data as interleaved double pairs), complex Z_S from the mixed factors in
// v.fac, C = Z^H X_hat_S (I_n x R complex row-major)
void launch_cfft_mode(const DctPlan& pl, const double* in_real, const double* in_c, double* out_c, double* out_real,
                      i64 st, i64 nfib, const double* sign, int forward, const double* col_div, cudaStream_t stream);
// complex Z_S as the stacked real matrix [Re Z; Im Z] (2S x rt)
void launch_zc(const ModeView& v, int rt, double* zs, cudaStream_t stream);
// C = Z^H X_hat_S: split-K partials (<= rhsc_splits(in, s, sms) x I_n x R
// complex, in part) reduced in split order into out
int rhsc_splits(i64 in, int s, int sms);
void launch_rhsc(const double* xh, const i64* base, i64 st, i64 in, int s, const double* zs, int rt, int r,
                 double* part, double* out, int sms, cudaStream_t stream);
// TMA-fed forward pass (mixtma.cu); false when the shape does not suit it
bool launch_mix_tma(const DctPlan& p, double* x, i64 st, i64 nfib, const double* sign, cudaStream_t stream,
                    bool prepare_only);
// register four-step pass (mixreg.cu) for strided modes; false when the shape does not suit it
bool launch_mix_reg(const DctPlan& p, double* x, i64 st, i64 nfib, const double* sign, cudaStream_t stream,
                    bool prepare_only);
// prepare_only: load and configure the kernel the call would launch, no launch
void launch_mix_pass(const DctPlan& p, const double* in, double* out, i64 st, i64 nfib, const double* sign,
                     int forward, cudaStream_t stream, bool prepare_only = false);
// MIX path: RHS (I_n x R row-major) = D_n C^T (sum_ks part_rhs) per column
void launch_reduce_rhs(const double* part_rhs, int ks, i64 in, int r, double* out,
                       cudaStream_t st);
// the same, or (QR mode, w.info[2] set by the fallback) the QR solution rows
void launch_reduce_rhs_qr(const ModeWork& w, i64 in, int r, double* out, cudaStream_t st);

// ---- slab sharding (shard.cu) ---------------------------------------------
void launch_gather_z_rows(const double* z, const int* idx, int cnt, int rt, double* out, cudaStream_t st);
// slab [M][L] <-> P row blocks packed back to back (distributed last-mode mixing)
void launch_slab_blocks(double* x, double* buf, i64 m, i64 l, i64 mb, int pack, cudaStream_t st);
int apply_rows_grid(i64 rows, int r);
void launch_apply_rows(i64 rows, int r, const double* rhs, const double* ginv, double* a_out, double* ssq_part,
                       cudaStream_t st);
void launch_col_ssq(const double* part, int nparts, int r, double* out, cudaStream_t st);
void launch_norms_from_ssq(const double* ssq, int r, i64 rows, double* a, double* norms, double* lambda,
                           int first_of_pass, unsigned long long* rng_state, cudaStream_t st);
// out[j] = x[loc[j]], or 0 where loc[j] < 0 (entry outside this slab)
void launch_gather_values_masked(const double* x, const i64* loc, i64 n, double* out, cudaStream_t st);

// ---- synthetic generator (synth.cu) ------------------------------------
void launch_synth(double* x, int order, const i64* dims, int r, const double* const* fac_dev,
                  double eta, unsigned long long seed, double* scratch, cudaStream_t st, i64 last_off = 0,
                  i64 global_last = 0, const std::function<void(double*)>& reduce_sums = nullptr);

// ---- persistent per-iteration kernel (fused.cu) -------------------------
// One cooperative launch per outer iteration runs every mode update and the
// fit: grid barriers separate Z -> (Gram + inverse on one CTA, GEMM on the
// rest) -> apply (+ norms on the last CTA) -> next mode. Used when every
// mode reads its fibers in place (mode 1 / replicas).
struct FusedMode {
  ModeView v;            // x / base: in-place fiber source and row offsets
  int vec16;
  i64 est;               // MIX kernel: element stride of the fibers (1: mode 1 / replica)
  int mtiles, ks, ks_len;
  int gparts, gklen;
  double tol;
  double qtol;           // QR path rank threshold max(S, R) * eps
  double* a;             // A_un of this mode
  double* norms;         // its column norms
  double* mixed;         // MIX: mixed image of the factor
  const double* sign;    // MIX: D_n
  DctArgs plan;          // MIX: DCT plan of I_n
  int dctF;              // MIX: fibers per CTA in the transform
  int tail1;             // MIX: one CTA runs unmix -> apply -> norms -> mix (small I_n x R)
  // CPRAND kernel (fused_rand_kernel): 64-row x tklen-sample tiles
  int tm, tk, tklen;     // row blocks, sample splits, samples per split
  int nblk;              // upper 8 x 8 Gram blocks
  int zcap;              // Z rows the tile's shared memory holds
  unsigned* mt_cnt;      // [tm] splits finished per row block                      (stride kCS)
  unsigned* kb_cnt;      // [tk] CTAs that wrote their share of split kb's Z rows   (stride kCS)
  unsigned* gm_cnt;      // [tm] splits whose Gram blocks of row block mt are written  (stride kCS)
  int dist_gram;         // 1: tile (mt, tk-1) sums row block mt's Gram blocks (one tile per CTA)
  unsigned* grdy;        // [kRep] replicas of the "Gram inverse ready" flag      (stride kCS)
  unsigned* adone;       // [kRep] replicas: tile CTAs whose factor rows are written (epoch count)
  unsigned* gdone;       // [kRep] replicas: Gram blocks summed (dist_gram)
  unsigned* nready;      // [kRep] replicas: this mode's norms / lambda are formed (epoch count)
  i64 in_full;           // rows of the whole factor (a sharded last mode: I_N, not the slab)
  // peer path (slab-sharded CPRAND kernel, np > 1), modes n < N-1: the
  // sample list is ordered by owner rank (the same order on every rank), so
  // this rank's fibers are the contiguous range [loff, loff + lcnt); the RHS
  // tiles cut it into tk local splits of tkllen samples
  int loff, lcnt, tkllen;
  unsigned* mcnt;        // [0] Gram blocks summed (or tiles written), [1] inverse ready,
                         // [2] tile CTAs whose sums of squares are written        (stride kCS)
};
// Inter-CTA counters live one per 128-byte line (atomics and polling on a
// shared line serialize): kCS words apart.
constexpr int kCS = 32;
constexpr int kRep = 16;  // replicas of widely polled flags
constexpr int kMaxPeer = 8;  // ranks of the peer path
constexpr int kSyncWords = 3 * kCS + 128 * kCS + kRep * kCS;  // gram_done, barrier, tickets, group tickets, gen replicas
struct FusedIter;
struct FusedIter {
  int order, r, first_mode_first_of_pass;
  FusedMode mode[kMaxOrder];
  double *z, *part_gram, *ginv, *gfull, *part_rhs, *ssq, *rhs_full, *lambda;
  double *gpart, *gsum;
  double* qrws;          // QR path workspace (qr.cuh), or null  // CPRAND kernel: Gram block partials [nblk][tk][64], reduced Gram [RT][RT]
  int* info;
  unsigned long long* rng;
  unsigned* ticket;      // [0] norm ticket, [1] fit ticket
  unsigned* gram_done;
  unsigned* bar;         // [0] count, [1] generation
  unsigned* lbar;        // MIX kernel: this launch's own grid-barrier arrival counter (zeroed once)
  const int* stop;
  int has_fit;
  // CPRAND kernel, bench mode (no fit): the last mode's norms are formed at
  // the next launch's mode 0 (or by fused_finish before the model is read):
  // mode 0's Z_S reads the last factor unnormalized, like every mode n >= 1
  // reads mode n-1's. npend: device flag "the last launch's norms are pending".
  int lazy_last;
  int* npend;
  int grid;  // CTAs of the persistent launch (the finishing kernel's ssq layout)
  FitArgs fit;
  unsigned long long* phase_t;  // optional: CTA 0 stamps globaltimer at phase edges [order][16]
  // CPRAND kernel roles: the Gram-inverse CTA and an idle CTA sharing its SM
  // (-1: none), chosen from a census launch (census != null: every CTA writes
  // its SM id to census[blockIdx] and returns).
  int inv_cta, idle_cta;
  int* census;
  unsigned* grp_cnt;             // CPRAND kernel: ssq group tickets [grid / 16] (stride kCS)
  const FusedIter* next;         // next iteration's arguments (L2 prefetch of its tables)
  unsigned* gen_rep;             // CPRAND kernel: [kRep] replicas of the mode-release generation
  unsigned seq;                  // CPRAND kernel: 1-based launch sequence (epoch of adone / nready)
  int gram_first;                // CPRAND kernel: RHS tiles wait for the summed Gram
  int gram_atomic;               // CPRAND kernel: tiles add their Gram blocks into gsum[n & 1] (L2 fp64 adds)
  unsigned long long* cta_t;  // debug: per-CTA stamps of mode 1 [grid][16] (CPRAND_DEBUG_CTA)
  // ---- peer path: the slab-sharded CPRAND kernel exchanging through peer
  // memory (NVLink P2P stores of CUDA-IPC-mapped buffers, one process per
  // GPU; or P rank groups of one launch on one device in the tests).
  // Pointers [q] are rank q's buffers as this rank addresses them.
  int np, prank;                 // ranks, this rank (np = 1: no exchange)
  double* precv[kMaxPeer];       // rank q's RHS receive buffer [np][rcv_ld] (block p from rank p)
  unsigned* prcnt[kMaxPeer];     // rank q's per-(mode, tile) arrival counters [order][ptiles] (stride kCS)
  double* pfac[kMaxPeer];        // rank q's last-mode factor A_un [I_N][r]
  double* pssq[kMaxPeer];        // rank q's last-mode column sums of squares [np][Gw][r]
  unsigned* pdone[kMaxPeer];     // rank q's last-mode apply counter replicas [kRep] (stride kCS)
  i64 rcv_ld;                    // doubles per sender block of precv
  int ptiles;                    // tile slots per mode in prcnt
  unsigned lastw;                // last-mode apply signals per launch, all ranks (sum of Gw)
  i64 slab_off;                  // first row of this rank's slab in the last mode
  int* perr;                     // set when a peer wait timed out (the host raises)
};
// One launch of the CPRAND kernel: `groups` rank groups of gridDim.x / groups
// CTAs, group g running a[g] (groups > 1: the peer path's one-device test
// harness; production launches one group per GPU).
struct FusedLaunch {
  const FusedIter* a[kMaxPeer];
  int groups;
};
size_t fused_smem_bytes(int rt, bool mix, int max_dim);
// CPRAND kernel: Z rows per tile, its dynamic shared memory, and the tiling
// of one mode over gw tile CTAs.
int fused_rand_zcap(int rt);
size_t fused_rand_smem(int rt, int zcap);
void fused_rand_tiles(i64 in, int s, int gw, int zcap, int* tm, int* tk, int* tklen);
// Largest co-resident grid for the fused kernel (0 when cooperative launch
// is unavailable).
int fused_max_grid(int rt, bool mix, size_t smem, int device);
void launch_fused_iteration(const FusedIter* dev_args, int rt, bool mix, int grid, size_t smem,
                            cudaStream_t st, bool gram_atomic = false);
// lazy_last: form the last launch's pending last-mode norms (one CTA)
void launch_fused_finish(const FusedIter* dev_args, int rt, cudaStream_t st);
// The peer path's CPRAND kernel (grid = groups x group size).
void launch_fused_peer(const FusedLaunch& l, int rt, int grid, size_t smem, cudaStream_t st, bool mix = false);

}  // namespace cpb
