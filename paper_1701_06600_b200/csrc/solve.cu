// sm_100a kernels of one sampled mode update (the CPRAND inner step,
// sampling.hpp:283-290; MIX variant mixing.hpp:286-298), as standalone
// launches; the phase logic lives in phases.cuh and is shared with the
// persistent per-iteration kernel (fused.cu).
//
//   z_kernel        Z_S rows (sampling.hpp:82-90), factors read A_un / norm
//   gram_kernel     split-K Z_S^T Z_S partials                 (stream s2)
//   gram_inverse    inverse of the Gram: Gauss-Jordan with a pivot test,
//                   then the QR-path factorization kernel (qr.cuh) or, where
//                   no workspace is given, a pivoted-Cholesky fallback  (s2)
//   rhs_gemm        split-K Z_S^T X_S^T partials, FP64 FMA
//   mode_apply      A_un = RHS * pinv(G), column norms, lambda rule
//                   (kruskal.hpp:51-67), zero-column refill
//
// The reference solves min ||Z_S A^T - X_S^T|| by pivoted QR
// (kr_linalg.hpp:105-118); the normal equations used here agree with it to
// ~kappa(Z_S)^2 eps, inside the 1e-10 parity bar while every Gauss-Jordan
// pivot is above kNeTol * d_max; below, the mode takes the QR path.
// Reductions run in a fixed order, so results are bitwise reproducible.
#include "phases.cuh"
#include "qr.cuh"

namespace cpb {

namespace {

constexpr int kThreads = 256;
using ph::GBK;
using ph::GBM;
using ph::GS;
using ph::GSTAGES;

template <int RT>
__global__ void __launch_bounds__(kThreads) z_kernel(ModeView v, double* __restrict__ z, const int* stop) {
  if (stop && *stop) return;
  ph::z_range<RT>(v, z, static_cast<i64>(blockIdx.x) * kThreads + threadIdx.x,
                  static_cast<i64>(gridDim.x) * kThreads);
}

template <int RT>
__global__ void __launch_bounds__(kThreads) gram_kernel(const double* __restrict__ z, int s_total, int klen,
                                                        double* __restrict__ part, const int* stop) {
  if (stop && *stop) return;
  extern __shared__ __align__(16) double sh[];  // GS x RT
  const int s0 = blockIdx.x * klen;
  ph::gram_chunk<RT>(z, s0, min(s_total, s0 + klen), part + static_cast<i64>(blockIdx.x) * RT * RT, sh);
}

constexpr int kInvThreads = 512;

template <int RT>
__global__ void __launch_bounds__(kInvThreads) gram_inverse_kernel(const double* __restrict__ part, int nparts,
                                                                   int r, double tol, double* __restrict__ ginv,
                                                                   double* __restrict__ gfull, int* info,
                                                                   const int* stop) {
  if (stop && *stop) return;
  __shared__ double sh[16 * RT + 40];
  ph::inverse_cta<RT, kInvThreads>(part, nparts, r, tol, ginv, gfull, info, sh);
}

// Rank-deficient Gram (rare): exits at once unless the inverse flagged
// failure; its matrices live in global scratch, so the launch reserves
// almost no shared memory.
template <int RT>
__global__ void __launch_bounds__(kThreads) gram_pinv_fallback_kernel(double* gfull, int r, double tol,
                                                                      double* __restrict__ ginv, int* info,
                                                                      const int* stop) {
  if (stop && *stop) return;
  if (info[0] >= 0) return;
  __shared__ int perm[RT];
  ph::pinv_fallback<RT>(gfull, r, tol, ginv, info, perm);
}

// QR path (qr.cuh): exits at once unless the inverse's pivot test failed
template <int RT>
__global__ void __launch_bounds__(kThreads) qr_fallback_kernel(const double* __restrict__ z, int s, int r,
                                                               double qtol, double* ws, double* __restrict__ ginv,
                                                               int* info, const int* stop) {
  if (stop && *stop) return;
  if (info[0] >= 0) return;
  extern __shared__ __align__(16) double qsm[];
  ph::qr_factor<RT>(z, s, r, qtol, ws, ginv, info, qsm);
}

template <int RT, bool VEC16>
__global__ void __launch_bounds__(kThreads) rhs_gemm_kernel(const double* __restrict__ xs, i64 ld,
                                                            const i64* __restrict__ row_off,
                                                            const double* __restrict__ z, i64 in, int s_total,
                                                            int r, int ks_len, double* __restrict__ part,
                                                            const int* stop) {
  if (stop && *stop) return;
  extern __shared__ __align__(16) double gsm[];
  ph::gemm_tile<RT, VEC16>(xs, ld, row_off, z, in, s_total, r, ks_len, part, blockIdx.x, blockIdx.y, gsm);
}

constexpr int kApplyThreads = 1024;
template <int RT>
constexpr int apply_gi_doubles() {
  return RT * (RT + 1) > ph::qr_rows_smem_doubles<RT, kApplyThreads>() ? RT * (RT + 1)
                                                                     : ph::qr_rows_smem_doubles<RT, kApplyThreads>();
}
template <int RT>
constexpr size_t apply_smem() {
  return static_cast<size_t>(apply_gi_doubles<RT>() + (kApplyThreads / RT) * (RT + 1)) * sizeof(double);
}

template <int RT>
__global__ void __launch_bounds__(kApplyThreads) mode_apply_kernel(i64 in, int r, ModeWork w,
                                                                   const double* __restrict__ rhs_full,
                                                                   int first_of_pass,
                                                                   unsigned long long* rng_state) {
  if (w.stop && *w.stop) return;
  constexpr int BI = kApplyThreads / RT;
  extern __shared__ __align__(16) double asm_[];
  double* gi = asm_;                       // the inverse, or the QR rows' staging (apply_gi_doubles)
  double* rh = asm_ + apply_gi_doubles<RT>();  // BI x (RT + 1)
  __shared__ bool s_last;
  // QR mode (the MIX path brings its QR rows in rhs_full, times ginv = I)
  const bool qr = w.qrws && !rhs_full && __ldcg(w.info + 2) != 0;
  if (!qr) ph::load_ginv<RT, kApplyThreads>(w.ginv, r, gi);
  __syncthreads();
  const i64 i0 = static_cast<i64>(blockIdx.x) * BI;
  const double q = qr ? ph::apply_block_qr<RT, kApplyThreads>(in, r, w, i0, rh, gi)
                      : ph::apply_block<RT, kApplyThreads>(in, r, w, rhs_full, i0, gi, rh);
  ph::ssq_store<RT, kApplyThreads>(q, r, w.ssq + static_cast<i64>(blockIdx.x) * r, rh);
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = (atomicAdd(&w.ticket[1], 1u) == gridDim.x - 1u);
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  ph::norms_final<RT, kApplyThreads>(r, in, w, gridDim.x, first_of_pass, rng_state, rh);
  if (threadIdx.x == 0) w.ticket[1] = 0u;
}

// ------------------------------------------------------- mode-n replica
// y = X_(n) stored column-major (I_n x P/I_n): for every hi-slab the
// [i_n][lo] block (I_n x st_n, lo fastest) becomes [lo][i_n] (i_n fastest),
// through 32 x 32 shared-memory tiles (coalesced reads and writes). Column j
// of the unfolding (unfold_column_index, tensor.hpp:92-106) = lo + st_n hi,
// so a sampled fiber becomes the contiguous row y + I_n * j.
// Tiles of TI = 64 tensor rows (mode-n index i) x 32 fastest-index columns:
// 8 loads of 256-byte row runs per thread in flight, 512-byte runs written.
__global__ void __launch_bounds__(256) replica_kernel(const double* __restrict__ x, i64 in, i64 st,
                                                      i64 nhi, double* __restrict__ y, i64 i0, i64 i1) {
  constexpr int TI = 64;
  __shared__ double tile[TI][33];
  const i64 tiles_lo = (st + 31) / 32, tiles_i = (i1 - i0 + TI - 1) / TI;
  const i64 per_hi = tiles_lo * tiles_i;
  const int tx = threadIdx.x % 32, ty = threadIdx.x / 32;  // 32 x 8
  for (i64 blk = blockIdx.x; blk < nhi * per_hi; blk += gridDim.x) {
    const i64 hi = blk / per_hi, rem = blk % per_hi;
    const i64 ti = rem / tiles_lo, tl = rem % tiles_lo;
    const double* src = x + hi * st * in;
    double* dst = y + hi * st * in;
    double v[TI / 8];
#pragma unroll
    for (int q = 0; q < TI / 8; ++q) {
      const i64 i = i0 + ti * TI + ty + 8 * q, lo = tl * 32 + tx;
      v[q] = (i < i1 && lo < st) ? __ldcs(src + i * st + lo) : 0.0;
    }
#pragma unroll
    for (int q = 0; q < TI / 8; ++q) tile[ty + 8 * q][tx] = v[q];
    __syncthreads();
    // column lo of the tile: TI consecutive i, written as two 32-lane runs
#pragma unroll
    for (int q = 0; q < 32 / 8; ++q) {
      const i64 lo = tl * 32 + ty + 8 * q;
#pragma unroll
      for (int h = 0; h < TI / 32; ++h) {
        const i64 i = i0 + ti * TI + 32 * h + tx;
        if (i < i1 && lo < st) __stcs(dst + lo * in + i, tile[32 * h + tx][ty + 8 * q]);
      }
    }
    __syncthreads();
  }
}

}  // namespace

// Small host -> device copy by a kernel reading mapped pinned memory over
// PCIe (Session::h2d): while a tensor upload keeps the copy engine busy, a
// cudaMemcpyAsync on another stream is not served until the upload stream
// drains (measured), and everything ordered behind it would wait with it.
template <class W>
__global__ void __launch_bounds__(256) stage_copy_kernel(const W* __restrict__ src, W* __restrict__ dst, size_t n) {
  for (size_t e = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
       e += static_cast<size_t>(gridDim.x) * blockDim.x)
    dst[e] = src[e];
}

void launch_stage_copy(void* dst, const void* src_mapped_dev, size_t bytes, cudaStream_t stream) {
  if (bytes == 0) return;
  const size_t al = reinterpret_cast<size_t>(dst) | reinterpret_cast<size_t>(src_mapped_dev) | bytes;
  const size_t w = (al % 16 == 0) ? 16 : (al % 4 == 0) ? 4 : 1;
  const size_t n = bytes / w;
  const int grid = static_cast<int>(std::min<size_t>(32, std::max<size_t>(1, (n + 255) / 256)));
  if (w == 16)
    stage_copy_kernel<uint4><<<grid, 256, 0, stream>>>(static_cast<const uint4*>(src_mapped_dev), static_cast<uint4*>(dst), n);
  else if (w == 4)
    stage_copy_kernel<unsigned><<<grid, 256, 0, stream>>>(static_cast<const unsigned*>(src_mapped_dev),
                                                          static_cast<unsigned*>(dst), n);
  else
    stage_copy_kernel<unsigned char><<<grid, 256, 0, stream>>>(static_cast<const unsigned char*>(src_mapped_dev),
                                                               static_cast<unsigned char*>(dst), n);
  CPB_LAUNCH_CHECK();
}

void launch_replica(const double* x, i64 in, i64 st, i64 p, double* y, cudaStream_t stream) {
  if (p == 0) return;  // an empty slab
  const i64 nhi = p / (st * in);
  replica_kernel<<<148 * 8, 256, 0, stream>>>(x, in, st, nhi, y, 0, in);
  CPB_LAUNCH_CHECK();
}

void launch_replica_rows(const double* x, i64 in, i64 st, i64 p, double* y, i64 i0, i64 i1, cudaStream_t stream) {
  if (p == 0 || i0 >= i1) return;
  const i64 nhi = p / (st * in);
  replica_kernel<<<148 * 8, 256, 0, stream>>>(x, in, st, nhi, y, i0, i1);
  CPB_LAUNCH_CHECK();
}

// ------------------------------------------------------------ launchers
int rank_bucket(int r) {
  if (r <= 16) return 16;
  if (r <= 32) return 32;
  if (r <= 64) return 64;
  if (r <= 128) return 128;
  throw Unsupported("rank > 128 is not supported by the sm_100a kernels");
}

void mode_splits(i64 in, int s, int rt, int* ks, int* ks_len, int sms) {
  (void)rt;
  const int mtiles = ceil_div(in, GBM);
  const int want = sms;  // ~1 CTA per SM (each holds 2 CTA slots): fewer partials for apply
  int k = ceil_div(want, mtiles);
  const int tiles = ceil_div(s, GBK);
  if (k > tiles) k = tiles;
  if (k > 64) k = 64;
  if (k < 1) k = 1;
  const int len = ceil_div(ceil_div(s, k), GBK) * GBK;
  *ks = ceil_div(s, len);
  *ks_len = len;
}

void gram_splits(int s, int* parts, int* klen) {
  // one CTA per chunk of >= GS samples, at most 32 partials for the inverse to sum
  int k = ceil_div(s, GS);
  if (k > 32) k = 32;
  if (k < 1) k = 1;
  const int len = ceil_div(ceil_div(s, k), GS) * GS;
  *parts = ceil_div(s, len);
  *klen = len;
}

template <int RT>
static void z_t(const ModeView& v, double* z, const int* stop, cudaStream_t st) {
  z_kernel<RT><<<ceil_div(static_cast<i64>(v.s) * RT, kThreads), kThreads, 0, st>>>(v, z, stop);
  CPB_LAUNCH_CHECK();
}

void launch_z(const ModeView& v, double* z, const int* stop, cudaStream_t st) {
  if (v.s <= 0) return;
  switch (rank_bucket(v.r)) {
    case 16: z_t<16>(v, z, stop, st); break;
    case 32: z_t<32>(v, z, stop, st); break;
    case 64: z_t<64>(v, z, stop, st); break;
    default: z_t<128>(v, z, stop, st); break;
  }
}

template <int RT>
static void gram_t(const double* z, int s, double* part, const int* stop, cudaStream_t st) {
  int parts, klen;
  gram_splits(s, &parts, &klen);
  const size_t sm = static_cast<size_t>(GS) * RT * sizeof(double);
  static bool configured = false;
  if (!configured) {
    CPB_CUDA(cudaFuncSetAttribute(gram_kernel<RT>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm)));
    configured = true;
  }
  gram_kernel<RT><<<parts, kThreads, sm, st>>>(z, s, klen, part, stop);
  CPB_LAUNCH_CHECK();
}

void launch_gram(const double* z, int s, int r, double* part, const int* stop, cudaStream_t st) {
  switch (rank_bucket(r)) {
    case 16: gram_t<16>(z, s, part, stop, st); break;
    case 32: gram_t<32>(z, s, part, stop, st); break;
    case 64: gram_t<64>(z, s, part, stop, st); break;
    default: gram_t<128>(z, s, part, stop, st); break;
  }
}

template <int RT>
static void inverse_t(const double* pg, int nparts, int r, double tol, double* ginv, double* gfull,
                      int* info, const int* stop, cudaStream_t st, const double* z, int s, double qtol,
                      double* qrws) {
  gram_inverse_kernel<RT><<<1, kInvThreads, 0, st>>>(pg, nparts, r, tol, ginv, gfull, info, stop);
  CPB_LAUNCH_CHECK();
  if (qrws) {
    const size_t sm = static_cast<size_t>(ph::qr_factor_smem_doubles<RT>()) * sizeof(double);
    static bool configured = false;
    if (!configured) {
      CPB_CUDA(cudaFuncSetAttribute(qr_fallback_kernel<RT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(sm)));
      configured = true;
    }
    qr_fallback_kernel<RT><<<1, kThreads, sm, st>>>(z, s, r, qtol, qrws, ginv, info, stop);
  } else {
    gram_pinv_fallback_kernel<RT><<<1, kThreads, 0, st>>>(gfull, r, tol, ginv, info, stop);
  }
  CPB_LAUNCH_CHECK();
}

void launch_gram_inverse(const double* part_gram, int nparts, int r, double tol, double* ginv,
                         double* gfull, int* info, const int* stop, cudaStream_t st, const double* z, int s,
                         double qtol, double* qrws) {
  switch (rank_bucket(r)) {
    case 16: inverse_t<16>(part_gram, nparts, r, tol, ginv, gfull, info, stop, st, z, s, qtol, qrws); break;
    case 32: inverse_t<32>(part_gram, nparts, r, tol, ginv, gfull, info, stop, st, z, s, qtol, qrws); break;
    case 64: inverse_t<64>(part_gram, nparts, r, tol, ginv, gfull, info, stop, st, z, s, qtol, qrws); break;
    default:  // (R > 64: the pivoted-Cholesky fallback; the QR path's one-CTA factorization stops at 64)
      inverse_t<128>(part_gram, nparts, r, tol, ginv, gfull, info, stop, st, z, s, qtol, nullptr);
      break;
  }
}

template <int RT, bool V>
static void gemm_t(const double* xs, i64 ld, const i64* row_off, const double* z, i64 in, int s, int r,
                   int ks, int ks_len, double* part, const int* stop, cudaStream_t st) {
  const size_t sm = static_cast<size_t>(GSTAGES * GBK * (GBM + RT)) * sizeof(double);
  static bool configured = false;
  if (!configured) {
    CPB_CUDA(cudaFuncSetAttribute(rhs_gemm_kernel<RT, V>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(sm)));
    configured = true;
  }
  rhs_gemm_kernel<RT, V><<<dim3(ceil_div(in, GBM), ks), kThreads, sm, st>>>(xs, ld, row_off, z, in, s, r,
                                                                            ks_len, part, stop);
  CPB_LAUNCH_CHECK();
}

void launch_rhs_gemm(const double* xs, i64 ld, const i64* row_off, bool vec16, const double* z, i64 in,
                     int s, int r, int ks, int ks_len, double* part, const int* stop, cudaStream_t st) {
  switch (rank_bucket(r)) {
    case 16:
      vec16 ? gemm_t<16, true>(xs, ld, row_off, z, in, s, r, ks, ks_len, part, stop, st)
            : gemm_t<16, false>(xs, ld, row_off, z, in, s, r, ks, ks_len, part, stop, st);
      break;
    case 32:
      vec16 ? gemm_t<32, true>(xs, ld, row_off, z, in, s, r, ks, ks_len, part, stop, st)
            : gemm_t<32, false>(xs, ld, row_off, z, in, s, r, ks, ks_len, part, stop, st);
      break;
    case 64:
      vec16 ? gemm_t<64, true>(xs, ld, row_off, z, in, s, r, ks, ks_len, part, stop, st)
            : gemm_t<64, false>(xs, ld, row_off, z, in, s, r, ks, ks_len, part, stop, st);
      break;
    default:
      vec16 ? gemm_t<128, true>(xs, ld, row_off, z, in, s, r, ks, ks_len, part, stop, st)
            : gemm_t<128, false>(xs, ld, row_off, z, in, s, r, ks, ks_len, part, stop, st);
      break;
  }
}

i64 gram_scratch_doubles(int r) {
  const i64 rt = rank_bucket(r);
  return static_cast<i64>(r) * r + 2 * rt * (rt + 1) + 2 * rt;
}

int apply_grid(i64 in, int r) { return ceil_div(in, kApplyThreads / rank_bucket(r)); }

template <int RT>
static void apply_t(int grid, i64 in, int r, const ModeWork& w, const double* rhs_override, int first_of_pass,
                    unsigned long long* rng_state, cudaStream_t st) {
  constexpr size_t sm = apply_smem<RT>();
  static bool configured = false;
  if (!configured) {
    CPB_CUDA(cudaFuncSetAttribute(mode_apply_kernel<RT>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm)));
    configured = true;
  }
  mode_apply_kernel<RT><<<grid, kApplyThreads, sm, st>>>(in, r, w, rhs_override, first_of_pass, rng_state);
}

void launch_mode_apply(i64 in, int r, const ModeWork& w, const double* rhs_override,
                       int first_of_pass, unsigned long long* rng_state, cudaStream_t st) {
  const int rt = rank_bucket(r);
  const int grid = ceil_div(in, kApplyThreads / rt);
  switch (rt) {
    case 16: apply_t<16>(grid, in, r, w, rhs_override, first_of_pass, rng_state, st); break;
    case 32: apply_t<32>(grid, in, r, w, rhs_override, first_of_pass, rng_state, st); break;
    case 64: apply_t<64>(grid, in, r, w, rhs_override, first_of_pass, rng_state, st); break;
    default: apply_t<128>(grid, in, r, w, rhs_override, first_of_pass, rng_state, st); break;
  }
  CPB_LAUNCH_CHECK();
}

}  // namespace cpb
