// Whole-tensor mixing pass v4 (mix_tensor, mixing.hpp:130-156: every
// mode-m fiber gets sign then the orthonormal DCT-II), in place, one HBM
// read and one HBM write per element (16 B).
//
// Tiles of 2 NSEQ adjacent fibers; fiber pairs are the interleaved complex
// sequences of Makhoul's DCT (one complex FFT per pair, as in dct.cuh). The
// FFT is a four-step (two stages, n = N1 N2) or six-step (three stages,
// n = R1 R2 R3) FFT whose small DFTs run in registers:
//   * strided modes (mix_reg2_kernel, mix_reg3_kernel): the first stage's
//     threads load their points straight from global (a warp instruction
//     reads whole 256-byte rows of the tile), the results go straight back
//     in 256-byte row stores;
//   * mode 1, contiguous fibers (mix_reg2c_kernel): the tile streams into
//     shared memory with cp.async in [row][pair] order, the epilogue's lanes
//     take consecutive rows of one fiber for coalesced stores.
// Each stage reads and writes a thread's own point slots (slot k1 + N1 (n2 |
// k2) ...), so a stage needs no barrier between its reads and writes; every
// shared-memory access is consecutive in the pair index (no bank conflicts).
// Measured on B200 (tests/micro/mix_rate.py, 16 B / element): C5 (n = 320)
// 3.7 TB/s on mode 1 and 4.4-4.6 TB/s on the strided modes (v2: 2.2 / 3.2);
// n = 256: 4.2 / 5.0-5.2; C4 (n = 1000) strided 3.0 TB/s (v3: 2.2-2.3).
// Round 2: every kernel but the strided three-stage one prefetches its next
// tile into L2 while the current tile runs (one CTA per SM leaves no other
// tile to hide the DRAM latency of the loads): C5 strided modes 4.5 -> 4.8-
// 5.2 TB/s, C5 mode 1 3.7 -> 4.1; the strided three-stage kernel lost with it
// (rows 8 MB apart) and does not. Mode 1 of n = 1000 runs the three-stage FFT
// from a cp.async-staged tile (mix_reg3c_kernel: C4 mode 1 2.16 -> 3.4 TB/s).
// Rounding differs from v2 / v3 in the FFT order only (parity tests: 1e-12).
#include <algorithm>
#include <cmath>
#include <vector>

#include "dct.cuh"
#include "devutil.cuh"

namespace cpb {

namespace {

constexpr int kSeq = 16;  // complex sequences (fiber pairs) per tile: 32 fibers

__device__ __forceinline__ double2 cmulw(double2 a, double2 w) {
  return make_double2(a.x * w.x - a.y * w.y, a.x * w.y + a.y * w.x);
}

template <int N>
constexpr int first_radix() {
  if constexpr (N % 4 == 0 && N != 4 && N != 8) return 4;
  if constexpr (N % 5 == 0 && N != 5) return 5;
  if constexpr (N % 2 == 0 && N != 2) return 2;
  if constexpr (N % 3 == 0 && N != 3) return 3;
  return N;
}

// The DFT's internal twiddles W_N^j for the register DFT lengths the kernels
// use, in constant memory: with the indices compile-time constants they are
// instruction operands, not shared-memory loads (the MIO queue bounds these
// kernels). Filled once per device by init_wconst.
__constant__ double2 c_w10[10];
__constant__ double2 c_w16[16];
__constant__ double2 c_w20[20];
template <int N>
constexpr bool has_wconst() {
  return N == 10 || N == 16 || N == 20;
}
template <int N>
__device__ __forceinline__ double2 wconst(int j) {
  if constexpr (N == 10) return c_w10[j];
  else if constexpr (N == 16) return c_w16[j];
  else return c_w20[j];
}

// forward DFT of N points in registers (mixed radix, decimation in time);
// roots: the n-th roots exp(-2 pi i t / n) (shared memory, broadcast reads),
// N divides n, rs = n / N
template <int N>
__device__ __forceinline__ void dft_reg(double2 (&v)[N], const double2* roots, int rs) {
  if constexpr (N == 1) {
  } else if constexpr (N == 2 || N == 3 || N == 4 || N == 5 || N == 8) {
    dct::dft<N>(v, false);
  } else {
    constexpr int R = first_radix<N>(), M = N / R;
    double2 sub[R][M];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int m = 0; m < M; ++m) sub[r][m] = v[r + R * m];
#pragma unroll
    for (int r = 0; r < R; ++r) dft_reg<M>(sub[r], roots, rs * R);
#pragma unroll
    for (int k = 0; k < M; ++k) {
      double2 t[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (r == 0 || k == 0)
          t[r] = sub[r][k];
        else if constexpr (has_wconst<N>())
          t[r] = cmulw(sub[r][k], wconst<N>((r * k) % N));  // = roots[r k rs]
        else
          t[r] = cmulw(sub[r][k], roots[r * k * rs]);
      }
      dct::dft<R>(t, false);
#pragma unroll
      for (int u = 0; u < R; ++u) v[k + M * u] = t[u];
    }
  }
}

// Makhoul's reorder: permuted point m holds input element src(m)
__device__ __forceinline__ int makhoul_src(int m, int n) { return 2 * m < n ? 2 * m : 2 * (n - 1 - m) + 1; }

// L2 prefetch of a strided tile (n rows of w doubles at stride st): the next
// tile's DRAM reads overlap this tile's FFT stages, and its first stage then
// loads from L2 (one CTA per SM leaves no other tile to hide the latency).
// Two lines per row cover a row segment that straddles a 128-byte line.
__device__ __forceinline__ void prefetch_rows_l2(const double* base, int n, i64 st, int w, int tid, int nt) {
  for (int e = tid; e < 2 * n; e += nt) {
    const double* p = base + static_cast<i64>(e >> 1) * st + ((e & 1) ? w - 1 : 0);
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
  }
}

// Two-stage variant (four-step FFT n = N1 * N2, all points of a DFT in one
// thread's registers): stage 1 thread (q, n2) loads its N1 points from
// global, DFT_N1, twiddle W_n^(n2 k1), one store; stage 2 thread (q, k1)
// reads its N2 points, DFT_N2, one store in natural order. Fewer barriers
// and shared-memory round trips than barrier-separated radix passes
// (measured: a register Stockham pass sequence ran at 2.6-2.8 TB/s on C5's
// n = 320 against 4.5 for this kernel).
template <int N1, int N2, int NSEQ>
constexpr int two_threads() {
  return NSEQ * (N1 > N2 ? N1 : N2);
}
template <int N1, int N2, int NSEQ, int MB>
__global__ void __launch_bounds__(two_threads<N1, N2, NSEQ>(), MB)
    mix_reg2_kernel(double* __restrict__ x, i64 st, i64 tiles_per_slab, i64 ntiles, const double* __restrict__ sign,
                    const double2* __restrict__ tw, const double2* __restrict__ phase, double s0, double sk) {
  constexpr int N = N1 * N2, NT = two_threads<N1, N2, NSEQ>();
  extern __shared__ __align__(16) double2 rsm[];
  double2* buf = rsm;                // [N][NSEQ]
  double2* stw = rsm + N * NSEQ;     // [N]
  double2* sph = stw + N;            // [N]
  double* ssg = reinterpret_cast<double*>(sph + N);  // [N]
  const int tid = threadIdx.x;
  for (int e = tid; e < N; e += NT) {
    stw[e] = tw[e];
    sph[e] = phase[e];
    ssg[e] = sign[e];
  }
  __syncthreads();
  const int q = tid % NSEQ, part = tid / NSEQ;
  for (i64 t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const i64 hi = t / tiles_per_slab;
    const i64 lo0 = (t - hi * tiles_per_slab) * (2 * NSEQ);
    double* base = x + hi * st * N + lo0;
    if (t + gridDim.x < ntiles) {
      const i64 tn = t + gridDim.x, hn = tn / tiles_per_slab, ln = (tn - hn * tiles_per_slab) * (2 * NSEQ);
      prefetch_rows_l2(x + hn * st * N + ln, N, st, static_cast<int>(st - ln < 2 * NSEQ ? st - ln : 2 * NSEQ), tid,
                       NT);
    }
    // 16-byte pair loads / stores need even row offsets (st even)
    const bool full = (st & 1) == 0 && lo0 + 2 * NSEQ <= st;
    const bool lo_ok = lo0 + 2 * q < st, hi_ok = lo0 + 2 * q + 1 < st;
    if (part < N2) {  // stage 1: points n2 + N2 n1 of sequence q, DFT over n1
      const int n2 = part;
      double2 v[N1];
      if (full) {  // (the loop is duplicated so the common case issues only 16-byte loads)
#pragma unroll
        for (int n1 = 0; n1 < N1; ++n1)
          v[n1] = __ldcs(reinterpret_cast<const double2*>(base + static_cast<i64>(makhoul_src(n2 + N2 * n1, N)) * st + 2 * q));
      } else {
#pragma unroll
        for (int n1 = 0; n1 < N1; ++n1) {
          const double* p = base + static_cast<i64>(makhoul_src(n2 + N2 * n1, N)) * st + 2 * q;
          v[n1].x = lo_ok ? __ldcs(p) : 0.0;
          v[n1].y = hi_ok ? __ldcs(p + 1) : 0.0;
        }
      }
#pragma unroll
      for (int n1 = 0; n1 < N1; ++n1) {
        const double sg = ssg[makhoul_src(n2 + N2 * n1, N)];
        v[n1] = make_double2(v[n1].x * sg, v[n1].y * sg);
      }
      dft_reg<N1>(v, stw, N2);
      // slot k1 + N1 n2: stage 2's thread k1 reads its points from the slots
      // its results go to (k1 + N1 k2), so it transforms in place
#pragma unroll
      for (int k1 = 0; k1 < N1; ++k1)
        buf[(k1 + N1 * n2) * NSEQ + q] = (k1 == 0 || n2 == 0) ? v[k1] : cmulw(v[k1], stw[(n2 * k1) % N]);
    }
    __syncthreads();
    if (part < N1) {  // stage 2: for k1, the N2 points over n2, DFT over n2
      const int k1 = part;
      double2 v[N2];
#pragma unroll
      for (int n2 = 0; n2 < N2; ++n2) v[n2] = buf[(k1 + N1 * n2) * NSEQ + q];
      dft_reg<N2>(v, stw, N1);
#pragma unroll
      for (int k2 = 0; k2 < N2; ++k2) buf[(k1 + N1 * k2) * NSEQ + q] = v[k2];
    }
    __syncthreads();
    auto out = [&](int k) {  // epilogue value of row k, pair q (dct::transform_group's formulas)
      const double2 z = buf[k * NSEQ + q];
      const double2 zc = buf[((N - k) % N) * NSEQ + q];
      const double2 ph = sph[k];
      const double sc = k == 0 ? s0 : sk;
      const double ex = 0.5 * (z.x + zc.x), ey = 0.5 * (z.y - zc.y);
      const double ox = 0.5 * (z.y + zc.y), oy = -0.5 * (z.x - zc.x);
      return make_double2(sc * (ph.x * ex - ph.y * ey), sc * (ph.x * ox - ph.y * oy));
    };
    if (full) {
      for (int k = part; k < N; k += NT / NSEQ)
        __stcs(reinterpret_cast<double2*>(base + static_cast<i64>(k) * st + 2 * q), out(k));
    } else {
      for (int k = part; k < N; k += NT / NSEQ) {
        const double2 o = out(k);
        double* p = base + static_cast<i64>(k) * st + 2 * q;
        if (lo_ok) __stcs(p, o.x);
        if (hi_ok) __stcs(p + 1, o.y);
      }
    }
    __syncthreads();
  }
}

// Three-stage variant for longer fibers, n = R1 R2 R3, every stage in place:
// point slot k1 + R1 (n2 | k2) + R1 R2 (n3 | k3). Stage A thread (q, n2, n3)
// loads its R1 points from global (n = n3 + R3 n2 + R2 R3 n1), DFT_R1,
// twiddle W_n^((n3 + R3 n2) k1); stage B thread (q, k1, n3): DFT_R2 over n2,
// twiddle W_n^(R1 n3 k2); stage C thread (q, k1, k2): DFT_R3 over n3, which
// leaves natural order. One barrier per stage.
template <int R1, int R2, int R3, int NSEQ>
constexpr int three_threads() {
  constexpr int a = R2 * R3, b = R1 * R3, c = R1 * R2;
  return NSEQ * (a > b ? (a > c ? a : c) : (b > c ? b : c));
}
template <int R1, int R2, int R3, int NSEQ, int MB>
__global__ void __launch_bounds__(three_threads<R1, R2, R3, NSEQ>(), MB)
    mix_reg3_kernel(double* __restrict__ x, i64 st, i64 tiles_per_slab, i64 ntiles, const double* __restrict__ sign,
                    const double2* __restrict__ tw, const double2* __restrict__ phase, double s0, double sk) {
  constexpr int N = R1 * R2 * R3, NT = three_threads<R1, R2, R3, NSEQ>();
  extern __shared__ __align__(16) double2 rsm[];
  double2* buf = rsm;                // [N][NSEQ]
  double2* stw = rsm + N * NSEQ;     // [N]
  double2* sph = stw + N;            // [N]
  double* ssg = reinterpret_cast<double*>(sph + N);  // [N]
  const int tid = threadIdx.x;
  for (int e = tid; e < N; e += NT) {
    stw[e] = tw[e];
    sph[e] = phase[e];
    ssg[e] = sign[e];
  }
  __syncthreads();
  const int q = tid % NSEQ, part = tid / NSEQ;
  for (i64 t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const i64 hi = t / tiles_per_slab;
    const i64 lo0 = (t - hi * tiles_per_slab) * (2 * NSEQ);
    double* base = x + hi * st * N + lo0;
    // 16-byte pair loads / stores need even row offsets (st even)
    const bool full = (st & 1) == 0 && lo0 + 2 * NSEQ <= st;
    const bool lo_ok = lo0 + 2 * q < st, hi_ok = lo0 + 2 * q + 1 < st;
    if (part < R2 * R3) {  // stage A
      const int n3 = part % R3, n2 = part / R3, m0 = n3 + R3 * n2;
      double2 v[R1];
      if (full) {
#pragma unroll
        for (int n1 = 0; n1 < R1; ++n1)
          v[n1] = __ldcs(reinterpret_cast<const double2*>(
              base + static_cast<i64>(makhoul_src(m0 + R2 * R3 * n1, N)) * st + 2 * q));
      } else {
#pragma unroll
        for (int n1 = 0; n1 < R1; ++n1) {
          const double* p = base + static_cast<i64>(makhoul_src(m0 + R2 * R3 * n1, N)) * st + 2 * q;
          v[n1].x = lo_ok ? __ldcs(p) : 0.0;
          v[n1].y = hi_ok ? __ldcs(p + 1) : 0.0;
        }
      }
#pragma unroll
      for (int n1 = 0; n1 < R1; ++n1) {
        const double sg = ssg[makhoul_src(m0 + R2 * R3 * n1, N)];
        v[n1] = make_double2(v[n1].x * sg, v[n1].y * sg);
      }
      dft_reg<R1>(v, stw, N / R1);
#pragma unroll
      for (int k1 = 0; k1 < R1; ++k1)
        buf[(k1 + R1 * n2 + R1 * R2 * n3) * NSEQ + q] =
            (k1 == 0 || m0 == 0) ? v[k1] : cmulw(v[k1], stw[(m0 * k1) % N]);
    }
    __syncthreads();
    if (part < R1 * R3) {  // stage B (in place)
      const int k1 = part % R1, n3 = part / R1;
      double2 v[R2];
#pragma unroll
      for (int n2 = 0; n2 < R2; ++n2) v[n2] = buf[(k1 + R1 * n2 + R1 * R2 * n3) * NSEQ + q];
      dft_reg<R2>(v, stw, N / R2);
#pragma unroll
      for (int k2 = 0; k2 < R2; ++k2)
        buf[(k1 + R1 * k2 + R1 * R2 * n3) * NSEQ + q] =
            (k2 == 0 || n3 == 0) ? v[k2] : cmulw(v[k2], stw[(R1 * n3 * k2) % N]);
    }
    __syncthreads();
    if (part < R1 * R2) {  // stage C (in place, natural order)
      const int k1 = part % R1, k2 = part / R1;
      double2 v[R3];
#pragma unroll
      for (int n3 = 0; n3 < R3; ++n3) v[n3] = buf[(k1 + R1 * k2 + R1 * R2 * n3) * NSEQ + q];
      dft_reg<R3>(v, stw, N / R3);
#pragma unroll
      for (int k3 = 0; k3 < R3; ++k3) buf[(k1 + R1 * k2 + R1 * R2 * k3) * NSEQ + q] = v[k3];
    }
    __syncthreads();
    auto out = [&](int k) {
      const double2 z = buf[k * NSEQ + q];
      const double2 zc = buf[((N - k) % N) * NSEQ + q];
      const double2 ph = sph[k];
      const double sc = k == 0 ? s0 : sk;
      const double ex = 0.5 * (z.x + zc.x), ey = 0.5 * (z.y - zc.y);
      const double ox = 0.5 * (z.y + zc.y), oy = -0.5 * (z.x - zc.x);
      return make_double2(sc * (ph.x * ex - ph.y * ey), sc * (ph.x * ox - ph.y * oy));
    };
    if (full) {
      for (int k = part; k < N; k += NT / NSEQ)
        __stcs(reinterpret_cast<double2*>(base + static_cast<i64>(k) * st + 2 * q), out(k));
    } else {
      for (int k = part; k < N; k += NT / NSEQ) {
        const double2 o = out(k);
        double* p = base + static_cast<i64>(k) * st + 2 * q;
        if (lo_ok) __stcs(p, o.x);
        if (hi_ok) __stcs(p + 1, o.y);
      }
    }
    __syncthreads();
  }
}

template <int R1, int R2, int R3, int NSEQ, int MB>
bool launch_reg3_t(const DctPlan& pl, double* x, i64 st, i64 nfib, const double* sign, cudaStream_t stream,
                   bool prepare_only) {
  constexpr int N = R1 * R2 * R3, NT = three_threads<R1, R2, R3, NSEQ>();
  auto* fn = mix_reg3_kernel<R1, R2, R3, NSEQ, MB>;
  const size_t smem = (static_cast<size_t>(N) * NSEQ + 2 * N) * sizeof(double2) + static_cast<size_t>(N) * sizeof(double);
  static bool configured = false;
  if (!configured) {
    CPB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    configured = true;
  }
  if (prepare_only) return true;
  const i64 slabs = nfib / st;
  const i64 tps = (st + 2 * NSEQ - 1) / (2 * NSEQ);
  const i64 ntiles = slabs * tps;
  int dev = 0, sms = 148, per_sm = 1;
  CPB_CUDA(cudaGetDevice(&dev));
  CPB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CPB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, NT, smem));
  const int grid = static_cast<int>(std::min<i64>(ntiles, static_cast<i64>(std::max(per_sm, 1)) * sms));
  fn<<<grid, NT, smem, stream>>>(x, st, tps, ntiles, sign, pl.tw, pl.phase, pl.s0, pl.sk);
  CPB_LAUNCH_CHECK();
  return true;
}

// Mode 1 (contiguous fibers): the tile (2 NSEQ whole fibers, one contiguous
// block) streams into shared memory with 8-byte cp.async in a [row][pair]
// layout (row stride 2 NSEQ + 1 doubles: conflict-free), the same two
// stages run from there (rows of NSEQ + 1 points: the epilogue's k-strided
// reads are conflict-free too), and the epilogue's lanes take consecutive
// rows k, so each fiber's results go out in coalesced 256-byte stores.
template <int N1, int N2, int NSEQ, int MB, bool DB>
__global__ void __launch_bounds__(two_threads<N1, N2, NSEQ>(), MB)
    mix_reg2c_kernel(double* __restrict__ x, i64 nfib, const double* __restrict__ sign,
                     const double2* __restrict__ tw, const double2* __restrict__ phase, double s0, double sk) {
  constexpr int N = N1 * N2, NT = two_threads<N1, N2, NSEQ>(), W = 2 * NSEQ;
  constexpr int LDS = W + 1;   // staging row stride (doubles)
  constexpr int LDB = NSEQ + 1; // point-row stride of the stage buffer (double2)
  extern __shared__ __align__(16) double2 rsm[];
  constexpr int BUFD = N * LDS > 2 * N * LDB ? N * LDS : 2 * N * LDB;  // doubles
  constexpr int BUFA = (BUFD + 1) / 2 * 2;
  double* raw0 = reinterpret_cast<double*>(rsm);
  double2* stw = reinterpret_cast<double2*>(raw0 + (DB ? 2 : 1) * BUFA);
  double2* sph = stw + N;
  double* ssg = reinterpret_cast<double*>(sph + N);
  const int tid = threadIdx.x;
  for (int e = tid; e < N; e += NT) {
    stw[e] = tw[e];
    sph[e] = phase[e];
    ssg[e] = sign[e];
  }
  __syncthreads();
  const int q = tid % NSEQ, part = tid / NSEQ;
  const i64 ntiles = (nfib + W - 1) / W;
  // stream tile t in: element e = f N + i -> raw[i LDS + f]
  auto fetch = [&](i64 t, double* raw) {
    const i64 f0 = t * W;
    const int nf = static_cast<int>(nfib - f0 < W ? nfib - f0 : W);
    const double* src = x + f0 * N;
    for (int e = tid; e < W * N; e += NT) {
      const int f = e / N, i = e - f * N;
      cp_async8(raw + i * LDS + f, f < nf ? src + e : src, f < nf ? 8 : 0);
    }
  };
  int cur = 0;
  if (DB && static_cast<i64>(blockIdx.x) < ntiles) fetch(blockIdx.x, raw0);
  cp_async_commit();
  for (i64 t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const i64 f0 = t * W;
    const int nf = static_cast<int>(nfib - f0 < W ? nfib - f0 : W);
    double* raw = raw0 + (DB ? cur * BUFA : 0);
    double2* buf = reinterpret_cast<double2*>(raw);
    if constexpr (DB) {  // the next tile streams into the other buffer meanwhile
      if (t + gridDim.x < ntiles) fetch(t + gridDim.x, raw0 + (cur ^ 1) * BUFA);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      fetch(t, raw);
      cp_async_commit();
      // the next tile (one contiguous block) streams into L2 meanwhile
      if (t + gridDim.x < ntiles) {
        const i64 fn = (t + gridDim.x) * W;
        const i64 nb = (nfib - fn < W ? nfib - fn : W) * N * 8;
        const char* src = reinterpret_cast<const char*>(x + fn * N);
        for (i64 o = static_cast<i64>(tid) * 128; o < nb; o += static_cast<i64>(NT) * 128)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(src + o));
      }
      cp_async_wait<0>();
    }
    __syncthreads();
    if (part < N2) {  // stage 1
      const int n2 = part;
      double2 v[N1];
#pragma unroll
      for (int n1 = 0; n1 < N1; ++n1) {
        const int i = makhoul_src(n2 + N2 * n1, N);
        const double sg = ssg[i];
        v[n1] = make_double2(raw[i * LDS + 2 * q] * sg, raw[i * LDS + 2 * q + 1] * sg);
      }
      dft_reg<N1>(v, stw, N2);
      __syncthreads();  // every stage-1 read of the staging rows is done
#pragma unroll
      for (int k1 = 0; k1 < N1; ++k1)
        buf[(k1 + N1 * n2) * LDB + q] = (k1 == 0 || n2 == 0) ? v[k1] : cmulw(v[k1], stw[(n2 * k1) % N]);
    } else {
      __syncthreads();
    }
    __syncthreads();
    if (part < N1) {  // stage 2 (in place)
      const int k1 = part;
      double2 v[N2];
#pragma unroll
      for (int n2 = 0; n2 < N2; ++n2) v[n2] = buf[(k1 + N1 * n2) * LDB + q];
      dft_reg<N2>(v, stw, N1);
#pragma unroll
      for (int k2 = 0; k2 < N2; ++k2) buf[(k1 + N1 * k2) * LDB + q] = v[k2];
    }
    __syncthreads();
    // ---- epilogue into registers, then fiber-major into shared memory
    // epilogue: lane l of the warp group takes row k = k0 + l (consecutive
    // rows), pair q of the group; rows k and N - k from the same two points
    double* dst = x + f0 * N;
    for (int e = tid; e < NSEQ * (N / 2 + 1); e += NT) {
      const int qq = e / (N / 2 + 1), k = e - qq * (N / 2 + 1);
      const double2 z = buf[k * LDB + qq];
      const double2 zc = buf[((N - k) % N) * LDB + qq];
      auto val = [&](int kk, double2 a, double2 b) {
        const double2 ph = sph[kk];
        const double sc = kk == 0 ? s0 : sk;
        const double ex = 0.5 * (a.x + b.x), ey = 0.5 * (a.y - b.y);
        const double ox = 0.5 * (a.y + b.y), oy = -0.5 * (a.x - b.x);
        return make_double2(sc * (ph.x * ex - ph.y * ey), sc * (ph.x * ox - ph.y * oy));
      };
      const bool f_ok = 2 * qq < nf, g_ok = 2 * qq + 1 < nf;
      const double2 o = val(k, z, zc);
      if (f_ok) __stcs(dst + static_cast<i64>(2 * qq) * N + k, o.x);
      if (g_ok) __stcs(dst + static_cast<i64>(2 * qq + 1) * N + k, o.y);
      if (k != 0 && 2 * k != N) {
        const double2 o2 = val(N - k, zc, z);
        if (f_ok) __stcs(dst + static_cast<i64>(2 * qq) * N + N - k, o2.x);
        if (g_ok) __stcs(dst + static_cast<i64>(2 * qq + 1) * N + N - k, o2.y);
      }
    }
    __syncthreads();
    cur ^= 1;
  }
  cp_async_wait<0>();
}

template <int N1, int N2, int NSEQ, int MB, bool DB = false>
bool launch_reg2c_t(const DctPlan& pl, double* x, i64 nfib, const double* sign, cudaStream_t stream, bool prepare_only) {
  constexpr int N = N1 * N2, NT = two_threads<N1, N2, NSEQ>(), W = 2 * NSEQ;
  constexpr size_t bufd = std::max<size_t>(static_cast<size_t>(N) * (W + 1), 2 * static_cast<size_t>(N) * (NSEQ + 1));
  const size_t smem = (DB ? 2 : 1) * ((bufd + 1) / 2 * 2) * sizeof(double) + 2 * N * sizeof(double2) + N * sizeof(double);
  auto* fn = mix_reg2c_kernel<N1, N2, NSEQ, MB, DB>;
  static bool configured = false;
  if (!configured) {
    CPB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    configured = true;
  }
  if (prepare_only) return true;
  const i64 ntiles = (nfib + W - 1) / W;
  int dev = 0, sms = 148, per_sm = 1;
  CPB_CUDA(cudaGetDevice(&dev));
  CPB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CPB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, NT, smem));
  const int grid = static_cast<int>(std::min<i64>(ntiles, static_cast<i64>(std::max(per_sm, 1)) * sms));
  fn<<<grid, NT, smem, stream>>>(x, nfib, sign, pl.tw, pl.phase, pl.s0, pl.sk);
  CPB_LAUNCH_CHECK();
  return true;
}

// Mode 1 with the three-stage FFT (n = R1 R2 R3, e.g. C4's n = 1000): the
// tile of 2 NSEQ whole fibers streams into shared memory with 8-byte
// cp.async in the [row][pair] layout of mix_reg2c_kernel, stages A, B, C
// run as in mix_reg3_kernel on point rows of NSEQ + 1 (conflict-free
// k-strided epilogue reads), and the epilogue stores each fiber's results
// in coalesced runs. One CTA per SM (the staging / stage buffer of a
// 1000-point tile is 144 KB).
template <int R1, int R2, int R3, int NSEQ, int MB>
__global__ void __launch_bounds__(three_threads<R1, R2, R3, NSEQ>(), MB)
    mix_reg3c_kernel(double* __restrict__ x, i64 nfib, const double* __restrict__ sign,
                     const double2* __restrict__ tw, const double2* __restrict__ phase, double s0, double sk) {
  constexpr int N = R1 * R2 * R3, NT = three_threads<R1, R2, R3, NSEQ>(), W = 2 * NSEQ;
  constexpr int LDS = W + 1;    // staging row stride (doubles)
  constexpr int LDB = NSEQ + 1; // point-row stride of the stage buffer (double2)
  extern __shared__ __align__(16) double2 rsm[];
  constexpr int BUFD = N * LDS > 2 * N * LDB ? N * LDS : 2 * N * LDB;  // doubles
  constexpr int BUFA = (BUFD + 1) / 2 * 2;
  double* raw = reinterpret_cast<double*>(rsm);
  double2* buf = rsm;
  double2* stw = reinterpret_cast<double2*>(raw + BUFA);
  double2* sph = stw + N;
  double* ssg = reinterpret_cast<double*>(sph + N);
  const int tid = threadIdx.x;
  for (int e = tid; e < N; e += NT) {
    stw[e] = tw[e];
    sph[e] = phase[e];
    ssg[e] = sign[e];
  }
  const int q = tid % NSEQ, part = tid / NSEQ;
  const i64 ntiles = (nfib + W - 1) / W;
  // (measured: double-buffered 8-fiber tiles, 2.3 TB/s on n = 1000, lose to
  // one 16-fiber tile at a time, 2.9: the FFT stages, not the loads, bound it)
  for (i64 t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const i64 f0 = t * W;
    const int nf = static_cast<int>(nfib - f0 < W ? nfib - f0 : W);
    {  // element e = f N + i -> raw[i LDS + f]
      const double* src = x + f0 * N;
      for (int e = tid; e < W * N; e += NT) {
        const int f = e / N, i = e - f * N;
        cp_async8(raw + i * LDS + f, f < nf ? src + e : src, f < nf ? 8 : 0);
      }
      cp_async_commit();
      if (t + gridDim.x < ntiles) {  // the next tile streams into L2 meanwhile
        const i64 fn = (t + gridDim.x) * W;
        const i64 nb = (nfib - fn < W ? nfib - fn : W) * N * 8;
        const char* nsrc = reinterpret_cast<const char*>(x + fn * N);
        for (i64 o = static_cast<i64>(tid) * 128; o < nb; o += static_cast<i64>(NT) * 128)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(nsrc + o));
      }
      cp_async_wait<0>();
    }
    __syncthreads();
    if (part < R2 * R3) {  // stage A: points m0 + R2 R3 n1, DFT over n1
      const int n3 = part % R3, n2 = part / R3, m0 = n3 + R3 * n2;
      double2 v[R1];
      auto ld = [&](int n1) {
        const int i = makhoul_src(m0 + R2 * R3 * n1, N);
        const double sg = ssg[i];
        return make_double2(raw[i * LDS + 2 * q] * sg, raw[i * LDS + 2 * q + 1] * sg);
      };
      if constexpr (R1 % 2 == 0) {
        // points n1 < R1 / 2 sit on even staging rows, the others on odd
        // rows; odd parts take the halves in the other order, so each load
        // instruction of a warp (four parts) reads two even and two odd rows
        // (two wavefronts instead of four with row stride 2 W + 1)
        const bool odd = part & 1;
#pragma unroll
        for (int h = 0; h < R1 / 2; ++h) {
          const double2 a = ld(odd ? h + R1 / 2 : h), b2 = ld(odd ? h : h + R1 / 2);
          v[h] = odd ? b2 : a;
          v[h + R1 / 2] = odd ? a : b2;
        }
      } else {
#pragma unroll
        for (int n1 = 0; n1 < R1; ++n1) v[n1] = ld(n1);
      }
      dft_reg<R1>(v, stw, N / R1);
      __syncthreads();  // every stage-A read of the staging rows is done
#pragma unroll
      for (int k1 = 0; k1 < R1; ++k1)
        buf[(k1 + R1 * n2 + R1 * R2 * n3) * LDB + q] = (k1 == 0 || m0 == 0) ? v[k1] : cmulw(v[k1], stw[(m0 * k1) % N]);
    } else {
      __syncthreads();
    }
    __syncthreads();
    if (part < R1 * R3) {  // stage B (in place)
      const int k1 = part % R1, n3 = part / R1;
      double2 v[R2];
#pragma unroll
      for (int n2 = 0; n2 < R2; ++n2) v[n2] = buf[(k1 + R1 * n2 + R1 * R2 * n3) * LDB + q];
      dft_reg<R2>(v, stw, N / R2);
#pragma unroll
      for (int k2 = 0; k2 < R2; ++k2)
        buf[(k1 + R1 * k2 + R1 * R2 * n3) * LDB + q] = (k2 == 0 || n3 == 0) ? v[k2] : cmulw(v[k2], stw[(R1 * n3 * k2) % N]);
    }
    __syncthreads();
    if (part < R1 * R2) {  // stage C (in place, natural order)
      const int k1 = part % R1, k2 = part / R1;
      double2 v[R3];
#pragma unroll
      for (int n3 = 0; n3 < R3; ++n3) v[n3] = buf[(k1 + R1 * k2 + R1 * R2 * n3) * LDB + q];
      dft_reg<R3>(v, stw, N / R3);
#pragma unroll
      for (int k3 = 0; k3 < R3; ++k3) buf[(k1 + R1 * k2 + R1 * R2 * k3) * LDB + q] = v[k3];
    }
    __syncthreads();
    // epilogue: consecutive threads take consecutive rows k of one pair
    double* dst = x + f0 * N;
    for (int e = tid; e < NSEQ * (N / 2 + 1); e += NT) {
      const int qq = e / (N / 2 + 1), k = e - qq * (N / 2 + 1);
      const double2 z = buf[k * LDB + qq];
      const double2 zc = buf[((N - k) % N) * LDB + qq];
      auto val = [&](int kk, double2 a, double2 b) {
        const double2 ph = sph[kk];
        const double sc = kk == 0 ? s0 : sk;
        const double ex = 0.5 * (a.x + b.x), ey = 0.5 * (a.y - b.y);
        const double ox = 0.5 * (a.y + b.y), oy = -0.5 * (a.x - b.x);
        return make_double2(sc * (ph.x * ex - ph.y * ey), sc * (ph.x * ox - ph.y * oy));
      };
      const bool f_ok = 2 * qq < nf, g_ok = 2 * qq + 1 < nf;
      const double2 o = val(k, z, zc);
      if (f_ok) __stcs(dst + static_cast<i64>(2 * qq) * N + k, o.x);
      if (g_ok) __stcs(dst + static_cast<i64>(2 * qq + 1) * N + k, o.y);
      if (k != 0 && 2 * k != N) {
        const double2 o2 = val(N - k, zc, z);
        if (f_ok) __stcs(dst + static_cast<i64>(2 * qq) * N + N - k, o2.x);
        if (g_ok) __stcs(dst + static_cast<i64>(2 * qq + 1) * N + N - k, o2.y);
      }
    }
    __syncthreads();
  }
}

template <int R1, int R2, int R3, int NSEQ, int MB>
bool launch_reg3c_t(const DctPlan& pl, double* x, i64 nfib, const double* sign, cudaStream_t stream, bool prepare_only) {
  constexpr int N = R1 * R2 * R3, NT = three_threads<R1, R2, R3, NSEQ>(), W = 2 * NSEQ;
  constexpr size_t bufd = std::max<size_t>(static_cast<size_t>(N) * (W + 1), 2 * static_cast<size_t>(N) * (NSEQ + 1));
  const size_t smem = ((bufd + 1) / 2 * 2) * sizeof(double) + 2 * N * sizeof(double2) + N * sizeof(double);
  auto* fn = mix_reg3c_kernel<R1, R2, R3, NSEQ, MB>;
  static bool configured = false;
  if (!configured) {
    CPB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    configured = true;
  }
  if (prepare_only) return true;
  const i64 ntiles = (nfib + W - 1) / W;
  int dev = 0, sms = 148, per_sm = 1;
  CPB_CUDA(cudaGetDevice(&dev));
  CPB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CPB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, NT, smem));
  const int grid = static_cast<int>(std::min<i64>(ntiles, static_cast<i64>(std::max(per_sm, 1)) * sms));
  fn<<<grid, NT, smem, stream>>>(x, nfib, sign, pl.tw, pl.phase, pl.s0, pl.sk);
  CPB_LAUNCH_CHECK();
  return true;
}

template <int N1, int N2, int NSEQ, int MB>
bool launch_reg2_t(const DctPlan& pl, double* x, i64 st, i64 nfib, const double* sign, cudaStream_t stream,
                   bool prepare_only) {
  constexpr int N = N1 * N2, NT = two_threads<N1, N2, NSEQ>();
  auto* fn = mix_reg2_kernel<N1, N2, NSEQ, MB>;
  const size_t smem = (static_cast<size_t>(N) * NSEQ + 2 * N) * sizeof(double2) + static_cast<size_t>(N) * sizeof(double);
  static bool configured = false;
  if (!configured) {
    CPB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    configured = true;
  }
  if (prepare_only) return true;
  const i64 slabs = nfib / st;
  const i64 tps = (st + 2 * NSEQ - 1) / (2 * NSEQ);
  const i64 ntiles = slabs * tps;
  int dev = 0, sms = 148, per_sm = 1;
  CPB_CUDA(cudaGetDevice(&dev));
  CPB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CPB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, NT, smem));
  const int grid = static_cast<int>(std::min<i64>(ntiles, static_cast<i64>(std::max(per_sm, 1)) * sms));
  fn<<<grid, NT, smem, stream>>>(x, st, tps, ntiles, sign, pl.tw, pl.phase, pl.s0, pl.sk);
  CPB_LAUNCH_CHECK();
  return true;
}

// W_N^j = exp(-2 pi i j / N), rounded from long double as make_dct_plan rounds its tables
void init_wconst() {
  int dev = 0;
  CPB_CUDA(cudaGetDevice(&dev));
  static unsigned long long done = 0;  // devices initialized (host code runs these launches in order)
  if (dev < 64 && ((done >> dev) & 1ull)) return;
  const long double pi = 3.141592653589793238462643383279502884L;
  auto fill = [&](const void* sym, int n) {
    std::vector<double2> w(static_cast<size_t>(n));
    for (int j = 0; j < n; ++j) {
      const long double a = 2.0L * pi * static_cast<long double>(j) / static_cast<long double>(n);
      w[static_cast<size_t>(j)] = make_double2(static_cast<double>(cosl(a)), static_cast<double>(-sinl(a)));
    }
    CPB_CUDA(cudaMemcpyToSymbol(sym, w.data(), sizeof(double2) * n));
  };
  fill(c_w10, 10);
  fill(c_w16, 16);
  fill(c_w20, 20);
  if (dev < 64) done |= 1ull << dev;
}

}  // namespace

// v4 whole-tensor pass for a strided mode (st >= 32) of a supported length;
// false when the shape does not suit it.
bool launch_mix_reg(const DctPlan& pl, double* x, i64 st, i64 nfib, const double* sign, cudaStream_t stream,
                    bool prepare_only) {
  if (pl.kind != 1) return false;
  if (std::getenv("CPRAND_MIX_V2") || std::getenv("CPRAND_MIX_TMA")) return false;
  init_wconst();
  if (st == 1) {  // mode 1: contiguous fibers
    switch (pl.n) {
      case 256: return launch_reg2c_t<16, 16, 16, 2>(pl, x, nfib, sign, stream, prepare_only);
      case 320: return launch_reg2c_t<16, 20, 16, 2>(pl, x, nfib, sign, stream, prepare_only);
      case 1000: return launch_reg3c_t<10, 10, 10, 8, 1>(pl, x, nfib, sign, stream, prepare_only);
      default: return false;
    }
  }
  if (st < 2 * kSeq || nfib % st != 0) return false;
  switch (pl.n) {  // (short fibers: the v2 pass is faster, measured at n = 80)
    case 256: return launch_reg2_t<16, 16, 16, 2>(pl, x, st, nfib, sign, stream, prepare_only);
    case 320: return launch_reg2_t<16, 20, 16, 2>(pl, x, st, nfib, sign, stream, prepare_only);
    case 1000: return launch_reg3_t<10, 10, 10, 8, 1>(pl, x, st, nfib, sign, stream, prepare_only);
    default: return false;
  }
}

}  // namespace cpb
