// sm_100a kernels for the CPRAND hot path: sampled-fiber gather, fused
// SKR + Gram + RHS, pivoted Gram inverse, row solve + column norms,
// normalization (incl. the device normalize RNG), and the sampled fit.
//
// Reference behaviour (paths under /root/reference/proj/include/cprand/):
//   gather_fibers  tensor.hpp:188-212      skr            sampling.hpp:74-92
//   least_squares  kr_linalg.hpp:105-118   normalize      kruskal.hpp:51-67
//   estimate_fit   sampling.hpp:191-210    should_stop    sampling.hpp:237-251
// Bit-exactness: gathers and Z_S copy / multiply in the reference's order
// (no FMA can form: pure products), so they match the oracle bit for bit.
// Solves use the normal equations (Gram + pivoted Cholesky), which agree
// with the reference's pivoted-QR solve to ~kappa(Z)^2 eps (1e-10 bar).
#include <cfloat>
#include <cstdio>

#include "kernels.cuh"

namespace cpb {

namespace {

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// ------------------------------------------------------------- gather
__global__ void gather_fibers_kernel(const double* __restrict__ x, i64 in, i64 stride,
                                     const i64* __restrict__ base, int s,
                                     double* __restrict__ out) {
  // one CTA per sample column, threads over the fiber
  const int col = blockIdx.x;
  if (col >= s) return;
  const i64 b = base[col];
  for (i64 i = threadIdx.x; i < in; i += blockDim.x) out[col * in + i] = x[b + i * stride];
}

__global__ void base_offsets_kernel(const int* __restrict__ rows, int kept, int s,
                                    i64 k0, i64 k1, i64 k2, i64 k3, i64 k4, i64 k5, i64 k6,
                                    i64* __restrict__ base) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= s) return;
  const i64 ks[7] = {k0, k1, k2, k3, k4, k5, k6};
  i64 b = 0;
  for (int c = 0; c < kept; ++c) b += static_cast<i64>(rows[c * s + j]) * ks[c];
  base[j] = b;
}

// Z(s, r): ones, then *= factor rows in ascending kept mode (sampling.hpp:82-90).
__device__ __forceinline__ double skr_entry(const ModeView& v, int s, int r) {
  double z = 1.0;
  for (int c = 0; c < v.kept; ++c) z = __dmul_rn(z, v.fac[c][static_cast<i64>(v.rows[c][s]) * v.r + r]);
  return z;
}

__global__ void skr_kernel(ModeView v, double* __restrict__ out) {
  const i64 e = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= static_cast<i64>(v.s) * v.r) return;
  const int s = static_cast<int>(e % v.s), r = static_cast<int>(e / v.s);
  out[e] = skr_entry(v, s, r);  // column-major S x R
}

constexpr int kThreads = 256;

// Pivoted Cholesky of the R x R Gram in shared memory (warp 0), then its
// (pseudo-)inverse. g: [RT][RT+1]; w: [RT][RT+1] scratch. On exit ginv
// (global, R x R row-major) holds pinv(G) and info[0] the numerical rank.
template <int RT>
__device__ void gram_pinv(double* g, double* w, int* perm, int r, double tol, double* ginv,
                          int* info) {
  constexpr int LD = RT + 1;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  __shared__ int s_rank;
  if (warp == 0) {
    for (int t = lane; t < RT; t += 32) perm[t] = t;
    __syncwarp();
    int rank = r;
    double d0 = 0.0;
    for (int k = 0; k < r; ++k) {
      double bv = -1.0;
      int bj = RT;
      for (int j = lane; j < r; j += 32)
        if (j >= k) {
          const double dv = g[j * LD + j];
          if (dv > bv || (dv == bv && j < bj)) {
            bv = dv;
            bj = j;
          }
        }
      for (int off = 16; off > 0; off >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, off);
        const int oj = __shfl_xor_sync(0xffffffffu, bj, off);
        if (ov > bv || (ov == bv && oj < bj)) {
          bv = ov;
          bj = oj;
        }
      }
      if (k == 0) d0 = bv;
      if (!(bv > tol * d0) || !(bv > 0.0)) {
        rank = k;
        break;
      }
      const int p = bj;
      if (p != k) {
        for (int t = lane; t < r; t += 32) {
          const double a = g[k * LD + t];
          g[k * LD + t] = g[p * LD + t];
          g[p * LD + t] = a;
        }
        __syncwarp();
        for (int t = lane; t < r; t += 32) {
          const double a = g[t * LD + k];
          g[t * LD + k] = g[t * LD + p];
          g[t * LD + p] = a;
        }
        if (lane == 0) {
          const int q = perm[k];
          perm[k] = perm[p];
          perm[p] = q;
        }
        __syncwarp();
      }
      const double lkk = sqrt(g[k * LD + k]);
      __syncwarp();
      for (int t = lane; t < r; t += 32)
        if (t > k) g[t * LD + k] = g[t * LD + k] / lkk;
      __syncwarp();
      if (lane == 0) g[k * LD + k] = lkk;
      __syncwarp();
      for (int j = lane; j < r; j += 32)
        if (j > k) {
          const double ljk = g[j * LD + k];
          for (int i = k + 1; i < r; ++i) g[i * LD + j] -= g[i * LD + k] * ljk;
        }
      __syncwarp();
    }
    if (lane == 0) s_rank = rank;
  }
  __syncthreads();
  const int rank = s_rank;
  // w <- inverse of the leading rank x rank lower factor L (column j per thread)
  for (int j = tid; j < rank; j += blockDim.x) {
    for (int i = 0; i < rank; ++i) {
      if (i < j) {
        w[i * LD + j] = 0.0;
        continue;
      }
      double sacc = (i == j) ? 1.0 : 0.0;
      for (int m = j; m < i; ++m) sacc -= g[i * LD + m] * w[m * LD + j];
      w[i * LD + j] = sacc / g[i * LD + i];
    }
  }
  __syncthreads();
  if (rank == r) {
    // pinv = P L^-T L^-1 P^T
    for (int e = tid; e < r * r; e += blockDim.x) {
      const int a = e / r, b = e % r;
      const int lo = a > b ? a : b;
      double sacc = 0.0;
      for (int m = lo; m < r; ++m) sacc += w[m * LD + a] * w[m * LD + b];
      ginv[perm[a] * r + perm[b]] = sacc;
    }
  } else {
    // rank-deficient: G ~= M M^T, M = P L[:, :k]; pinv = B B^T with
    // B = M (M^T M)^{-1}. Rare path, single thread.
    if (tid == 0) {
      const int k = rank;
      // C = L1^T L1 (k x k) over all r rows of the factored columns, into w
      for (int a = 0; a < k; ++a)
        for (int b = 0; b <= a; ++b) {
          double sacc = 0.0;
          for (int m = a; m < r; ++m) sacc += g[m * LD + a] * g[m * LD + b];
          w[a * LD + b] = sacc;
          w[b * LD + a] = sacc;
        }
      // Cholesky of C in place (lower), into w
      for (int j = 0; j < k; ++j) {
        double d = w[j * LD + j];
        for (int m = 0; m < j; ++m) d -= w[j * LD + m] * w[j * LD + m];
        d = sqrt(d > 0.0 ? d : DBL_MIN);
        w[j * LD + j] = d;
        for (int i = j + 1; i < k; ++i) {
          double sacc = w[i * LD + j];
          for (int m = 0; m < j; ++m) sacc -= w[i * LD + m] * w[j * LD + m];
          w[i * LD + j] = sacc / d;
        }
      }
      for (int e = 0; e < r * r; ++e) ginv[e] = 0.0;
      // rows of B: b_t = C^{-1} m_t with m_t = row t of L1 (k entries);
      // scratch vectors live in shared memory right after w
      double* bt = w + RT * LD;
      double* bu = bt + RT;
      for (int t = 0; t < r; ++t) {
        for (int a = 0; a < k; ++a) bt[a] = (t >= a) ? g[t * LD + a] : 0.0;
        for (int a = 0; a < k; ++a) {
          double sacc = bt[a];
          for (int m = 0; m < a; ++m) sacc -= w[a * LD + m] * bt[m];
          bt[a] = sacc / w[a * LD + a];
        }
        for (int a = k - 1; a >= 0; --a) {
          double sacc = bt[a];
          for (int m = a + 1; m < k; ++m) sacc -= w[m * LD + a] * bt[m];
          bt[a] = sacc / w[a * LD + a];
        }
        for (int u = 0; u <= t; ++u) {
          for (int a = 0; a < k; ++a) bu[a] = (u >= a) ? g[u * LD + a] : 0.0;
          for (int a = 0; a < k; ++a) {
            double sacc = bu[a];
            for (int m = 0; m < a; ++m) sacc -= w[a * LD + m] * bu[m];
            bu[a] = sacc / w[a * LD + a];
          }
          for (int a = k - 1; a >= 0; --a) {
            double sacc = bu[a];
            for (int m = a + 1; m < k; ++m) sacc -= w[m * LD + a] * bu[m];
            bu[a] = sacc / w[a * LD + a];
          }
          double dot = 0.0;
          for (int a = 0; a < k; ++a) dot += bt[a] * bu[a];
          ginv[perm[t] * r + perm[u]] = dot;
          ginv[perm[u] * r + perm[t]] = dot;
        }
      }
    }
  }
  if (tid == 0) info[0] = rank;
}

// ---------------------------------------------- Z_S + Gram partials
// One CTA per SB samples: Z rows (ones, then *= factor rows in ascending
// mode, sampling.hpp:82-90) written to a dense [S][RT] buffer (zero padded
// for r >= R) and Z_tile^T Z_tile accumulated into a per-CTA Gram partial.
// Loads are issued mode by mode for all of a thread's entries at once so the
// index -> factor-row dependency costs two load latencies per mode, not two
// per entry.
constexpr int SB = 64;

template <int RT>
__global__ void __launch_bounds__(kThreads) skr_gram_kernel(ModeView v, double* __restrict__ z,
                                                            double* __restrict__ part_gram,
                                                            const int* stop) {
  if (stop && *stop) return;
  constexpr int Q = SB * RT / kThreads;  // entries per thread
  constexpr int GP = RT * RT / kThreads;
  __shared__ double zt[SB][RT];
  const int tid = threadIdx.x;
  const int s0 = blockIdx.x * SB;
  double zv[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) zv[q] = 1.0;
  for (int c = 0; c < v.kept; ++c) {
    int row[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const int e = tid + q * kThreads, s = s0 + e / RT;
      row[q] = (s < v.s) ? __ldg(v.rows[c] + s) : 0;
    }
    double f[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const int e = tid + q * kThreads, rr = e % RT;
      f[q] = (rr < v.r) ? __ldg(v.fac[c] + static_cast<i64>(row[q]) * v.r + rr) : 0.0;
    }
#pragma unroll
    for (int q = 0; q < Q; ++q) zv[q] = __dmul_rn(zv[q], f[q]);
  }
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int e = tid + q * kThreads, sl = e / RT, rr = e % RT, s = s0 + sl;
    const double val = (s < v.s && rr < v.r) ? zv[q] : 0.0;
    zt[sl][rr] = val;
    if (s < v.s) z[static_cast<i64>(s) * RT + rr] = val;
  }
  __syncthreads();
  double g[GP];
#pragma unroll
  for (int q = 0; q < GP; ++q) g[q] = 0.0;
  for (int sl = 0; sl < SB; ++sl) {
#pragma unroll
    for (int q = 0; q < GP; ++q) {
      const int e = tid + q * kThreads;
      g[q] = fma(zt[sl][e / RT], zt[sl][e % RT], g[q]);
    }
  }
  double* pg = part_gram + static_cast<i64>(blockIdx.x) * RT * RT;
#pragma unroll
  for (int q = 0; q < GP; ++q) pg[tid + q * kThreads] = g[q];
}

// ---------------------------------------------- Gram pseudo-inverse
// One CTA: G = sum of the Gram partials (fixed order); in-place
// Gauss-Jordan inversion (SPD, no pivoting) with every pivot checked against
// tol * max diag; a failed check (numerical rank < R) falls back to the
// pivoted Cholesky pseudo-inverse (gram_pinv).
template <int RT>
__global__ void __launch_bounds__(kThreads) gram_inverse_kernel(const double* __restrict__ part_gram,
                                                                int nparts, int r, double tol,
                                                                double* __restrict__ ginv, int* info,
                                                                const int* stop) {
  if (stop && *stop) return;
  constexpr int LD = RT + 1;
  extern __shared__ __align__(16) double sm[];
  double* a = sm;             // working copy [RT][LD]
  double* g0 = sm + RT * LD;  // original G (for the fallback)
  double* wk = g0 + RT * LD;  // fallback scratch [RT][LD] + 2 RT
  __shared__ double col[RT], rowk[RT];
  __shared__ int perm[RT];
  __shared__ int s_fail;
  __shared__ double s_dmax;
  const int tid = threadIdx.x;
  for (int e = tid; e < r * r; e += blockDim.x) {
    const int i = e / r, j = e % r;
    double s = 0.0;
    for (int k = 0; k < nparts; ++k) s += part_gram[static_cast<i64>(k) * RT * RT + i * RT + j];
    a[i * LD + j] = s;
    g0[i * LD + j] = s;
  }
  if (tid == 0) s_fail = 0;
  __syncthreads();
  if (tid == 0) {
    double d = 0.0;
    for (int i = 0; i < r; ++i) d = fmax(d, a[i * LD + i]);
    s_dmax = d;
  }
  __syncthreads();
  const double thr = tol * s_dmax;
  for (int k = 0; k < r; ++k) {
    const double piv = a[k * LD + k];
    if (!(piv > thr) || !(piv > 0.0)) {
      if (tid == 0) s_fail = 1;
      break;  // uniform: every thread reads the same pivot
    }
    const double p = 1.0 / piv;
    for (int i = tid; i < r; i += blockDim.x) {
      col[i] = a[i * LD + k];
      rowk[i] = (i == k) ? p : a[k * LD + i] * p;
    }
    __syncthreads();
    for (int e = tid; e < r * r; e += blockDim.x) {
      const int i = e / r, j = e % r;
      double v;
      if (i == k) v = rowk[j];
      else if (j == k) v = -col[i] * p;
      else v = a[i * LD + j] - col[i] * rowk[j];
      a[i * LD + j] = v;
    }
    __syncthreads();
  }
  __syncthreads();
  if (!s_fail) {
    for (int e = tid; e < r * r; e += blockDim.x) ginv[e] = a[(e / r) * LD + (e % r)];
    if (tid == 0) info[0] = r;
    return;
  }
  // rank-deficient (or numerically so): pivoted Cholesky pseudo-inverse
  for (int e = tid; e < RT * LD; e += blockDim.x) a[e] = (e % LD < r && e / LD < r) ? g0[e] : 0.0;
  __syncthreads();
  gram_pinv<RT>(a, wk, perm, r, tol, ginv, info);
}

// ---------------------------------------------- sampled-fiber gather
// X_S rows (one per sample, the fiber contiguous, ld >= I_n) straight from
// the tensor: coalesced along i for mode 1, one 32 B sector per element for
// strided modes. Streaming loads (evict-first) keep the random tensor
// traffic from displacing the X_S ring in L2. Pure copies: bit-exact.
constexpr int kGatherThreads = 256;
constexpr int kGatherUnroll = 4;

__global__ void __launch_bounds__(kGatherThreads) gather_rows_kernel(
    const double* __restrict__ x, i64 in, i64 stride, const i64* __restrict__ base, int s,
    double* __restrict__ xs, i64 ld) {
  const int row = blockIdx.y;
  const i64 b = base[row];
  const double* src = x + b;
  double* dst = xs + static_cast<i64>(row) * ld;
  for (i64 i0 = static_cast<i64>(blockIdx.x) * kGatherThreads * kGatherUnroll + threadIdx.x; i0 < in;
       i0 += static_cast<i64>(gridDim.x) * kGatherThreads * kGatherUnroll) {
    double v[kGatherUnroll];
#pragma unroll
    for (int u = 0; u < kGatherUnroll; ++u) {
      const i64 i = i0 + u * kGatherThreads;
      v[u] = (i < in) ? __ldcs(src + i * stride) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kGatherUnroll; ++u) {
      const i64 i = i0 + u * kGatherThreads;
      if (i < in) dst[i] = v[u];
    }
  }
}

// ---------------------------------------------- RHS GEMM (split-K)
// part[kb](i, r) = sum_{s in split kb} X_S(s, i) Z(s, r): M = I_n, N = R
// (padded RT), K = S. CTA tile 64 x RT x 16, two-stage cp.async pipeline,
// 4 x RT/16 register tile per thread, FP64 FMA. Deterministic: fixed
// per-thread accumulation order, splits reduced in order by mode_apply.
constexpr int GBM = 64;
constexpr int GBK = 16;

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc, int src_bytes) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(gsrc), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

template <int RT>
__global__ void __launch_bounds__(kThreads) rhs_gemm_kernel(const double* __restrict__ xs, i64 ld,
                                                            const double* __restrict__ z, i64 in,
                                                            int s_total, int r, int ks_len,
                                                            double* __restrict__ part,
                                                            const int* stop) {
  if (stop && *stop) return;
  constexpr int TN = RT / 16, TM = GBM / 16;
  __shared__ __align__(16) double as[2][GBK][GBM];
  __shared__ __align__(16) double bs[2][GBK][RT];
  const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
  const i64 i0 = static_cast<i64>(blockIdx.x) * GBM;
  const int kb = blockIdx.y;
  const int s_begin = kb * ks_len;
  const int s_end = min(s_total, s_begin + ks_len);
  const int ntiles = (s_end - s_begin + GBK - 1) / GBK;

  auto load_tile = [&](int t, int buf) {
    const int sbase = s_begin + t * GBK;
    // A: GBK rows x 64 doubles = 512 chunks of 16 B (2 per thread)
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int c = tid + q * kThreads;
      const int sl = c / 32, ic = (c % 32) * 2;
      const int s = sbase + sl;
      const i64 i = i0 + ic;
      const bool ok = (s < s_end) && (i < ld);
      const double* src = ok ? xs + static_cast<i64>(s) * ld + i : xs;
      cp_async16(&as[buf][sl][ic], src, ok ? 16 : 0);
    }
    // B: GBK rows x RT doubles = GBK*RT/2 chunks
    for (int c = tid; c < GBK * RT / 2; c += kThreads) {
      const int sl = c / (RT / 2), rc = (c % (RT / 2)) * 2;
      const int s = sbase + sl;
      const bool ok = s < s_end;
      const double* src = ok ? z + static_cast<i64>(s) * RT + rc : z;
      cp_async16(&bs[buf][sl][rc], src, ok ? 16 : 0);
    }
    cp_async_commit();
  };

  double acc[TM][TN];
#pragma unroll
  for (int a = 0; a < TM; ++a)
#pragma unroll
    for (int b = 0; b < TN; ++b) acc[a][b] = 0.0;

  if (ntiles > 0) load_tile(0, 0);
  for (int t = 0; t < ntiles; ++t) {
    const int buf = t & 1;
    if (t + 1 < ntiles) {
      load_tile(t + 1, buf ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < GBK; ++kk) {
      double af[TM], bf[TN];
#pragma unroll
      for (int a = 0; a < TM; ++a) af[a] = as[buf][kk][ty * TM + a];
#pragma unroll
      for (int b = 0; b < TN; ++b) bf[b] = bs[buf][kk][tx * TN + b];
#pragma unroll
      for (int a = 0; a < TM; ++a)
#pragma unroll
        for (int b = 0; b < TN; ++b) acc[a][b] = fma(af[a], bf[b], acc[a][b]);
    }
    __syncthreads();
  }
  double* pr = part + static_cast<i64>(kb) * in * r;
#pragma unroll
  for (int a = 0; a < TM; ++a) {
    const i64 i = i0 + ty * TM + a;
    if (i >= in) continue;
#pragma unroll
    for (int b = 0; b < TN; ++b) {
      const int rr = tx * TN + b;
      if (rr < r) pr[i * r + rr] = acc[a][b];
    }
  }
}

// A_un(i, :) = (sum_ks part_rhs(ks, i, :)) * Ginv; column sum-of-squares
// partials; the last CTA forms the norms and the lambda update.
constexpr int BI = 16;  // rows per CTA

template <int RT>
__global__ void __launch_bounds__(kThreads) mode_apply_kernel(i64 in, int r, ModeWork w,
                                                              const double* __restrict__ rhs_full,
                                                              int first_of_pass) {
  if (w.stop && *w.stop) return;
  constexpr int TN = RT / 16;
  __shared__ double gi[RT][RT + 1];
  __shared__ double rh[BI][RT + 1];
  __shared__ bool s_last;
  auto& red = rh;  // reused after the products are formed
  const int tid = threadIdx.x;
  const i64 i0 = static_cast<i64>(blockIdx.x) * BI;
  for (int e = tid; e < RT * RT; e += kThreads) {
    const int a = e / RT, b = e % RT;
    gi[a][b] = (a < r && b < r) ? w.ginv[a * r + b] : 0.0;
  }
  for (int e = tid; e < BI * RT; e += kThreads) {
    const int il = e / RT, c = e % RT;
    const i64 i = i0 + il;
    double sacc = 0.0;
    if (i < in && c < r) {
      if (rhs_full) {
        sacc = rhs_full[i * r + c];
      } else {
        for (int k = 0; k < w.ks; ++k) sacc += w.part_rhs[(static_cast<i64>(k) * in + i) * r + c];
      }
    }
    rh[il][c] = sacc;
  }
  __syncthreads();
  const int il = tid / 16, tx = tid % 16;
  const i64 i = i0 + il;
  double out[TN];
#pragma unroll
  for (int b = 0; b < TN; ++b) out[b] = 0.0;
  for (int c = 0; c < r; ++c) {
    const double rv = rh[il][c];
#pragma unroll
    for (int b = 0; b < TN; ++b) out[b] = fma(rv, gi[c][tx * TN + b], out[b]);
  }
  __syncthreads();
#pragma unroll
  for (int b = 0; b < TN; ++b) {
    const int cc = tx * TN + b;
    const bool ok = (i < in && cc < r);
    if (ok) w.a[i * r + cc] = out[b];
    red[il][cc] = ok ? out[b] * out[b] : 0.0;
  }
  __syncthreads();
  if (tid < RT) {
    double sacc = 0.0;
    for (int q = 0; q < BI; ++q) sacc += red[q][tid];
    if (tid < r) w.ssq[static_cast<i64>(blockIdx.x) * r + tid] = sacc;
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    const unsigned t = atomicAdd(&w.ticket[1], 1u);
    s_last = (t == gridDim.x - 1u);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (tid < r) {
    double sacc = 0.0;
    for (unsigned b = 0; b < gridDim.x; ++b) sacc += w.ssq[static_cast<i64>(b) * r + tid];
    const double nrm = sqrt(sacc);
    w.norms[tid] = nrm;
    // kruskal.hpp:57-66: zero column -> lambda 0 (refilled by normalize)
    w.lambda[tid] = (nrm == 0.0) ? 0.0 : (first_of_pass ? w.lambda[tid] * nrm : nrm);
  }
  if (tid == 0) w.ticket[1] = 0u;
}

// ---------------------------------------------- device normalize RNG
// std::mt19937_64 (state words 0..311, index in word 312) and the libstdc++
// Marsaglia-polar normal_distribution (random.tcc:1811-1844), one fresh
// distribution object per call, as kruskal.hpp:53 constructs it.
struct DevMt {
  unsigned long long* s;
  __device__ void seed(unsigned long long v) {
    s[0] = v;
    for (int i = 1; i < 312; ++i) s[i] = 6364136223846793005ULL * (s[i - 1] ^ (s[i - 1] >> 62)) + i;
    s[312] = 312;
  }
  __device__ unsigned long long next() {
    unsigned long long idx = s[312];
    if (idx >= 312) {
      const unsigned long long um = 0xFFFFFFFF80000000ULL, lm = 0x7FFFFFFFULL;
      for (int i = 0; i < 312; ++i) {
        const unsigned long long y = (s[i] & um) | (s[(i + 1) % 312] & lm);
        unsigned long long xa = y >> 1;
        if (y & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
        s[i] = s[(i + 156) % 312] ^ xa;
      }
      idx = 0;
    }
    unsigned long long z = s[idx];
    s[312] = idx + 1;
    z ^= (z >> 29) & 0x5555555555555555ULL;
    z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
    z ^= (z << 37) & 0xFFF7EEE000000000ULL;
    z ^= (z >> 43);
    return z;
  }
  __device__ double canonical() {  // generate_canonical<double, 53>
    double v = __dmul_rn(__ull2double_rn(next()), 0x1.0p-64);
    if (v >= 1.0) v = 0x1.fffffffffffffp-1;
    return v;
  }
};

struct DevNormal {
  bool saved_ok = false;
  double saved = 0.0;
  __device__ double operator()(DevMt& g) {
    if (saved_ok) {
      saved_ok = false;
      return saved;
    }
    double x, y, r2;
    do {
      x = __dsub_rn(__dmul_rn(2.0, g.canonical()), 1.0);
      y = __dsub_rn(__dmul_rn(2.0, g.canonical()), 1.0);
      r2 = __dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y));
    } while (r2 > 1.0 || r2 == 0.0);
    const double mult = sqrt(__ddiv_rn(__dmul_rn(-2.0, log(r2)), r2));
    saved = __dmul_rn(x, mult);
    saved_ok = true;
    return __dmul_rn(y, mult);
  }
};

__device__ double dev_stable_norm(const double* v, i64 n, i64 inc) {
  double scale = 0.0, ssq = 1.0;
  for (i64 i = 0; i < n; ++i) {
    const double a = fabs(v[i * inc]);
    if (a != 0.0) {
      if (scale < a) {
        const double q = scale / a;
        ssq = 1.0 + ssq * q * q;
        scale = a;
      } else {
        const double q = a / scale;
        ssq += q * q;
      }
    }
  }
  return scale * sqrt(ssq);
}

__global__ void rng_seed_kernel(unsigned long long* state, unsigned long long v) {
  DevMt g{state};
  g.seed(v);
}

__global__ void rng_normals_kernel(unsigned long long* state, int n, double* out) {
  DevMt g{state};
  DevNormal d;
  for (int i = 0; i < n; ++i) out[i] = d(g);
}

__global__ void normalize_kernel(double* __restrict__ a, i64 in, int r,
                                 const double* __restrict__ norms, const int* stop,
                                 unsigned long long* rng_state) {
  if (stop && *stop) return;
  const i64 e = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e < in * r) {
    const int c = static_cast<int>(e % r);
    const double nv = norms[c];
    if (nv != 0.0) a[e] = a[e] / nv;  // true division, as Eigen's col /= norm
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    bool any = false;
    for (int c = 0; c < r; ++c) any |= (norms[c] == 0.0);
    if (!any) return;
    // kruskal.hpp:57-63, columns in order, one distribution per call
    DevMt g{rng_state};
    DevNormal gauss;
    for (int c = 0; c < r; ++c) {
      if (norms[c] != 0.0) continue;
      for (i64 i = 0; i < in; ++i) a[i * r + c] = gauss(g);
      const double fn = dev_stable_norm(a + c, in, r);
      for (i64 i = 0; i < in; ++i) a[i * r + c] = a[i * r + c] / fn;
    }
  }
}

// ------------------------------------------------------------ fit
__global__ void gather_values_kernel(const double* __restrict__ x, const i64* __restrict__ off,
                                     i64 n, double* __restrict__ out) {
  const i64 j = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j < n) out[j] = x[off[j]];
}

__global__ void sumsq_partial_kernel(const double* __restrict__ x, i64 n, double* partials) {
  __shared__ double red[kThreads];
  double acc = 0.0;
  const i64 per = (n + gridDim.x - 1) / gridDim.x;
  const i64 lo = per * blockIdx.x, hi = min(n, lo + per);
  // vectorized main body when 16 B aligned
  i64 i = lo + threadIdx.x;
  for (; i < hi; i += blockDim.x) {
    const double v = x[i];
    acc = fma(v, v, acc);
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s = kThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) partials[blockIdx.x] = red[0];
}

__global__ void sum_partials_kernel(const double* partials, int n, double* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += partials[i];
    *out = s;
  }
}

__global__ void stamp_start_kernel(FitState* s) {
  s->t_start_ns = static_cast<long long>(globaltimer());
}

__global__ void __launch_bounds__(kThreads) estimate_fit_kernel(FitArgs a) {
  if (a.state->stopped) return;
  __shared__ double red[kThreads];
  __shared__ bool s_last;
  const i64 j = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  double e2 = 0.0;
  if (j < a.phat) {
    double sum = 0.0;
    // model_entry (kruskal.hpp:37-44): lambda_r * prod_n A_n(i_n, r), summed over r
    for (int q = 0; q < a.r; ++q) {
      double p = a.lambda[q];
      for (int n = 0; n < a.order; ++n)
        p = __dmul_rn(p, a.fac[n][static_cast<i64>(a.idx[n][j]) * a.r + q]);
      sum = __dadd_rn(sum, p);
    }
    const double e = a.values[j] - sum;
    e2 = e * e;
  }
  red[threadIdx.x] = e2;
  __syncthreads();
  for (int s = kThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    a.partials[blockIdx.x] = red[0];
    __threadfence();
    const unsigned t = atomicAdd(a.ticket, 1u);
    s_last = (t == gridDim.x - 1u);
  }
  __syncthreads();
  if (!s_last || threadIdx.x != 0) return;
  __threadfence();
  double sq = 0.0;
  for (unsigned b = 0; b < gridDim.x; ++b) sq += a.partials[b];
  *a.ticket = 0u;
  // sampling.hpp:192, :207-209
  double fit;
  if (a.x_norm == 0.0) {
    fit = 1.0;
  } else {
    const double mu = sq / static_cast<double>(a.phat);
    fit = 1.0 - sqrt(a.total * mu) / a.x_norm;
  }
  // should_stop (sampling.hpp:237-251)
  FitState* st = a.state;
  if (fit > st->best_fit) {
    st->best_fit = fit;
    st->stall_count = 0;
  } else {
    st->stall_count += 1;
  }
  int stop = 0, reason = 0;
  if (a.has_threshold && fit >= a.threshold) {
    stop = 1;
    reason = 2;  // fit_threshold
  } else if (st->stall_count >= a.stall_limit) {
    stop = 1;
    reason = 3;  // best_fit_stall
  } else if (a.iteration >= a.max_iters) {
    stop = 1;
    reason = 0;  // max_iterations
  }
  st->iterations = a.iteration;
  TraceRec& tr = a.trace[a.iteration - 1];
  tr.iteration = a.iteration;
  tr.t_ns = static_cast<long long>(globaltimer()) - st->t_start_ns;
  tr.fit = fit;
  tr.best_fit = st->best_fit;
  if (stop) {
    st->reason = reason;
    __threadfence_system();
    st->stopped = 1;
    if (a.stop_host_mapped) *reinterpret_cast<volatile int*>(a.stop_host_mapped) = 1;
  }
}

}  // namespace

// ---------------------------------------------------------------- launchers
void launch_gather_fibers(const double* x, i64 in, i64 stride, const i64* base, int s,
                          double* out, cudaStream_t st) {
  if (s <= 0) return;
  const int threads = in >= 256 ? 256 : (in >= 64 ? 128 : 32);
  gather_fibers_kernel<<<s, threads, 0, st>>>(x, in, stride, base, s, out);
  CPB_LAUNCH_CHECK();
}

void launch_skr(const ModeView& v, double* out, cudaStream_t st) {
  const i64 n = static_cast<i64>(v.s) * v.r;
  if (n == 0) return;
  skr_kernel<<<ceil_div(n, 256), 256, 0, st>>>(v, out);
  CPB_LAUNCH_CHECK();
}

void launch_base_offsets(const int* rows, int kept, int s, const i64* ks, i64* base,
                         cudaStream_t st) {
  if (kept > 7) throw Unsupported("base_offsets: order > 8");
  i64 k[7] = {0, 0, 0, 0, 0, 0, 0};
  for (int c = 0; c < kept; ++c) k[c] = ks[c];
  base_offsets_kernel<<<ceil_div(s, 256), 256, 0, st>>>(rows, kept, s, k[0], k[1], k[2], k[3],
                                                        k[4], k[5], k[6], base);
  CPB_LAUNCH_CHECK();
}

int rank_bucket(int r) {
  if (r <= 16) return 16;
  if (r <= 32) return 32;
  if (r <= 64) return 64;
  throw Unsupported("rank > 64 is not supported by the fused sm_100a kernels");
}

void mode_splits(i64 in, int s, int rt, int* ks, int* ks_len, int sms) {
  (void)rt;
  const int mtiles = ceil_div(in, GBM);
  const int want = 2 * sms;  // ~2 CTAs per SM
  int k = ceil_div(want, mtiles);
  const int tiles = ceil_div(s, GBK);
  if (k > tiles) k = tiles;
  if (k > 64) k = 64;
  if (k < 1) k = 1;
  const int len = ceil_div(ceil_div(s, k), GBK) * GBK;
  *ks = ceil_div(s, len);
  *ks_len = len;
}

int skr_gram_parts(int s) { return ceil_div(s, SB); }

template <int RT>
static void skr_gram_t(const ModeView& v, double* z, double* pg, const int* stop, cudaStream_t st) {
  skr_gram_kernel<RT><<<ceil_div(v.s, SB), kThreads, 0, st>>>(v, z, pg, stop);
  CPB_LAUNCH_CHECK();
}

void launch_skr_gram(const ModeView& v, double* z, double* part_gram, const int* stop,
                     cudaStream_t st) {
  switch (rank_bucket(v.r)) {
    case 16: skr_gram_t<16>(v, z, part_gram, stop, st); break;
    case 32: skr_gram_t<32>(v, z, part_gram, stop, st); break;
    default: skr_gram_t<64>(v, z, part_gram, stop, st); break;
  }
}

template <int RT>
static void gram_inverse_t(const double* pg, int nparts, int r, double tol, double* ginv, int* info,
                           const int* stop, cudaStream_t st) {
  const size_t sm = static_cast<size_t>(3 * RT * (RT + 1) + 2 * RT) * sizeof(double);
  static bool configured = false;
  if (!configured) {
    CPB_CUDA(cudaFuncSetAttribute(gram_inverse_kernel<RT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(sm)));
    configured = true;
  }
  gram_inverse_kernel<RT><<<1, kThreads, sm, st>>>(pg, nparts, r, tol, ginv, info, stop);
  CPB_LAUNCH_CHECK();
}

void launch_gram_inverse(const double* part_gram, int nparts, int r, double tol, double* ginv,
                         int* info, const int* stop, cudaStream_t st) {
  switch (rank_bucket(r)) {
    case 16: gram_inverse_t<16>(part_gram, nparts, r, tol, ginv, info, stop, st); break;
    case 32: gram_inverse_t<32>(part_gram, nparts, r, tol, ginv, info, stop, st); break;
    default: gram_inverse_t<64>(part_gram, nparts, r, tol, ginv, info, stop, st); break;
  }
}

void launch_gather_rows(const double* x, i64 in, i64 stride, const i64* base, int s, double* xs,
                        i64 ld, cudaStream_t st) {
  if (s <= 0) return;
  const int per = kGatherThreads * kGatherUnroll;
  int gx = ceil_div(in, per);
  if (gx > 64) gx = 64;
  int rows = s;
  for (int r0 = 0; r0 < s; r0 += 65535) {
    const int ny = (s - r0) < 65535 ? (s - r0) : 65535;
    gather_rows_kernel<<<dim3(gx, ny), kGatherThreads, 0, st>>>(x, in, stride, base + r0, ny,
                                                                xs + static_cast<i64>(r0) * ld, ld);
    CPB_LAUNCH_CHECK();
  }
  (void)rows;
}

void launch_rhs_gemm(const double* xs, i64 ld, const double* z, i64 in, int s, int r, int ks,
                     int ks_len, double* part, const int* stop, cudaStream_t st) {
  const dim3 grid(ceil_div(in, GBM), ks);
  switch (rank_bucket(r)) {
    case 16: rhs_gemm_kernel<16><<<grid, kThreads, 0, st>>>(xs, ld, z, in, s, r, ks_len, part, stop); break;
    case 32: rhs_gemm_kernel<32><<<grid, kThreads, 0, st>>>(xs, ld, z, in, s, r, ks_len, part, stop); break;
    default: rhs_gemm_kernel<64><<<grid, kThreads, 0, st>>>(xs, ld, z, in, s, r, ks_len, part, stop); break;
  }
  CPB_LAUNCH_CHECK();
}

void launch_mode_apply(const ModeView& v, const ModeWork& w, const double* rhs_override,
                       int first_of_pass, cudaStream_t st) {
  const int grid = ceil_div(v.in, BI);
  switch (rank_bucket(v.r)) {
    case 16: mode_apply_kernel<16><<<grid, kThreads, 0, st>>>(v.in, v.r, w, rhs_override, first_of_pass); break;
    case 32: mode_apply_kernel<32><<<grid, kThreads, 0, st>>>(v.in, v.r, w, rhs_override, first_of_pass); break;
    default: mode_apply_kernel<64><<<grid, kThreads, 0, st>>>(v.in, v.r, w, rhs_override, first_of_pass); break;
  }
  CPB_LAUNCH_CHECK();
}

void launch_normalize(const ModeWork& w, i64 in, int r, unsigned long long* rng_state,
                      cudaStream_t st) {
  const i64 n = in * r;
  normalize_kernel<<<ceil_div(n, 256), 256, 0, st>>>(w.a, in, r, w.norms, w.stop, rng_state);
  CPB_LAUNCH_CHECK();
}

void launch_gather_values(const double* x, const i64* off, i64 n, double* out, cudaStream_t st) {
  if (n <= 0) return;
  gather_values_kernel<<<ceil_div(n, 256), 256, 0, st>>>(x, off, n, out);
  CPB_LAUNCH_CHECK();
}

void launch_sumsq(const double* x, i64 n, double* partials, int nparts, double* out,
                  cudaStream_t st) {
  sumsq_partial_kernel<<<nparts, kThreads, 0, st>>>(x, n, partials);
  CPB_LAUNCH_CHECK();
  sum_partials_kernel<<<1, 32, 0, st>>>(partials, nparts, out);
  CPB_LAUNCH_CHECK();
}

void launch_estimate_fit(const FitArgs& a, cudaStream_t st) {
  estimate_fit_kernel<<<ceil_div(a.phat, kThreads), kThreads, 0, st>>>(a);
  CPB_LAUNCH_CHECK();
}

void launch_stamp_start(FitState* s, cudaStream_t st) {
  stamp_start_kernel<<<1, 1, 0, st>>>(s);
  CPB_LAUNCH_CHECK();
}

void launch_rng_seed(unsigned long long* state, unsigned long long v, cudaStream_t st) {
  rng_seed_kernel<<<1, 1, 0, st>>>(state, v);
  CPB_LAUNCH_CHECK();
}

void launch_rng_normals(unsigned long long* state, int n, double* out, cudaStream_t st) {
  rng_normals_kernel<<<1, 1, 0, st>>>(state, n, out);
  CPB_LAUNCH_CHECK();
}

}  // namespace cpb
