// CTA-level device functions of one sampled mode update, shared by the
// standalone kernels (solve.cu) and the persistent per-iteration kernel
// (fused.cu). Every function takes its shared-memory scratch from the
// caller, so a persistent kernel can reuse one buffer across phases.
//
// Reference steps (paths under /root/reference/proj/include/cprand/):
//   Z_S rows            skr            sampling.hpp:74-92
//   LS solve            least_squares  kr_linalg.hpp:105-118 (normal equations here)
//   column norms/lambda normalize      kruskal.hpp:51-67
#pragma once

#include <cfloat>
#include <type_traits>

#include "devutil.cuh"
#include "kernels.cuh"

#ifndef CPB_INV_STAMP
#define CPB_INV_STAMP(k)  // micro-benchmark hooks (tests/micro/inv_bench.cu)
#define CPB_INV_STAMP_AT(k, s, lane0)
#endif

namespace cpb {
namespace ph {

// ------------------------------------------------------------------ Z_S
// ones, then *= factor rows in ascending kept mode; factors are kept as
// A_un with column norms, and A_un / norm is the exact value the reference
// stores after col /= norm.
__device__ __forceinline__ double z_entry(const ModeView& v, int s, int rr) {
  double zv = 1.0;
  for (int c = 0; c < v.kept; ++c) {
    const int row = __ldg(v.rows[c] + s);
    CPB_DCHECK(v.kdim[c] == 0 || (row >= 0 && row < v.kdim[c]), "z_entry: sampled row");
    double a = __ldcg(v.fac[c] + static_cast<i64>(row) * v.r + rr);  // written earlier in a persistent launch
    if (v.nrm[c]) a = a / __ldcg(v.nrm[c] + rr);
    zv = __dmul_rn(zv, a);
  }
  return zv;
}

// Z[s][RT] for entries e in [g, S*RT) step G
template <int RT>
__device__ __forceinline__ void z_range(const ModeView& v, double* __restrict__ z, i64 g, i64 G) {
  const i64 total = static_cast<i64>(v.s) * RT;
  for (i64 e = g; e < total; e += G) {
    const int s = static_cast<int>(e / RT), rr = static_cast<int>(e % RT);
    z[e] = (rr < v.r) ? z_entry(v, s, rr) : 0.0;
  }
}

// ------------------------------------------------------------------ Gram
// RT x RT partial sum_{s in [s0,s1)} Z(s,:)^T Z(s,:) by one CTA of 256
// threads (4 x RT/16 register tile for RT = 64). sh: GS x RT doubles.
constexpr int GS = 64;

template <int RT>
__device__ void gram_chunk(const double* __restrict__ z, int s0, int s1, double* __restrict__ out,
                           double* sh) {
  constexpr int NT = 256;
  constexpr int GPT = RT * RT / NT;
  constexpr int TA = RT >= 32 ? 4 : 1;
  constexpr int TB = GPT / TA;
  double(*zs)[RT] = reinterpret_cast<double(*)[RT]>(sh);
  const int tid = threadIdx.x;
  const int ra = (tid / (RT / TB)) * TA, cb = tid % (RT / TB);
  double acc[TA][TB];
#pragma unroll
  for (int x = 0; x < TA; ++x)
#pragma unroll
    for (int y = 0; y < TB; ++y) acc[x][y] = 0.0;
  for (int sc = s0; sc < s1; sc += GS) {
    constexpr int PER = GS * RT / NT;
    double v[PER];
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int e = tid + q * NT, sl = e / RT, c = e % RT, s = sc + sl;
      v[q] = (s < s1) ? z[static_cast<i64>(s) * RT + c] : 0.0;
    }
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int e = tid + q * NT;
      zs[e / RT][e % RT] = v[q];
    }
    __syncthreads();
#pragma unroll 4
    for (int sl = 0; sl < GS; ++sl) {
      double xa[TA], xb[TB];
#pragma unroll
      for (int x = 0; x < TA; ++x) xa[x] = zs[sl][ra + x];
#pragma unroll
      for (int y = 0; y < TB; ++y) xb[y] = zs[sl][cb + (RT / TB) * y];
#pragma unroll
      for (int x = 0; x < TA; ++x)
#pragma unroll
        for (int y = 0; y < TB; ++y) acc[x][y] = fma(xa[x], xb[y], acc[x][y]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int x = 0; x < TA; ++x)
#pragma unroll
    for (int y = 0; y < TB; ++y) out[(ra + x) * RT + cb + (RT / TB) * y] = acc[x][y];
}

// ------------------------------------------------ pivoted-Cholesky pinv
// Rank-deficient fallback (kr_linalg.hpp:113-117 analogue): pivoted
// Cholesky of G (warp 0), pinv = P L^-T L^-1 P^T at full rank, else
// B B^T with B = M (M^T M)^-1, M = P L[:, :rank]. g, w: [RT][RT+1] (any
// memory), w followed by 2 RT scratch doubles; perm: RT ints (shared).
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
  for (int j = tid; j < rank; j += blockDim.x) {  // w <- L^-1 (column j per thread)
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
    for (int e = tid; e < r * r; e += blockDim.x) {
      const int a = e / r, b = e % r;
      const int lo = a > b ? a : b;
      double sacc = 0.0;
      for (int m = lo; m < r; ++m) sacc += w[m * LD + a] * w[m * LD + b];
      ginv[perm[a] * r + perm[b]] = sacc;
    }
  } else if (tid == 0) {
    const int k = rank;
    for (int a = 0; a < k; ++a)
      for (int b = 0; b <= a; ++b) {
        double sacc = 0.0;
        for (int m = a; m < r; ++m) sacc += g[m * LD + a] * g[m * LD + b];
        w[a * LD + b] = sacc;
        w[b * LD + a] = sacc;
      }
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
  if (tid == 0) {
    info[0] = rank;
    info[1] += 1;  // fallback count (diagnostics)
  }
}

// Fallback driver: G from gfull, working matrices in global scratch after it.
template <int RT>
__device__ void pinv_fallback(double* gfull, int r, double tol, double* ginv, int* info, int* perm_sh) {
  constexpr int LD = RT + 1;
  double* g = gfull + r * r;
  double* wk = g + RT * LD;
  for (int e = threadIdx.x; e < RT * LD; e += blockDim.x) {
    const int x = e / LD, y = e % LD;
    g[e] = (x < r && y < r) ? gfull[x * r + y] : 0.0;
  }
  __threadfence_block();
  __syncthreads();
  gram_pinv<RT>(g, wk, perm_sh, r, tol, ginv, info);
}

// ------------------------------------------------------ Gram inverse
// In-place block Gauss-Jordan (4 x 4 pivot blocks, no pivoting: the Gram
// is SPD) by one CTA of NTH threads. Warp w owns rows w + W t, lane l owns
// columns l + 32 u; elements live in registers. The matrix is padded to a
// multiple of 4 with d_max on the padding diagonal. Step s (K = [4s,4s+4)):
// with P^-1 the inverse of the current pivot block, X = a with rows and
// columns K zeroed, C(i) = a(i,K) (-e on rows K) and M(j) = P^-1 a(K,j)
// (column j - 4s of P^-1 on columns K), a' = X - C M covers all four
// Gauss-Jordan block rules with 4 FMAs per element. The owners of the next
// block's rows/columns publish them (double-buffered); thread 0 inverts the
// next pivot block (scalar pivots tested against tol * d_max). Returns true
// (uniformly) on failure, after writing the reduced Gram to gfull for the
// pivoted fallback. sh: 16 RT + 40 doubles.
template <int RT, int NTH>
__device__ bool inverse_cta(const double* __restrict__ part, int nparts, int r, double tol,
                            double* __restrict__ ginv, double* __restrict__ gfull, int* info,
                            double* sh) {
  constexpr int W = NTH / 32;
  constexpr int TR = RT / W > 0 ? RT / W : 1;  // rows per warp
  constexpr int TC = RT >= 32 ? RT / 32 : 1;   // columns per lane
  double* colB = sh;              // [2][RT][4]  column block of the next step
  double* rowB = sh + 8 * RT;     // [2][4][RT]  row block of the next step
  double* pinv = sh + 16 * RT;    // [2][16]
  double* misc = pinv + 32;       // [0] d_max, [1] thr, [2..3] fail flags
  const int tid = threadIdx.x, w = tid / 32, l = tid % 32;
  const int r4 = (r + 3) & ~3;
  double a[TR][TC];
  int row[TR], col[TC];
#pragma unroll
  for (int t = 0; t < TR; ++t) row[t] = w + W * t;
#pragma unroll
  for (int u = 0; u < TC; ++u) col[u] = l + 32 * u;
#pragma unroll
  for (int t = 0; t < TR; ++t)
#pragma unroll
    for (int u = 0; u < TC; ++u) a[t][u] = 0.0;
  {  // G = sum of the split partials in split order, PB partials per batch
     // (about 32 loads in flight per thread; the last batch predicated)
    constexpr int PB = TR * TC >= 32 ? 1 : ((32 / (TR * TC)) > 4 ? (32 / (TR * TC)) : 4);
    for (int k = 0; k < nparts; k += PB) {
      double v[PB][TR][TC];
#pragma unroll
      for (int x = 0; x < PB; ++x)
#pragma unroll
        for (int t = 0; t < TR; ++t)
#pragma unroll
          for (int u = 0; u < TC; ++u)
            v[x][t][u] = (k + x < nparts && row[t] < r && col[u] < r)
                             ? __ldcg(part + static_cast<i64>(k + x) * RT * RT + row[t] * RT + col[u])
                             : 0.0;
#pragma unroll
      for (int x = 0; x < PB; ++x)
        if (k + x < nparts)
#pragma unroll
          for (int t = 0; t < TR; ++t)
#pragma unroll
            for (int u = 0; u < TC; ++u) a[t][u] += v[x][t][u];
    }
  }
  // d_max for the threshold and the padding diagonal
  if (tid == 0) misc[0] = 0.0;
  __syncthreads();
#pragma unroll
  for (int t = 0; t < TR; ++t)
#pragma unroll
    for (int u = 0; u < TC; ++u) {
      if (row[t] < r && col[u] < r) gfull[row[t] * r + col[u]] = a[t][u];
      if (row[t] == col[u] && row[t] < r)
        atomicMax(reinterpret_cast<unsigned long long*>(misc), __double_as_longlong(fmax(a[t][u], 0.0)));
    }
  __syncthreads();
  const double dmax = misc[0];
  const double thr = tol * dmax;
#pragma unroll
  for (int t = 0; t < TR; ++t)
#pragma unroll
    for (int u = 0; u < TC; ++u) {
      if (row[t] >= r && row[t] < r4 && row[t] == col[u]) a[t][u] = dmax;  // padding diagonal
      if (row[t] < 4 && col[u] < RT) rowB[row[t] * RT + col[u]] = a[t][u];
      if (col[u] < 4 && row[t] < RT) colB[row[t] * 4 + col[u]] = a[t][u];
    }
  __syncthreads();
  auto invert_block = [&](const double* cb, int k0, double* out, double* failp) {
    // unpivoted 4 x 4 Gauss-Jordan of rows/cols K of the current matrix
    double p[4][4];
    for (int x = 0; x < 4; ++x)
      for (int y = 0; y < 4; ++y) p[x][y] = cb[(k0 + x) * 4 + y];
    bool bad = false;
    for (int k = 0; k < 4; ++k) {
      const double piv = p[k][k];
      if (!(piv > thr) || !(piv > 0.0)) bad = true;
      const double q = 1.0 / piv;
      double rk[4], ck[4];
      for (int y = 0; y < 4; ++y) rk[y] = (y == k) ? q : p[k][y] * q;
      for (int x = 0; x < 4; ++x) ck[x] = (x == k) ? -1.0 : p[x][k];
      for (int x = 0; x < 4; ++x)
        for (int y = 0; y < 4; ++y) {
          const double xv = (x == k || y == k) ? 0.0 : p[x][y];
          p[x][y] = fma(-ck[x], rk[y], xv);
        }
    }
    for (int x = 0; x < 4; ++x)
      for (int y = 0; y < 4; ++y) out[x * 4 + y] = p[x][y];
    *failp = bad ? 1.0 : 0.0;
  };
  if (tid == 0) invert_block(colB, 0, pinv, misc + 2);
  __syncthreads();
  bool fail = false;
  for (int k0 = 0; k0 < r4; k0 += 4) {
    const int b = (k0 >> 2) & 1, nb = b ^ 1;
    if (misc[2 + b] != 0.0) {
      fail = true;  // uniform
      break;
    }
    const double* P = pinv + 16 * b;
    const double* cb = colB + b * RT * 4;
    const double* rb = rowB + b * 4 * RT;
    double m[TC][4];
#pragma unroll
    for (int u = 0; u < TC; ++u) {
      const int j = col[u];
      const bool jk = (j >= k0 && j < k0 + 4);
      double rv[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) rv[q] = rb[q * RT + (j < RT ? j : 0)];
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        const double mv = P[x * 4 + 0] * rv[0] + P[x * 4 + 1] * rv[1] + P[x * 4 + 2] * rv[2] + P[x * 4 + 3] * rv[3];
        m[u][x] = jk ? P[x * 4 + (j - k0)] : mv;
      }
    }
#pragma unroll
    for (int t = 0; t < TR; ++t) {
      const int i = row[t];
      const bool ik = (i >= k0 && i < k0 + 4);
      double c[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) c[q] = ik ? (i - k0 == q ? -1.0 : 0.0) : cb[(i < RT ? i : 0) * 4 + q];
#pragma unroll
      for (int u = 0; u < TC; ++u) {
        const bool jk = (col[u] >= k0 && col[u] < k0 + 4);
        double v = (ik || jk) ? 0.0 : a[t][u];
        v = fma(-c[0], m[u][0], v);
        v = fma(-c[1], m[u][1], v);
        v = fma(-c[2], m[u][2], v);
        v = fma(-c[3], m[u][3], v);
        a[t][u] = v;
      }
    }
    // publish the next step's row and column blocks
    const int n0 = k0 + 4;
    if (n0 < r4) {
#pragma unroll
      for (int t = 0; t < TR; ++t)
#pragma unroll
        for (int u = 0; u < TC; ++u) {
          const int i = row[t], j = col[u];
          if (j >= n0 && j < n0 + 4 && i < RT) colB[nb * RT * 4 + i * 4 + (j - n0)] = a[t][u];
          if (i >= n0 && i < n0 + 4 && j < RT) rowB[nb * 4 * RT + (i - n0) * RT + j] = a[t][u];
        }
    }
    __syncthreads();
    if (n0 < r4) {
      if (tid == 0) invert_block(colB + nb * RT * 4, n0, pinv + 16 * nb, misc + 2 + nb);
      __syncthreads();
    }
  }
  CPB_INV_STAMP(30);
  if (!fail) {
#pragma unroll
    for (int t = 0; t < TR; ++t)
#pragma unroll
      for (int u = 0; u < TC; ++u)
        if (row[t] < r && col[u] < r) ginv[row[t] * r + col[u]] = a[t][u];
  }
  if (tid == 0) {
    info[0] = fail ? -1 : r;
    info[2] = 0;  // normal-equations mode (qr_factor sets 1)
  }
  __syncthreads();
  CPB_INV_STAMP(31);
  return fail;
}

// ---------------------------------------------- 4 x 4 pivot inverse
// 1/d to full precision: hardware approximation + two Newton steps (the
// inverse is not a bit-parity quantity; 1e-16 relative is what matters).
__device__ __forceinline__ double rcp_nr(double d) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;\n" : "=d"(y) : "d"(d));
  double e = fma(-d, y, 1.0);
  y = fma(y, e, y);
  e = fma(-d, y, 1.0);
  return fma(y, e, y);
}
// Unpivoted 4 x 4 Gauss-Jordan inverse by lanes 0..15 of a warp (lane
// 4 x + y holds p(x, y) in and p^-1(x, y) out); all 32 lanes must call.
// ok = false when a pivot is <= thr (or not positive).
__device__ __forceinline__ double invert4_lanes(double p, double thr, bool& ok) {
  const int l = threadIdx.x & 31, x = (l >> 2) & 3, y = l & 3;
  ok = true;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const double pkk = __shfl_sync(0xffffffffu, p, k * 5);
    const double pky = __shfl_sync(0xffffffffu, p, k * 4 + y);
    const double pxk = __shfl_sync(0xffffffffu, p, x * 4 + k);
    if (!(pkk > thr) || !(pkk > 0.0)) ok = false;
    const double q = rcp_nr(pkk);
    const double rk = (y == k) ? q : pky * q;
    const double ck = (x == k) ? -1.0 : pxk;
    const double xv = (x == k || y == k) ? 0.0 : p;
    p = fma(-ck, rk, xv);
  }
  return p;
}

// ------------------------------------------- Gram inverse, look-ahead
// 4 x 4 inverse by the 2 x 2-minor (Laplace) expansion: every entry is a
// short independent expression, so the latency is ~6 dependent FP64 ops and
// one reciprocal instead of four chained pivot divisions. The unpivoted
// Gauss-Jordan pivots are d_k / d_{k-1} (leading principal minors), so the
// rank test pivot_k > thr becomes d_k > thr d_{k-1} without divisions.
__device__ __forceinline__ bool inv4_minors(const double* a, double* out, double thr) {
  const double a00 = a[0], a01 = a[1], a02 = a[2], a03 = a[3];
  const double a10 = a[4], a11 = a[5], a12 = a[6], a13 = a[7];
  const double a20 = a[8], a21 = a[9], a22 = a[10], a23 = a[11];
  const double a30 = a[12], a31 = a[13], a32 = a[14], a33 = a[15];
  const double s0 = fma(a00, a11, -a10 * a01), s1 = fma(a00, a12, -a10 * a02);
  const double s2 = fma(a00, a13, -a10 * a03), s3 = fma(a01, a12, -a11 * a02);
  const double s4 = fma(a01, a13, -a11 * a03), s5 = fma(a02, a13, -a12 * a03);
  const double c5 = fma(a22, a33, -a32 * a23), c4 = fma(a21, a33, -a31 * a23);
  const double c3 = fma(a21, a32, -a31 * a22), c2 = fma(a20, a33, -a30 * a23);
  const double c1 = fma(a20, a32, -a30 * a22), c0 = fma(a20, a31, -a30 * a21);
  const double det = (fma(s0, c5, -s1 * c4) + fma(s2, c3, s3 * c2)) + fma(-s4, c1, s5 * c0);
  // leading principal minors d1 = a00, d2 = s0, d3 = det(a[0..2][0..2])
  const double d3 = fma(a20, s3, fma(-a21, s1, a22 * s0));
  const bool ok = (a00 > thr) && (s0 > thr * a00) && (d3 > thr * s0) && (det > thr * d3) && (a00 > 0.0) &&
                  (s0 > 0.0) && (d3 > 0.0) && (det > 0.0);
  const double id = 1.0 / det;
  out[0] = (fma(a11, c5, -a12 * c4) + a13 * c3) * id;
  out[1] = (fma(-a01, c5, a02 * c4) - a03 * c3) * id;
  out[2] = (fma(a31, s5, -a32 * s4) + a33 * s3) * id;
  out[3] = (fma(-a21, s5, a22 * s4) - a23 * s3) * id;
  out[4] = (fma(-a10, c5, a12 * c2) - a13 * c1) * id;
  out[5] = (fma(a00, c5, -a02 * c2) + a03 * c1) * id;
  out[6] = (fma(-a30, s5, a32 * s2) - a33 * s1) * id;
  out[7] = (fma(a20, s5, -a22 * s2) + a23 * s1) * id;
  out[8] = (fma(a10, c4, -a11 * c2) + a13 * c0) * id;
  out[9] = (fma(-a00, c4, a01 * c2) - a03 * c0) * id;
  out[10] = (fma(a30, s4, -a31 * s2) + a33 * s0) * id;
  out[11] = (fma(-a20, s4, a21 * s2) - a23 * s0) * id;
  out[12] = (fma(-a10, c3, a11 * c1) - a12 * c0) * id;
  out[13] = (fma(a00, c3, -a01 * c1) + a02 * c0) * id;
  out[14] = (fma(-a30, s3, a31 * s1) - a32 * s0) * id;
  out[15] = (fma(a20, s3, -a21 * s1) + a22 * s0) * id;
  return ok;
}

// 4 x 4 inverse by cofactors, one entry per lane (lanes 0..15; all 32 lanes
// must call): lane 4 i + j forms the 3 x 3 minor of P without row j and
// column i from p (row-major, shared memory), det P from the row-0
// cofactors (shuffles), and returns P^-1(i, j) = C_ji / det. The rank test
// uses the leading principal minors d_k (pivot_k = d_k / d_{k-1}) without
// divisions; ok is uniform over the warp.
__device__ __forceinline__ double inv4_cofactor(const double* p, double thr, bool& ok, int ld = 4) {
  const int l = threadIdx.x & 31, i = (l >> 2) & 3, j = l & 3;
  const int r0 = (0 >= j) ? 1 : 0, r1 = (1 >= j) ? 2 : 1, r2 = (2 >= j) ? 3 : 2;
  const int c0 = (0 >= i) ? 1 : 0, c1 = (1 >= i) ? 2 : 1, c2 = (2 >= i) ? 3 : 2;
  const double m00 = p[r0 * ld + c0], m01 = p[r0 * ld + c1], m02 = p[r0 * ld + c2];
  const double m10 = p[r1 * ld + c0], m11 = p[r1 * ld + c1], m12 = p[r1 * ld + c2];
  const double m20 = p[r2 * ld + c0], m21 = p[r2 * ld + c1], m22 = p[r2 * ld + c2];
  const double det3 = fma(m00, fma(m11, m22, -m12 * m21), fma(-m01, fma(m10, m22, -m12 * m20), m02 * fma(m10, m21, -m11 * m20)));
  const double cof = ((i + j) & 1) ? -det3 : det3;  // C_ji
  // det P = sum_k P(0, k) C_0k (C_0k lives on lane 4 k)
  const double q0 = __shfl_sync(0xffffffffu, cof, 0), q1 = __shfl_sync(0xffffffffu, cof, 4);
  const double q2 = __shfl_sync(0xffffffffu, cof, 8), q3 = __shfl_sync(0xffffffffu, cof, 12);
  const double d3 = __shfl_sync(0xffffffffu, cof, 15);  // C_33 = det P[0..2][0..2]
  const double det = fma(p[0], q0, p[1] * q1) + fma(p[2], q2, p[3] * q3);
  const double d1 = p[0], d2 = fma(p[0], p[ld + 1], -p[1] * p[ld]);
  ok = (d1 > thr) && (d2 > thr * d1) && (d3 > thr * d2) && (det > thr * d3) && (d1 > 0.0) && (d2 > 0.0) &&
       (d3 > 0.0) && (det > 0.0);
  return cof * rcp_nr(det);
}

// Block Gauss-Jordan inverse (4 x 4 pivot blocks, no pivoting: the Gram is
// SPD) by one CTA of 256 threads, one barrier per step.
//  * Warps 0-6 hold the matrix as FP64 MMA accumulator fragments (warp w:
//    8-column tiles w and w + 7, every 8-row tile) and do step s as one
//    m8n8k4 MMA per tile: a' = X + (-C) M, where X = a with rows/columns K
//    zeroed, -C(i) = -a(i, K) (+e on rows K) comes from the published column
//    block and M(j) = P^-1 a(K, j) from the published row block, whose K
//    columns hold the identity (so M = P^-1 e_j there): the four
//    Gauss-Jordan block rules in one form.
//  * After the MMAs the owners publish step s+1's row/column blocks and
//    zero rows/columns K_{s+1} (X of the next step). The step loop is fully
//    unrolled, so every tile index is a compile-time constant.
//  * Warp 7 meanwhile forms the NEXT pivot block (rows/columns K_{s+1} after
//    step s, from the raw rows K_s, K_{s+1}) and inverts it (inv4_minors):
//    the pivot inversion is off the workers' critical path.
// g: RT x RT Gram (ld RT; entries outside [0, r) ignored). Returns true
// (uniformly) on a pivot <= tol * d_max, after writing the Gram to gfull
// (r x r) for the pivoted fallback. sh: 24 RT + 64 doubles.
template <int RT>
__device__ bool inverse_la(const double* __restrict__ g, int r, double tol, double* __restrict__ ginv,
                           double* __restrict__ gfull, int* info, double* sh,
                           unsigned long long* stamps = nullptr) {
  constexpr int NTI = RT / 8;
  constexpr int NSMAX = RT / 4;
  static_assert(NTI <= 8, "one 8-column tile per warp");
  double* rbs = sh;              // [2][8][RT] rows K_s (identity on K_s columns), raw rows K_{s+1}
  double* cbs = rbs + 16 * RT;   // [2][RT][4] -a(i, K_s), +e on rows K_s
  double* pin = cbs + 8 * RT;    // [2][16]    inverse of the pivot block of step s
  double* misc = pin + 32;       // [2..3] fail flags, [4..5] warp maxima
  double* tmp = misc + 8;        // [16] next pivot block
  const int tid = threadIdx.x, w = tid / 32, l = tid % 32;
  const int lr = l >> 2, lc = (l & 3) * 2, lk = l & 3;
  const int r4 = (r + 3) & ~3;
  const int nt = (r + 7) / 8;
  const int nsteps = r4 / 4;
  const bool worker = w < nt;  // warp w owns 8-column tile w
  const int ct = w;
  double acc[NTI][2];
#pragma unroll
  for (int mt = 0; mt < NTI; ++mt) {
    const int row = mt * 8 + lr, col = ct * 8 + lc;
    const bool ok = worker && row < r;
    acc[mt][0] = (ok && col < r) ? __ldcg(g + row * RT + col) : 0.0;
    acc[mt][1] = (ok && col + 1 < r) ? __ldcg(g + row * RT + col + 1) : 0.0;
  }
  {  // d_max: largest (clamped) diagonal entry
    double dv = (tid < r) ? fmax(__ldcg(g + tid * (RT + 1)), 0.0) : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dv = fmax(dv, __shfl_xor_sync(0xffffffffu, dv, o));
    if (l == 0 && w < 2) misc[4 + w] = dv;
  }
  __syncthreads();
  const double dmax = RT > 32 ? fmax(misc[4], misc[5]) : misc[4];
  const double thr = tol * dmax;
#pragma unroll
  for (int mt = 0; mt < NTI; ++mt) {
    const int row = mt * 8 + lr;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int col = ct * 8 + lc + e;
      if (!worker) continue;
      if (row < r && col < r) gfull[row * r + col] = acc[mt][e];
      if (row == col && row >= r && row < r4) acc[mt][e] = dmax;  // padding diagonal
    }
  }
  CPB_INV_STAMP(1);
  // Publish rows K (identity on K x K) and the raw rows K+ after them into
  // rb, -a(., K) (+e on rows K) into cb (owner warp of the K columns), and
  // zero rows/columns K. Fragment slot p holds row tile (T + p) % NTI (the
  // slots rotate once per tile), so every slot index here is compile-time:
  // rows K are local rows RK..RK+3 of slot PK, rows K+ local rows RKK.. of
  // slot PKK, columns K local columns 4 CH..4 CH+3 of the owner.
  auto publish = [&](auto pk, auto rk0, auto pkk, auto rkk0, auto ch, int T, bool own, double* rb, double* cb,
                     bool first) {
    constexpr int PK = decltype(pk)::value, RK = decltype(rk0)::value;
    constexpr int PKK = decltype(pkk)::value, RKK = decltype(rkk0)::value, CH = decltype(ch)::value;
    if (!worker) return;  // warp-uniform
    const int col = ct * 8 + lc;
    const bool inK = (lr >= RK && lr < RK + 4);
    const bool inKK = (lr >= RKK && lr < RKK + 4) && (((T + PKK) % NTI) * 8 + lr < r4);
    const bool ck = (lk >> 1) == CH;  // my two columns are in K (owner warp only)
    {  // rows K (slot PK)
      const int qi = lr - RK;
      if (inK) {
        const double v0 = acc[PK][0], v1 = acc[PK][1];
        if (first && own && ck) {
          tmp[qi * 4 + (lc & 3)] = v0;
          tmp[qi * 4 + (lc & 3) + 1] = v1;
        }
        double2 o;
        o.x = (own && ck) ? (qi == (lc & 3) ? 1.0 : 0.0) : v0;
        o.y = (own && ck) ? (qi == (lc & 3) + 1 ? 1.0 : 0.0) : v1;
        *reinterpret_cast<double2*>(rb + qi * RT + col) = o;
      }
    }
    if (inKK)  // raw rows K+ (slot PKK)
      *reinterpret_cast<double2*>(rb + (4 + lr - RKK) * RT + col) = make_double2(acc[PKK][0], acc[PKK][1]);
    if (own && ck) {  // column block K, every slot
#pragma unroll
      for (int p = 0; p < NTI; ++p) {
        const int row = ((T + p) % NTI) * 8 + lr;
        const bool rkk = (p == PK) && inK;
        const int q0 = (lc & 3);
        double2 o;
        o.x = rkk ? ((lr - RK) == q0 ? 1.0 : 0.0) : -acc[p][0];
        o.y = rkk ? ((lr - RK) == q0 + 1 ? 1.0 : 0.0) : -acc[p][1];
        *reinterpret_cast<double2*>(cb + row * 4 + q0) = o;
        acc[p][0] = 0.0;
        acc[p][1] = 0.0;
      }
    }
    if (inK) {
      acc[PK][0] = 0.0;
      acc[PK][1] = 0.0;
    }
  };
  using I0 = std::integral_constant<int, 0>;
  using I1 = std::integral_constant<int, 1>;
  using I4 = std::integral_constant<int, 4>;
  publish(I0{}, I0{}, I0{}, I4{}, I0{}, 0, ct == 0, rbs, cbs, true);
  __syncthreads();
  if (w == 7) {
    bool ok;
    const double v = inv4_cofactor(tmp, thr, ok);
    if (l < 16) pin[l] = v;
    if (l == 0) misc[2] = ok ? 0.0 : 1.0;
  }
  __syncthreads();
  CPB_INV_STAMP(2);
  if (stamps && tid == 0) stamps[0] = globaltimer();
  bool fail = false;
  int T = 0;
#pragma unroll 1
  for (; T < nt && !fail; ++T) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int s = 2 * T + h;
      if (s >= nsteps) break;  // uniform
      CPB_INV_STAMP(3 + s);
      const int pb = s & 1, k0 = 4 * s;
      if (misc[2 + pb] != 0.0) {
        fail = true;  // uniform
        break;
      }
      const double* P = pin + 16 * pb;
      const double* rb = rbs + pb * 8 * RT;
      const double* cb = cbs + pb * RT * 4;
      if (w == 7 && k0 + 4 < r4) {
        // warp 7: pivot block of step s+1 = rows/columns K_{s+1} after step s
        if (l < 16) {
          const int x = l >> 2, y = l & 3;
          const int jj = k0 + 4 + y;
          const double* rn = rb + (4 + x) * RT;  // raw row k0 + 4 + x
          double mv[4];
#pragma unroll
          for (int q = 0; q < 4; ++q)
            mv[q] = fma(P[q * 4], rb[jj], P[q * 4 + 1] * rb[RT + jj]) +
                    fma(P[q * 4 + 2], rb[2 * RT + jj], P[q * 4 + 3] * rb[3 * RT + jj]);
          tmp[l] = (rn[jj] - fma(rn[k0], mv[0], rn[k0 + 1] * mv[1])) - fma(rn[k0 + 2], mv[2], rn[k0 + 3] * mv[3]);
        }
        __syncwarp();
        CPB_INV_STAMP_AT(43, s, l == 0);
        {
          bool ok;
          const double v = inv4_cofactor(tmp, thr, ok);
          if (l < 16) pin[16 * (pb ^ 1) + l] = v;
          if (l == 0) misc[2 + (pb ^ 1)] = ok ? 0.0 : 1.0;
        }
        CPB_INV_STAMP_AT(44, s, l == 0);
      }
      if (worker) {
        // all fragment operands are loaded before the first MMA
        const double2 p01 = *reinterpret_cast<const double2*>(P + lk * 4);
        const double2 p23 = *reinterpret_cast<const double2*>(P + lk * 4 + 2);
        double am[NTI];
#pragma unroll
        for (int p = 0; p < NTI; ++p) am[p] = cb[(((T + p) % NTI) * 8 + lr) * 4 + lk];  // rows >= r4 hold zeros
        const int j = ct * 8 + lr;  // B fragment (k = l % 4, n = l / 4)
        const double bm = fma(p01.x, rb[j], p01.y * rb[RT + j]) + fma(p23.x, rb[2 * RT + j], p23.y * rb[3 * RT + j]);
#pragma unroll
        for (int p = 0; p < NTI; ++p)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                       : "+d"(acc[p][0]), "+d"(acc[p][1])
                       : "d"(am[p]), "d"(bm));
        CPB_INV_STAMP_AT(41, s, tid == 0);
        if (k0 + 4 < r4) {
          double* rbn = rbs + (pb ^ 1) * 8 * RT;
          double* cbn = cbs + (pb ^ 1) * RT * 4;
          if (h == 0)  // K' = rows 4..7 of tile T (slot 0), K'' = rows 0..3 of tile T+1 (slot 1)
            publish(I0{}, I4{}, I1{}, I0{}, I1{}, T, ct == T, rbn, cbn, false);
          else  // K' = rows 0..3 of tile T+1 (slot 1), K'' = rows 4..7 of tile T+1
            publish(I1{}, I0{}, I1{}, I4{}, I0{}, T, ct == T + 1, rbn, cbn, false);
        }
      }
      CPB_INV_STAMP_AT(42, s, tid == 0);
      CPB_INV_STAMP_AT(45, s, tid == 224);
      __syncthreads();
    }
    // rotate the slots: slot 0 <- tile T + 1
    double f0 = acc[0][0], f1 = acc[0][1];
#pragma unroll
    for (int p = 0; p + 1 < NTI; ++p) {
      acc[p][0] = acc[p + 1][0];
      acc[p][1] = acc[p + 1][1];
    }
    acc[NTI - 1][0] = f0;
    acc[NTI - 1][1] = f1;
  }
  CPB_INV_STAMP(30);
  if (stamps && tid == 0) stamps[1] = globaltimer();
  if (!fail && worker) {
#pragma unroll
    for (int p = 0; p < NTI; ++p) {
      const int mt = (T + p) % NTI;
      const int row = mt * 8 + lr, col = ct * 8 + lc;
      if (mt >= nt || row >= r) continue;
      if (col + 1 < r && !(r & 1))
        *reinterpret_cast<double2*>(ginv + row * r + col) = make_double2(acc[p][0], acc[p][1]);
      else {
        if (col < r) ginv[row * r + col] = acc[p][0];
        if (col + 1 < r) ginv[row * r + col + 1] = acc[p][1];
      }
    }
  }
  if (tid == 0) {
    info[0] = fail ? -1 : r;
    info[2] = 0;  // normal-equations mode (qr_factor sets 1)
  }
  __syncthreads();
  CPB_INV_STAMP(31);
  return fail;
}

// ------------------------------------------------------------ RHS GEMM
// part[kb](i, c) = sum_{s in split kb} X_S(s, i) Z(s, c) for the 128-row
// tile mt: 256 threads, 8 x RT/16 register tile (columns strided by 16 for
// conflict-free loads), 3-stage cp.async pipeline. A rows at
// xs + row_off[s] (fibers read in place) or xs + s * ld (gathered X_S);
// element i of a row at + i * est (est > 1: a strided mode read in place
// from the tensor itself, one 8-byte cp.async per element, !VEC16 only).
// sh: GSTAGES * GBK * (GBM + RT) doubles.
constexpr int GBM = 128, GBK = 16, GSTAGES = 3;

template <int RT, bool VEC16>
__device__ void gemm_tile(const double* __restrict__ xs, i64 ld, const i64* __restrict__ row_off,
                          const double* __restrict__ z, i64 in, int s_total, int r, int ks_len,
                          double* __restrict__ part, int mt, int kb, double* sh, i64 est = 1) {
  constexpr int NT = 256;
  constexpr int TN = RT / 16, TM = GBM / 16;
  double* as = sh;                        // [GSTAGES][GBK][GBM]
  double* bs = sh + GSTAGES * GBK * GBM;  // [GSTAGES][GBK][RT]
  const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
  const i64 i0 = static_cast<i64>(mt) * GBM;
  const int s_begin = kb * ks_len;
  const int s_end = min(s_total, s_begin + ks_len);
  const int ntiles = (s_end - s_begin + GBK - 1) / GBK;

  auto load_tile = [&](int t, int st) {
    const int sbase = s_begin + t * GBK;
    double* ab = as + st * GBK * GBM;
    double* bb = bs + st * GBK * RT;
    if constexpr (VEC16) {
#pragma unroll
      for (int q = 0; q < GBK * GBM / 2 / NT; ++q) {
        const int c = tid + q * NT;
        const int sl = c / (GBM / 2), ic = (c % (GBM / 2)) * 2;
        const int s = sbase + sl;
        const i64 i = i0 + ic;
        const i64 lim = row_off ? in : ld;  // gathered rows are zero padded to ld
        const bool ok = (s < s_end) && (i < lim);
        const i64 ro = (s < s_end) ? (row_off ? row_off[s] : static_cast<i64>(s) * ld) : 0;
        const int bytes = !ok ? 0 : (i + 1 < lim ? 16 : 8);
        cp_async16(ab + sl * GBM + ic, ok ? xs + ro + i : xs, bytes);
      }
    } else {
#pragma unroll
      for (int q = 0; q < GBK * GBM / NT; ++q) {
        const int c = tid + q * NT;
        const int sl = c / GBM, ic = c % GBM;
        const int s = sbase + sl;
        const i64 i = i0 + ic;
        const bool ok = (s < s_end) && (i < in);
        const i64 ro = (s < s_end) ? (row_off ? row_off[s] : static_cast<i64>(s) * ld) : 0;
        cp_async8(ab + sl * GBM + ic, ok ? xs + ro + i * est : xs, ok ? 8 : 0);
      }
    }
    for (int c = tid; c < GBK * RT / 2; c += NT) {
      const int sl = c / (RT / 2), rc = (c % (RT / 2)) * 2;
      const int s = sbase + sl;
      const bool ok = s < s_end;
      cp_async16(bb + sl * RT + rc, ok ? z + static_cast<i64>(s) * RT + rc : z, ok ? 16 : 0);
    }
  };

  double acc[TM][TN];
#pragma unroll
  for (int a = 0; a < TM; ++a)
#pragma unroll
    for (int b = 0; b < TN; ++b) acc[a][b] = 0.0;
#pragma unroll
  for (int t = 0; t < GSTAGES - 1; ++t) {
    if (t < ntiles) load_tile(t, t);
    cp_async_commit();
  }
  for (int t = 0; t < ntiles; ++t) {
    cp_async_wait<GSTAGES - 2>();
    __syncthreads();
    const int nt = t + GSTAGES - 1;
    if (nt < ntiles) load_tile(nt, nt % GSTAGES);
    cp_async_commit();
    const double* ab = as + (t % GSTAGES) * GBK * GBM;
    const double* bb = bs + (t % GSTAGES) * GBK * RT;
#pragma unroll
    for (int kk = 0; kk < GBK; ++kk) {
      double af[TM], bf[TN];
#pragma unroll
      for (int a = 0; a < TM; ++a) af[a] = ab[kk * GBM + ty * TM + a];
#pragma unroll
      for (int b = 0; b < TN; ++b) bf[b] = bb[kk * RT + tx + 16 * b];
#pragma unroll
      for (int a = 0; a < TM; ++a)
#pragma unroll
        for (int b = 0; b < TN; ++b) acc[a][b] = fma(af[a], bf[b], acc[a][b]);
    }
  }
  cp_async_wait<0>();
  __syncthreads();  // the smem stages may be reused by the caller's next tile
  double* pr = part + static_cast<i64>(kb) * in * r;
#pragma unroll
  for (int a = 0; a < TM; ++a) {
    const i64 i = i0 + ty * TM + a;
    if (i >= in) continue;
#pragma unroll
    for (int b = 0; b < TN; ++b) {
      const int rr = tx + 16 * b;
      if (rr < r) pr[i * r + rr] = acc[a][b];
    }
  }
}

// --------------------------------------------------------- apply + norms
// One block of BI = NTH / RT factor rows starting at i0: RHS rows (split
// partials summed in split order, or the unmixed rhs_full), times Ginv
// (gi: RT x (RT+1) in shared memory, loaded by load_ginv). Writes A_un and
// returns this thread's out^2 (0 outside the matrix). rh: BI x (RT+1).
template <int RT, int NTH>
__device__ void load_ginv(const double* __restrict__ ginv, int r, double* gi) {
  for (int e = threadIdx.x; e < RT * RT; e += NTH) {
    const int x = e / RT, y = e % RT;
    gi[x * (RT + 1) + y] = (x < r && y < r) ? __ldcg(ginv + x * r + y) : 0.0;
  }
}

template <int RT, int NTH>
__device__ double apply_block(i64 in, int r, const ModeWork& w, const double* __restrict__ rhs_full,
                              i64 i0, const double* gi, double* rh) {
  constexpr int LD = RT + 1;
  const int tid = threadIdx.x;
  const int il = tid / RT, c = tid % RT;
  const i64 i = i0 + il;
  double s = 0.0;
  if (i < in && c < r) {
    if (rhs_full) {
      s = __ldcg(rhs_full + i * r + c);
    } else {
      const double* p = w.part_rhs + i * r + c;
      const i64 step = in * r;
      // 16 partials in flight per round trip, summed in split order
      int k = 0;
      for (; k + 16 <= w.ks; k += 16) {
        double v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) v[u] = __ldcg(p + (k + u) * step);
#pragma unroll
        for (int u = 0; u < 16; ++u) s += v[u];
      }
      if (k < w.ks) {
        double v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) v[u] = (k + u < w.ks) ? __ldcg(p + (k + u) * step) : 0.0;
#pragma unroll
        for (int u = 0; u < 16; ++u)
          if (k + u < w.ks) s += v[u];
      }
    }
  }
  rh[il * LD + c] = s;
  __syncthreads();
  double out = 0.0;
  for (int cc = 0; cc < r; ++cc) out = fma(rh[il * LD + cc], gi[cc * LD + c], out);
  __syncthreads();  // rh may be rewritten by the caller's next block
  const bool ok = (i < in && c < r);
  if (ok) w.a[i * r + c] = out;
  return ok ? out * out : 0.0;
}

// Per-CTA column sums of squares: thread (il, c) holds q; writes ssq[part][c].
template <int RT, int NTH>
__device__ void ssq_store(double q, int r, double* ssq_part, double* red) {
  constexpr int BI = NTH / RT;
  const int tid = threadIdx.x, il = tid / RT, c = tid % RT;
  red[il * (RT + 1) + c] = q;
  __syncthreads();
  if (tid < RT) {
    double t = 0.0;
#pragma unroll 8
    for (int x = 0; x < BI; ++x) t += red[x * (RT + 1) + tid];
    if (tid < r) ssq_part[tid] = t;
  }
  __syncthreads();
}

// Column norms from nparts per-CTA partials (interleaved sums, combined in
// fixed order), the lambda rule (kruskal.hpp:57-66) and the zero-column
// refill from the device normalize RNG. One CTA of NTH threads.
// red: (NTH / RT) x (RT + 1) doubles. Returns (uniformly) the mask of the
// columns that were zero and refilled.
template <int RT, int NTH>
__device__ unsigned long long norms_final(int r, i64 in, const ModeWork& w, int nparts, int first_of_pass,
                            unsigned long long* rng_state, double* red, unsigned long long* dbg = nullptr,
                            const double* lam_scale = nullptr) {
  constexpr int NP = NTH / RT;
  const int tid = threadIdx.x, part = tid / RT, c = tid % RT;
  __shared__ int s_zero;
  __shared__ unsigned long long s_zmask;
  // thread (part, c) sums a contiguous range of partials, 32 loads in flight;
  // the parts are then combined in order (deterministic)
  double q = 0.0;
  if (c < r && part < nparts) {
    const int len = (nparts + NP - 1) / NP;
    const int b0 = part * len, b1 = min(nparts, b0 + len);
    const double* p = w.ssq + static_cast<i64>(b0) * r + c;
    for (int k = 0; k < b1 - b0; k += 32) {
      double v[32];
#pragma unroll
      for (int u = 0; u < 32; ++u) v[u] = (k + u < b1 - b0) ? p[static_cast<i64>(k + u) * r] : 0.0;  // after an acquire
#pragma unroll
      for (int u = 0; u < 32; ++u)
        if (k + u < b1 - b0) q += v[u];
    }
  }
  red[part * (RT + 1) + c] = q;
  if (tid == 0) {
    s_zero = 0;
    s_zmask = 0ull;
  }
  if (dbg && tid == 0) dbg[0] = globaltimer();
  __syncthreads();
  if (dbg && tid == 0) dbg[1] = globaltimer();
  if (tid < r) {
    double t = 0.0;
    for (int x = 0; x < NP; ++x) t += red[x * (RT + 1) + tid];
    const double nrm = sqrt(t);
    w.norms[tid] = nrm;
    if (nrm == 0.0) {
      w.lambda[tid] = 0.0;
      atomicOr(&s_zero, 1);
    } else {
      // lam_scale: column scale the solution carried (the previous mode's norms
      // when its factor entered Z_S unnormalized)
      const double full = lam_scale ? nrm * __ldcg(lam_scale + tid) : nrm;
      w.lambda[tid] = first_of_pass ? __ldcg(w.lambda + tid) * full : full;
    }
  }
  __syncthreads();
  if (dbg && tid == 0) dbg[2] = globaltimer() | (s_zero ? (1ULL << 63) : 0ULL);
  if (tid == 0 && s_zero) {
    // zero columns (kruskal.hpp:57-63): N(0,1) column from the normalize
    // stream, one distribution object per call, columns in order
    DevMt g{rng_state};
    DevNormal gauss;
    for (int col = 0; col < r; ++col) {
      if (w.norms[col] != 0.0) continue;
      for (i64 t = 0; t < in; ++t) w.a[t * r + col] = gauss(g);
      w.norms[col] = dev_stable_norm(w.a + col, in, r);
      s_zmask |= 1ull << col;
    }
  }
  __syncthreads();
  return s_zmask;
}

// ------------------------------------------------------------ fit
// Squared error over the 256 sampled entries of virtual block vb (one
// thread per entry, fixed tree reduction); model_entry kruskal.hpp:37-44.
// red: 256 doubles. Result valid in thread 0.
// 256 sampled entries per block: 32 groups of 8 lanes, each group takes 8
// entries, U at a time. A group reads an entry's factor rows with its 8
// lanes on consecutive columns (q = lane, lane + 8, ...: 64-byte runs, so a
// warp load touches 4-8 sectors, not 32 lines), each lane multiplies its
// columns, the group sums them with three shuffles. The model value is
// sum_q lambda_q prod_n A_un(i_n, q) / norm_n(q) (kruskal.hpp:37-44,
// sampling.hpp:191-210); the column scale lambda_q / prod_n norm_n(q) is
// formed once per block in shared memory (red[256..]), so a term costs N
// multiplies instead of N divisions (a reassociation: the estimate agrees
// with the reference's to a few ulp). red: 256 + 128 doubles.
template <int KM, int QC, int U>
__device__ inline double fit_block_t(const FitArgs& a, i64 vb, double* red) {
  const int r = a.r, N = a.order;
  double* s_sc = red + 256;  // [r <= 128]
  for (int q = threadIdx.x; q < r; q += blockDim.x) {
    double den = 1.0;
    for (int n = 0; n < N; ++n)
      if (a.nrm[n]) den *= __ldcg(a.nrm[n] + q);
    s_sc[q] = __ldcg(a.lambda + q) / den;
  }
  const double* fac[KM];
#pragma unroll
  for (int n = 0; n < KM; ++n) fac[n] = n < N ? a.fac[n] : nullptr;
  __syncthreads();
  const int grp = threadIdx.x / 8, l = threadIdx.x % 8;
  double part = 0.0;  // lane 0: the group's squared residuals, entries in order
  for (int k = 0; k < 8; k += U) {
    i64 row[U][KM];
    bool ok[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const i64 j = vb * 256 + grp * 8 + k + u;
      ok[u] = j < a.phat;
#pragma unroll
      for (int n = 0; n < KM; ++n) row[u][n] = (ok[u] && n < N) ? static_cast<i64>(__ldg(a.idx[n] + j)) * r : 0;
    }
    double s[U];
#pragma unroll
    for (int u = 0; u < U; ++u) s[u] = 0.0;
    for (int q0 = l; q0 < r; q0 += 8 * QC) {
      double f[U][QC][KM];
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int c = 0; c < QC; ++c)
#pragma unroll
          for (int n = 0; n < KM; ++n)
            f[u][c][n] = (ok[u] && n < N && q0 + 8 * c < r) ? __ldcg(fac[n] + row[u][n] + q0 + 8 * c) : 1.0;
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int c = 0; c < QC; ++c) {
          const int q = q0 + 8 * c;
          if (q >= r) break;
          double p = s_sc[q];
#pragma unroll
          for (int n = 0; n < KM; ++n) {
            if (n >= N) break;
            p = __dmul_rn(p, f[u][c][n]);
          }
          s[u] = __dadd_rn(s[u], p);
        }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      double v = s[u];
      v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, 4));
      v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, 2));
      v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, 1));
      if (ok[u]) {
        const double e = a.values[vb * 256 + grp * 8 + k + u] - v;
        part += e * e;
      }
    }
  }
  red[threadIdx.x] = (l == 0) ? part : 0.0;
  __syncthreads();
  for (int st = 128; st > 0; st >>= 1) {
    if (threadIdx.x < st) red[threadIdx.x] += red[threadIdx.x + st];
    __syncthreads();
  }
  const double out = red[0];
  __syncthreads();
  return out;
}

constexpr int kFitSmemDoubles = 256 + 128;

__device__ inline double fit_block(const FitArgs& a, i64 vb, double* red) {
  return a.order <= 4 ? fit_block_t<4, 4, 2>(a, vb, red) : fit_block_t<kMaxOrder, 1, 2>(a, vb, red);
}

// Fit from the block partials (in order), sampling.hpp:192,207-209, and the
// stop rule should_stop (sampling.hpp:237-251); one thread.
// Whole CTA (blockDim 256): the block partials summed by a fixed tree (each
// thread adds partials t, t + 256, ... in order first); thread 0 then
// finishes. red: >= 256 doubles of shared memory.
__device__ inline void fit_final(const FitArgs& a, i64 nblocks, double* red) {
  double t = 0.0;
  for (i64 b = threadIdx.x; b < nblocks; b += blockDim.x) t += __ldcg(a.partials + b);
  red[threadIdx.x] = t;
  __syncthreads();
  for (int st = 128; st > 0; st >>= 1) {
    if (static_cast<int>(threadIdx.x) < st) red[threadIdx.x] += red[threadIdx.x + st];
    __syncthreads();
  }
  if (threadIdx.x != 0) return;
  const double sq = red[0];
  double fit;
  if (a.x_norm == 0.0) {
    fit = 1.0;
  } else {
    const double mu = sq / static_cast<double>(a.phat);
    fit = 1.0 - sqrt(a.total * mu) / a.x_norm;
  }
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
    if (a.stop_host_mapped) reinterpret_cast<volatile int*>(a.stop_host_mapped)[a.iteration] = 1;
  }
}

}  // namespace ph
}  // namespace cpb
