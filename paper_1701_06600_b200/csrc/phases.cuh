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

#include "devutil.cuh"
#include "kernels.cuh"

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
    double a = __ldg(v.fac[c] + static_cast<i64>(row) * v.r + rr);
    if (v.nrm[c]) a = a / __ldg(v.nrm[c] + rr);
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
  if (tid == 0) info[0] = rank;
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
  {  // G = sum of the split partials in split order, 4 partials per batch
    int k = 0;
    for (; k + 4 <= nparts; k += 4) {
      double v[4][TR][TC];
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int t = 0; t < TR; ++t)
#pragma unroll
          for (int u = 0; u < TC; ++u)
            v[x][t][u] = (row[t] < r && col[u] < r) ? part[static_cast<i64>(k + x) * RT * RT + row[t] * RT + col[u]]
                                                    : 0.0;
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int t = 0; t < TR; ++t)
#pragma unroll
          for (int u = 0; u < TC; ++u) a[t][u] += v[x][t][u];
    }
    for (; k < nparts; ++k)
#pragma unroll
      for (int t = 0; t < TR; ++t)
#pragma unroll
        for (int u = 0; u < TC; ++u)
          if (row[t] < r && col[u] < r) a[t][u] += part[static_cast<i64>(k) * RT * RT + row[t] * RT + col[u]];
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
  if (!fail) {
#pragma unroll
    for (int t = 0; t < TR; ++t)
#pragma unroll
      for (int u = 0; u < TC; ++u)
        if (row[t] < r && col[u] < r) ginv[row[t] * r + col[u]] = a[t][u];
  }
  if (tid == 0) info[0] = fail ? -1 : r;
  __syncthreads();
  return fail;
}

// ------------------------------------------------------------ RHS GEMM
// part[kb](i, c) = sum_{s in split kb} X_S(s, i) Z(s, c) for the 128-row
// tile mt: 256 threads, 8 x RT/16 register tile (columns strided by 16 for
// conflict-free loads), 3-stage cp.async pipeline. A rows at
// xs + row_off[s] (fibers read in place) or xs + s * ld (gathered X_S).
// sh: GSTAGES * GBK * (GBM + RT) doubles.
constexpr int GBM = 128, GBK = 16, GSTAGES = 3;

template <int RT, bool VEC16>
__device__ void gemm_tile(const double* __restrict__ xs, i64 ld, const i64* __restrict__ row_off,
                          const double* __restrict__ z, i64 in, int s_total, int r, int ks_len,
                          double* __restrict__ part, int mt, int kb, double* sh) {
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
        cp_async8(ab + sl * GBM + ic, ok ? xs + ro + i : xs, ok ? 8 : 0);
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
    gi[x * (RT + 1) + y] = (x < r && y < r) ? ginv[x * r + y] : 0.0;
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
      s = rhs_full[i * r + c];
    } else {
      const double* p = w.part_rhs + i * r + c;
      const i64 step = in * r;
      int k = 0;
      for (; k + 6 <= w.ks; k += 6) {
        const double v0 = p[k * step], v1 = p[(k + 1) * step], v2 = p[(k + 2) * step];
        const double v3 = p[(k + 3) * step], v4 = p[(k + 4) * step], v5 = p[(k + 5) * step];
        s = (((((s + v0) + v1) + v2) + v3) + v4) + v5;
      }
      for (; k < w.ks; ++k) s += p[k * step];
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
// red: (NTH / RT) x (RT + 1) doubles.
template <int RT, int NTH>
__device__ void norms_final(int r, i64 in, const ModeWork& w, int nparts, int first_of_pass,
                            unsigned long long* rng_state, double* red) {
  constexpr int NP = NTH / RT;
  const int tid = threadIdx.x, part = tid / RT, c = tid % RT;
  __shared__ int s_zero;
  double q = 0.0;
  if (c < r)
    for (int b = part; b < nparts; b += NP) q += w.ssq[static_cast<i64>(b) * r + c];
  red[part * (RT + 1) + c] = q;
  if (tid == 0) s_zero = 0;
  __syncthreads();
  if (tid < r) {
    double t = 0.0;
    for (int x = 0; x < NP; ++x) t += red[x * (RT + 1) + tid];
    const double nrm = sqrt(t);
    w.norms[tid] = nrm;
    if (nrm == 0.0) {
      w.lambda[tid] = 0.0;
      atomicOr(&s_zero, 1);
    } else {
      w.lambda[tid] = first_of_pass ? w.lambda[tid] * nrm : nrm;
    }
  }
  __syncthreads();
  if (tid == 0 && s_zero) {
    // zero columns (kruskal.hpp:57-63): N(0,1) column from the normalize
    // stream, one distribution object per call, columns in order
    DevMt g{rng_state};
    DevNormal gauss;
    for (int col = 0; col < r; ++col) {
      if (w.norms[col] != 0.0) continue;
      for (i64 t = 0; t < in; ++t) w.a[t * r + col] = gauss(g);
      w.norms[col] = dev_stable_norm(w.a + col, in, r);
    }
  }
  __syncthreads();
}

// ------------------------------------------------------------ fit
// Squared error over the 256 sampled entries of virtual block vb (one
// thread per entry, fixed tree reduction); model_entry kruskal.hpp:37-44.
// red: 256 doubles. Result valid in thread 0.
__device__ inline double fit_block(const FitArgs& a, i64 vb, double* red) {
  const i64 j = vb * 256 + threadIdx.x;
  double e2 = 0.0;
  if (j < a.phat) {
    double sum = 0.0;
    for (int q = 0; q < a.r; ++q) {
      double p = a.lambda[q];
      for (int n = 0; n < a.order; ++n) {
        double f = a.fac[n][static_cast<i64>(a.idx[n][j]) * a.r + q];
        if (a.nrm[n]) f = f / a.nrm[n][q];
        p = __dmul_rn(p, f);
      }
      sum = __dadd_rn(sum, p);
    }
    const double e = a.values[j] - sum;
    e2 = e * e;
  }
  red[threadIdx.x] = e2;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  const double out = red[0];
  __syncthreads();
  return out;
}

// Fit from the block partials (in order), sampling.hpp:192,207-209, and the
// stop rule should_stop (sampling.hpp:237-251); one thread.
__device__ inline void fit_final(const FitArgs& a, i64 nblocks) {
  double sq = 0.0;
  for (i64 b = 0; b < nblocks; ++b) sq += a.partials[b];
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
    if (a.stop_host_mapped) *reinterpret_cast<volatile int*>(a.stop_host_mapped) = 1;
  }
}

}  // namespace ph
}  // namespace cpb
