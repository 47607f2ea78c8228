// QR path of the sampled least-squares step: the reference's algorithm
// (least_squares, kr_linalg.hpp:105-118: Eigen ColPivHouseholderQR with
// threshold max(S,R)*eps, CompleteOrthogonalDecomposition when rank
// deficient) restated on the device for the modes whose normal equations
// are not accurate enough.
//
// The fast path solves the normal equations (Gram Z^T Z, Gauss-Jordan
// inverse). Their forward error grows like cond(Z)^2 * eps, so when a
// Gauss-Jordan pivot falls below kNeTol * max diag(G) (cond(Z) beyond about
// 1e3) the mode switches to this path:
//
//  1. qr_factor (one CTA): column-pivoted Householder QR of Z_S (S x r) with
//     Eigen's pivot order, norm downdates and rank rule (oracle PivQR,
//     cprand_oracle.cpp), then COD's RZ step when rank < r. The result is
//     compiled into two r x r matrices so that the solution row of factor
//     row i is linear in the sampled fiber values b = X_S(i, :):
//        c = (Q^T b)[0:r] = b[0:r] - V0 T^T (V^T b)        (compact WY:
//            Q = H_0 ... H_{r-1} = I - V T V^T, V0 = V[0:r, :])
//        x = L c  (L = P R11^-1, or the COD minimum-norm map)
//     so x^T = b[0:r]^T L^T - (V^T b)^T K L^T with K = T V0^T.
//  2. qr_rows (every CTA of the apply phase): for its factor rows, w = V^T b
//     by one pass over the sampled fibers, then c and x as above. The rows
//     replace the RHS rows of the fast path and ginv is set to the identity,
//     so the apply / normalize code downstream is unchanged.
//
// Workspace (doubles, qr_ws_doubles): V [S][RT] row-major (zero padded,
// unit diagonal), the column-major working copy M [RT][S], K [RT][RT],
// LT = L^T [RT][RT], T [RT][RT], scratch [RT][RT].
#pragma once

#include <cfloat>

#include "phases.cuh"

namespace cpb {
namespace ph {

struct QrPtrs {
  double *V, *M, *K, *LT, *T, *X;
};
__device__ __forceinline__ QrPtrs qr_ptrs(double* ws, int s, int rt) {
  QrPtrs p;
  p.V = ws;
  p.M = ws + static_cast<i64>(s) * rt;
  p.K = p.M + static_cast<i64>(s) * rt;
  p.LT = p.K + rt * rt;
  p.T = p.LT + rt * rt;
  p.X = p.T + rt * rt;
  return p;
}

// shared memory qr_factor needs (doubles)
template <int RT>
__host__ __device__ constexpr int qr_factor_smem_doubles() {
  return GS * RT + RT * (RT + 1) + 4 * RT + 64;
}

template <int NTH>
__device__ __forceinline__ double block_sum(double v, double* red) {
  constexpr int NW = NTH / 32;
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();  // red may still be read by a previous call
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double t = 0.0;
#pragma unroll
  for (int w = 0; w < NW; ++w) t += red[w];
  return t;
}

// Column-pivoted Householder QR of z (S x r, row-major ld RT) + COD, compiled
// into V, K, LT (see above). One CTA of 256 threads. Sets ginv (r x r) to the
// identity, info[0] = numerical rank, info[1] += 1, info[2] = 1 (QR mode).
// sh: qr_factor_smem_doubles<RT>().
template <int RT>
__device__ void qr_factor(const double* z, int s, int r, double qtol, double* ws, double* ginv, int* info,
                          double* sh) {
  constexpr int NTH = 256, NW = NTH / 32, LDR = RT + 1;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const QrPtrs P = qr_ptrs(ws, s, RT);
  double* gsh = sh;                     // GS x RT (gram_chunk staging)
  double* upd = sh + GS * RT;           // RT
  double* dir = upd + RT;               // RT
  double* hc = dir + RT;                // RT: tau_k
  int* perm = reinterpret_cast<int*>(hc + RT);  // RT ints
  double* red = hc + RT + RT / 2 + 1;   // NW
  double* Rt = sh + GS * RT + 4 * RT + 64;  // [RT][RT+1] top r x r block of M (after the sweep)
  __shared__ int s_big, s_nz, s_rank;
  __shared__ double s_maxpivot, s_thr_helper;
  const double eps = DBL_EPSILON;
  // ---- M = Z[:, 0:r] column-major
  for (i64 e = tid; e < static_cast<i64>(s) * r; e += NTH) {
    const int j = static_cast<int>(e / s);
    const i64 i = e - static_cast<i64>(j) * s;
    P.M[static_cast<i64>(j) * s + i] = __ldcg(z + i * RT + j);
  }
  if (tid < RT) perm[tid] = tid;
  __syncthreads();
  for (int j = warp; j < r; j += NW) {
    const double* c = P.M + static_cast<i64>(j) * s;
    double a = 0.0;
    for (int i = lane; i < s; i += 32) a += c[i] * c[i];
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (lane == 0) dir[j] = upd[j] = sqrt(a);
  }
  __syncthreads();
  if (tid == 0) {
    double mx = 0.0;
    for (int j = 0; j < r; ++j) mx = fmax(mx, upd[j]);
    s_thr_helper = (mx * eps) * (mx * eps) / static_cast<double>(s);
    s_nz = r;
    s_maxpivot = 0.0;
  }
  __syncthreads();
  // ---- the sweep (oracle PivQR::compute; Eigen ColPivHouseholderQR)
  for (int k = 0; k < r; ++k) {
    if (tid == 0) {
      int big = k;
      for (int j = k + 1; j < r; ++j)
        if (upd[j] > upd[big]) big = j;
      const double big_sq = upd[big] * upd[big];
      if (s_nz == r && big_sq < s_thr_helper * static_cast<double>(s - k)) s_nz = k;
      if (big != k) {
        double t = upd[k]; upd[k] = upd[big]; upd[big] = t;
        t = dir[k]; dir[k] = dir[big]; dir[big] = t;
        const int q = perm[k]; perm[k] = perm[big]; perm[big] = q;
      }
      s_big = big;
    }
    __syncthreads();
    const int big = s_big;
    double* ck = P.M + static_cast<i64>(k) * s;
    if (big != k) {
      double* cb = P.M + static_cast<i64>(big) * s;
      for (int i = tid; i < s; i += NTH) {
        const double t = ck[i];
        ck[i] = cb[i];
        cb[i] = t;
      }
      __syncthreads();
    }
    // Householder vector of column k, rows k..s-1 (make_householder)
    double tl = 0.0;
    for (int i = k + 1 + tid; i < s; i += NTH) tl += ck[i] * ck[i];
    const double tail = block_sum<NTH>(tl, red);
    const double c0 = ck[k];
    double tau, beta;
    if (tail <= DBL_MIN) {
      tau = 0.0;
      beta = c0;
      for (int i = k + 1 + tid; i < s; i += NTH) ck[i] = 0.0;
    } else {
      beta = sqrt(c0 * c0 + tail);
      if (c0 >= 0.0) beta = -beta;
      const double den = c0 - beta;
      for (int i = k + 1 + tid; i < s; i += NTH) ck[i] /= den;
      tau = (beta - c0) / beta;
    }
    __syncthreads();
    if (tid == 0) {
      ck[k] = beta;
      hc[k] = tau;
      if (fabs(beta) > s_maxpivot) s_maxpivot = fabs(beta);
    }
    // apply H_k to columns j > k (a warp per column) and downdate their norms
    // (M lives in global memory, S x r doubles: a warp's columns are taken CB
    // at a time and U rows per lane per pass, so CB * U + U loads are in
    // flight instead of two; every lane still adds its own rows in ascending
    // order, so the sums are the ones the one-column loop formed)
    constexpr int CB = 4, U = 4;
    double ckjs[((RT + NW - 1) / NW + CB - 1) / CB * CB];
    if (tau != 0.0) {
      for (int jb = k + 1 + warp, q0 = 0; jb < r; jb += NW * CB, q0 += CB) {
        double* cjp[CB];
        double t[CB];
#pragma unroll
        for (int c = 0; c < CB; ++c) {
          const int j = jb + NW * c;
          cjp[c] = P.M + static_cast<i64>(j < r ? j : jb) * s;
          t[c] = 0.0;
        }
        for (int i0 = k + 1 + lane; i0 < s; i0 += 32 * U) {
          double a[U], b[CB][U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int i = i0 + 32 * u;
            a[u] = i < s ? ck[i] : 0.0;
#pragma unroll
            for (int c = 0; c < CB; ++c) b[c][u] = i < s ? cjp[c][i] : 0.0;
          }
#pragma unroll
          for (int u = 0; u < U; ++u)
            if (i0 + 32 * u < s)
#pragma unroll
              for (int c = 0; c < CB; ++c) t[c] += a[u] * b[c][u];
        }
#pragma unroll
        for (int c = 0; c < CB; ++c) {
          for (int o = 16; o > 0; o >>= 1) t[c] += __shfl_xor_sync(0xffffffffu, t[c], o);
          const double ckj0 = cjp[c][k];
          t[c] = (t[c] + ckj0) * tau;
          ckjs[q0 + c] = ckj0 - t[c];
        }
        for (int i0 = k + 1 + lane; i0 < s; i0 += 32 * U) {
          double a[U], b[CB][U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int i = i0 + 32 * u;
            a[u] = i < s ? ck[i] : 0.0;
#pragma unroll
            for (int c = 0; c < CB; ++c) b[c][u] = i < s ? cjp[c][i] : 0.0;
          }
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int i = i0 + 32 * u;
            if (i < s)
#pragma unroll
              for (int c = 0; c < CB; ++c)
                if (jb + NW * c < r) cjp[c][i] = b[c][u] - t[c] * a[u];
          }
        }
        __syncwarp();
        if (lane == 0)
#pragma unroll
          for (int c = 0; c < CB; ++c)
            if (jb + NW * c < r) cjp[c][k] = ckjs[q0 + c];
      }
    }
    for (int j = k + 1 + warp, q = 0; j < r; j += NW, ++q) {
      double* cj = P.M + static_cast<i64>(j) * s;
      const double ckj = tau != 0.0 ? ckjs[q] : cj[k];
      const double u = upd[j];
      if (u != 0.0) {
        double t = fabs(ckj) / u;
        t = (1.0 + t) * (1.0 - t);
        t = t < 0.0 ? 0.0 : t;
        const double ratio = u / dir[j];
        const double t2 = t * ratio * ratio;
        if (t2 <= sqrt(eps)) {
          double a = 0.0;
          for (int i = k + 1 + lane; i < s; i += 32) a += cj[i] * cj[i];
          for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
          __syncwarp();
          if (lane == 0) dir[j] = upd[j] = sqrt(a);
        } else if (lane == 0) {
          upd[j] = u * sqrt(t);
        }
      }
    }
    __syncthreads();
  }
  // ---- rank (PivQR::rank) and the top r x r block in shared memory
  if (tid == 0) {
    const double pre = fabs(s_maxpivot) * qtol;
    int rk = 0;
    for (int i = 0; i < s_nz; ++i) rk += fabs(P.M[static_cast<i64>(i) * s + i]) > pre;
    s_rank = rk;
  }
  __syncthreads();
  const int rk = s_rank;
  // ---- V row-major (unit diagonal, zeros above), consumed by qr_rows
  for (i64 e = tid; e < static_cast<i64>(s) * RT; e += NTH) {
    const i64 i = e / RT;
    const int j = static_cast<int>(e - i * RT);
    double v = 0.0;
    if (j < r) v = i < j ? 0.0 : (i == j ? 1.0 : P.M[static_cast<i64>(j) * s + i]);
    P.V[e] = v;
  }
  __syncthreads();
  // VtV (RT x RT) -> X, by the Gram routine
  gram_chunk<RT>(P.V, 0, s, P.X, gsh);
  __syncthreads();
  for (int e = tid; e < RT * LDR; e += NTH) {
    const int i = e / LDR, j = e - i * LDR;
    Rt[e] = (i < r && j < r) ? P.M[static_cast<i64>(j) * s + i] : 0.0;
  }
  // T (compact WY, forward): T_kk = tau_k, T[0:k, k] = -tau_k T[0:k,0:k] VtV[0:k, k]
  for (int e = tid; e < RT * RT; e += NTH) P.T[e] = 0.0;
  __syncthreads();
  for (int k = 0; k < r; ++k) {
    if (tid < k) {
      double t = 0.0;
      for (int m = tid; m < k; ++m) t += P.T[tid * RT + m] * P.X[m * RT + k];
      P.T[tid * RT + k] = -hc[k] * t;
    } else if (tid == k) {
      P.T[k * RT + k] = hc[k];
    }
    __syncthreads();
  }
  // K = T V0^T: K[j][c] = sum_m T[j][m] V[c][m]
  for (int e = tid; e < RT * RT; e += NTH) {
    const int j = e / RT, c = e - j * RT;
    double t = 0.0;
    if (j < r && c < r)
      for (int m = j; m < r; ++m) t += P.T[j * RT + m] * P.V[static_cast<i64>(c) * RT + m];
    P.K[e] = t;
  }
  // ---- COD's RZ reduction of rows [0, rk) when rank deficient (oracle COD::compute)
  if (rk < r && tid == 0) {
    double* zc = hc;  // tau no longer needed: zcoeffs
    for (int k = rk - 1; k >= 0; --k) {
      if (k != rk - 1)
        for (int i = 0; i <= k; ++i) {
          const double t = Rt[i * LDR + k]; Rt[i * LDR + k] = Rt[i * LDR + rk - 1]; Rt[i * LDR + rk - 1] = t;
        }
      // make_householder over [X(k, rk-1), X(k, rk..r)]
      const int n = r - rk + 1;
      double tail = 0.0;
      for (int q = 1; q < n; ++q) tail += Rt[k * LDR + rk - 1 + q] * Rt[k * LDR + rk - 1 + q];
      const double x0 = Rt[k * LDR + rk - 1];
      double tau, beta;
      if (tail <= DBL_MIN) {
        tau = 0.0;
        beta = x0;
        for (int q = 1; q < n; ++q) Rt[k * LDR + rk - 1 + q] = 0.0;
      } else {
        beta = sqrt(x0 * x0 + tail);
        if (x0 >= 0.0) beta = -beta;
        for (int q = 1; q < n; ++q) Rt[k * LDR + rk - 1 + q] /= (x0 - beta);
        tau = (beta - x0) / beta;
      }
      Rt[k * LDR + rk - 1] = beta;
      zc[k] = tau;
      if (k > 0 && tau != 0.0)
        for (int i = 0; i < k; ++i) {
          double t = Rt[i * LDR + rk - 1];
          for (int j = rk; j < r; ++j) t += Rt[i * LDR + j] * Rt[k * LDR + j];
          t *= tau;
          Rt[i * LDR + rk - 1] -= t;
          for (int j = rk; j < r; ++j) Rt[i * LDR + j] -= t * Rt[k * LDR + j];
        }
      if (k != rk - 1)
        for (int i = 0; i <= k; ++i) {
          const double t = Rt[i * LDR + k]; Rt[i * LDR + k] = Rt[i * LDR + rk - 1]; Rt[i * LDR + rk - 1] = t;
        }
    }
  }
  __syncthreads();
  // ---- L: column j = the solve applied to e_j (PivQR::solve / COD::solve),
  // LT[j][perm[i]] = dst(i); columns j >= rank are zero
  for (int e = tid; e < RT * RT; e += NTH) P.LT[e] = 0.0;
  __syncthreads();
  if (tid < rk) {
    const int j = tid;
    double* dst = P.X + static_cast<i64>(j) * RT;  // VtV no longer needed: one row per thread
    for (int i = 0; i < RT; ++i) dst[i] = 0.0;
    for (int i = rk - 1; i >= 0; --i) {
      double sum = (i == j) ? 1.0 : 0.0;
      for (int k = i + 1; k < rk; ++k) sum -= Rt[i * LDR + k] * dst[k];
      dst[i] = sum / Rt[i * LDR + i];
    }
    if (rk < r)
      for (int k = 0; k < rk; ++k) {
        const double tau = hc[k];
        if (tau == 0.0) continue;
        double t = dst[k];
        for (int i = rk; i < r; ++i) t += Rt[k * LDR + i] * dst[i];
        t *= tau;
        dst[k] -= t;
        for (int i = rk; i < r; ++i) dst[i] -= t * Rt[k * LDR + i];
      }
    for (int i = 0; i < r; ++i) P.LT[j * RT + perm[i]] = dst[i];
  }
  for (int e = tid; e < r * r; e += NTH) ginv[e] = (e / r == e % r) ? 1.0 : 0.0;
  if (tid == 0) {
    info[0] = rk;
    info[1] += 1;  // fallback count (diagnostics)
    info[2] = 1;   // QR mode: the apply takes its rows from qr_rows
  }
  __threadfence();
  __syncthreads();
}

template <int RT, int NTH>
__host__ __device__ constexpr int qr_rows_smem_doubles() {
  return (NTH / RT) * 33 + 32 * RT > 2 * (NTH / RT) * (RT + 1) ? (NTH / RT) * 33 + 32 * RT
                                                               : 2 * (NTH / RT) * (RT + 1);
}

// Solution rows i0 .. i0 + nrow - 1 (nrow <= NTH / RT) of the QR path into
// out[il * ldo + c], c < r (rows outside the matrix are not written). stage: qr_rows_smem_doubles.
template <int RT, int NTH>
__device__ void qr_rows(const QrSrc& q, const double* ws, int r, i64 in, i64 i0, int nrow, double* out, int ldo,
                        double* stage) {
  constexpr int BI = NTH / RT, SC = 32, LX = SC + 1, LR = RT + 1;
  const int tid = threadIdx.x, il = tid / RT, c = tid % RT;
  const QrPtrs P = qr_ptrs(const_cast<double*>(ws), q.s, RT);
  const i64 i = i0 + il;
  const bool ok = il < nrow && i < in;
  double* xb = stage;           // [BI][LX]
  double* vb = stage + BI * LX; // [SC][RT]
  auto xat = [&](int s_, i64 row) { return __ldcg(q.x + (q.row_off ? __ldg(q.row_off + s_) : s_ * q.ld) + row * q.est); };
  // w = V^T b, one pass over the sampled fibers (SC samples per stage)
  double acc = 0.0;
  for (int s0 = 0; s0 < q.s; s0 += SC) {
    for (int e = tid; e < BI * SC; e += NTH) {
      const int a = e % BI, sl = e / BI, ss = s0 + sl;
      const i64 ii = i0 + a;
      xb[a * LX + sl] = (a < nrow && ii < in && ss < q.s) ? xat(ss, ii) : 0.0;
    }
    for (int e = tid; e < SC * RT; e += NTH) {
      const int ss = s0 + e / RT;
      vb[e] = ss < q.s ? __ldcg(P.V + static_cast<i64>(ss) * RT + (e % RT)) : 0.0;
    }
    __syncthreads();
#pragma unroll 8
    for (int sl = 0; sl < SC; ++sl) acc = fma(xb[il * LX + sl], vb[sl * RT + c], acc);
    __syncthreads();
  }
  double* wv = stage;             // [BI][LR]
  double* cf = stage + BI * LR;   // [BI][LR]
  wv[il * LR + c] = (ok && c < r) ? acc : 0.0;
  __syncthreads();
  // c = b[0:r] - w^T K
  double cv = 0.0;
  if (ok && c < r) {
    cv = xat(c, i);
    for (int k = 0; k < r; ++k) cv -= wv[il * LR + k] * __ldcg(P.K + k * RT + c);
  }
  cf[il * LR + c] = cv;
  __syncthreads();
  // x = c^T L^T
  double xv = 0.0;
  if (ok && c < r)
    for (int k = 0; k < r; ++k) xv = fma(cf[il * LR + k], __ldcg(P.LT + k * RT + c), xv);
  if (ok && c < r) out[il * ldo + c] = xv;
  __syncthreads();
}

// apply_block (phases.cuh) in QR mode: the block's BI = NTH / RT factor
// rows from qr_rows (ginv is the identity then, so they are the rows of
// A_un); writes A_un and returns this thread's out^2. rh: BI x (RT+1),
// stage: qr_rows_smem_doubles.
template <int RT, int NTH>
__device__ double apply_block_qr(i64 in, int r, const ModeWork& w, i64 i0, double* rh, double* stage) {
  constexpr int LD = RT + 1, BI = NTH / RT;
  qr_rows<RT, NTH>(w.q, w.qrws, r, in, i0, BI, rh, LD, stage);
  const int il = threadIdx.x / RT, c = threadIdx.x % RT;
  const i64 i = i0 + il;
  const bool ok = i < in && c < r;
  const double out = ok ? rh[il * LD + c] : 0.0;
  if (ok) w.a[i * r + c] = out;
  __syncthreads();
  return ok ? out * out : 0.0;
}

}  // namespace ph
}  // namespace cpb
