// Measured-and-dropped Gram inverse variants with 8 x 8 pivot blocks (the
// product uses ph::inverse_la, 4 x 4 pivots with look-ahead; phases.cuh).
// Kept for tests/micro/inv_bench.cu only: 11.9 us (inverse_b8) against
// 10.3 us for the product's inverse on C4's 50 x 50 Gram.
#pragma once
#include "phases.cuh"

namespace cpb {
namespace ph {

// ------------------------------------------- Gram inverse, 8-wide steps
// Unpivoted 8 x 8 Gauss-Jordan inverse by one warp: lane l holds
// p[0] = P(l/4, l%4) and p[1] = P(l/4, l%4 + 4), in and out. ok = false
// when a pivot is <= thr (or not positive).
__device__ __forceinline__ void inv8_warp(double (&p)[2], double thr, bool& ok) {
  const int l = threadIdx.x & 31, x = l >> 2, y = l & 3;
  ok = true;
#pragma unroll 1
  for (int k = 0; k < 8; ++k) {
    const int ks = k >> 2, kl = k & 3;
    const double pk0 = __shfl_sync(0xffffffffu, p[0], k * 4 + kl);
    const double pk1 = __shfl_sync(0xffffffffu, p[1], k * 4 + kl);
    const double rk0 = __shfl_sync(0xffffffffu, p[0], k * 4 + y);
    const double rk1 = __shfl_sync(0xffffffffu, p[1], k * 4 + y);
    const double cx0 = __shfl_sync(0xffffffffu, p[0], x * 4 + kl);
    const double cx1 = __shfl_sync(0xffffffffu, p[1], x * 4 + kl);
    const double pkk = ks ? pk1 : pk0;
    if (!(pkk > thr) || !(pkk > 0.0)) ok = false;
    const double q = rcp_nr(pkk);
    const double ck = (x == k) ? -1.0 : (ks ? cx1 : cx0);
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int col = y + 4 * e;
      const double rkv = (col == k) ? q : (e ? rk1 : rk0) * q;
      const double xv = (x == k || col == k) ? 0.0 : p[e];
      p[e] = fma(-ck, rkv, xv);
    }
  }
}

// Block Gauss-Jordan inverse with 8 x 8 pivot blocks (no pivoting: the Gram
// is SPD, padded to a multiple of 8 with d_max on the padding diagonal) by
// one CTA of 256 threads, one barrier per step; step s pivots on tile s.
//  * Warp w holds 8-column tile w as FP64 MMA accumulator fragments (every
//    8-row tile) and does step s as two m8n8k4 MMAs per tile:
//    a' = X + (-C) M, X = a with rows/columns K zeroed, -C(i) = -a(i, K)
//    (+e on rows K) from the published column block, M(j) = P^-1 a(K, j)
//    from the published row block whose K columns hold the identity: the
//    four Gauss-Jordan block rules in one form.
//  * After its MMAs each warp publishes its part of the next row block
//    (identity on the next K) and the raw row block after it; the owner of
//    the next column tile publishes -C; rows/columns of the next K are
//    zeroed in the fragments. The step loop is unrolled (compile-time tiles).
//  * Warp 7 (first, when it also owns a tile) forms the next pivot block from
//    the raw rows and inverts it (inv8_warp), off the workers' critical path.
// g: RT x RT Gram (ld RT; entries outside [0, r) ignored). Returns true
// (uniformly) on a pivot <= tol * d_max, after writing the Gram to gfull
// (r x r) for the pivoted fallback. sh: 48 RT + 256 doubles.
template <int RT>
__device__ bool inverse_b8(const double* __restrict__ g, int r, double tol, double* __restrict__ ginv,
                           double* __restrict__ gfull, int* info, double* sh,
                           unsigned long long* stamps = nullptr) {
  constexpr int NTI = RT / 8;
  static_assert(NTI <= 8, "one 8-column tile per warp");
  double* rbs = sh;              // [2][16][RT] rows K_s (identity on K_s columns), raw rows K_{s+1}
  double* cbs = rbs + 32 * RT;   // [2][RT][8]  -a(i, K_s), +e on rows K_s
  double* pin = cbs + 16 * RT;   // [2][64]     inverse of the pivot block of step s
  double* mtmp = pin + 128;      // [64]        look-ahead scratch
  double* misc = mtmp + 64;      // [2..3] fail flags, [4..5] warp maxima
  const int tid = threadIdx.x, w = tid / 32, l = tid % 32;
  const int lr = l >> 2, lc = (l & 3) * 2, lk = l & 3;
  const int r8 = (r + 7) & ~7;
  const int nt = r8 / 8;
  const bool worker = w < nt;  // warp w owns 8-column tile w
  double acc[NTI][2];
#pragma unroll
  for (int mt = 0; mt < NTI; ++mt) {
    const int row = mt * 8 + lr, col = w * 8 + lc;
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
  CPB_INV_STAMP(1);
  if (worker) {
#pragma unroll
    for (int mt = 0; mt < NTI; ++mt) {
      const int row = mt * 8 + lr;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int col = w * 8 + lc + e;
        if (row < r && col < r) gfull[row * r + col] = acc[mt][e];
        if (row == col && row >= r && row < r8) acc[mt][e] = dmax;  // padding diagonal
      }
    }
  }
  // publish step n's blocks (tile n; runtime n, fragments selected by
  // compile-time tile loops so nothing is indexed dynamically)
  auto publish = [&](const int n, double* rb, double* cb) {
    if (!worker) return;  // warp-uniform
    const bool own = (w == n);
#pragma unroll
    for (int mt = 0; mt < NTI; ++mt) {
      const int row = mt * 8 + lr;
      if (own) {
        double2 o;
        o.x = (mt == n) ? (lr == lc ? 1.0 : 0.0) : -acc[mt][0];
        o.y = (mt == n) ? (lr == lc + 1 ? 1.0 : 0.0) : -acc[mt][1];
        *reinterpret_cast<double2*>(cb + row * 8 + lc) = o;
      }
      if (mt == n) {
        double2 o;
        o.x = own ? (lr == lc ? 1.0 : 0.0) : acc[mt][0];
        o.y = own ? (lr == lc + 1 ? 1.0 : 0.0) : acc[mt][1];
        *reinterpret_cast<double2*>(rb + lr * RT + w * 8 + lc) = o;
      }
      if (mt == n + 1 && mt < nt)
        *reinterpret_cast<double2*>(rb + (8 + lr) * RT + w * 8 + lc) = make_double2(acc[mt][0], acc[mt][1]);
      if (mt == n || own) acc[mt][0] = acc[mt][1] = 0.0;
    }
  };
  // raw first pivot block (tile 0 of warp 0) for warp 7
  if (w == 0) *reinterpret_cast<double2*>(mtmp + lr * 8 + lc) = make_double2(acc[0][0], acc[0][1]);
  publish(0, rbs, cbs);
  __syncthreads();
  if (w == 7) {
    double p[2] = {mtmp[lr * 8 + lk], mtmp[lr * 8 + lk + 4]};
    bool ok;
    inv8_warp(p, thr, ok);
    pin[lr * 8 + lk] = p[0];
    pin[lr * 8 + lk + 4] = p[1];
    if (l == 0) misc[2] = ok ? 0.0 : 1.0;
  }
  __syncthreads();
  CPB_INV_STAMP(2);
  if (stamps && tid == 0) stamps[0] = globaltimer();
  bool fail = false;
#pragma unroll 1
  for (int s = 0; s < nt; ++s) {
    CPB_INV_STAMP(3 + s);
    const int pb = s & 1;
    if (misc[2 + pb] != 0.0) {
      fail = true;  // uniform
      break;
    }
    const double* P = pin + 64 * pb;
    const double* rb = rbs + pb * 16 * RT;
    const double* cb = cbs + pb * RT * 8;
    if (w == 7 && s + 1 < nt) {
      // look-ahead: pivot block of step s+1 = rows/columns of tile s+1 after step s
      const int k0 = 8 * s, k1 = 8 * (s + 1);
      {  // M_q(j) = sum_t P(q, t) a(K_t, j) for q = l/4, j = k1 + l%4 (+4)
        const int q = lr;
        double m0 = 0.0, m1 = 0.0;
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          const double pq = P[q * 8 + t];
          m0 = fma(pq, rb[t * RT + k1 + lk], m0);
          m1 = fma(pq, rb[t * RT + k1 + lk + 4], m1);
        }
        mtmp[q * 8 + lk] = m0;
        mtmp[q * 8 + lk + 4] = m1;
      }
      __syncwarp();
      double p[2];
      {
        const double* rn = rb + (8 + lr) * RT;  // raw row k1 + x
        double v0 = rn[k1 + lk], v1 = rn[k1 + lk + 4];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const double c = rn[k0 + q];
          v0 = fma(-c, mtmp[q * 8 + lk], v0);
          v1 = fma(-c, mtmp[q * 8 + lk + 4], v1);
        }
        p[0] = v0;
        p[1] = v1;
      }
      bool ok;
      CPB_INV_STAMP_AT(43, s, l == 0);
      inv8_warp(p, thr, ok);
      CPB_INV_STAMP_AT(44, s, l == 0);
      pin[64 * (pb ^ 1) + lr * 8 + lk] = p[0];
      pin[64 * (pb ^ 1) + lr * 8 + lk + 4] = p[1];
      if (l == 0) misc[2 + (pb ^ 1)] = ok ? 0.0 : 1.0;
      __syncwarp();
    }
    if (worker) {
      // all fragment operands are loaded before the first MMA
      double pr0[8], pr1[8];  // rows l%4 and l%4 + 4 of P^-1
#pragma unroll
      for (int t = 0; t < 8; t += 2) {
        const double2 a = *reinterpret_cast<const double2*>(P + lk * 8 + t);
        const double2 c = *reinterpret_cast<const double2*>(P + (lk + 4) * 8 + t);
        pr0[t] = a.x;
        pr0[t + 1] = a.y;
        pr1[t] = c.x;
        pr1[t + 1] = c.y;
      }
      const int j = w * 8 + lr;  // B fragment (k = l % 4 (+4), n = l / 4)
      double bm0 = 0.0, bm1 = 0.0;
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const double rv = rb[t * RT + j];
        bm0 = fma(pr0[t], rv, bm0);
        bm1 = fma(pr1[t], rv, bm1);
      }
      double am[NTI][2];
#pragma unroll
      for (int mt = 0; mt < NTI; ++mt) {
        am[mt][0] = cb[(mt * 8 + lr) * 8 + lk];
        am[mt][1] = cb[(mt * 8 + lr) * 8 + lk + 4];
      }
#pragma unroll
      for (int mt = 0; mt < NTI; ++mt) {
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(acc[mt][0]), "+d"(acc[mt][1])
                     : "d"(am[mt][0]), "d"(bm0));
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(acc[mt][0]), "+d"(acc[mt][1])
                     : "d"(am[mt][1]), "d"(bm1));
      }
      CPB_INV_STAMP_AT(41, s, tid == 0);
      if (s + 1 < nt) publish(s + 1, rbs + (pb ^ 1) * 16 * RT, cbs + (pb ^ 1) * RT * 8);
    }
    CPB_INV_STAMP_AT(42, s, tid == 0);
    CPB_INV_STAMP_AT(45, s, tid == 224);
    __syncthreads();
  }
  CPB_INV_STAMP(30);
  if (stamps && tid == 0) stamps[1] = globaltimer();
  if (!fail && worker) {
#pragma unroll
    for (int mt = 0; mt < NTI; ++mt) {
      const int row = mt * 8 + lr, col = w * 8 + lc;
      if (mt >= nt || row >= r) continue;
      if (col + 1 < r && !(r & 1))
        *reinterpret_cast<double2*>(ginv + row * r + col) = make_double2(acc[mt][0], acc[mt][1]);
      else {
        if (col < r) ginv[row * r + col] = acc[mt][0];
        if (col + 1 < r) ginv[row * r + col + 1] = acc[mt][1];
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

// ------------------------------------------ Gram inverse, 8-wide steps
// 8 x 8 inverse of a pivot block P (row-major, shared memory) by one warp,
// through its 4 x 4 blocks [A B; C D]: A^-1 and the Schur complement
// S = D - C A^-1 B by cofactors (inv4_cofactor), then
//   P^-1 = [A^-1 + A^-1 B S^-1 C A^-1, -A^-1 B S^-1; -S^-1 C A^-1, S^-1].
// The unpivoted pivots of P are those of A followed by those of S, so the
// rank test is the two cofactor tests. scr: 80 doubles. All lanes call.
__device__ __forceinline__ void inv8_schur(const double* p, double thr, double* out, double* scr, bool& ok) {
  const int l = threadIdx.x & 31, i = (l >> 2) & 3, j = l & 3;
  double* ai = scr;        // A^-1
  double* ca = scr + 16;   // C A^-1
  double* ab = scr + 32;   // A^-1 B
  double* sm = scr + 48;   // S, then S^-1
  double* tr = scr + 64;   // -A^-1 B S^-1
  bool ok1, ok2;
  const double av = inv4_cofactor(p, thr, ok1, 8);
  if (l < 16) ai[l] = av;
  __syncwarp();
  if (l < 16) {  // C A^-1
    double v = 0.0;
#pragma unroll
    for (int k = 0; k < 4; ++k) v = fma(p[(4 + i) * 8 + k], ai[k * 4 + j], v);
    ca[l] = v;
  } else {       // A^-1 B
    double v = 0.0;
#pragma unroll
    for (int k = 0; k < 4; ++k) v = fma(ai[i * 4 + k], p[k * 8 + 4 + j], v);
    ab[l - 16] = v;
  }
  __syncwarp();
  if (l < 16) {  // S = D - (C A^-1) B
    double v = p[(4 + i) * 8 + 4 + j];
#pragma unroll
    for (int k = 0; k < 4; ++k) v = fma(-ca[i * 4 + k], p[k * 8 + 4 + j], v);
    sm[l] = v;
  }
  __syncwarp();
  const double sv = inv4_cofactor(sm, thr, ok2, 4);
  __syncwarp();
  if (l < 16) {
    sm[l] = sv;
    out[(4 + i) * 8 + 4 + j] = sv;
  }
  __syncwarp();
  if (l < 16) {  // top right: -(A^-1 B) S^-1
    double v = 0.0;
#pragma unroll
    for (int k = 0; k < 4; ++k) v = fma(-ab[i * 4 + k], sm[k * 4 + j], v);
    tr[l] = v;
    out[i * 8 + 4 + j] = v;
  } else {       // bottom left: -S^-1 (C A^-1)
    double v = 0.0;
#pragma unroll
    for (int k = 0; k < 4; ++k) v = fma(-sm[i * 4 + k], ca[k * 4 + j], v);
    out[(4 + i) * 8 + j] = v;
  }
  __syncwarp();
  if (l < 16) {  // top left: A^-1 - (top right) (C A^-1)
    double v = ai[l];
#pragma unroll
    for (int k = 0; k < 4; ++k) v = fma(-tr[i * 4 + k], ca[k * 4 + j], v);
    out[i * 8 + j] = v;
  }
  ok = ok1 && ok2;
  __syncwarp();
}

// Block Gauss-Jordan inverse with 8 x 8 pivot blocks, one 8-row tile per
// step (see inverse_la for the scheme; here K is tile s, every step is two
// m8n8k4 MMAs per tile, and the fragment slots rotate every step so slot 0
// holds tile s). g: RT x RT Gram (ld RT). sh: 48 RT + 256 doubles.
template <int RT>
__device__ bool inverse_b8r(const double* __restrict__ g, int r, double tol, double* __restrict__ ginv,
                            double* __restrict__ gfull, int* info, double* sh,
                            unsigned long long* stamps = nullptr) {
  constexpr int NTI = RT / 8;
  static_assert(NTI <= 8, "one 8-column tile per warp");
  double* rbs = sh;              // [2][16][RT] rows K (identity on K columns), raw rows K+
  double* cbs = rbs + 32 * RT;   // [2][RT][8]  -a(i, K), +e on rows K
  double* pin = cbs + 16 * RT;   // [2][64]     inverse of the pivot block of step s
  double* pv = pin + 128;        // [64]        next pivot block (look-ahead)
  double* scr = pv + 64;         // [80]        look-ahead scratch
  double* misc = scr + 80;       // [2..3] fail flags, [4..5] warp maxima
  const int tid = threadIdx.x, w = tid / 32, l = tid % 32;
  const int lr = l >> 2, lc = (l & 3) * 2, lk = l & 3;
  const int r8 = (r + 7) & ~7;
  const int nt = r8 / 8;
  const bool worker = w < nt;  // warp w owns 8-column tile w
  double acc[NTI][2];          // slot p: rows of tile (s + p) % NTI at step s
#pragma unroll
  for (int mt = 0; mt < NTI; ++mt) {
    const int row = mt * 8 + lr, col = w * 8 + lc;
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
  if (worker) {
#pragma unroll
    for (int mt = 0; mt < NTI; ++mt) {
      const int row = mt * 8 + lr;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int col = w * 8 + lc + e;
        if (row < r && col < r) gfull[row * r + col] = acc[mt][e];
        if (row == col && row >= r && row < r8) acc[mt][e] = dmax;  // padding diagonal
      }
    }
  }
  // publish tile T's blocks (slot PK holds tile T, slot PKK tile T+1); the
  // owner of tile T's columns publishes -C; rows/columns of tile T zeroed
  auto publish = [&](auto pk, auto pkk, int T, double* rb, double* cb, bool first) {
    constexpr int PK = decltype(pk)::value, PKK = decltype(pkk)::value;
    if (!worker) return;  // warp-uniform
    const bool own = (w == T);
    const int col = w * 8 + lc;
    if (first && own) *reinterpret_cast<double2*>(pv + lr * 8 + lc) = make_double2(acc[PK][0], acc[PK][1]);
    double2 o;
    o.x = own ? (lr == lc ? 1.0 : 0.0) : acc[PK][0];
    o.y = own ? (lr == lc + 1 ? 1.0 : 0.0) : acc[PK][1];
    *reinterpret_cast<double2*>(rb + lr * RT + col) = o;
    if (T + 1 < nt) *reinterpret_cast<double2*>(rb + (8 + lr) * RT + col) = make_double2(acc[PKK][0], acc[PKK][1]);
    if (own) {
#pragma unroll
      for (int p = 0; p < NTI; ++p) {
        const int row = ((T - PK + p + NTI) % NTI) * 8 + lr;
        double2 c;
        c.x = (p == PK) ? (lr == lc ? 1.0 : 0.0) : -acc[p][0];
        c.y = (p == PK) ? (lr == lc + 1 ? 1.0 : 0.0) : -acc[p][1];
        *reinterpret_cast<double2*>(cb + row * 8 + lc) = c;
        acc[p][0] = acc[p][1] = 0.0;
      }
    }
    acc[PK][0] = acc[PK][1] = 0.0;
  };
  using I0 = std::integral_constant<int, 0>;
  using I1 = std::integral_constant<int, 1>;
  using I2 = std::integral_constant<int, 2>;
  publish(I0{}, I1{}, 0, rbs, cbs, true);
  __syncthreads();
  if (w == 7) {
    bool ok;
    inv8_schur(pv, thr, pin, scr, ok);
    if (l == 0) misc[2] = ok ? 0.0 : 1.0;
  }
  __syncthreads();
  if (stamps && tid == 0) stamps[0] = globaltimer();
  bool fail = false;
  int s = 0;
#pragma unroll 1
  for (; s < nt; ++s) {
    const int pb = s & 1;
    if (misc[2 + pb] != 0.0) {
      fail = true;  // uniform
      break;
    }
    const double* P = pin + 64 * pb;
    const double* rb = rbs + pb * 16 * RT;
    const double* cb = cbs + pb * RT * 8;
    if (w == 7 && s + 1 < nt) {
      // look-ahead: pivot block of step s+1 (tile s+1 after step s) and its inverse
      const int k0 = 8 * s, k1 = 8 * (s + 1);
      {  // M_q(j) = sum_t P^-1(q, t) a(K_t, j), j in tile s+1: lane (q = l/4, j = l%4 (+4))
        double m0 = 0.0, m1 = 0.0;
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          const double pq = P[lr * 8 + t];
          m0 = fma(pq, rb[t * RT + k1 + lk], m0);
          m1 = fma(pq, rb[t * RT + k1 + lk + 4], m1);
        }
        scr[lr * 8 + lk] = m0;
        scr[lr * 8 + lk + 4] = m1;
      }
      __syncwarp();
      {
        const double* rn = rb + (8 + lr) * RT;  // raw row k1 + l/4
        double v0 = rn[k1 + lk], v1 = rn[k1 + lk + 4];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const double c = rn[k0 + q];
          v0 = fma(-c, scr[q * 8 + lk], v0);
          v1 = fma(-c, scr[q * 8 + lk + 4], v1);
        }
        __syncwarp();
        pv[lr * 8 + lk] = v0;
        pv[lr * 8 + lk + 4] = v1;
      }
      __syncwarp();
      bool ok;
      inv8_schur(pv, thr, pin + 64 * (pb ^ 1), scr, ok);
      if (l == 0) misc[2 + (pb ^ 1)] = ok ? 0.0 : 1.0;
    }
    if (worker) {
      double pr0[8], pr1[8];  // rows l%4 and l%4 + 4 of P^-1
#pragma unroll
      for (int t = 0; t < 8; t += 2) {
        const double2 a = *reinterpret_cast<const double2*>(P + lk * 8 + t);
        const double2 c = *reinterpret_cast<const double2*>(P + (lk + 4) * 8 + t);
        pr0[t] = a.x;
        pr0[t + 1] = a.y;
        pr1[t] = c.x;
        pr1[t + 1] = c.y;
      }
      const int j = w * 8 + lr;  // B fragment (k = l % 4 (+4), n = l / 4)
      double bm0 = 0.0, bm1 = 0.0;
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const double rv = rb[t * RT + j];
        bm0 = fma(pr0[t], rv, bm0);
        bm1 = fma(pr1[t], rv, bm1);
      }
      double am[NTI][2];
#pragma unroll
      for (int p = 0; p < NTI; ++p) {
        const int row = ((s + p) % NTI) * 8 + lr;
        am[p][0] = cb[row * 8 + lk];
        am[p][1] = cb[row * 8 + lk + 4];
      }
#pragma unroll
      for (int p = 0; p < NTI; ++p) {
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(acc[p][0]), "+d"(acc[p][1])
                     : "d"(am[p][0]), "d"(bm0));
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(acc[p][0]), "+d"(acc[p][1])
                     : "d"(am[p][1]), "d"(bm1));
      }
      if (s + 1 < nt) publish(I1{}, I2{}, s + 1, rbs + (pb ^ 1) * 16 * RT, cbs + (pb ^ 1) * RT * 8, false);
      // rotate: slot 0 <- tile s + 1
      const double f0 = acc[0][0], f1 = acc[0][1];
#pragma unroll
      for (int p = 0; p + 1 < NTI; ++p) {
        acc[p][0] = acc[p + 1][0];
        acc[p][1] = acc[p + 1][1];
      }
      acc[NTI - 1][0] = f0;
      acc[NTI - 1][1] = f1;
    }
    __syncthreads();
  }
  if (stamps && tid == 0) stamps[1] = globaltimer();
  if (!fail && worker) {
#pragma unroll
    for (int p = 0; p < NTI; ++p) {
      const int mt = (s + p) % NTI;
      const int row = mt * 8 + lr, col = w * 8 + lc;
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
  return fail;
}


}  // namespace ph
}  // namespace cpb
