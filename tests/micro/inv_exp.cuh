// Experimental copy of ph::inverse_la for timing variants (not the product).
#pragma once
namespace cpb {
namespace phx {
using ph::inv4_cofactor;
template <int RT, int VAR>
__device__ bool inverse_x(const double* __restrict__ g, int r, double tol, double* __restrict__ ginv,
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
  double Pr[16];  // VAR & 2: warp 7 keeps the current pivot inverse in registers (every lane)
  if (w == 7) {
    if constexpr (VAR & 2) {
      double tv[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) tv[e] = tmp[e];
      const bool ok = ph::inv4_minors(tv, Pr, thr);
      if (l == 0) {
#pragma unroll
        for (int e = 0; e < 16; ++e) pin[e] = Pr[e];
        misc[2] = ok ? 0.0 : 1.0;
      }
    } else {
      bool ok;
      const double v = inv4_cofactor(tmp, thr, ok);
      if (l < 16) pin[l] = v;
      if (l == 0) misc[2] = ok ? 0.0 : 1.0;
    }
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
      if constexpr ((VAR & 2) != 0) {
        if (w == 7 && k0 + 4 < r4) {
          // every lane: the next pivot block T = RAW(K+, K+) - RAW(K+, K) P ROWS_K(K+)
          // and its inverse, all in registers (no shared-memory round trip)
          double Rr[4][4], Wn[4][4], Wk[4][4];
#pragma unroll
          for (int k = 0; k < 4; ++k)
#pragma unroll
            for (int y = 0; y < 4; ++y) {
              Rr[k][y] = rb[k * RT + k0 + 4 + y];
              Wn[k][y] = rb[(4 + k) * RT + k0 + 4 + y];
              Wk[k][y] = rb[(4 + k) * RT + k0 + y];
            }
          double Q[4][4];
#pragma unroll
          for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int y = 0; y < 4; ++y)
              Q[q][y] = fma(Pr[q * 4], Rr[0][y], Pr[q * 4 + 1] * Rr[1][y]) + fma(Pr[q * 4 + 2], Rr[2][y], Pr[q * 4 + 3] * Rr[3][y]);
          double Tm[16];
#pragma unroll
          for (int x = 0; x < 4; ++x)
#pragma unroll
            for (int y = 0; y < 4; ++y)
              Tm[x * 4 + y] = (Wn[x][y] - fma(Wk[x][0], Q[0][y], Wk[x][1] * Q[1][y])) - fma(Wk[x][2], Q[2][y], Wk[x][3] * Q[3][y]);
          CPB_INV_STAMP_AT(43, s, l == 0);
          const bool ok = ph::inv4_minors(Tm, Pr, thr);
          if (l == 0) {
#pragma unroll
            for (int e = 0; e < 16; ++e) pin[16 * (pb ^ 1) + e] = Pr[e];
            misc[2 + (pb ^ 1)] = ok ? 0.0 : 1.0;
          }
          CPB_INV_STAMP_AT(44, s, l == 0);
        }
      } else if (w == 7 && k0 + 4 < r4) {
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
      if (worker && !(VAR & 1)) {
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


}  // namespace phx
}  // namespace cpb
