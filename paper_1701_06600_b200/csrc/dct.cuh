// Mixing-transform engine (sign + orthonormal DCT-II / DCT-III along a
// mode), shared by the standalone transform kernel (mix.cu) and the
// persistent per-iteration kernel (fused.cu). See mix.cu for the method.
#pragma once

#include "kernels.cuh"

namespace cpb {
namespace dct {

using PlanArgs = DctArgs;

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }

// e^{-2 pi i u r / R} multiply-accumulate DFT of R points (R in {2,3,4,5,8});
// inverse uses the conjugate roots.
template <int R>
__device__ __forceinline__ void dft(double2 (&v)[R], bool inv) {
  if constexpr (R == 2) {
    const double2 a = v[0], b = v[1];
    v[0] = cadd(a, b);
    v[1] = csub(a, b);
  } else if constexpr (R == 4) {
    const double2 a = cadd(v[0], v[2]), b = csub(v[0], v[2]);
    const double2 c = cadd(v[1], v[3]), e = csub(v[1], v[3]);
    const double2 ej = inv ? make_double2(-e.y, e.x) : make_double2(e.y, -e.x);
    v[0] = cadd(a, c);
    v[2] = csub(a, c);
    v[1] = cadd(b, ej);
    v[3] = csub(b, ej);
  } else if constexpr (R == 8) {
    // two radix-4 on even/odd, twiddle the odd half by W8^k, combine
    double2 e[4] = {v[0], v[2], v[4], v[6]}, o[4] = {v[1], v[3], v[5], v[7]};
    dft<4>(e, inv);
    dft<4>(o, inv);
    const double h = 0.70710678118654752440;
    // W8^1 = (1 - i)/sqrt2 (forward), W8^2 = -i, W8^3 = (-1 - i)/sqrt2
    const double2 o1 = inv ? make_double2(h * (o[1].x - o[1].y), h * (o[1].x + o[1].y))
                           : make_double2(h * (o[1].x + o[1].y), h * (o[1].y - o[1].x));
    const double2 o2 = inv ? make_double2(-o[2].y, o[2].x) : make_double2(o[2].y, -o[2].x);
    const double2 o3 = inv ? make_double2(-h * (o[3].x + o[3].y), h * (o[3].x - o[3].y))
                           : make_double2(h * (o[3].y - o[3].x), -h * (o[3].x + o[3].y));
    v[0] = cadd(e[0], o[0]);
    v[4] = csub(e[0], o[0]);
    v[1] = cadd(e[1], o1);
    v[5] = csub(e[1], o1);
    v[2] = cadd(e[2], o2);
    v[6] = csub(e[2], o2);
    v[3] = cadd(e[3], o3);
    v[7] = csub(e[3], o3);
  } else if constexpr (R == 3) {
    const double c1 = -0.5, s1 = inv ? 0.86602540378443864676 : -0.86602540378443864676;
    const double2 a = v[0], b = v[1], c = v[2];
    const double2 sbc = cadd(b, c), dbc = csub(b, c);
    v[0] = cadd(a, sbc);
    const double2 t = make_double2(a.x + c1 * sbc.x, a.y + c1 * sbc.y);
    // (b - c) * i s1
    const double2 u = make_double2(-s1 * dbc.y, s1 * dbc.x);
    v[1] = cadd(t, u);
    v[2] = csub(t, u);
  } else {  // R == 5
    const double c1 = 0.30901699437494742410, c2 = -0.80901699437494742410;
    const double s1 = inv ? 0.95105651629515357212 : -0.95105651629515357212;
    const double s2 = inv ? 0.58778525229247312917 : -0.58778525229247312917;
    const double2 a = v[0];
    const double2 p1 = cadd(v[1], v[4]), m1 = csub(v[1], v[4]);
    const double2 p2 = cadd(v[2], v[3]), m2 = csub(v[2], v[3]);
    v[0] = make_double2(a.x + p1.x + p2.x, a.y + p1.y + p2.y);
    const double2 t1 = make_double2(a.x + c1 * p1.x + c2 * p2.x, a.y + c1 * p1.y + c2 * p2.y);
    const double2 t2 = make_double2(a.x + c2 * p1.x + c1 * p2.x, a.y + c2 * p1.y + c1 * p2.y);
    // i (s1 m1 + s2 m2), i (s2 m1 - s1 m2)
    const double2 u1 = make_double2(-(s1 * m1.y + s2 * m2.y), s1 * m1.x + s2 * m2.x);
    const double2 u2 = make_double2(-(s2 * m1.y - s1 * m2.y), s2 * m1.x - s1 * m2.x);
    v[1] = cadd(t1, u1);
    v[4] = csub(t1, u1);
    v[2] = cadd(t2, u2);
    v[3] = csub(t2, u2);
  }
}

// root(t) = exp(-+2 pi i t / n), t taken mod n
__device__ __forceinline__ double2 root(const PlanArgs& p, int t, bool inv) {
  const double2 w = p.tw[t];
  return inv ? cconj(w) : w;
}

// One Stockham pass of radix R over `np` sequences of length n.
template <int R>
__device__ inline void stockham_pass(const PlanArgs& p, const double2* src, double2* dst, int np, int ns,
                              bool inv) {
  const int n = p.n, m = n / R;
  const int step = n / (ns * R);
  for (int t = threadIdx.x; t < np * m; t += blockDim.x) {
    const int q = t / m, j = t - q * m;
    const double2* s = src + q * n;
    double2* d = dst + q * n;
    const int k = j % ns;
    double2 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = s[j + r * m];
    if (ns > 1) {
#pragma unroll
      for (int r = 1; r < R; ++r) v[r] = cmul(v[r], root(p, r * k * step, inv));
    }
    double2 o[R];
    if constexpr (R == 2 || R == 3 || R == 4 || R == 5 || R == 8) {
      dft<R>(v, inv);  // closed-form butterflies
#pragma unroll
      for (int u = 0; u < R; ++u) o[u] = v[u];
    } else {
#pragma unroll
      for (int u = 0; u < R; ++u) {
        double2 acc = v[0];
#pragma unroll
        for (int r = 1; r < R; ++r) acc = cadd(acc, cmul(v[r], root(p, ((u * r) % R) * m, inv)));
        o[u] = acc;
      }
    }
    const int idx = (j / ns) * ns * R + k;
#pragma unroll
    for (int r = 0; r < R; ++r) d[idx + r * ns] = o[r];
  }
}

// Generic radix (any prime): O(R) per output, reads src directly.
__device__ inline void stockham_pass_generic(const PlanArgs& p, int R, const double2* src, double2* dst,
                                      int np, int ns, bool inv) {
  const int n = p.n, m = n / R;
  const int step = n / (ns * R);
  for (int t = threadIdx.x; t < np * m * R; t += blockDim.x) {
    const int q = t / (m * R);
    const int rem = t - q * m * R;
    const int j = rem / R, u = rem - (rem / R) * R;
    const double2* s = src + q * n;
    const int k = j % ns;
    double2 acc = make_double2(0.0, 0.0);
    for (int r = 0; r < R; ++r) {
      double2 v = s[j + r * m];
      if (ns > 1 && r > 0) v = cmul(v, root(p, r * k * step, inv));
      acc = cadd(acc, r == 0 ? v : cmul(v, root(p, ((u * r) % R) * m, inv)));
    }
    dst[q * n + (j / ns) * ns * R + k + u * ns] = acc;
  }
}

// Runs the full FFT on np sequences in buffers a/b; returns the buffer
// holding the result.
__device__ inline double2* fft_smem(const PlanArgs& p, double2* a, double2* b, int np, bool inv) {
  int ns = 1;
  double2* src = a;
  double2* dst = b;
  for (int st = 0; st < p.nrad; ++st) {
    const int R = p.radix[st];
    switch (R) {
      case 2: stockham_pass<2>(p, src, dst, np, ns, inv); break;
      case 3: stockham_pass<3>(p, src, dst, np, ns, inv); break;
      case 4: stockham_pass<4>(p, src, dst, np, ns, inv); break;
      case 5: stockham_pass<5>(p, src, dst, np, ns, inv); break;
      case 7: stockham_pass<7>(p, src, dst, np, ns, inv); break;
      default: stockham_pass_generic(p, R, src, dst, np, ns, inv); break;
    }
    __syncthreads();
    ns *= R;
    double2* t = src;
    src = dst;
    dst = t;
  }
  return src;
}

__device__ __forceinline__ i64 fib_addr(i64 f, i64 i, i64 st, int n) {
  if (f < st) return f + i * st;  // first slab (every fiber of a factor matrix): no division
  const i64 hi = f / st, lo = f - hi * st;
  return hi * st * n + lo + i * st;
}

// Fibers [f0, f0 + F) (F even), packed in F/2 complex sequences; sbuf
// holds F * n double2. CTA-level; callable from any kernel.
__device__ inline void transform_group(const PlanArgs& p, const double* in, double* out, i64 st, i64 nfib,
                                       i64 f0, int F, const double* sign, int forward, const double* col_div,
                                       double2* sbuf) {
  const int n = p.n, np = F / 2;
  double2* b0 = sbuf;
  double2* b1 = sbuf + np * n;
  const int total = F * n;
  const bool contig = (st == 1);
  // Two real fibers share one complex FFT, which leaks rounding between
  // them; a fiber that is exactly zero must stay exactly zero, as in the
  // reference's per-fiber transform (a zero factor column is refilled only
  // when its norm is exactly 0, kruskal.hpp:57-63). Bit fl of s_nz: fiber
  // f0 + fl has a nonzero entry (groups of more than 64 fibers: not tracked).
  __shared__ unsigned long long s_nz;
  if (threadIdx.x == 0) s_nz = F > 64 ? ~0ull : 0ull;
  __syncthreads();
  unsigned long long nz = 0ull;
  // ---- load (coalesced along i for contiguous fibers, along f otherwise)
  for (int t = threadIdx.x; t < total; t += blockDim.x) {
    int fl, i;
    if (contig) {
      fl = t / n;
      i = t - fl * n;
    } else {
      i = t / F;
      fl = t - i * F;
    }
    const i64 f = f0 + fl;
    double v = 0.0;
    if (f < nfib) {
      v = in[fib_addr(f, i, st, n)];
      if (col_div) v = v / col_div[f];  // lazily normalized factor column
      if (v != 0.0 && fl < 64) nz |= 1ull << fl;
    }
    const int q = fl >> 1;
    if (forward) {
      v *= sign[i];  // D_n first (mixing.hpp:148)
      const int d = (i & 1) ? (n - 1 - (i >> 1)) : (i >> 1);
      double* slot = reinterpret_cast<double*>(&b0[q * n + d]);
      slot[fl & 1] = v;
    } else {
      double* slot = reinterpret_cast<double*>(&b1[q * n + i]);
      slot[fl & 1] = v;
    }
  }
  if (nz) atomicOr(&s_nz, nz);
  __syncthreads();
  double2* res;
  if (forward) {
    res = fft_smem(p, b0, b1, np, false);
  } else {
    // W_k = V1_k + i V2_k, V_k = e^{+i pi k / 2n} (C_k - i C_{n-k}), C = Y / s
    const double inv0 = 1.0 / p.s0, invk = 1.0 / p.sk;
    for (int t = threadIdx.x; t < np * n; t += blockDim.x) {
      const int q = t / n, k = t - q * n;
      const double2 yk = b1[q * n + k];
      const double2 ynk = (k == 0) ? make_double2(0.0, 0.0) : b1[q * n + (n - k)];
      const double ik = (k == 0) ? inv0 : invk;
      const double ink = invk;
      const double2 ph = cconj(p.phase[k]);
      const double2 u1 = make_double2(yk.x * ik, -ynk.x * ink);
      const double2 u2 = make_double2(yk.y * ik, -ynk.y * ink);
      const double2 v1 = cmul(ph, u1), v2 = cmul(ph, u2);
      b0[q * n + k] = make_double2(v1.x - v2.y, v1.y + v2.x);
    }
    __syncthreads();
    res = fft_smem(p, b0, b1, np, true);
  }
  // ---- epilogue + store
  const double invn = 1.0 / static_cast<double>(n);
  for (int t = threadIdx.x; t < total; t += blockDim.x) {
    int fl, i;
    if (contig) {
      fl = t / n;
      i = t - fl * n;
    } else {
      i = t / F;
      fl = t - i * F;
    }
    const i64 f = f0 + fl;
    if (f >= nfib) continue;
    const int q = fl >> 1;
    double v;
    if (forward) {
      const double2 z = res[q * n + i];
      const double2 zc = res[q * n + ((n - i) % n)];
      const double2 ph = p.phase[i];
      const double sc = (i == 0) ? p.s0 : p.sk;
      if ((fl & 1) == 0) {
        const double vx = 0.5 * (z.x + zc.x), vy = 0.5 * (z.y - zc.y);
        v = sc * (ph.x * vx - ph.y * vy);
      } else {
        const double vx = 0.5 * (z.y + zc.y), vy = -0.5 * (z.x - zc.x);
        v = sc * (ph.x * vx - ph.y * vy);
      }
    } else {
      const int m = (i & 1) ? (n - 1 - (i >> 1)) : (i >> 1);
      const double2 z = res[q * n + m];
      v = ((fl & 1) ? z.y : z.x) * invn;
      v *= sign[i];  // D_n after the adjoint (mixing.hpp:231)
    }
    if (fl < 64 && !((s_nz >> fl) & 1ull)) v = 0.0;
    out[fib_addr(f, i, st, n)] = v;
  }
  __syncthreads();  // sbuf may be reused by the caller
}

}  // namespace dct
}  // namespace cpb
