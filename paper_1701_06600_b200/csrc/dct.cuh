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
    if (R == 2) {
      o[0] = cadd(v[0], v[1]);
      o[1] = csub(v[0], v[1]);
    } else if (R == 4) {
      const double2 a = cadd(v[0], v[2]), b = csub(v[0], v[2]);
      const double2 c = cadd(v[1], v[3]), e = csub(v[1], v[3]);
      // forward: multiply e by -i; inverse: by +i
      const double2 ej = inv ? make_double2(-e.y, e.x) : make_double2(e.y, -e.x);
      o[0] = cadd(a, c);
      o[2] = csub(a, c);
      o[1] = cadd(b, ej);
      o[3] = csub(b, ej);
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
    out[fib_addr(f, i, st, n)] = v;
  }
  __syncthreads();  // sbuf may be reused by the caller
}

}  // namespace dct
}  // namespace cpb
