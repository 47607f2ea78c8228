// CPRAND-MIX transforms on sm_100a (mixing.hpp:130-236, transforms.hpp:124-166).
//
// forward  = sign then orthonormal DCT-II   (mix_tensor / mix_factor)
// adjoint  = orthonormal DCT-III then sign  (unmix_sampled_rhs / unmix_factor)
//
// The reference evaluates the DCT through a length-2n complex FFT (Bluestein
// when 2n is not a power of two). Here each CTA stages F fibers of a mode in
// shared memory and runs Makhoul's n-point form: the even/odd reordering of
// a real fiber, one complex FFT of length n (two real fibers packed as
// re/im of one complex sequence), and a quarter-wave phase. The FFT is a
// mixed-radix Stockham autosort over radices {4, 2, 3, 5, 7, any prime};
// twiddles come from a table of n-th roots computed once in long double.
// Same transform, different rounding: parity with the reference is
// tolerance level (1e-12 rel, test_mixing.cpp:90-137).
#include <cmath>
#include <vector>

#include "kernels.cuh"

namespace cpb {

namespace {

constexpr int kMixThreads = 256;

struct PlanArgs {
  int n;
  int nrad;
  int radix[24];
  const double2* tw;
  const double2* phase;
  double s0, sk;
};

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
__device__ void stockham_pass(const PlanArgs& p, const double2* src, double2* dst, int np, int ns,
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
__device__ void stockham_pass_generic(const PlanArgs& p, int R, const double2* src, double2* dst,
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
__device__ double2* fft_smem(const PlanArgs& p, double2* a, double2* b, int np, bool inv) {
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

// F fibers (F even) per CTA, packed in F/2 complex sequences.
__global__ void __launch_bounds__(kMixThreads) mode_transform_kernel(PlanArgs p, const double* in,
                                                                    double* out, i64 st, i64 nfib,
                                                                    int F, const double* sign,
                                                                    int forward,
                                                                    const double* col_div) {
  extern __shared__ __align__(16) double2 sbuf[];
  const int n = p.n, np = F / 2;
  double2* b0 = sbuf;
  double2* b1 = sbuf + np * n;
  const i64 f0 = static_cast<i64>(blockIdx.x) * F;
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
}

__global__ void reduce_rhs_kernel(const double* __restrict__ part, int ks, i64 in, int r,
                                  double* __restrict__ out) {
  const i64 e = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= in * r) return;
  double s = 0.0;
  for (int k = 0; k < ks; ++k) s += part[static_cast<i64>(k) * in * r + e];
  out[e] = s;
}

}  // namespace

DctPlan make_dct_plan(int n) {
  if (n < 1) throw InvalidArgument("dct length must be >= 1");
  DctPlan p;
  p.n = n;
  int m = n;
  while (m % 4 == 0) {
    p.radix[p.nrad++] = 4;
    m /= 4;
  }
  while (m % 2 == 0) {
    p.radix[p.nrad++] = 2;
    m /= 2;
  }
  for (int f = 3; f <= m; f += 2)
    while (m % f == 0) {
      if (p.nrad >= 24) throw Unsupported("dct length has too many factors");
      if (f > 61) throw Unsupported("dct length has a prime factor > 61");
      p.radix[p.nrad++] = f;
      m /= f;
    }
  const long double pi = 3.141592653589793238462643383279502884L;
  std::vector<double2> tw(static_cast<size_t>(n)), ph(static_cast<size_t>(n));
  for (int t = 0; t < n; ++t) {
    const long double a = 2.0L * pi * static_cast<long double>(t) / static_cast<long double>(n);
    tw[static_cast<size_t>(t)] = make_double2(static_cast<double>(cosl(a)), static_cast<double>(-sinl(a)));
    const long double b = pi * static_cast<long double>(t) / (2.0L * static_cast<long double>(n));
    ph[static_cast<size_t>(t)] = make_double2(static_cast<double>(cosl(b)), static_cast<double>(-sinl(b)));
  }
  CPB_CUDA(cudaMalloc(&p.tw, sizeof(double2) * n));
  CPB_CUDA(cudaMalloc(&p.phase, sizeof(double2) * n));
  CPB_CUDA(cudaMemcpy(p.tw, tw.data(), sizeof(double2) * n, cudaMemcpyHostToDevice));
  CPB_CUDA(cudaMemcpy(p.phase, ph.data(), sizeof(double2) * n, cudaMemcpyHostToDevice));
  p.s0 = std::sqrt(1.0 / static_cast<double>(n));
  p.sk = std::sqrt(2.0 / static_cast<double>(n));
  return p;
}

void free_dct_plan(DctPlan& p) {
  if (p.tw) cudaFree(p.tw);
  if (p.phase) cudaFree(p.phase);
  p.tw = p.phase = nullptr;
}

void launch_mode_transform(const DctPlan& p, const double* in, double* out, i64 st, i64 nfib,
                           const double* sign, int forward, const double* col_div,
                           cudaStream_t stream) {
  if (nfib <= 0) return;
  PlanArgs a;
  a.n = p.n;
  a.nrad = p.nrad;
  for (int i = 0; i < 24; ++i) a.radix[i] = p.radix[i];
  a.tw = p.tw;
  a.phase = p.phase;
  a.s0 = p.s0;
  a.sk = p.sk;
  // fibers per CTA: even, smem 16 B x F x n (two buffers of F/2 sequences)
  const size_t budget = 96 * 1024;
  int F = static_cast<int>(budget / (16 * static_cast<size_t>(p.n)));
  F = F > 32 ? 32 : F;
  F &= ~1;
  if (F < 2) F = 2;
  const size_t smem = static_cast<size_t>(F) * p.n * 16;
  if (smem > 227 * 1024) throw Unsupported("mode length too large for the in-SMEM transform");
  static size_t configured = 0;
  if (smem > 48 * 1024 && smem > configured) {
    CPB_CUDA(cudaFuncSetAttribute(mode_transform_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    configured = smem;
  }
  const i64 blocks = (nfib + F - 1) / F;
  if (blocks > 0x7fffffffLL) throw Unsupported("too many fibers for one launch");
  mode_transform_kernel<<<static_cast<unsigned>(blocks), kMixThreads, smem, stream>>>(
      a, in, out, st, nfib, F, sign, forward, col_div);
  CPB_LAUNCH_CHECK();
}

void launch_reduce_rhs(const double* part_rhs, int ks, i64 in, int r, double* out,
                       cudaStream_t st) {
  const i64 n = in * r;
  reduce_rhs_kernel<<<ceil_div(n, 256), 256, 0, st>>>(part_rhs, ks, in, r, out);
  CPB_LAUNCH_CHECK();
}

}  // namespace cpb
