// The CPRAND-MIX preprocessing pass over a whole tensor (mix_tensor,
// mixing.hpp:130-156): along one mode, every fiber gets sign then the
// orthonormal DCT-II (forward) or DCT-III then sign (adjoint). HBM bound:
// each element is read once and written once per mode (16 B).
//
// Persistent CTAs (one per SM, 512 threads). Each CTA loops over groups of
// F = 4 fibers, packed as two complex sequences of length n (Makhoul's
// even/odd reordering, then one complex FFT, then a quarter-wave phase: the
// same transform as dct.cuh).
//  * The next group's fibers stream into a second staging buffer with
//    cp.async while the current group is transformed.
//  * Strided modes: the 4 fibers of a group are adjacent in the fastest
//    index, so every row of the group is one 32-byte sector.
//  * The twiddles, phases and signs sit in shared memory.
//  * The Stockham passes use compile-time radices 8 / 5 / 4 / 3 / 2 with
//    division-free indexing.
// Same algorithm and rounding structure as dct.cuh's transform_group; parity
// with the oracle's Bluestein DCT is at tolerance (1e-12 relative).
#include "dct.cuh"
#include "devutil.cuh"

namespace cpb {

namespace {

constexpr int kPassThreads = 512;
constexpr int kGroup = 4;  // fibers per group (two complex sequences)

using dct::PlanArgs;

// e^{-2 pi i u r / R} multiply-accumulate DFT of R points (R in {2,3,4,5,8});
// inverse uses the conjugate roots.
template <int R>
__device__ __forceinline__ void dft(double2 (&v)[R], bool inv) {
  if constexpr (R == 2) {
    const double2 a = v[0], b = v[1];
    v[0] = dct::cadd(a, b);
    v[1] = dct::csub(a, b);
  } else if constexpr (R == 4) {
    const double2 a = dct::cadd(v[0], v[2]), b = dct::csub(v[0], v[2]);
    const double2 c = dct::cadd(v[1], v[3]), e = dct::csub(v[1], v[3]);
    const double2 ej = inv ? make_double2(-e.y, e.x) : make_double2(e.y, -e.x);
    v[0] = dct::cadd(a, c);
    v[2] = dct::csub(a, c);
    v[1] = dct::cadd(b, ej);
    v[3] = dct::csub(b, ej);
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
    v[0] = dct::cadd(e[0], o[0]);
    v[4] = dct::csub(e[0], o[0]);
    v[1] = dct::cadd(e[1], o1);
    v[5] = dct::csub(e[1], o1);
    v[2] = dct::cadd(e[2], o2);
    v[6] = dct::csub(e[2], o2);
    v[3] = dct::cadd(e[3], o3);
    v[7] = dct::csub(e[3], o3);
  } else if constexpr (R == 3) {
    const double c1 = -0.5, s1 = inv ? 0.86602540378443864676 : -0.86602540378443864676;
    const double2 a = v[0], b = v[1], c = v[2];
    const double2 sbc = dct::cadd(b, c), dbc = dct::csub(b, c);
    v[0] = dct::cadd(a, sbc);
    const double2 t = make_double2(a.x + c1 * sbc.x, a.y + c1 * sbc.y);
    // (b - c) * i s1
    const double2 u = make_double2(-s1 * dbc.y, s1 * dbc.x);
    v[1] = dct::cadd(t, u);
    v[2] = dct::csub(t, u);
  } else {  // R == 5
    const double c1 = 0.30901699437494742410, c2 = -0.80901699437494742410;
    const double s1 = inv ? 0.95105651629515357212 : -0.95105651629515357212;
    const double s2 = inv ? 0.58778525229247312917 : -0.58778525229247312917;
    const double2 a = v[0];
    const double2 p1 = dct::cadd(v[1], v[4]), m1 = dct::csub(v[1], v[4]);
    const double2 p2 = dct::cadd(v[2], v[3]), m2 = dct::csub(v[2], v[3]);
    v[0] = make_double2(a.x + p1.x + p2.x, a.y + p1.y + p2.y);
    const double2 t1 = make_double2(a.x + c1 * p1.x + c2 * p2.x, a.y + c1 * p1.y + c2 * p2.y);
    const double2 t2 = make_double2(a.x + c2 * p1.x + c1 * p2.x, a.y + c2 * p1.y + c1 * p2.y);
    // i (s1 m1 + s2 m2), i (s2 m1 - s1 m2)
    const double2 u1 = make_double2(-(s1 * m1.y + s2 * m2.y), s1 * m1.x + s2 * m2.x);
    const double2 u2 = make_double2(-(s2 * m1.y - s1 * m2.y), s2 * m1.x - s1 * m2.x);
    v[1] = dct::cadd(t1, u1);
    v[4] = dct::csub(t1, u1);
    v[2] = dct::cadd(t2, u2);
    v[3] = dct::csub(t2, u2);
  }
}

// One Stockham pass of radix R over two sequences of length n (src -> dst),
// twiddles tw (shared, e^{-2 pi i t / n}).
template <int R>
__device__ void pass(int n, const double2* tw, const double2* src, double2* dst, int ns, bool inv) {
  const int m = n / R;
  const int step = n / (ns * R);
  for (int t = threadIdx.x; t < 2 * m; t += kPassThreads) {
    const int q = t >= m ? 1 : 0, j = t - q * m;
    const int jj = j / ns, k = j - jj * ns;
    const double2* s = src + q * n + j;
    double2 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = s[r * m];
    if (ns > 1) {
#pragma unroll
      for (int r = 1; r < R; ++r) {
        const double2 w = tw[r * k * step];
        v[r] = dct::cmul(v[r], inv ? dct::cconj(w) : w);
      }
    }
    dft<R>(v, inv);
    double2* d = dst + q * n + jj * ns * R + k;
#pragma unroll
    for (int r = 0; r < R; ++r) d[r * ns] = v[r];
  }
}

__device__ double2* fft2(const PlanArgs& p, const double2* tw, double2* a, double2* b, bool inv) {
  int ns = 1;
  double2* src = a;
  double2* dst = b;
  for (int st = 0; st < p.nrad; ++st) {
    const int R = p.radix[st];
    switch (R) {
      case 2: pass<2>(p.n, tw, src, dst, ns, inv); break;
      case 3: pass<3>(p.n, tw, src, dst, ns, inv); break;
      case 4: pass<4>(p.n, tw, src, dst, ns, inv); break;
      case 5: pass<5>(p.n, tw, src, dst, ns, inv); break;
      default: pass<8>(p.n, tw, src, dst, ns, inv); break;
    }
    __syncthreads();
    ns *= R;
    double2* t = src;
    src = dst;
    dst = t;
  }
  return src;
}

__global__ void __launch_bounds__(kPassThreads, 1) mix_pass_kernel(PlanArgs p, const double* in, double* out, i64 st,
                                                                  i64 nfib, const double* __restrict__ sign,
                                                                  int forward) {
  extern __shared__ __align__(16) double2 psm[];
  const int n = p.n, tid = threadIdx.x;
  double2* tw = psm;                                              // [n]
  double2* ph = tw + n;                                           // [n]
  double2* b0 = ph + n;                                           // [2 * n]
  double2* b1 = b0 + 2 * n;                                       // [2 * n]
  double* stage = reinterpret_cast<double*>(b1 + 2 * n);          // [2][kGroup * n]
  double* sg = stage + 2 * kGroup * n;                            // [n]
  __shared__ i64 fbase[2][kGroup];
  for (int i = tid; i < n; i += kPassThreads) {
    tw[i] = p.tw[i];
    ph[i] = p.phase[i];
    sg[i] = sign ? sign[i] : 1.0;
  }
  const i64 ng = (nfib + kGroup - 1) / kGroup;
  const bool contig = (st == 1);
  // issue the cp.async loads of group g into stage buffer bi
  auto load = [&](i64 g, int bi) {
    double* dstb = stage + bi * kGroup * n;
    const i64 f0 = g * kGroup;
    if (tid < kGroup) {
      const i64 f = f0 + tid;
      const i64 hi = f / st, lo = f - hi * st;
      fbase[bi][tid] = (f < nfib) ? hi * st * n + lo : -1;
    }
    __syncthreads();
    if (contig) {
      // fibers f0.. are consecutive runs of n: one stretch of kGroup * n
      // (fibers past nfib are zero-filled: they share a complex sequence)
      const i64 cnt = min(static_cast<i64>(kGroup), nfib - f0) * n;
      const double* srcp = in + f0 * n;
      const bool al = ((reinterpret_cast<uintptr_t>(srcp) & 15) == 0);
      const int tot = kGroup * n;
      if (al) {
        for (int e = 2 * tid; e < tot; e += 2 * kPassThreads) {
          const i64 rem = cnt - e;
          cp_async16(dstb + e, rem > 0 ? srcp + e : in, rem >= 2 ? 16 : (rem == 1 ? 8 : 0));
        }
      } else {
        for (int e = tid; e < tot; e += kPassThreads) cp_async8(dstb + e, e < cnt ? srcp + e : in, e < cnt ? 8 : 0);
      }
    } else {
      // element i of fiber fl at fbase[fl] + i * st; stage layout [i][fl]
      const bool adj = fbase[bi][0] >= 0 && fbase[bi][kGroup - 1] == fbase[bi][0] + (kGroup - 1) &&
                       ((fbase[bi][0] & 1) == 0) && ((reinterpret_cast<uintptr_t>(in) & 15) == 0);
      if (adj) {
        for (int e = tid; e < n * 2; e += kPassThreads) {
          const int i = e >> 1, h = e & 1;
          cp_async16(dstb + i * kGroup + 2 * h, in + fbase[bi][0] + static_cast<i64>(i) * st + 2 * h, 16);
        }
      } else {
        for (int e = tid; e < n * kGroup; e += kPassThreads) {
          const int i = e / kGroup, fl = e - i * kGroup;
          const i64 b = fbase[bi][fl];
          cp_async8(dstb + e, b >= 0 ? in + b + static_cast<i64>(i) * st : in, b >= 0 ? 8 : 0);
        }
      }
    }
    cp_async_commit();
  };
  int it = 0;
  if (static_cast<i64>(blockIdx.x) < ng) load(blockIdx.x, 0);
  for (i64 g = blockIdx.x; g < ng; g += gridDim.x, ++it) {
    const int bi = it & 1;
    const i64 gn = g + gridDim.x;
    if (gn < ng) load(gn, bi ^ 1);
    else cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const double* sb = stage + bi * kGroup * n;
    // stage -> complex sequences (fibers 0,1 -> sequence 0; 2,3 -> 1)
    for (int e0 = tid; e0 < n * kGroup; e0 += kPassThreads) {
      // contiguous: e0 walks fiber-major as (fl, i) without a division
      int i, fl, e;
      if (contig) {
        fl = e0 & (kGroup - 1);
        i = e0 >> 2;
        e = fl * n + i;
      } else {
        i = e0 >> 2;
        fl = e0 & (kGroup - 1);
        e = e0;
      }
      double v = sb[e];
      const int q = fl >> 1;
      if (forward) {
        v *= sg[i];  // D_n first (mixing.hpp:148)
        const int d = (i & 1) ? (n - 1 - (i >> 1)) : (i >> 1);
        reinterpret_cast<double*>(&b0[q * n + d])[fl & 1] = v;
      } else {
        reinterpret_cast<double*>(&b1[q * n + i])[fl & 1] = v;
      }
    }
    __syncthreads();
    double2* res;
    if (forward) {
      res = fft2(p, tw, b0, b1, false);
    } else {
      const double inv0 = 1.0 / p.s0, invk = 1.0 / p.sk;
      for (int t = tid; t < 2 * n; t += kPassThreads) {
        const int q = t >= n ? 1 : 0, k = t - q * n;
        const double2 yk = b1[q * n + k];
        const double2 ynk = (k == 0) ? make_double2(0.0, 0.0) : b1[q * n + (n - k)];
        const double ik = (k == 0) ? inv0 : invk;
        const double2 phc = dct::cconj(ph[k]);
        const double2 u1 = make_double2(yk.x * ik, -ynk.x * invk);
        const double2 u2 = make_double2(yk.y * ik, -ynk.y * invk);
        const double2 v1 = dct::cmul(phc, u1), v2 = dct::cmul(phc, u2);
        b0[q * n + k] = make_double2(v1.x - v2.y, v1.y + v2.x);
      }
      __syncthreads();
      res = fft2(p, tw, b0, b1, true);
    }
    // epilogue + store (same formulas as dct::transform_group)
    const double invn = 1.0 / static_cast<double>(n);
    for (int e0 = tid; e0 < n * kGroup; e0 += kPassThreads) {
      int i, fl;
      if (contig) {  // consecutive threads along i: coalesced stores
        fl = e0 / n;
        i = e0 - fl * n;
      } else {
        i = e0 >> 2;
        fl = e0 & (kGroup - 1);
      }
      const i64 b = fbase[bi][fl];
      if (b < 0) continue;
      const int q = fl >> 1;
      double v;
      if (forward) {
        const double2 z = res[q * n + i];
        const double2 zc = res[q * n + (i == 0 ? 0 : n - i)];
        const double2 w = ph[i];
        const double sc = (i == 0) ? p.s0 : p.sk;
        if ((fl & 1) == 0) {
          const double vx = 0.5 * (z.x + zc.x), vy = 0.5 * (z.y - zc.y);
          v = sc * (w.x * vx - w.y * vy);
        } else {
          const double vx = 0.5 * (z.y + zc.y), vy = -0.5 * (z.x - zc.x);
          v = sc * (w.x * vx - w.y * vy);
        }
      } else {
        const int mm = (i & 1) ? (n - 1 - (i >> 1)) : (i >> 1);
        const double2 z = res[q * n + mm];
        v = ((fl & 1) ? z.y : z.x) * invn;
        v *= sg[i];  // D_n after the adjoint (mixing.hpp:231)
      }
      out[b + static_cast<i64>(i) * st] = v;
    }
    __syncthreads();
  }
  cp_async_wait<0>();
}

}  // namespace

size_t mix_pass_smem(int n) {
  return static_cast<size_t>(n) * (16 + 16 + 32 + 32 + 2 * kGroup * 8 + 8);
}

bool mix_pass_supported(const DctPlan& p) {
  for (int i = 0; i < p.nrad; ++i)
    if (p.radix[i] != 2 && p.radix[i] != 3 && p.radix[i] != 4 && p.radix[i] != 5 && p.radix[i] != 8) return false;
  return mix_pass_smem(p.n) <= 220 * 1024;
}

void launch_mix_pass(const DctPlan& pl, const double* in, double* out, i64 st, i64 nfib, const double* sign,
                     int forward, cudaStream_t stream) {
  PlanArgs a = dct_args(pl);
  const size_t smem = mix_pass_smem(pl.n);
  static size_t configured = 0;
  if (smem > configured) {
    CPB_CUDA(cudaFuncSetAttribute(mix_pass_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    configured = smem;
  }
  int dev = 0, sms = 148;
  CPB_CUDA(cudaGetDevice(&dev));
  CPB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const i64 ng = (nfib + kGroup - 1) / kGroup;
  const int grid = static_cast<int>(std::min<i64>(ng, sms));
  mix_pass_kernel<<<grid, kPassThreads, smem, stream>>>(a, in, out, st, nfib, sign, forward);
  CPB_LAUNCH_CHECK();
}

}  // namespace cpb
