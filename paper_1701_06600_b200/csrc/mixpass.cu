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
#include <algorithm>

#include "dct.cuh"
#include "devutil.cuh"

namespace cpb {

namespace {

constexpr int kPassThreads = 512;
constexpr int kGroup = 4;  // fibers per group (two complex sequences)

using dct::PlanArgs;

using dct::dft;

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

// ---------------------------------------------------------------------------
// Forward pass, groups of 2 SEQ fibers (SEQ complex sequences; SEQ grows as
// the fibers get shorter so a pass keeps ~NT butterflies per barrier), NT =
// 256 threads per CTA for SEQ = 2 (two CTAs per SM: independent barrier
// domains) and 512 above:
//  * the first radix pass reads its butterfly inputs straight from global
//    memory into registers (sign and the even/odd reorder folded into the
//    addressing): no staging buffer, no packing pass;
//  * those loads are issued one group ahead, so they stream in while the
//    current group's remaining passes and epilogue run;
//  * per-pass index constants (multiply-high magics instead of divisions)
//    are formed once per CTA.

// j / d for j * d < 2^32, with M = floor((2^32 - 1) / d) + 1
__device__ __forceinline__ int udiv(int j, unsigned M) { return static_cast<int>(__umulhi(static_cast<unsigned>(j), M)); }
__host__ __device__ constexpr unsigned umagic(int d) { return 0xffffffffu / static_cast<unsigned>(d) + 1u; }

struct PassK {  // one Stockham pass: butterflies per sequence m, ns, twiddle step, magics
  int m, ns, step;
  unsigned Mm, Mns;
};

template <int SEQ>
constexpr int fwd_threads() { return SEQ == 2 ? 256 : 512; }

template <int R, int SEQ>
__device__ void pass_seq(const PassK& c, int ss, const double2* tw, const double2* src, double2* dst) {
  constexpr int NT = fwd_threads<SEQ>();
  const int m = c.m, ns = c.ns, step = c.step;
  for (int t = threadIdx.x; t < SEQ * m; t += NT) {
    const int q = udiv(t, c.Mm), j = t - q * m;
    const int jj = udiv(j, c.Mns), k = j - jj * ns;
    const double2* sp = src + q * ss + j;
    double2 v[R], w[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = sp[r * m];
#pragma unroll
    for (int r = 1; r < R; ++r) w[r] = tw[r * k * step];
#pragma unroll
    for (int r = 1; r < R; ++r) v[r] = dct::cmul(v[r], w[r]);
    dft<R>(v, false);
    double2* d = dst + q * ss + jj * ns * R + k;
#pragma unroll
    for (int r = 0; r < R; ++r) d[r * ns] = v[r];
  }
}

// STG (contiguous fibers only): the group's FIB * n doubles are one
// contiguous range; it streams into a shared staging buffer with cp.async
// (fully coalesced) instead of the strided per-butterfly register loads.
template <int R1, int SEQ, bool STG>
__global__ void __launch_bounds__(fwd_threads<SEQ>(), 512 / fwd_threads<SEQ>()) mix_pass_fwd_kernel(
    PlanArgs p, const double* in, double* out, i64 st, i64 nfib, const double* __restrict__ sign) {
  constexpr int NT = fwd_threads<SEQ>(), FIB = 2 * SEQ;
  extern __shared__ __align__(16) double2 psm[];
  const int n = p.n, tid = threadIdx.x;
  const int ss = n + 1;                                   // sequence stride (banks)
  double2* tw = psm;                                      // [n]
  double2* ph = tw + n;                                   // [n]
  double2* b0 = ph + n;                                   // [SEQ * ss]
  double2* b1 = b0 + SEQ * ss;                            // [SEQ * ss]
  double* sg = reinterpret_cast<double*>(b1 + SEQ * ss);  // [n]
  double* stg = sg + n + (n & 1);                         // STG: [2][FIB * n] (16-byte aligned)
  __shared__ i64 fbase[2][FIB];
  __shared__ PassK pk[24];
  for (int i = tid; i < n; i += NT) {
    tw[i] = p.tw[i];
    ph[i] = p.phase[i];
    sg[i] = sign ? sign[i] : 1.0;
  }
  if (tid == 0) {
    int ns = R1;
    for (int q = 1; q < p.nrad; ++q) {
      const int R = p.radix[q];
      PassK c;
      c.m = n / R;
      c.ns = ns;
      c.step = n / (ns * R);
      c.Mm = umagic(c.m);
      c.Mns = umagic(ns);
      pk[q] = c;
      ns *= R;
    }
  }
  const i64 ng = (nfib + FIB - 1) / FIB;
  const bool contig = (st == 1);
  // this thread's first-pass butterfly (fixed for every group): sequence bq,
  // index bj, and the fiber element feeding each of its R1 inputs
  // (contiguous fibers: consecutive lanes along j; strided: the SEQ
  // sequences of one j in adjacent lanes, so a warp reads whole rows)
  const int m1 = n / R1;
  const bool bact = tid < SEQ * m1;
  const int bq = !bact ? 0 : (contig ? udiv(tid, umagic(m1)) : (tid & (SEQ - 1)));
  const int bj = !bact ? 0 : (contig ? tid - bq * m1 : (tid / SEQ));
  int ei[R1];
#pragma unroll
  for (int r = 0; r < R1; ++r) {
    const int d = bj + r * m1;
    ei[r] = (d < (n + 1) / 2) ? 2 * d : 2 * (n - 1 - d) + 1;  // Makhoul reorder, inverted
  }
  auto bases = [&](i64 g, int slot) {
    if (tid < FIB) {
      const i64 f = g * FIB + tid;
      const i64 hi = f / st, lo = f - hi * st;
      fbase[slot][tid] = (g < ng && f < nfib) ? hi * st * n + lo : -1;
    }
  };
  double va[R1], vb[R1];  // first-pass inputs of the group in flight
  const bool in16 = (reinterpret_cast<uintptr_t>(in) & 15) == 0;
  auto stage = [&](i64 g, int slot) {  // STG: group g's fibers -> stg[slot]
    double* d = stg + slot * FIB * n;
    const i64 f0 = g * FIB;
    const i64 cnt = g < ng ? min(static_cast<i64>(FIB), nfib - f0) * n : 0;  // doubles present
    const double* srcp = in + f0 * n;
    if (in16) {
      for (int e = 2 * tid; e < FIB * n; e += 2 * NT) {
        const i64 rem = cnt - e;
        cp_async16(d + e, rem > 0 ? srcp + e : in, rem >= 2 ? 16 : (rem == 1 ? 8 : 0));
      }
    } else {
      for (int e = tid; e < FIB * n; e += NT) cp_async8(d + e, e < cnt ? srcp + e : in, e < cnt ? 8 : 0);
    }
    cp_async_commit();
  };
  auto load_stg = [&](int slot) {  // STG: first-pass inputs from the staging buffer
    const double* d = stg + slot * FIB * n + 2 * bq * n;
#pragma unroll
    for (int r = 0; r < R1; ++r) {
      va[r] = d[ei[r]];
      vb[r] = d[n + ei[r]];
    }
  };
  auto load = [&](int slot) {
    const i64 ba = bact ? fbase[slot][2 * bq] : -1, bb = bact ? fbase[slot][2 * bq + 1] : -1;
    if (!contig && in16 && ba >= 0 && bb == ba + 1 && (ba & 1) == 0 && (st & 1) == 0) {
      // the pair of fibers is adjacent and aligned: one 16-byte load per row
#pragma unroll
      for (int r = 0; r < R1; ++r) {
        const double2 t = __ldcg(reinterpret_cast<const double2*>(in + ba + static_cast<i64>(ei[r]) * st));
        va[r] = t.x;
        vb[r] = t.y;
      }
    } else {
#pragma unroll
      for (int r = 0; r < R1; ++r) {
        // L1-cached: contiguous fibers read every other element per lane
        // (the reorder), the other half hits in L1 from a neighbouring warp.
        // Safe in place: a fiber is read once, by this CTA, before it is
        // written, and no CTA re-reads another group's bytes.
        const i64 off = static_cast<i64>(ei[r]) * st;
        va[r] = ba >= 0 ? in[ba + off] : 0.0;
        vb[r] = bb >= 0 ? in[bb + off] : 0.0;
      }
    }
  };
  bases(blockIdx.x, 0);
  if constexpr (STG) {
    stage(blockIdx.x, 0);
  } else {
    __syncthreads();
    load(0);
  }
  int it = 0;
  for (i64 g = blockIdx.x; g < ng; g += gridDim.x, ++it) {
    const int cur = it & 1;
    bases(g + gridDim.x, cur ^ 1);
    if constexpr (STG) {
      cp_async_wait<0>();
      __syncthreads();
      if (bact) load_stg(cur);
    }
    // first pass (ns = 1: no twiddles): sign, reorder, DFT_R1 -> b0
    if (bact) {
      double2 v[R1];
#pragma unroll
      for (int r = 0; r < R1; ++r) {
        const double sgn = sg[ei[r]];
        v[r] = make_double2(sgn * va[r], sgn * vb[r]);
      }
      dft<R1>(v, false);
      double2* d = b0 + bq * ss + bj * R1;
#pragma unroll
      for (int r = 0; r < R1; ++r) d[r] = v[r];
    }
    __syncthreads();
    // the next group streams in behind the remaining passes
    if constexpr (STG)
      stage(g + gridDim.x, cur ^ 1);
    else
      load(cur ^ 1);
    double2* src = b0;
    double2* dst = b1;
    for (int stg = 1; stg < p.nrad; ++stg) {
      const PassK c = pk[stg];
      switch (p.radix[stg]) {
        case 2: pass_seq<2, SEQ>(c, ss, tw, src, dst); break;
        case 3: pass_seq<3, SEQ>(c, ss, tw, src, dst); break;
        case 4: pass_seq<4, SEQ>(c, ss, tw, src, dst); break;
        case 5: pass_seq<5, SEQ>(c, ss, tw, src, dst); break;
        default: pass_seq<8, SEQ>(c, ss, tw, src, dst); break;
      }
      __syncthreads();
      double2* t = src;
      src = dst;
      dst = t;
    }
    const double2* res = src;
    // epilogue (dct::transform_group's forward formulas) + store
    auto emit = [&](int i, int fl) {
      const i64 b = fbase[cur][fl];
      if (b < 0) return;
      const int q = fl >> 1;
      const double2 z = res[q * ss + i];
      const double2 zc = res[q * ss + (i == 0 ? 0 : n - i)];
      const double2 w = ph[i];
      const double sc = (i == 0) ? p.s0 : p.sk;
      double vx, vy;
      if ((fl & 1) == 0) {
        vx = 0.5 * (z.x + zc.x);
        vy = 0.5 * (z.y - zc.y);
      } else {
        vx = 0.5 * (z.y + zc.y);
        vy = -0.5 * (z.x - zc.x);
      }
      out[b + static_cast<i64>(i) * st] = sc * (w.x * vx - w.y * vy);
    };
    if (contig) {  // consecutive threads along i (fibers back to back): coalesced stores
      const unsigned Mn = umagic(n);
      for (int e = tid; e < FIB * n; e += NT) {
        const int fl = udiv(e, Mn);
        emit(e - fl * n, fl);
      }
    } else {  // consecutive threads along the adjacent fibers
      for (int e0 = tid; e0 < n * FIB; e0 += NT) emit(e0 / FIB, e0 & (FIB - 1));
    }
    __syncthreads();
  }
}

template <int SEQ>
size_t mix_pass_fwd_smem(int n, bool stg) {
  return static_cast<size_t>(n) * (16 + 16 + 8) + 8 + 2 * SEQ * static_cast<size_t>(n + 1) * 16 +
         (stg ? 2 * 2 * SEQ * static_cast<size_t>(n) * 8 : 0);
}

// radices for the forward kernel: 8s first, then 4, 2, 5, 3, largest first
// (0 entries: n has another prime factor)
int fwd_radices(int n, int* rad) {
  int k = 0, m = n;
  while (m % 8 == 0) { rad[k++] = 8; m /= 8; }
  while (m % 4 == 0) { rad[k++] = 4; m /= 4; }
  while (m % 2 == 0) { rad[k++] = 2; m /= 2; }
  while (m % 5 == 0) { rad[k++] = 5; m /= 5; }
  while (m % 3 == 0) { rad[k++] = 3; m /= 3; }
  if (m != 1 || k > 24) return 0;
  std::sort(rad, rad + k, [](int a, int b) { return a > b; });
  return k;
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

namespace {
template <int SEQ>
bool launch_fwd(PlanArgs a, int nr, const int* rad, const double* in, double* out, i64 st, i64 nfib,
                const double* sign, cudaStream_t stream, bool stg, bool prep) {
  constexpr int NT = fwd_threads<SEQ>();
  const int n = a.n, r1 = rad[0];
  const int per_sm = 512 / NT;
  if (SEQ * (n / r1) > NT || per_sm * mix_pass_fwd_smem<SEQ>(n, stg) > 220 * 1024) return false;
  a.nrad = nr;
  for (int i = 0; i < nr; ++i) a.radix[i] = rad[i];
  void* fn = nullptr;
#define CPB_FWD(R) (stg ? reinterpret_cast<void*>(&mix_pass_fwd_kernel<R, SEQ, true>) \
                        : reinterpret_cast<void*>(&mix_pass_fwd_kernel<R, SEQ, false>))
  switch (r1) {
    case 2: fn = CPB_FWD(2); break;
    case 3: fn = CPB_FWD(3); break;
    case 4: fn = CPB_FWD(4); break;
    case 5: fn = CPB_FWD(5); break;
    default: fn = CPB_FWD(8); break;
  }
#undef CPB_FWD
  const size_t smem = mix_pass_fwd_smem<SEQ>(n, stg);
  CPB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  int dev = 0, sms = 148, per = 1;
  CPB_CUDA(cudaGetDevice(&dev));
  CPB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CPB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, NT, smem));
  if (prep) return true;  // the kernel is loaded and configured
  const i64 ng = (nfib + 2 * SEQ - 1) / (2 * SEQ);
  const int grid = static_cast<int>(std::min<i64>(ng, static_cast<i64>(sms) * std::max(per, 1)));
  void* args[] = {&a, const_cast<double**>(&in), &out, &st, &nfib, const_cast<double**>(&sign)};
  CPB_CUDA(cudaLaunchKernel(fn, dim3(grid), dim3(NT), args, smem, stream));
  return true;
}

// sequences per group: contiguous fibers of length >= 512 use 2 (two CTAs
// per SM, direct loads); otherwise the most (<= 32) whose first pass fits 512
// threads (contiguous fibers through the staging buffer)
bool launch_fwd_any(PlanArgs a, int nr, const int* rad, const double* in, double* out, i64 st, i64 nfib,
                    const double* sign, cudaStream_t stream, bool prep) {
  const int m1 = a.n / rad[0];
  if (st == 1 && a.n >= 512) return launch_fwd<2>(a, nr, rad, in, out, st, nfib, sign, stream, false, prep);
  const bool stg = st == 1;
  if (32 * m1 <= 512 && launch_fwd<32>(a, nr, rad, in, out, st, nfib, sign, stream, stg, prep)) return true;
  if (16 * m1 <= 512 && launch_fwd<16>(a, nr, rad, in, out, st, nfib, sign, stream, stg, prep)) return true;
  if (8 * m1 <= 512 && launch_fwd<8>(a, nr, rad, in, out, st, nfib, sign, stream, stg, prep)) return true;
  if (4 * m1 <= 512 && launch_fwd<4>(a, nr, rad, in, out, st, nfib, sign, stream, stg, prep)) return true;
  return launch_fwd<2>(a, nr, rad, in, out, st, nfib, sign, stream, stg, prep);
}
}  // namespace

void launch_mix_pass(const DctPlan& pl, const double* in, double* out, i64 st, i64 nfib, const double* sign,
                     int forward, cudaStream_t stream, bool prepare_only) {
  // v4: register four-step FFT for strided modes of supported lengths (mixreg.cu)
  if (forward && in == out && launch_mix_reg(pl, out, st, nfib, sign, stream, prepare_only)) return;
  // v3: TMA-fed in-place pipeline (mixtma.cu) when the shape suits it
  if (forward && in == out && launch_mix_tma(pl, out, st, nfib, sign, stream, prepare_only)) return;
  PlanArgs a = dct_args(pl);
  int rad[24];
  const int nr = fwd_radices(pl.n, rad);
  if (forward && nr > 0 && launch_fwd_any(a, nr, rad, in, out, st, nfib, sign, stream, prepare_only)) return;
  const size_t smem = mix_pass_smem(pl.n);
  static size_t configured = 0;
  if (smem > configured) {
    CPB_CUDA(cudaFuncSetAttribute(mix_pass_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    configured = smem;
  }
  if (prepare_only) return;
  int dev = 0, sms = 148;
  CPB_CUDA(cudaGetDevice(&dev));
  CPB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const i64 ng = (nfib + kGroup - 1) / kGroup;
  const int grid = static_cast<int>(std::min<i64>(ng, sms));
  mix_pass_kernel<<<grid, kPassThreads, smem, stream>>>(a, in, out, st, nfib, sign, forward);
  CPB_LAUNCH_CHECK();
}

}  // namespace cpb
