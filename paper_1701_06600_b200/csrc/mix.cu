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

#include "dct.cuh"
#include "qr.cuh"
#include <algorithm>

namespace cpb {

namespace {

constexpr int kMixThreads = 256;
using dct::PlanArgs;

__global__ void __launch_bounds__(kMixThreads) mode_transform_kernel(PlanArgs p, const double* in,
                                                                    double* out, i64 st, i64 nfib,
                                                                    int F, const double* sign,
                                                                    int forward,
                                                                    const double* col_div) {
  extern __shared__ __align__(16) double2 sbuf[];
  dct::transform_group(p, in, out, st, nfib, static_cast<i64>(blockIdx.x) * F, F, sign, forward, col_div, sbuf);
}

// Walsh-Hadamard mixing (transforms.hpp:170-197): natural (Hadamard) order,
// butterflies x[i+k] = u + v, x[i+k+len] = u - v for len = 1, 2, 4, ..., then
// the 1/sqrt(n) scale: the reference's operations in its order, so the
// result is bit-identical. forward: sign first; adjoint (= forward): sign
// after. F fibers per CTA in shared memory.
__global__ void __launch_bounds__(kMixThreads) wht_mode_kernel(int n, const double* in, double* out, i64 st,
                                                              i64 nfib, int F, const double* __restrict__ sign,
                                                              int forward, const double* __restrict__ col_div,
                                                              double scale) {
  extern __shared__ __align__(16) double wbuf[];
  const i64 f0 = static_cast<i64>(blockIdx.x) * F;
  const int cnt = static_cast<int>(min(static_cast<i64>(F), nfib - f0));
  const bool contig = (st == 1);
  for (int t = threadIdx.x; t < F * n; t += blockDim.x) {
    int fl, i;
    if (contig) {
      fl = t / n;
      i = t - fl * n;
    } else {
      i = t / F;
      fl = t - i * F;
    }
    double v = 0.0;
    if (fl < cnt) {
      v = in[dct::fib_addr(f0 + fl, i, st, n)];
      if (col_div) v = v / col_div[f0 + fl];
      if (forward && sign) v = v * sign[i];
    }
    wbuf[fl * n + i] = v;
  }
  __syncthreads();
  const int half = n / 2;
  for (int len = 1; len < n; len <<= 1) {
    for (int t = threadIdx.x; t < F * half; t += blockDim.x) {
      const int fl = t / half, k2 = t - fl * half;
      const int i = (k2 / len) * 2 * len + (k2 % len);
      double* x = wbuf + fl * n;
      const double u = x[i], v = x[i + len];
      x[i] = u + v;
      x[i + len] = u - v;
    }
    __syncthreads();
  }
  for (int t = threadIdx.x; t < F * n; t += blockDim.x) {
    int fl, i;
    if (contig) {
      fl = t / n;
      i = t - fl * n;
    } else {
      i = t / F;
      fl = t - i * F;
    }
    if (fl >= cnt) continue;
    double v = wbuf[fl * n + i] * scale;
    if (!forward && sign) v = v * sign[i];
    out[dct::fib_addr(f0 + fl, i, st, n)] = v;
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

// MIX chain: the RHS reduction, or in QR mode (qr.cuh) the QR solution rows
// of block b (BI = 256 / RT rows; the unmix transform and the apply with
// ginv = I follow as for the RHS)
template <int RT>
__global__ void __launch_bounds__(256) reduce_rhs_qr_kernel(ModeWork w, i64 in, int r, double* __restrict__ out) {
  if (w.stop && *w.stop) return;
  constexpr int BI = 256 / RT;
  if (w.qrws && __ldcg(w.info + 2) != 0) {
    __shared__ double st[ph::qr_rows_smem_doubles<RT, 256>()];
    __shared__ double rows[BI * (RT + 1)];
    const i64 i0 = static_cast<i64>(blockIdx.x) * BI;
    if (i0 >= in) return;  // uniform per block
    ph::qr_rows<RT, 256>(w.q, w.qrws, r, in, i0, BI, rows, RT + 1, st);
    const int il = threadIdx.x / RT, c = threadIdx.x % RT;
    if (i0 + il < in && c < r) out[(i0 + il) * r + c] = rows[il * (RT + 1) + c];
    return;
  }
  const i64 e = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= in * r) return;
  double s = 0.0;
  for (int k = 0; k < w.ks; ++k) s += w.part_rhs[static_cast<i64>(k) * in * r + e];
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
      // any prime: radices above 8 run dct.cuh's generic O(R) Stockham pass
      // (the reference's Bluestein FFT, transforms.hpp:27-118, computes the
      // same DFT; the fast whole-tensor passes take smooth lengths only)
      if (p.nrad >= 24) throw Unsupported("dct length has too many factors");
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

DctPlan make_mix_plan(int kind, int n) {
  if (kind == 2) {
    if (n < 1 || (n & (n - 1)) != 0) throw InvalidArgument("wht requires power-of-two mode lengths");
    DctPlan p;
    p.kind = 2;
    p.n = n;
    return p;
  }
  return make_dct_plan(n);
}

void free_dct_plan(DctPlan& p) {
  if (p.tw) cudaFree(p.tw);
  if (p.phase) cudaFree(p.phase);
  p.tw = p.phase = nullptr;
}

DctArgs dct_args(const DctPlan& p) {
  DctArgs a;
  a.n = p.n;
  a.nrad = p.nrad;
  for (int i = 0; i < 24; ++i) a.radix[i] = p.radix[i];
  a.tw = p.tw;
  a.phase = p.phase;
  a.s0 = p.s0;
  a.sk = p.sk;
  return a;
}

int dct_fibers_per_cta(int n, size_t budget) {
  int F = static_cast<int>(budget / (16 * static_cast<size_t>(n)));
  F = F > 32 ? 32 : F;
  F &= ~1;
  return F < 2 ? 2 : F;
}

void prepare_mode_transform(const DctPlan& p, i64 st, i64 nfib, int forward) {
  if (p.kind == 2) return;
  if (nfib >= 4096 && mix_pass_supported(p)) launch_mix_pass(p, nullptr, nullptr, st, nfib, nullptr, forward, nullptr, true);
}

void launch_mode_transform(const DctPlan& p, const double* in, double* out, i64 st, i64 nfib,
                           const double* sign, int forward, const double* col_div,
                           cudaStream_t stream) {
  if (nfib <= 0) return;
  if (p.kind == 2) {
    int F = static_cast<int>((96 * 1024) / (8 * static_cast<size_t>(p.n)));
    F = F > 32 ? 32 : (F < 1 ? 1 : F);
    const size_t smem = static_cast<size_t>(F) * p.n * sizeof(double);
    static size_t configured = 0;
    if (smem > configured) {
      CPB_CUDA(cudaFuncSetAttribute(wht_mode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
      configured = smem;
    }
    const double scale = 1.0 / std::sqrt(static_cast<double>(p.n));
    wht_mode_kernel<<<static_cast<unsigned>((nfib + F - 1) / F), kMixThreads, smem, stream>>>(
        p.n, in, out, st, nfib, F, sign, forward, col_div, scale);
    CPB_LAUNCH_CHECK();
    return;
  }
  if (nfib >= 4096 && col_div == nullptr && in == out && mix_pass_supported(p)) {
    launch_mix_pass(p, in, out, st, nfib, sign, forward, stream);  // whole-tensor pass
    return;
  }
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

void launch_reduce_rhs_qr(const ModeWork& w, i64 in, int r, double* out, cudaStream_t st) {
  const int rt = rank_bucket(r);
  const int grid = std::max(ceil_div(in * r, 256), ceil_div(in, 256 / rt));
  switch (rt) {
    case 16: reduce_rhs_qr_kernel<16><<<grid, 256, 0, st>>>(w, in, r, out); break;
    case 32: reduce_rhs_qr_kernel<32><<<grid, 256, 0, st>>>(w, in, r, out); break;
    default: reduce_rhs_qr_kernel<64><<<grid, 256, 0, st>>>(w, in, r, out); break;
  }
  CPB_LAUNCH_CHECK();
}

void launch_reduce_rhs(const double* part_rhs, int ks, i64 in, int r, double* out,
                       cudaStream_t st) {
  const i64 n = in * r;
  reduce_rhs_kernel<<<ceil_div(n, 256), 256, 0, st>>>(part_rhs, ks, in, r, out);
  CPB_LAUNCH_CHECK();
}

}  // namespace cpb
