// CPRAND-MIX with the reference's default transform, the unitary FFT
// (mixing.hpp:326-345 -> cprand_mix_impl<Complex>, :258-318): the mixed
// tensor and the mixed factors are complex, the factors stay real.
//
// Per mode n the reference forms the complex Z_S from the mixed factors,
// gathers the complex fibers of X_hat, unmixes the S sampled right-hand-side
// rows (F^H then D_n, unmix_sampled_rhs :218-236) and solves the real-
// constrained least squares of the stacked system [Re Z; Im Z] A^T =
// [Re B; Im B] (real_least_squares :246-254). With B = G conj(F) D the
// normal equations of the stacked system are
//     Re(Z^H Z) A^T = D Re(F^H (Z^H X_S)^T)
// so this path contracts first (C = Z^H X_S, R x I_n complex, one pass over
// the sampled complex fibers), unmixes the R rows of C instead of the S rows
// of B, and keeps the real part. The Gram is Re(Z^H Z). Apply, norms and the
// lambda rule are the real path's (mode_apply_kernel); the new factor is
// mixed again with the forward FFT (mix_factor :159-174).
//
// The FFT is dct.cuh's mixed-radix Stockham (fft_smem) on complex fibers
// staged in shared memory, unitary scaling 1/sqrt(n) as ModeTransform.
#include <algorithm>
#include <cmath>

#include "dct.cuh"

namespace cpb {

namespace {

constexpr int kCThreads = 256;
using dct::PlanArgs;

// Fibers [f0, f0 + F) of a mode (length n, stride st) through the unitary FFT.
// forward: v = D x (x real or complex), FFT, / sqrt(n)      (mix_tensor, mix_factor)
// adjoint: inverse FFT / sqrt(n), then D                    (unmix_sampled_rhs)
// in_real (nullable): real input; col_div (nullable): input fiber f divided
// by col_div[f] first (lazy column norms of a factor, fiber = column);
// out_real (nullable): store the real part there instead of out_c.
__global__ void __launch_bounds__(kCThreads) cfft_mode_kernel(PlanArgs p, const double* __restrict__ in_real,
                                                               const double2* in_c, double2* out_c,
                                                               double* __restrict__ out_real, i64 st, i64 nfib,
                                                               int F, const double* __restrict__ sign, int forward,
                                                               const double* __restrict__ col_div) {
  extern __shared__ __align__(16) double2 cbuf[];
  const int n = p.n;
  double2* a = cbuf;
  double2* b = cbuf + static_cast<size_t>(F) * n;
  const i64 f0 = static_cast<i64>(blockIdx.x) * F;
  const int fl_cnt = static_cast<int>(min(static_cast<i64>(F), nfib - f0));
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
    double2 v = make_double2(0.0, 0.0);
    if (fl < fl_cnt) {
      const i64 addr = dct::fib_addr(f0 + fl, i, st, n);
      v = in_real ? make_double2(in_real[addr], 0.0) : in_c[addr];
      if (col_div) {
        const double d = col_div[f0 + fl];
        v = make_double2(v.x / d, v.y / d);
      }
      if (forward && sign) v = make_double2(v.x * sign[i], v.y * sign[i]);
    }
    a[fl * n + i] = v;
  }
  __syncthreads();
  const double2* res = dct::fft_smem(p, a, b, F, !forward);
  const double sc = 1.0 / sqrt(static_cast<double>(n));
  for (int t = threadIdx.x; t < F * n; t += blockDim.x) {
    int fl, i;
    if (contig) {
      fl = t / n;
      i = t - fl * n;
    } else {
      i = t / F;
      fl = t - i * F;
    }
    if (fl >= fl_cnt) continue;
    double2 v = res[fl * n + i];
    v = make_double2(v.x * sc, v.y * sc);
    if (!forward && sign) v = make_double2(v.x * sign[i], v.y * sign[i]);
    const i64 addr = dct::fib_addr(f0 + fl, i, st, n);
    if (out_real)
      out_real[addr] = v.x;
    else
      out_c[addr] = v;
  }
}

// Z_S(s, c) = prod over kept modes (ascending) of mixed_m(i_m(s), c), complex
// (skr, sampling.hpp:74-92, on Mat<Complex>); v.fac[k] = the kept modes'
// mixed factors, complex row-major [i][c]. Written as the stacked real
// matrix [Re Z; Im Z] (2S x RT, zero-padded columns): its Gram is
// Re(Z^H Z), the Gram of real_least_squares' stacked system, so the real
// path's Gram kernel and inverse run on it unchanged.
__global__ void zc_kernel(ModeView v, int rt, double* __restrict__ zs) {
  const i64 e = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= static_cast<i64>(v.s) * rt) return;
  const int s = static_cast<int>(e / rt), c = static_cast<int>(e - static_cast<i64>(s) * rt);
  double2 zv = make_double2(0.0, 0.0);
  if (c < v.r) {
    zv = make_double2(1.0, 0.0);
    for (int k = 0; k < v.kept; ++k) {
      const double2 a = reinterpret_cast<const double2*>(v.fac[k])[static_cast<i64>(v.rows[k][s]) * v.r + c];
      zv = dct::cmul(zv, a);
    }
  }
  zs[static_cast<i64>(s) * rt + c] = zv.x;
  zs[(static_cast<i64>(v.s) + s) * rt + c] = zv.y;
}

// Split-K partials of C(i, c) = sum_s conj(Z(s, c)) X_hat(base_s + i st),
// the complex RHS before unmixing: CTA (row block of 32, split kb) sums the
// samples [kb klen, ...) into part[kb] (I_n x R complex row-major). Z is read
// from the stacked real layout (Re rows 0..S-1, Im rows S..2S-1, ld rt).
constexpr int kRows = 32;
constexpr int kZChunk = 32;
__global__ void __launch_bounds__(kCThreads) rhsc_kernel(const double2* __restrict__ xh, const i64* __restrict__ base,
                                                          i64 st, i64 in, int s, int klen, const double* __restrict__ zs,
                                                          int rt, int r, double2* __restrict__ part) {
  __shared__ double2 zsm[kZChunk * 64];
  __shared__ double2 xsm[kZChunk * kRows];
  const i64 i0 = static_cast<i64>(blockIdx.x) * kRows;
  const int sb = blockIdx.y * klen, se = min(s, sb + klen);
  const int tid = threadIdx.x;
  const int il = tid % kRows, cg = tid / kRows;  // 8 column groups
  double2 acc[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) acc[q] = make_double2(0.0, 0.0);
  for (int s0 = sb; s0 < se; s0 += kZChunk) {
    const int cnt = min(kZChunk, se - s0);
    for (int e = tid; e < cnt * r; e += kCThreads) {
      const int sl = e / r, c = e - sl * r;
      zsm[e] = make_double2(zs[static_cast<i64>(s0 + sl) * rt + c], zs[static_cast<i64>(s + s0 + sl) * rt + c]);
    }
    for (int e = tid; e < cnt * kRows; e += kCThreads) {
      const int sl = e / kRows, ii = e - sl * kRows;
      const i64 i = i0 + ii;
      xsm[e] = (i < in) ? xh[base[s0 + sl] + i * st] : make_double2(0.0, 0.0);
    }
    __syncthreads();
    for (int sl = 0; sl < cnt; ++sl) {
      const double2 x = xsm[sl * kRows + il];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int c = cg + 8 * q;
        if (c < r) {
          const double2 zc = zsm[sl * r + c];
          // conj(z) * x
          acc[q].x = fma(zc.x, x.x, fma(zc.y, x.y, acc[q].x));
          acc[q].y = fma(zc.x, x.y, fma(-zc.y, x.x, acc[q].y));
        }
      }
    }
    __syncthreads();
  }
  const i64 i = i0 + il;
  if (i < in)
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int c = cg + 8 * q;
      if (c < r) part[(static_cast<i64>(blockIdx.y) * in + i) * r + c] = acc[q];
    }
}

// C = sum of the split partials in split order
__global__ void rhsc_reduce_kernel(const double2* __restrict__ part, int ks, i64 n, double2* __restrict__ out) {
  const i64 e = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= n) return;
  double2 a = part[e];
  for (int k = 1; k < ks; ++k) {
    const double2 b = part[static_cast<i64>(k) * n + e];
    a = make_double2(a.x + b.x, a.y + b.y);
  }
  out[e] = a;
}

int fibers_per_cta(int n) {
  int F = static_cast<int>((96 * 1024) / (32 * static_cast<size_t>(n)));  // two complex buffers
  F = F > 16 ? 16 : F;
  return F < 1 ? 1 : F;
}

}  // namespace

void launch_cfft_mode(const DctPlan& pl, const double* in_real, const double* in_c, double* out_c, double* out_real,
                      i64 st, i64 nfib, const double* sign, int forward, const double* col_div, cudaStream_t stream) {
  if (nfib <= 0) return;
  const int F = fibers_per_cta(pl.n);
  const size_t smem = 2 * static_cast<size_t>(F) * pl.n * sizeof(double2);
  if (smem > 200 * 1024) throw Unsupported("FFT mixing: mode length too large for one CTA");
  static size_t configured = 0;
  if (smem > configured) {
    CPB_CUDA(cudaFuncSetAttribute(cfft_mode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    configured = smem;
  }
  const i64 grid = (nfib + F - 1) / F;
  cfft_mode_kernel<<<static_cast<unsigned>(grid), kCThreads, smem, stream>>>(
      dct_args(pl), in_real, reinterpret_cast<const double2*>(in_c), reinterpret_cast<double2*>(out_c), out_real, st,
      nfib, F, sign, forward, col_div);
  CPB_LAUNCH_CHECK();
}

void launch_zc(const ModeView& v, int rt, double* zs, cudaStream_t stream) {
  const i64 tot = static_cast<i64>(v.s) * rt;
  zc_kernel<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, stream>>>(v, rt, zs);
  CPB_LAUNCH_CHECK();
}

int rhsc_splits(i64 in, int s, int sms) {
  const i64 rb = (in + kRows - 1) / kRows;
  i64 ks = std::max<i64>(1, (2 * static_cast<i64>(sms)) / rb);
  ks = std::min<i64>(ks, (s + kZChunk - 1) / kZChunk);
  return static_cast<int>(std::max<i64>(1, ks));
}

void launch_rhsc(const double* xh, const i64* base, i64 st, i64 in, int s, const double* zs, int rt, int r,
                 double* part, double* out, int sms, cudaStream_t stream) {
  if (r > 64) throw Unsupported("FFT mixing: rank > 64");
  const int ks = rhsc_splits(in, s, sms);
  const int klen = ((s + ks - 1) / ks + kZChunk - 1) / kZChunk * kZChunk;
  const int ksu = (s + klen - 1) / klen;
  dim3 grid(static_cast<unsigned>((in + kRows - 1) / kRows), static_cast<unsigned>(ksu));
  rhsc_kernel<<<grid, kCThreads, 0, stream>>>(reinterpret_cast<const double2*>(xh), base, st, in, s, klen, zs, rt, r,
                                              reinterpret_cast<double2*>(part));
  CPB_LAUNCH_CHECK();
  const i64 n = in * r;
  rhsc_reduce_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, stream>>>(
      reinterpret_cast<const double2*>(part), ksu, n, reinterpret_cast<double2*>(out));
  CPB_LAUNCH_CHECK();
}

}  // namespace cpb
