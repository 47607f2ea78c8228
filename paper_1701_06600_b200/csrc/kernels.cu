// sm_100a kernels for the CPRAND hot path outside the mode solve (solve.cu):
// sampled-fiber gathers, the sampled Khatri-Rao operator, the sampled fit
// with the device-side stop rule, norms, and the normalize-RNG self check.
//
// Reference behaviour (paths under /root/reference/proj/include/cprand/):
//   gather_fibers  tensor.hpp:188-212      skr            sampling.hpp:74-92
//   least_squares  kr_linalg.hpp:105-118   normalize      kruskal.hpp:51-67
//   estimate_fit   sampling.hpp:191-210    should_stop    sampling.hpp:237-251
// Bit-exactness: gathers and Z_S copy / multiply in the reference's order
// (no FMA can form: pure products), so they match the oracle bit for bit.
#include <cfloat>
#include <cstdio>

#include "phases.cuh"

namespace cpb {

namespace {

// ------------------------------------------------------------- gather
__global__ void gather_fibers_kernel(const double* __restrict__ x, i64 in, i64 stride,
                                     const i64* __restrict__ base, int s,
                                     double* __restrict__ out) {
  // one CTA per sample column, threads over the fiber
  const int col = blockIdx.x;
  if (col >= s) return;
  const i64 b = base[col];
  for (i64 i = threadIdx.x; i < in; i += blockDim.x) out[col * in + i] = x[b + i * stride];
}

__global__ void base_offsets_kernel(const int* __restrict__ rows, int kept, int s,
                                    i64 k0, i64 k1, i64 k2, i64 k3, i64 k4, i64 k5, i64 k6,
                                    i64* __restrict__ base) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= s) return;
  const i64 ks[7] = {k0, k1, k2, k3, k4, k5, k6};
  i64 b = 0;
  for (int c = 0; c < kept; ++c) b += static_cast<i64>(rows[c * s + j]) * ks[c];
  base[j] = b;
}

// Z(s, r): ones, then *= factor rows in ascending kept mode (sampling.hpp:82-90).
__device__ __forceinline__ double skr_entry(const ModeView& v, int s, int r) {
  double z = 1.0;
  for (int c = 0; c < v.kept; ++c) {
    double a = v.fac[c][static_cast<i64>(v.rows[c][s]) * v.r + r];
    if (v.nrm[c]) a = a / v.nrm[c][r];
    z = __dmul_rn(z, a);
  }
  return z;
}

__global__ void skr_kernel(ModeView v, double* __restrict__ out) {
  const i64 e = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= static_cast<i64>(v.s) * v.r) return;
  const int s = static_cast<int>(e % v.s), r = static_cast<int>(e / v.s);
  out[e] = skr_entry(v, s, r);  // column-major S x R
}

constexpr int kThreads = 256;

// ---------------------------------------------- sampled-fiber gather
// X_S rows (one per sample, the fiber contiguous, ld >= I_n) straight from
// the tensor: coalesced along i for mode 1, one 32 B sector per element for
// strided modes. Streaming loads (evict-first) keep the random tensor
// traffic from displacing the X_S ring in L2. Pure copies: bit-exact.
constexpr int kGatherThreads = 256;
constexpr int kGatherUnroll = 4;

__global__ void __launch_bounds__(kGatherThreads) gather_rows_kernel(
    const double* __restrict__ x, i64 in, i64 stride, const i64* __restrict__ base, int s,
    double* __restrict__ xs, i64 ld) {
  const int row = blockIdx.y;
  const i64 b = base[row];
  const double* src = x + b;
  double* dst = xs + static_cast<i64>(row) * ld;
  for (i64 i0 = static_cast<i64>(blockIdx.x) * kGatherThreads * kGatherUnroll + threadIdx.x; i0 < in;
       i0 += static_cast<i64>(gridDim.x) * kGatherThreads * kGatherUnroll) {
    double v[kGatherUnroll];
#pragma unroll
    for (int u = 0; u < kGatherUnroll; ++u) {
      const i64 i = i0 + u * kGatherThreads;
      v[u] = (i < in) ? __ldcs(src + i * stride) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kGatherUnroll; ++u) {
      const i64 i = i0 + u * kGatherThreads;
      if (i < in) dst[i] = v[u];
    }
  }
}

__global__ void rng_seed_kernel(unsigned long long* state, unsigned long long v) {
  DevMt g{state};
  g.seed(v);
}

__global__ void rng_normals_kernel(unsigned long long* state, int n, double* out) {
  DevMt g{state};
  DevNormal d;
  for (int i = 0; i < n; ++i) out[i] = d(g);
}

// ------------------------------------------------------------ fit
__global__ void gather_values_kernel(const double* __restrict__ x, const i64* __restrict__ off,
                                     i64 n, double* __restrict__ out) {
  const i64 j = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j < n) out[j] = x[off[j]];
}

__global__ void sumsq_partial_kernel(const double* __restrict__ x, i64 n, double* partials) {
  __shared__ double red[kThreads];
  double acc = 0.0;
  const i64 per = (n + gridDim.x - 1) / gridDim.x;
  const i64 lo = per * blockIdx.x, hi = min(n, lo + per);
  // vectorized main body when 16 B aligned
  i64 i = lo + threadIdx.x;
  for (; i < hi; i += blockDim.x) {
    const double v = x[i];
    acc = fma(v, v, acc);
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s = kThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) partials[blockIdx.x] = red[0];
}

__global__ void sum_partials_kernel(const double* partials, int n, double* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += partials[i];
    *out = s;
  }
}

__global__ void stamp_start_kernel(FitState* s) {
  s->t_start_ns = static_cast<long long>(globaltimer());
}

__global__ void __launch_bounds__(kThreads) estimate_fit_kernel(FitArgs a) {
  if (a.state->stopped) return;
  __shared__ double red[ph::kFitSmemDoubles];
  __shared__ bool s_last;
  const double part = ph::fit_block(a, blockIdx.x, red);
  if (threadIdx.x == 0) {
    a.partials[blockIdx.x] = part;
    __threadfence();
    s_last = (atomicAdd(a.ticket, 1u) == gridDim.x - 1u);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (threadIdx.x == 0) *a.ticket = 0u;
  ph::fit_final(a, gridDim.x, red);
}

}  // namespace

// ---------------------------------------------------------------- launchers
void launch_gather_fibers(const double* x, i64 in, i64 stride, const i64* base, int s,
                          double* out, cudaStream_t st) {
  if (s <= 0) return;
  const int threads = in >= 256 ? 256 : (in >= 64 ? 128 : 32);
  gather_fibers_kernel<<<s, threads, 0, st>>>(x, in, stride, base, s, out);
  CPB_LAUNCH_CHECK();
}

void launch_skr(const ModeView& v, double* out, cudaStream_t st) {
  const i64 n = static_cast<i64>(v.s) * v.r;
  if (n == 0) return;
  skr_kernel<<<ceil_div(n, 256), 256, 0, st>>>(v, out);
  CPB_LAUNCH_CHECK();
}

void launch_base_offsets(const int* rows, int kept, int s, const i64* ks, i64* base,
                         cudaStream_t st) {
  if (kept > 7) throw Unsupported("base_offsets: order > 8");
  i64 k[7] = {0, 0, 0, 0, 0, 0, 0};
  for (int c = 0; c < kept; ++c) k[c] = ks[c];
  base_offsets_kernel<<<ceil_div(s, 256), 256, 0, st>>>(rows, kept, s, k[0], k[1], k[2], k[3],
                                                        k[4], k[5], k[6], base);
  CPB_LAUNCH_CHECK();
}

void launch_gather_rows(const double* x, i64 in, i64 stride, const i64* base, int s, double* xs,
                        i64 ld, cudaStream_t st) {
  if (s <= 0) return;
  const int per = kGatherThreads * kGatherUnroll;
  int gx = ceil_div(in, per);
  if (gx > 64) gx = 64;
  int rows = s;
  for (int r0 = 0; r0 < s; r0 += 65535) {
    const int ny = (s - r0) < 65535 ? (s - r0) : 65535;
    gather_rows_kernel<<<dim3(gx, ny), kGatherThreads, 0, st>>>(x, in, stride, base + r0, ny,
                                                                xs + static_cast<i64>(r0) * ld, ld);
    CPB_LAUNCH_CHECK();
  }
  (void)rows;
}

void launch_gather_values(const double* x, const i64* off, i64 n, double* out, cudaStream_t st) {
  if (n <= 0) return;
  gather_values_kernel<<<ceil_div(n, 256), 256, 0, st>>>(x, off, n, out);
  CPB_LAUNCH_CHECK();
}

void launch_sumsq(const double* x, i64 n, double* partials, int nparts, double* out,
                  cudaStream_t st) {
  sumsq_partial_kernel<<<nparts, kThreads, 0, st>>>(x, n, partials);
  CPB_LAUNCH_CHECK();
  sum_partials_kernel<<<1, 32, 0, st>>>(partials, nparts, out);
  CPB_LAUNCH_CHECK();
}

void launch_estimate_fit(const FitArgs& a, cudaStream_t st) {
  estimate_fit_kernel<<<ceil_div(a.phat, kThreads), kThreads, 0, st>>>(a);
  CPB_LAUNCH_CHECK();
}

void launch_stamp_start(FitState* s, cudaStream_t st) {
  stamp_start_kernel<<<1, 1, 0, st>>>(s);
  CPB_LAUNCH_CHECK();
}

void launch_rng_seed(unsigned long long* state, unsigned long long v, cudaStream_t st) {
  rng_seed_kernel<<<1, 1, 0, st>>>(state, v);
  CPB_LAUNCH_CHECK();
}

void launch_rng_normals(unsigned long long* state, int n, double* out, cudaStream_t st) {
  rng_normals_kernel<<<1, 1, 0, st>>>(state, n, out);
  CPB_LAUNCH_CHECK();
}

}  // namespace cpb
