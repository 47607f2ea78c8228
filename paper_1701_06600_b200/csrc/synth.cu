// BASELINE.json synthetic tensors generated in HBM:
// X = X_true + eta * ||X_true|| / ||N|| * N, X_true = sum_r a_r^(1) o ... o a_r^(N)
// with lambda = 1, noise N from a counter-based Philox4x32-10 + Box-Muller
// keyed by the seed (the CPU oracle draws the identical integer stream;
// transcendental rounding may differ in the last ulp). Factors are drawn on
// the host (normal_distribution on seeded_engine(seed, kSynthStream)).
#include <functional>

#include "kernels.cuh"

namespace cpb {

namespace {

constexpr int kSynthThreads = 256;

struct SynthArgs {
  double* x;
  int order;
  i64 dims[kMaxOrder];   // of the tensor written (a slab of the last mode when sharded)
  i64 gstr[kMaxOrder];   // strides of the global tensor (Philox counter = global offset)
  i64 last_off;          // global index of the slab's first last-mode row
  int r;
  const double* fac[kMaxOrder];  // row-major I_n x R
  i64 p;
  unsigned long long seed;
  double* part_sig;
  double* part_noise;
};

__device__ __forceinline__ double philox_gauss(unsigned long long seed, unsigned long long ctr) {
  unsigned c0 = static_cast<unsigned>(ctr), c1 = static_cast<unsigned>(ctr >> 32);
  unsigned c2 = 0x6E6F6973u, c3 = 0u;
  unsigned k0 = static_cast<unsigned>(seed), k1 = static_cast<unsigned>(seed >> 32) ^ 0x5EEDu;
#pragma unroll
  for (int round = 0; round < 10; ++round) {
    const unsigned hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    const unsigned hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
    const unsigned n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  const unsigned long long w1 = ((static_cast<unsigned long long>(c0) << 32) | c1) >> 11;
  const unsigned long long w2 = ((static_cast<unsigned long long>(c2) << 32) | c3) >> 11;
  const double u1 = static_cast<double>(w1 + 1) * 0x1.0p-53;
  const double u2 = static_cast<double>(w2) * 0x1.0p-53;
  return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.141592653589793 * u2);
}

__global__ void __launch_bounds__(kSynthThreads) synth_pass1(SynthArgs a) {
  __shared__ double rs[kSynthThreads], rn[kSynthThreads];
  double sig = 0.0, noi = 0.0;
  const i64 per = (a.p + gridDim.x - 1) / gridDim.x;
  const i64 lo = per * blockIdx.x, hi = min(a.p, lo + per);
  for (i64 off = lo + threadIdx.x; off < hi; off += blockDim.x) {
    i64 rem = off, goff = 0;
    i64 idx[kMaxOrder];
    for (int k = 0; k < a.order; ++k) {
      idx[k] = rem % a.dims[k];
      rem /= a.dims[k];
    }
    idx[a.order - 1] += a.last_off;
    for (int k = 0; k < a.order; ++k) goff += idx[k] * a.gstr[k];
    double sum = 0.0;
    for (int q = 0; q < a.r; ++q) {
      double prod = a.fac[0][idx[0] * a.r + q];
      for (int k = 1; k < a.order; ++k) prod = __dmul_rn(prod, a.fac[k][idx[k] * a.r + q]);
      sum = __dadd_rn(sum, prod);
    }
    a.x[off] = sum;
    sig = fma(sum, sum, sig);
    if (a.part_noise) {
      const double z = philox_gauss(a.seed, static_cast<unsigned long long>(goff));
      noi = fma(z, z, noi);
    }
  }
  rs[threadIdx.x] = sig;
  rn[threadIdx.x] = noi;
  __syncthreads();
  for (int s = kSynthThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      rs[threadIdx.x] += rs[threadIdx.x + s];
      rn[threadIdx.x] += rn[threadIdx.x + s];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    a.part_sig[blockIdx.x] = rs[0];
    if (a.part_noise) a.part_noise[blockIdx.x] = rn[0];
  }
}

__global__ void synth_sums(const double* part_sig, const double* part_noise, int nb, double* out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double s = 0.0, n = 0.0;
  for (int i = 0; i < nb; ++i) {
    s += part_sig[i];
    n += part_noise[i];
  }
  out[0] = s;
  out[1] = n;
}

__global__ void synth_scale(double* sums, double eta) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const double signal = sqrt(sums[0]), nn = sqrt(sums[1]);
  sums[2] = (signal > 0.0 && nn > 0.0) ? eta * signal / nn : 0.0;
}

__global__ void synth_pass2(SynthArgs a, const double* scale) {
  const double sc = *scale;
  for (i64 off = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; off < a.p;
       off += static_cast<i64>(gridDim.x) * blockDim.x) {
    i64 rem = off, goff = 0;
    for (int k = 0; k < a.order; ++k) {
      i64 v = rem % a.dims[k];
      rem /= a.dims[k];
      if (k == a.order - 1) v += a.last_off;
      goff += v * a.gstr[k];
    }
    const double z = philox_gauss(a.seed, static_cast<unsigned long long>(goff));
    a.x[off] = __dadd_rn(a.x[off], __dmul_rn(sc, z));
  }
}

}  // namespace

// scratch: >= 2 * 4096 + 3 doubles. Slab form: dims are the slab's, the
// last mode starts at global row last_off of a tensor whose last dim is
// global_last; reduce_sums (nullable) sums [sig, noise] over the ranks.
void launch_synth(double* x, int order, const i64* dims, int r, const double* const* fac_dev,
                  double eta, unsigned long long seed, double* scratch, cudaStream_t st, i64 last_off,
                  i64 global_last, const std::function<void(double*)>& reduce_sums) {
  if (order > kMaxOrder) throw Unsupported("synth: order > 8");
  SynthArgs a{};
  a.x = x;
  a.order = order;
  a.p = 1;
  i64 gs = 1;
  for (int k = 0; k < order; ++k) {
    a.dims[k] = dims[k];
    a.fac[k] = fac_dev[k];
    a.p *= dims[k];
    a.gstr[k] = gs;
    gs *= (k == order - 1 && global_last > 0) ? global_last : dims[k];
  }
  a.last_off = last_off;
  a.r = r;
  a.seed = seed;
  const int nb = 4096;
  a.part_sig = scratch;
  a.part_noise = eta > 0.0 ? scratch + nb : nullptr;
  synth_pass1<<<nb, kSynthThreads, 0, st>>>(a);
  CPB_LAUNCH_CHECK();
  if (eta > 0.0) {
    double* sums = scratch + 2 * nb;
    synth_sums<<<1, 32, 0, st>>>(scratch, scratch + nb, nb, sums);
    CPB_LAUNCH_CHECK();
    if (reduce_sums) reduce_sums(sums);
    synth_scale<<<1, 32, 0, st>>>(sums, eta);
    CPB_LAUNCH_CHECK();
    synth_pass2<<<148 * 16, 256, 0, st>>>(a, sums + 2);
    CPB_LAUNCH_CHECK();
  }
}

}  // namespace cpb
