// Device utilities shared by the sm_100a kernels: timer, async-copy
// wrappers, and the device replica of the reference's normalize RNG.
#pragma once

#include "common.cuh"

namespace cpb {

// Device-check build (make checklib: -DCPB_DEVICE_CHECKS): bounds asserts on
// the sampled reads and a time-out on the persistent kernels' flag waits,
// both trapping with a message (compute-sanitizer is not available on the
// GPU pool). Compiles to nothing in the product build.
#ifdef CPB_DEVICE_CHECKS
#define CPB_DCHECK(cond, what)                                                                          \
  do {                                                                                                  \
    if (!(cond)) {                                                                                      \
      printf("CPB_DCHECK failed: %s (%s:%d) block %d thread %d\n", what, __FILE__, __LINE__,          \
             static_cast<int>(blockIdx.x), static_cast<int>(threadIdx.x));                              \
      __trap();                                                                                         \
    }                                                                                                   \
  } while (0)
#else
#define CPB_DCHECK(cond, what) \
  do {                         \
  } while (0)
#endif

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc, int src_bytes) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(gsrc), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gsrc, int src_bytes) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(gsrc), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// ---------------------------------------------- device normalize RNG
// std::mt19937_64 (state words 0..311, index in word 312) and the libstdc++
// Marsaglia-polar normal_distribution (random.tcc:1811-1844), one fresh
// distribution object per call, as kruskal.hpp:53 constructs it.
struct DevMt {
  unsigned long long* s;
  __device__ void seed(unsigned long long v) {
    s[0] = v;
    for (int i = 1; i < 312; ++i) s[i] = 6364136223846793005ULL * (s[i - 1] ^ (s[i - 1] >> 62)) + i;
    s[312] = 312;
  }
  __device__ unsigned long long next() {
    unsigned long long idx = s[312];
    if (idx >= 312) {
      const unsigned long long um = 0xFFFFFFFF80000000ULL, lm = 0x7FFFFFFFULL;
      for (int i = 0; i < 312; ++i) {
        const unsigned long long y = (s[i] & um) | (s[(i + 1) % 312] & lm);
        unsigned long long xa = y >> 1;
        if (y & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
        s[i] = s[(i + 156) % 312] ^ xa;
      }
      idx = 0;
    }
    unsigned long long z = s[idx];
    s[312] = idx + 1;
    z ^= (z >> 29) & 0x5555555555555555ULL;
    z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
    z ^= (z << 37) & 0xFFF7EEE000000000ULL;
    z ^= (z >> 43);
    return z;
  }
  __device__ double canonical() {  // generate_canonical<double, 53>
    double v = __dmul_rn(__ull2double_rn(next()), 0x1.0p-64);
    if (v >= 1.0) v = 0x1.fffffffffffffp-1;
    return v;
  }
};

struct DevNormal {
  bool saved_ok = false;
  double saved = 0.0;
  __device__ double operator()(DevMt& g) {
    if (saved_ok) {
      saved_ok = false;
      return saved;
    }
    double x, y, r2;
    do {
      x = __dsub_rn(__dmul_rn(2.0, g.canonical()), 1.0);
      y = __dsub_rn(__dmul_rn(2.0, g.canonical()), 1.0);
      r2 = __dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y));
    } while (r2 > 1.0 || r2 == 0.0);
    const double mult = sqrt(__ddiv_rn(__dmul_rn(-2.0, log(r2)), r2));
    saved = __dmul_rn(x, mult);
    saved_ok = true;
    return __dmul_rn(y, mult);
  }
};

__device__ inline double dev_stable_norm(const double* v, i64 n, i64 inc) {
  double scale = 0.0, ssq = 1.0;
  for (i64 i = 0; i < n; ++i) {
    const double a = fabs(v[i * inc]);
    if (a != 0.0) {
      if (scale < a) {
        const double q = scale / a;
        ssq = 1.0 + ssq * q * q;
        scale = a;
      } else {
        const double q = a / scale;
        ssq += q * q;
      }
    }
  }
  return scale * sqrt(ssq);
}


}  // namespace cpb
