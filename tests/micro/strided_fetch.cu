// DRAM fetch granularity of strided 8-byte gathers (not part of the
// product): C4 mode-3 fibers (1000 elements at 8 MB stride) of 20000 random
// samples, one CTA per fiber, with several load flavours; reports the time
// and the implied bytes per element at the measured HBM rate.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o strided_fetch strided_fetch.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda_runtime.h>

template <int K>
__device__ __forceinline__ double ld(const double* p) {
  double v;
  if constexpr (K == 0) v = __ldcs(p);
  else if constexpr (K == 1) v = __ldcg(p);
  else if constexpr (K == 2) v = __ldg(p);
  else if constexpr (K == 3) asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p));
  else if constexpr (K == 4) asm volatile("ld.global.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  else if constexpr (K == 5) asm volatile("ld.global.nc.L1::no_allocate.L2::64B.f64 %0, [%1];" : "=d"(v) : "l"(p));
  else asm volatile("ld.global.cv.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

template <int K>
__global__ void gather(const double* x, const int64_t* base, int64_t stride, int in, double* out) {
  const double* src = x + base[blockIdx.x];
  double v[4];
  for (int i0 = threadIdx.x; i0 < in; i0 += 4 * blockDim.x) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = i0 + u * blockDim.x;
      v[u] = i < in ? ld<K>(src + static_cast<int64_t>(i) * stride) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = i0 + u * blockDim.x;
      if (i < in) out[static_cast<int64_t>(blockIdx.x) * in + i] = v[u];
    }
  }
}

template <int K>
float run(const double* x, const int64_t* b, int64_t st, int in, int s, double* out) {
  cudaEvent_t a, c;
  cudaEventCreate(&a);
  cudaEventCreate(&c);
  gather<K><<<s, 256>>>(x, b, st, in, out);
  cudaEventRecord(a);
  for (int r = 0; r < 3; ++r) gather<K><<<s, 256>>>(x, b, st, in, out);
  cudaEventRecord(c);
  cudaEventSynchronize(c);
  float ms;
  cudaEventElapsedTime(&ms, a, c);
  return ms / 3;
}

int main() {
  const int64_t n = 1000, p = n * n * n;
  const int s = 20000;
  double* x;
  double* out;
  int64_t* b;
  cudaMalloc(&x, p * 8);
  cudaMemset(x, 0, p * 8);
  cudaMalloc(&out, int64_t(s) * n * 8);
  cudaMalloc(&b, s * 8);
  std::mt19937_64 g(1);
  std::vector<int64_t> hb(s);
  for (auto& v : hb) v = int64_t(g() % n) + int64_t(g() % n) * n;  // mode 3: base = i0 + i1 n, stride n^2
  cudaMemcpy(b, hb.data(), s * 8, cudaMemcpyHostToDevice);
  size_t lim = 0;
  cudaError_t e = cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, 32);
  cudaDeviceGetLimit(&lim, cudaLimitMaxL2FetchGranularity);
  printf("set L2 fetch granularity 32: %s, now %zu\n", cudaGetErrorString(e), lim);
  const char* names[] = {"ldcs", "ldcg", "ldg", "relaxed.gpu", "L1::no_allocate", "nc.L2::64B", "cv"};
  float t[7];
  t[0] = run<0>(x, b, n * n, n, s, out);
  t[1] = run<1>(x, b, n * n, n, s, out);
  t[2] = run<2>(x, b, n * n, n, s, out);
  t[3] = run<3>(x, b, n * n, n, s, out);
  t[4] = run<4>(x, b, n * n, n, s, out);
  t[5] = run<5>(x, b, n * n, n, s, out);
  t[6] = run<6>(x, b, n * n, n, s, out);
  for (int k = 0; k < 7; ++k)
    printf("%-16s %.3f ms  %.0f G elements/s  B_min (32 B) %.2f TB/s\n", names[k], t[k], s * n / (t[k] * 1e-3) / 1e9,
           32.0 * s * n / (t[k] * 1e-3) / 1e12);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
