// Microbenchmarks that decide the B200 design (not part of the product):
//  1. random 8 B gathers (one element per 32 B sector, no reuse) with several
//     load flavours and L2 fetch-granularity limits: time + (under ncu) DRAM bytes;
//  2. FP64 throughput: DFMA (FP64 pipe) vs DMMA (mma.sync m8n8k4 f64).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probe probe.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                               \
  do {                                                                      \
    cudaError_t e = (x);                                                    \
    if (e != cudaSuccess) {                                                 \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                              \
    }                                                                       \
  } while (0)

template <int KIND>
__global__ void gather(const double* __restrict__ x, const long long* __restrict__ off, long long n,
                       double* __restrict__ out) {
  const long long i0 = (long long)blockIdx.x * blockDim.x * 4 + threadIdx.x;
  double v[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const long long i = i0 + u * blockDim.x;
    if (i < n) {
      const double* p = x + off[i];
      if (KIND == 0) v[u] = *p;
      else if (KIND == 1) v[u] = __ldg(p);
      else if (KIND == 2) v[u] = __ldcs(p);
      else if (KIND == 3) asm volatile("ld.global.L1::no_allocate.f64 %0, [%1];" : "=d"(v[u]) : "l"(p));
      else if (KIND == 4) asm volatile("ld.global.nc.L1::no_allocate.L2::64B.f64 %0, [%1];" : "=d"(v[u]) : "l"(p));
      else asm volatile("ld.global.lu.f64 %0, [%1];" : "=d"(v[u]) : "l"(p));
    } else {
      v[u] = 0;
    }
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const long long i = i0 + u * blockDim.x;
    if (i < n) out[i] = v[u];
  }
}

__global__ void dfma_kernel(double* out, int iters) {
  double a0 = threadIdx.x * 1e-9, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6,
         a7 = a0 + 7;
  const double b = 0.999999, c = 1e-12;
  for (int i = 0; i < iters; ++i) {
    a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
    a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__global__ void dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-9 + 1.0, b = 0.5;
  double c[4][2] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int q = 0; q < 4; ++q)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[q][0]), "+d"(c[q][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
  for (int q = 0; q < 4; ++q) s += c[q][0] + c[q][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main(int argc, char** argv) {
  const long long P = 1000LL * 1000 * 1000;  // 8 GB tensor
  const long long n = 4LL << 20;             // 4M random elements
  double* x;
  CK(cudaMalloc(&x, P * 8));
  CK(cudaMemset(x, 0, P * 8));
  std::vector<long long> h(n);
  unsigned long long s = 88172645463325252ULL;
  for (long long i = 0; i < n; ++i) {
    s ^= s << 13; s ^= s >> 7; s ^= s << 17;
    h[i] = (long long)(s % (unsigned long long)(P / 4)) * 4;  // sector-aligned, one element per sector
  }
  long long* off;
  double* out;
  CK(cudaMalloc(&off, n * 8));
  CK(cudaMalloc(&out, n * 8));
  CK(cudaMemcpy(off, h.data(), n * 8, cudaMemcpyHostToDevice));
  size_t gran = 0;
  cudaDeviceGetLimit(&gran, cudaLimitMaxL2FetchGranularity);
  printf("default L2 fetch granularity limit: %zu\n", gran);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const char* names[] = {"ld.global", "ld.global.nc", "ld.global.cs", "L1::no_allocate", "nc.L2::64B", "ld.global.lu"};
  for (int g : {128, 64, 32}) {
    CK(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, g));
    cudaDeviceGetLimit(&gran, cudaLimitMaxL2FetchGranularity);
    for (int k = 0; k < 6; ++k) {
      auto launch = [&] {
        const int blocks = (int)((n + 1023) / 1024);
        switch (k) {
          case 0: gather<0><<<blocks, 256>>>(x, off, n, out); break;
          case 1: gather<1><<<blocks, 256>>>(x, off, n, out); break;
          case 2: gather<2><<<blocks, 256>>>(x, off, n, out); break;
          case 3: gather<3><<<blocks, 256>>>(x, off, n, out); break;
          case 4: gather<4><<<blocks, 256>>>(x, off, n, out); break;
          default: gather<5><<<blocks, 256>>>(x, off, n, out); break;
        }
      };
      launch();
      CK(cudaDeviceSynchronize());
      cudaEventRecord(a);
      for (int r = 0; r < 5; ++r) launch();
      cudaEventRecord(b);
      CK(cudaEventSynchronize(b));
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      ms /= 5;
      printf("gran=%zu %-18s %8.1f us  %7.1f Gelem/s  B_min(32B) %7.1f GB/s\n", gran, names[k], ms * 1e3,
             n / (ms * 1e-3) / 1e9, n * 32.0 / (ms * 1e-3) / 1e9);
    }
  }
  // FP64 throughput
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* o2;
  CK(cudaMalloc(&o2, (size_t)sms * 8 * 1024 * 8));
  const int it = 4096;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a);
    dfma_kernel<<<sms * 8, 256>>>(o2, it);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (rep) printf("DFMA: %.2f TFLOP/s\n", 2.0 * 8 * it * (double)sms * 8 * 256 / (ms * 1e-3) / 1e12);
    cudaEventRecord(a);
    dmma_kernel<<<sms * 8, 256>>>(o2, it);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    cudaEventElapsedTime(&ms, a, b);
    // per warp per mma: 8*8*4 FMAs = 256 FMA = 512 flop
    if (rep) printf("DMMA: %.2f TFLOP/s\n", 512.0 * 4 * it * (double)sms * 8 * 8 / (ms * 1e-3) / 1e12);
  }
  return 0;
}
