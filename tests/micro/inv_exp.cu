// Timing variants of the look-ahead Gram inverse (R = 50, RT = 64) on one
// CTA: the product's ph::inverse_la against experimental copies
// (tests/micro/inv_exp.cuh). Not part of the product.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 -I paper_1701_06600_b200/csrc -I tests/micro -o inv_exp tests/micro/inv_exp.cu
#include <cstdio>
#include <vector>

__device__ unsigned long long g_st[64];
#define CPB_INV_STAMP(k) \
  if (threadIdx.x == 0) g_st[k] = clock64();
#define CPB_INV_STAMP_AT(k, s, who) \
  if ((s) == 5 && (who)) g_st[(k) - 24] = clock64();
#include "phases.cuh"
#include "inv_exp.cuh"

using namespace cpb;

template <int KIND>
__global__ void __launch_bounds__(256) inv_kernel(const double* g, int r, double* ginv, double* gfull, int* info,
                                                  unsigned long long* t, int reps) {
  extern __shared__ double sh[];
  for (int k = 0; k < reps; ++k) {
    __syncthreads();
    if (threadIdx.x == 0) g_st[0] = clock64();
    const unsigned long long t0 = globaltimer();
    bool fail;
    if (KIND == 0)
      fail = ph::inverse_la<64>(g, r, 4.4e-13, ginv, gfull, info, sh);
    else
      fail = phx::inverse_x<64, KIND>(g, r, 4.4e-13, ginv, gfull, info, sh);
    __syncthreads();
    if (threadIdx.x == 0) t[k] = globaltimer() - t0 + (fail ? 1000000000ULL : 0);
  }
}

int main() {
  const int r = 50, RT = 64;
  std::vector<double> h(RT * RT, 0.0);
  unsigned long long s = 88172645463325252ULL;
  std::vector<double> B(200 * r);
  for (auto& v : B) {
    s ^= s << 13; s ^= s >> 7; s ^= s << 17;
    v = 0.5 + (double)(s % 1000000) / 1e6;
  }
  for (int i = 0; i < r; ++i)
    for (int j = 0; j < r; ++j) {
      double a = (i == j) ? 1.0 : 0.0;
      for (int k = 0; k < 200; ++k) a += B[k * r + i] * B[k * r + j];
      h[i * RT + j] = a;
    }
  double *g, *ginv, *gfull;
  int* info;
  unsigned long long* t;
  cudaMalloc(&g, RT * RT * 8);
  cudaMalloc(&ginv, r * r * 8);
  cudaMalloc(&gfull, 64 * 1024 * 8);
  cudaMalloc(&info, 16);
  cudaMalloc(&t, 64 * 8);
  cudaMemset(info, 0, 16);
  cudaMemcpy(g, h.data(), RT * RT * 8, cudaMemcpyHostToDevice);
  const int reps = 20;
  std::vector<unsigned long long> ht(reps);
  auto report = [&](const char* name) {
    cudaDeviceSynchronize();
    cudaMemcpy(ht.data(), t, reps * 8, cudaMemcpyDeviceToHost);
    unsigned long long best = ~0ULL;
    for (int k = 2; k < reps; ++k) best = ht[k] < best ? ht[k] : best;
    std::vector<double> gi(r * r);
    cudaMemcpy(gi.data(), ginv, r * r * 8, cudaMemcpyDeviceToHost);
    double err = 0;
    for (int i = 0; i < r; ++i)
      for (int j = 0; j < r; ++j) {
        double a = 0;
        for (int k = 0; k < r; ++k) a += h[i * RT + k] * gi[k * r + j];
        a -= (i == j);
        err = err > fabs(a) ? err : fabs(a);
      }
    unsigned long long st[64];
    cudaMemcpyFromSymbol(st, g_st, sizeof(st));
    printf("%-10s best %6.2f us |G Ginv - I| %.1e %s | prologue %llu first %llu steps:", name, best / 1e3, err,
           cudaGetErrorString(cudaGetLastError()), st[1] - st[0], st[2] - st[1]);
    for (int k = 3; k < 15; ++k) printf(" %llu", st[k + 1] - st[k]);
    printf(" | step5: mma %lld wend %lld w7T %lld w7inv %lld w7end %lld\n", (long long)(st[17] - st[8]),
           (long long)(st[18] - st[8]), (long long)(st[19] - st[8]), (long long)(st[20] - st[8]),
           (long long)(st[21] - st[8]));
  };
#define RUN(K, NAME)                                                                                 \
  cudaFuncSetAttribute(inv_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024); \
  inv_kernel<K><<<1, 256, 100 * 1024>>>(g, r, ginv, gfull, info, t, reps);                     \
  report(NAME);
  RUN(0, "la");
  RUN(1, "no-mma");
  RUN(2, "w7-regs");
  return 0;
}
