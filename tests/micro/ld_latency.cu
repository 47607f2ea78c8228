// L2-hit load latency under load: 288 CTAs x 256 threads, each thread does
// a dependent chain of n loads over a 400 KB array (L2 resident), comparing
// ld.global (default), ld.global.cg (__ldcg), ld.global.nc (__ldg).
#include <cstdio>
template <int K>
__global__ void chase(const long long* __restrict__ a, long long* out, int n, long long* cyc) {
  long long p = (blockIdx.x * 256 + threadIdx.x) * 97 % 51200;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    if (K == 0) p = a[p];
    else if (K == 1) p = __ldcg(a + p);
    else p = __ldg(a + p);
  }
  long long t1 = clock64();
  out[blockIdx.x * 256 + threadIdx.x] = p;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  const int N = 51200;  // 400 KB
  long long *a, *out, *cyc;
  cudaMalloc(&a, N * 8); cudaMalloc(&out, 288 * 256 * 8); cudaMallocManaged(&cyc, 8);
  long long* h = new long long[N];
  for (int i = 0; i < N; ++i) h[i] = (i * 7919LL + 13) % N;
  cudaMemcpy(a, h, N * 8, cudaMemcpyHostToDevice);
  const char* nm[] = {"ld.global", "ld.global.cg (__ldcg)", "ld.global.nc (__ldg)"};
  for (int grid : {1, 288}) {
    for (int k = 0; k < 3; ++k) {
      for (int rep = 0; rep < 2; ++rep) {
        if (k == 0) chase<0><<<grid, 256>>>(a, out, 100, cyc);
        if (k == 1) chase<1><<<grid, 256>>>(a, out, 100, cyc);
        if (k == 2) chase<2><<<grid, 256>>>(a, out, 100, cyc);
        cudaDeviceSynchronize();
      }
      printf("grid %3d %-24s %.0f cycles/load\n", grid, nm[k], *cyc / 100.0);
    }
  }
  return 0;
}
