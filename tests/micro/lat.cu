// Dependent-chain latencies on sm_100a (cycles per op, one warp unless noted):
// DFMA, DMUL, DMMA m8n8k4, rcp.approx.f64, IEEE 1.0/x, LDS, SHFL, and
// __syncthreads with 8 warps.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lat lat.cu
#include <cstdio>

__global__ void lat(double* out, long long* cyc, double seed, int n) {
  double a = seed + threadIdx.x * 1e-9, b = 1.0000001, c = 1e-12;
  __shared__ double sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = (i * 7) % 1024;
  __syncthreads();
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) a = fma(a, b, c);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = (t1 - t0);
  // DMUL chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) a = a * b;
  t1 = clock64();
  if (threadIdx.x == 0) cyc[1] = (t1 - t0);
  // DMMA chain (accumulator dependency)
  double d0 = a, d1 = a;
  t0 = clock64();
  for (int i = 0; i < n; ++i)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(b), "d"(c));
  t1 = clock64();
  if (threadIdx.x == 0) cyc[2] = (t1 - t0);
  // rcp.approx chain
  double x = a;
  t0 = clock64();
  for (int i = 0; i < n; ++i) asm volatile("rcp.approx.ftz.f64 %0, %0;" : "+d"(x));
  t1 = clock64();
  if (threadIdx.x == 0) cyc[3] = (t1 - t0);
  // IEEE reciprocal chain
  double y = a + 1.0;
  t0 = clock64();
  for (int i = 0; i < n; ++i) y = 1.0 / y;
  t1 = clock64();
  if (threadIdx.x == 0) cyc[4] = (t1 - t0);
  // LDS pointer chase
  int p = threadIdx.x;
  t0 = clock64();
  for (int i = 0; i < n; ++i) p = (int)sm[p & 1023];
  t1 = clock64();
  if (threadIdx.x == 0) cyc[5] = (t1 - t0);
  // SHFL chain
  double s = a;
  t0 = clock64();
  for (int i = 0; i < n; ++i) s = __shfl_sync(0xffffffffu, s, (threadIdx.x + 1) & 31) + 0.0;
  t1 = clock64();
  if (threadIdx.x == 0) cyc[6] = (t1 - t0);
  // __syncthreads
  t0 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  t1 = clock64();
  if (threadIdx.x == 0) cyc[7] = (t1 - t0);
  // DFMA throughput: 8 independent chains, one warp
  double e0 = a, e1 = a + 1, e2 = a + 2, e3 = a + 3, e4 = a + 4, e5 = a + 5, e6 = a + 6, e7 = a + 7;
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    e0 = fma(e0, b, c); e1 = fma(e1, b, c); e2 = fma(e2, b, c); e3 = fma(e3, b, c);
    e4 = fma(e4, b, c); e5 = fma(e5, b, c); e6 = fma(e6, b, c); e7 = fma(e7, b, c);
  }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[8] = (t1 - t0);
  out[threadIdx.x] = a + d0 + d1 + x + y + p + s + e0 + e1 + e2 + e3 + e4 + e5 + e6 + e7;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1024 * 8);
  cudaMallocManaged(&cyc, 16 * 8);
  const int n = 1000;
  const char* names[] = {"DFMA", "DMUL", "DMMA m8n8k4", "rcp.approx.f64", "IEEE 1/x", "LDS chase", "SHFL",
                         "__syncthreads (8 warps)", "DFMA x8 indep (per iter)"};
  for (int threads : {32, 256}) {
    lat<<<1, threads>>>(out, cyc, 1.0, n);
    cudaDeviceSynchronize();
    printf("block %d threads:\n", threads);
    for (int k = 0; k < 9; ++k) printf("  %-26s %6.1f cycles\n", names[k], (double)cyc[k] / n);
  }
  return 0;
}
