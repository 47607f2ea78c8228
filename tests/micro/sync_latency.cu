// Costs of the inter-CTA protocol pieces on sm_100a: __threadfence(),
// atomicAdd (returning) on a global counter, __nanosleep(32) actual sleep,
// and a flag hand-off between two CTAs (release -> acquire observed).
#include <cstdio>
__global__ void k(unsigned* cnt, unsigned* flag, long long* cyc, double* sink) {
  const int b = blockIdx.x, t = threadIdx.x;
  if (t != 0) return;
  long long t0, t1;
  volatile unsigned* vf = flag;
  if (b == 0) {
    // fence after a store
    sink[0] = 1.0;
    t0 = clock64();
    for (int i = 0; i < 100; ++i) { sink[i & 7] = i; __threadfence(); }
    t1 = clock64();
    cyc[0] = (t1 - t0) / 100;
    t0 = clock64();
    for (int i = 0; i < 100; ++i) atomicAdd(cnt, 1u);
    t1 = clock64();
    cyc[1] = (t1 - t0) / 100;
    unsigned v = 0;
    t0 = clock64();
    for (int i = 0; i < 100; ++i) v += atomicAdd(cnt, 1u);
    t1 = clock64();
    cyc[2] = (t1 - t0) / 100 + (v == 12345 ? 1 : 0);
    t0 = clock64();
    for (int i = 0; i < 100; ++i) __nanosleep(32);
    t1 = clock64();
    cyc[3] = (t1 - t0) / 100;
    t0 = clock64();
    for (int i = 0; i < 100; ++i) __nanosleep(1000);
    t1 = clock64();
    cyc[4] = (t1 - t0) / 100;
    // ping-pong with block 1: 50 round trips
    long long g0 = 0, g1 = 0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
    for (int i = 0; i < 50; ++i) {
      *vf = 2 * i + 1;
      __threadfence();
      while (*vf != 2 * i + 2) {}
    }
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
    cyc[5] = (g1 - g0) / 50;  // ns per round trip
  } else if (b == 1) {
    for (int i = 0; i < 50; ++i) {
      while (*vf != 2 * i + 1) {}
      *vf = 2 * i + 2;
      __threadfence();
    }
  }
}
int main() {
  unsigned *cnt, *flag; long long* cyc; double* sink;
  cudaMalloc(&cnt, 4); cudaMalloc(&flag, 4); cudaMallocManaged(&cyc, 64); cudaMalloc(&sink, 64);
  cudaMemset(cnt, 0, 4); cudaMemset(flag, 0, 4);
  k<<<2, 32>>>(cnt, flag, cyc, sink);
  cudaDeviceSynchronize();
  printf("fence after store: %lld cycles\natomicAdd (no use): %lld cycles\natomicAdd (returned): %lld cycles\n"
         "nanosleep(32): %lld cycles\nnanosleep(1000): %lld cycles\nflag ping-pong round trip: %lld ns  %s\n",
         cyc[0], cyc[1], cyc[2], cyc[3], cyc[4], cyc[5], cudaGetErrorString(cudaGetLastError()));
  return 0;
}
