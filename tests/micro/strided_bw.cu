// Micro-benchmark behind the mixing-pass layout (not part of the product):
// read + write every element of a 1000^3 fp64 tensor (8 GB) once, walking it
// in tiles of W adjacent fibers of one mode (W*8 contiguous bytes per row,
// rows `st` elements apart), the access pattern of a per-mode transform pass.
// Prints the achieved read+write GB/s per (mode stride, W).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o strided_bw strided_bw.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e = (x);                                                       \
    if (e != cudaSuccess) {                                                    \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                 \
    }                                                                          \
  } while (0)

// one CTA = one tile (W fibers x n rows) at a time; each thread moves double2s;
// U rows in flight per thread before the stores
template <int W, int U>
__global__ void __launch_bounds__(256) rw_tiles(double* x, long long st, int n, long long ntiles) {
  constexpr int TPR = W / 2;            // threads per row
  constexpr int RPI = 256 / TPR;        // rows per instruction
  const int tid = threadIdx.x;
  if (tid >= RPI * TPR) return;
  const int rr = tid / TPR, cc = (tid % TPR) * 2;
  const long long per_slab = st / W;    // tiles per slab of st * n elements
  for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const long long hi = t / per_slab, lo = t - hi * per_slab;
    double* base = x + hi * st * n + lo * W + cc;
    for (int r0 = rr; r0 < n; r0 += RPI * U) {
      double2 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int r = r0 + u * RPI;
        if (r < n) v[u] = __ldcs(reinterpret_cast<const double2*>(base + static_cast<long long>(r) * st));
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int r = r0 + u * RPI;
        if (r < n) {
          v[u].x *= 1.0000001;
          v[u].y *= 0.9999999;
          __stcs(reinterpret_cast<double2*>(base + static_cast<long long>(r) * st), v[u]);
        }
      }
    }
  }
}

template <int W>
void run(double* x, long long st, int n, long long total, int sms) {
  const long long ntiles = total / (static_cast<long long>(n) * W);
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  for (int occ : {4, 8}) {
    const int grid = sms * occ;
    rw_tiles<W, 8><<<grid, 256>>>(x, st, n, ntiles);
    CK(cudaEventRecord(a));
    for (int k = 0; k < 3; ++k) rw_tiles<W, 8><<<grid, 256>>>(x, st, n, ntiles);
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, a, b));
    ms /= 3;
    printf("stride %9lld  W %3d (%4d B rows)  CTAs/SM %d: %7.3f ms  %7.1f GB/s\n", st, W, W * 8, occ, ms,
           16.0 * total / (ms * 1e-3) / 1e9);
  }
}

int main() {
  const int n = 1000;
  const long long total = 1000LL * 1000 * 1000;
  double* x;
  CK(cudaMalloc(&x, total * 8));
  CK(cudaMemset(x, 0, total * 8));
  int sms = 148;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  for (long long st : {1000LL, 1000000LL}) {
    // W divides 1000: tiles never straddle a slab
    run<4>(x, st, n, total, sms);
    run<8>(x, st, n, total, sms);
    run<20>(x, st, n, total, sms);
    run<40>(x, st, n, total, sms);
  }
  // contiguous (mode 1) reference: a "tile" of 1000-element fibers
  run<40>(x, 40, n, total, sms);
  CK(cudaFree(x));
  return 0;
}
