// Checks tl::div_rn (Markstein quotient with a correctly rounded reciprocal)
// against IEEE division, bit for bit, over random and adversarial operands.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1701_06600_b200/csrc -o div_check div_check.cu
#include <cstdio>

#include "tile.cuh"

__device__ unsigned long long mix64(unsigned long long z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

__global__ void check(unsigned long long n, unsigned long long seed, unsigned long long* bad,
                      double* ex) {
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned long long u = mix64(seed * 0x1000003ULL + i), v = mix64(u ^ 0xABCDEF);
    double a, b;
    const int kind = (int)(i % 4);
    // exponents within +-40 of 0 (factor entries / norms), mantissas random,
    // all-ones, or just above 1
    unsigned long long ea = 1023 + (int)((u >> 52) % 81) - 40, eb = 1023 + (int)((v >> 52) % 81) - 40;
    unsigned long long ma = u & 0xFFFFFFFFFFFFFULL, mb = v & 0xFFFFFFFFFFFFFULL;
    if (kind == 1) mb = 0xFFFFFFFFFFFFFULL - (v & 0xFF);
    if (kind == 2) mb = v & 0xFF;
    if (kind == 3) ma = 0xFFFFFFFFFFFFFULL - (u & 0xFF);
    a = __longlong_as_double((long long)((ea << 52) | ma)) * ((u >> 63) ? -1.0 : 1.0);
    b = __longlong_as_double((long long)((eb << 52) | mb));
    const double y = __drcp_rn(b);
    const double q1 = cpb::tl::div_rn(a, b, y), q2 = a / b;
    if (__double_as_longlong(q1) != __double_as_longlong(q2)) {
      const unsigned long long k = atomicAdd(bad, 1ULL);
      if (k < 4) {
        ex[4 * k] = a;
        ex[4 * k + 1] = b;
        ex[4 * k + 2] = q1;
        ex[4 * k + 3] = q2;
      }
    }
  }
}

int main() {
  unsigned long long* bad;
  double* ex;
  cudaMallocManaged(&bad, 8);
  cudaMallocManaged(&ex, 16 * 8);
  *bad = 0;
  const unsigned long long n = 1ULL << 32;
  check<<<148 * 8, 256>>>(n, 12345, bad, ex);
  cudaDeviceSynchronize();
  printf("div_rn vs a/b: %llu mismatches in %llu\n", *bad, n);
  for (unsigned long long k = 0; k < *bad && k < 4; ++k)
    printf("  a=%a b=%a div_rn=%a ieee=%a\n", ex[4 * k], ex[4 * k + 1], ex[4 * k + 2], ex[4 * k + 3]);
  return *bad ? 1 : 0;
}
