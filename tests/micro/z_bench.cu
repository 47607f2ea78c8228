// Time of tl::z_tile alone: 288 CTAs (16 row blocks x 18 splits, C4 mode
// shape: S = 2000, R = 50, two kept modes of 1000 rows), factors in L2.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 -I paper_1701_06600_b200/csrc -o z_bench z_bench.cu
#include <cstdio>
#include <vector>

#include "tile.cuh"

using namespace cpb;

__global__ void __launch_bounds__(256, 2) zk(ModeView v, int tm, int tk, int tklen, int zcap, double* sink,
                                             unsigned long long* t) {
  extern __shared__ __align__(16) double sm[];
  const tl::TileSmem ts = tl::tile_smem<64>(sm, zcap);
  const int tt = blockIdx.x, kb = tt / tm;
  const int s0 = kb * tklen, cnt = min(v.s - s0, tklen);
  const int kpad = (cnt + tl::BK - 1) / tl::BK * tl::BK;
  const unsigned long long t0 = globaltimer();
  tl::z_tile<64>(v, s0, cnt, kpad, ts);
  const unsigned long long t1 = globaltimer();
  if (threadIdx.x == 0) {
    t[blockIdx.x] = t1 - t0;
    sink[blockIdx.x] = ts.zs[7];
  }
}

int main() {
  const int S = 2000, R = 50, I = 1000, tm = 16, tk = 18, tklen = 112, zcap = 112;
  std::vector<int> rows(2 * S);
  unsigned long long x = 88172645463325252ULL;
  for (auto& r : rows) {
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    r = (int)(x % I);
  }
  std::vector<double> fac(I * R), nrm(R, 3.0);
  for (auto& f : fac) {
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    f = (double)(x % 100000) / 1e5 + 0.01;
  }
  int* drows;
  double *dfac0, *dfac1, *dnrm, *sink;
  i64* dbase;
  unsigned long long* dt;
  cudaMalloc(&drows, rows.size() * 4);
  cudaMalloc(&dfac0, fac.size() * 8);
  cudaMalloc(&dfac1, fac.size() * 8);
  cudaMalloc(&dnrm, R * 8);
  cudaMalloc(&sink, 4096 * 8);
  cudaMalloc(&dbase, S * 8);
  cudaMalloc(&dt, 4096 * 8);
  cudaMemset(dbase, 0, S * 8);
  cudaMemcpy(drows, rows.data(), rows.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dfac0, fac.data(), fac.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dfac1, fac.data(), fac.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dnrm, nrm.data(), R * 8, cudaMemcpyHostToDevice);
  ModeView v{};
  v.in = I;
  v.s = S;
  v.r = R;
  v.kept = 2;
  v.rows[0] = drows;
  v.rows[1] = drows + S;
  v.fac[0] = dfac0;
  v.fac[1] = dfac1;
  v.nrm[0] = dnrm;
  v.nrm[1] = dnrm;
  v.base = dbase;
  const size_t smem = tl::tile_smem_doubles<64>(zcap) * 8;
  cudaFuncSetAttribute(zk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int rep = 0; rep < 4; ++rep) {
    if (rep == 3) {  // no normalization: factor loads + products only
      v.nrm[0] = nullptr;
      v.nrm[1] = nullptr;
    }
    cudaEventRecord(a);
    zk<<<tm * tk, 256, smem>>>(v, tm, tk, tklen, zcap, sink, dt);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    std::vector<unsigned long long> ht(tm * tk);
    cudaMemcpy(ht.data(), dt, ht.size() * 8, cudaMemcpyDeviceToHost);
    unsigned long long mx = 0, sum = 0;
    for (auto t : ht) {
      mx = t > mx ? t : mx;
      sum += t;
    }
    printf("z_tile x %d CTAs: kernel %.2f us, per-CTA z_tile mean %.2f us max %.2f us  %s\n", tm * tk, ms * 1e3,
           sum / 1e3 / ht.size(), mx / 1e3, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
