// Exact fit of a Kruskal model to a device tensor (solver.hpp:161-181, the
// reference's exact_fit): 1 - ||X - M|| / ||X|| through the Gram expansion
//   ||X - M||^2 = ||X||^2 - 2 <W, A_1 diag(lambda)> + lambda^T (V * A_1^T A_1) lambda
// with W = X_(1) (A_N (.) ... (.) A_2) the mode-1 MTTKRP and V the Hadamard
// product of the other modes' Grams. The tensor is never reconstructed: the
// MTTKRP streams it once, as the split-K RHS GEMM (the fibers of mode 1 are
// its contiguous columns), with the Khatri-Rao rows of each column chunk
// formed on the device. ||X||^2 is the deterministic sum-of-squares kernel.
#include <cmath>
#include <vector>

#include "session.hpp"

namespace cpb {

namespace {

// K[j][q] = prod_{n >= 1} A_n(i_n(c0 + j), q) for q < r, 0 for r <= q < rt;
// column c = i_1 + I_1 (i_2 + I_2 (...)) of the mode-1 unfolding
__global__ void krp_rows_kernel(i64 c0, i64 cs, int order, const i64* __restrict__ dims,
                                const double* const* __restrict__ fac, int r, int rt, double* __restrict__ k,
                                i64* __restrict__ offs, i64 i0) {
  const i64 e = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= cs * rt) return;
  const i64 j = e / rt;
  const int q = static_cast<int>(e - j * rt);
  double v = 0.0;
  if (q < r) {
    v = 1.0;
    i64 c = c0 + j;
    for (int n = 1; n < order; ++n) {
      const i64 d = dims[n], idx = c % d;
      c /= d;
      v *= fac[n][idx * r + q];
    }
  }
  k[e] = v;
  if (q == 0) offs[j] = (c0 + j) * i0;
}

}  // namespace

double device_exact_fit(const Tensor& t, const double* lambda, const double* const* factors, int r) {
  const int N = static_cast<int>(t.dims.size());
  if (r < 1) throw InvalidArgument("rank must be >= 1");
  CPB_CUDA(cudaSetDevice(t.device));
  cudaStream_t st;
  CPB_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  int sms = 148;
  CPB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, t.device));
  // ||X||^2
  const int nparts = 1024;
  double* red = nullptr;
  CPB_CUDA(cudaMalloc(&red, sizeof(double) * (nparts + 1)));
  launch_sumsq(t.d, t.p, red, nparts, red + nparts, st);
  double xx = 0.0;
  CPB_CUDA(cudaMemcpyAsync(&xx, red + nparts, sizeof(double), cudaMemcpyDeviceToHost, st));
  CPB_CUDA(cudaStreamSynchronize(st));
  cudaFree(red);
  if (xx == 0.0) {
    cudaStreamDestroy(st);
    return 1.0;
  }
  // factors row-major on the device (modes >= 1) and their Grams on the host
  std::vector<std::vector<double>> rm(static_cast<size_t>(N));
  for (int n = 0; n < N; ++n) {
    const i64 rows = t.dims[static_cast<size_t>(n)];
    rm[static_cast<size_t>(n)].resize(static_cast<size_t>(rows * r));
    for (int q = 0; q < r; ++q)
      for (i64 i = 0; i < rows; ++i)
        rm[static_cast<size_t>(n)][static_cast<size_t>(i * r + q)] = factors[n][i + q * rows];
  }
  std::vector<double*> dfac(static_cast<size_t>(N), nullptr);
  for (int n = 1; n < N; ++n) {
    CPB_CUDA(cudaMalloc(&dfac[static_cast<size_t>(n)], sizeof(double) * rm[static_cast<size_t>(n)].size()));
    CPB_CUDA(cudaMemcpyAsync(dfac[static_cast<size_t>(n)], rm[static_cast<size_t>(n)].data(),
                             sizeof(double) * rm[static_cast<size_t>(n)].size(), cudaMemcpyHostToDevice, st));
  }
  double** dfp = nullptr;
  i64* ddims = nullptr;
  CPB_CUDA(cudaMalloc(&dfp, sizeof(double*) * N));
  CPB_CUDA(cudaMalloc(&ddims, sizeof(i64) * N));
  CPB_CUDA(cudaMemcpyAsync(dfp, dfac.data(), sizeof(double*) * N, cudaMemcpyHostToDevice, st));
  CPB_CUDA(cudaMemcpyAsync(ddims, t.dims.data(), sizeof(i64) * N, cudaMemcpyHostToDevice, st));
  // W = mode-1 MTTKRP, column chunks of the unfolding through the split-K GEMM
  const int rt = rank_bucket(r);
  const i64 i0 = t.dims[0], S = t.p / i0;
  const i64 CS = std::min<i64>(S, i64{1} << 20);
  double *k = nullptr, *part = nullptr, *wd = nullptr;
  i64* offs = nullptr;
  CPB_CUDA(cudaMalloc(&k, sizeof(double) * CS * rt));
  CPB_CUDA(cudaMalloc(&offs, sizeof(i64) * CS));
  CPB_CUDA(cudaMalloc(&part, sizeof(double) * 64 * i0 * r));
  CPB_CUDA(cudaMalloc(&wd, sizeof(double) * i0 * r));
  std::vector<double> w(static_cast<size_t>(i0 * r), 0.0), wc(w.size());
  const bool vec16 = (i0 % 2 == 0);
  for (i64 c0 = 0; c0 < S; c0 += CS) {
    const i64 cs = std::min(CS, S - c0);
    krp_rows_kernel<<<static_cast<unsigned>((cs * rt + 255) / 256), 256, 0, st>>>(c0, cs, N, ddims, dfp, r, rt, k,
                                                                                  offs, i0);
    CPB_LAUNCH_CHECK();
    int ks = 1, ks_len = 16;
    mode_splits(i0, static_cast<int>(cs), rt, &ks, &ks_len, sms);
    launch_rhs_gemm(t.d, 0, offs, vec16, k, i0, static_cast<int>(cs), r, ks, ks_len, part, nullptr, st);
    launch_reduce_rhs(part, ks, i0, r, wd, st);
    CPB_CUDA(cudaMemcpyAsync(wc.data(), wd, sizeof(double) * wc.size(), cudaMemcpyDeviceToHost, st));
    CPB_CUDA(cudaStreamSynchronize(st));
    for (size_t e = 0; e < w.size(); ++e) w[e] += wc[e];  // chunks in order
  }
  for (int n = 1; n < N; ++n) cudaFree(dfac[static_cast<size_t>(n)]);
  cudaFree(dfp);
  cudaFree(ddims);
  cudaFree(k);
  cudaFree(offs);
  cudaFree(part);
  cudaFree(wd);
  cudaStreamDestroy(st);
  // cross = sum_i,q A_1(i, q) W(i, q) lambda_q; model^2 = lambda^T (V * A_1^T A_1) lambda
  double cross = 0.0;
  for (i64 i = 0; i < i0; ++i)
    for (int q = 0; q < r; ++q)
      cross += rm[0][static_cast<size_t>(i * r + q)] * w[static_cast<size_t>(i * r + q)] * lambda[q];
  std::vector<double> v(static_cast<size_t>(r * r), 1.0);
  for (int n = 0; n < N; ++n) {
    const i64 rows = t.dims[static_cast<size_t>(n)];
    for (int a = 0; a < r; ++a)
      for (int b = 0; b < r; ++b) {
        double g = 0.0;
        for (i64 i = 0; i < rows; ++i)
          g += rm[static_cast<size_t>(n)][static_cast<size_t>(i * r + a)] * rm[static_cast<size_t>(n)][static_cast<size_t>(i * r + b)];
        v[static_cast<size_t>(a * r + b)] *= g;
      }
  }
  double model_sq = 0.0;
  for (int a = 0; a < r; ++a)
    for (int b = 0; b < r; ++b) model_sq += lambda[a] * v[static_cast<size_t>(a * r + b)] * lambda[b];
  const double resid_sq = std::max(0.0, xx - 2.0 * cross + model_sq);
  return 1.0 - std::sqrt(resid_sq) / std::sqrt(xx);
}

}  // namespace cpb
