#include <algorithm>
// Kernels of the slab-sharded CPRAND loop (one process per GPU, tensor split
// along its last mode). The collectives between them are NCCL
// calls on the session stream (session.cu).
//
//   modes n < N-1   every sampled fiber lies in one slab: each rank contracts
//                   its local samples (Z rows gathered by gather_z_rows), the
//                   R x I_n right-hand sides are allreduced, every rank solves
//                   the same system (factors stay replicated)
//   mode N-1        every fiber spans the slabs: each rank forms the rows of
//                   its slab (apply_rows), the column sums of squares are
//                   allreduced (col_ssq), the factor slabs allgathered, and
//                   norms_from_ssq applies the lambda rule (kruskal.hpp:51-67)
#include "devutil.cuh"
#include "kernels.cuh"

namespace cpb {

namespace {

constexpr int kShardThreads = 256;

__global__ void gather_z_rows_kernel(const double* __restrict__ z, const int* __restrict__ idx, int cnt, int rt,
                                     double* __restrict__ out) {
  const i64 e = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= static_cast<i64>(cnt) * rt) return;
  const int j = static_cast<int>(e / rt), c = static_cast<int>(e % rt);
  out[e] = z[static_cast<i64>(idx[j]) * rt + c];
}

// out rows [0, rows) = rhs (rows x r, row-major) * ginv (r x r); per-CTA
// column sums of squares of the new rows -> ssq_part[cta][r].
template <int RT>
__global__ void __launch_bounds__(kShardThreads) apply_rows_kernel(i64 rows, int r, const double* __restrict__ rhs,
                                                                  const double* __restrict__ ginv,
                                                                  double* __restrict__ a_out,
                                                                  double* __restrict__ ssq_part) {
  constexpr int BI = kShardThreads / RT;
  constexpr int LD = RT + 1;
  __shared__ double gi[RT * LD];
  __shared__ double rh[BI * LD];
  const int tid = threadIdx.x, il = tid / RT, c = tid % RT;
  for (int e = tid; e < RT * RT; e += kShardThreads) {
    const int x = e / RT, y = e % RT;
    gi[x * LD + y] = (x < r && y < r) ? ginv[x * r + y] : 0.0;
  }
  double q = 0.0;
  for (i64 i0 = static_cast<i64>(blockIdx.x) * BI; i0 < rows; i0 += static_cast<i64>(gridDim.x) * BI) {
    const i64 i = i0 + il;
    __syncthreads();
    rh[il * LD + c] = (i < rows && c < r) ? rhs[i * r + c] : 0.0;
    __syncthreads();
    double o = 0.0;
    for (int cc = 0; cc < r; ++cc) o = fma(rh[il * LD + cc], gi[cc * LD + c], o);
    if (i < rows && c < r) {
      a_out[i * r + c] = o;
      q += o * o;
    }
  }
  __syncthreads();
  rh[il * LD + c] = q;
  __syncthreads();
  if (tid < r) {
    double t = 0.0;
    for (int x = 0; x < BI; ++x) t += rh[x * LD + tid];
    ssq_part[static_cast<i64>(blockIdx.x) * r + tid] = t;
  }
}

__global__ void col_ssq_kernel(const double* __restrict__ part, int nparts, int r, double* __restrict__ out) {
  const int c = threadIdx.x;
  if (c >= r) return;
  double t = 0.0;
  for (int b = 0; b < nparts; ++b) t += part[static_cast<i64>(b) * r + c];
  out[c] = t;
}

// norms = sqrt(ssq), lambda rule, zero columns refilled from the normalize
// stream over the full (gathered) factor, identically on every rank.
__global__ void norms_from_ssq_kernel(const double* __restrict__ ssq, int r, i64 rows, double* a, double* norms,
                                      double* lambda, int first_of_pass, unsigned long long* rng_state) {
  __shared__ int s_zero;
  const int c = threadIdx.x;
  if (c == 0) s_zero = 0;
  __syncthreads();
  if (c < r) {
    const double nrm = sqrt(ssq[c]);
    norms[c] = nrm;
    if (nrm == 0.0) {
      lambda[c] = 0.0;
      atomicOr(&s_zero, 1);
    } else {
      lambda[c] = first_of_pass ? lambda[c] * nrm : nrm;
    }
  }
  __syncthreads();
  if (c == 0 && s_zero) {
    DevMt g{rng_state};
    DevNormal gauss;
    for (int col = 0; col < r; ++col) {
      if (norms[col] != 0.0) continue;
      for (i64 t = 0; t < rows; ++t) a[t * r + col] = gauss(g);
      norms[col] = dev_stable_norm(a + col, rows, r);
    }
  }
}

__global__ void gather_values_masked_kernel(const double* __restrict__ x, const i64* __restrict__ loc, i64 n,
                                            double* __restrict__ out) {
  const i64 j = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const i64 o = loc[j];
  out[j] = (o >= 0) ? x[o] : 0.0;
}

}  // namespace

// Block transpose for the distributed last-mode transform: the slab X
// (column-major [M][L], M = product of the leading modes) cut into P row
// blocks q = [q Mb, min(M, (q+1) Mb)); block q is packed contiguously
// ([Mq][L], column-major) at offset q Mb L of buf. unpack is the inverse.
__global__ void slab_blocks_kernel(double* __restrict__ x, double* __restrict__ buf, i64 m, i64 l, i64 mb,
                                   int pack) {
  const i64 tot = m * l;
  for (i64 e = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; e < tot;
       e += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 col = e / m, row = e - col * m;
    const i64 q = row / mb, mq = min(mb, m - q * mb);
    const i64 b = q * mb * l + col * mq + (row - q * mb);
    if (pack)
      buf[b] = x[e];
    else
      x[e] = buf[b];
  }
}

void launch_slab_blocks(double* x, double* buf, i64 m, i64 l, i64 mb, int pack, cudaStream_t st) {
  const i64 tot = m * l;
  if (tot == 0) return;
  const int grid = static_cast<int>(std::min<i64>((tot + 255) / 256, 148 * 16));
  slab_blocks_kernel<<<grid, 256, 0, st>>>(x, buf, m, l, mb, pack);
  CPB_LAUNCH_CHECK();
}

void launch_gather_z_rows(const double* z, const int* idx, int cnt, int rt, double* out, cudaStream_t st) {
  const i64 n = static_cast<i64>(cnt) * rt;
  if (n == 0) return;
  gather_z_rows_kernel<<<ceil_div(n, 256), 256, 0, st>>>(z, idx, cnt, rt, out);
  CPB_LAUNCH_CHECK();
}

int apply_rows_grid(i64 rows, int r) {
  const int bi = kShardThreads / rank_bucket(r);
  return std::max(1, std::min(ceil_div(rows, bi), 1024));
}

void launch_apply_rows(i64 rows, int r, const double* rhs, const double* ginv, double* a_out, double* ssq_part,
                       cudaStream_t st) {
  const int grid = apply_rows_grid(rows, r);
  switch (rank_bucket(r)) {
    case 16: apply_rows_kernel<16><<<grid, kShardThreads, 0, st>>>(rows, r, rhs, ginv, a_out, ssq_part); break;
    case 32: apply_rows_kernel<32><<<grid, kShardThreads, 0, st>>>(rows, r, rhs, ginv, a_out, ssq_part); break;
    default: apply_rows_kernel<64><<<grid, kShardThreads, 0, st>>>(rows, r, rhs, ginv, a_out, ssq_part); break;
  }
  CPB_LAUNCH_CHECK();
}

void launch_col_ssq(const double* part, int nparts, int r, double* out, cudaStream_t st) {
  col_ssq_kernel<<<1, 64, 0, st>>>(part, nparts, r, out);
  CPB_LAUNCH_CHECK();
}

void launch_norms_from_ssq(const double* ssq, int r, i64 rows, double* a, double* norms, double* lambda,
                           int first_of_pass, unsigned long long* rng_state, cudaStream_t st) {
  norms_from_ssq_kernel<<<1, 64, 0, st>>>(ssq, r, rows, a, norms, lambda, first_of_pass, rng_state);
  CPB_LAUNCH_CHECK();
}

void launch_gather_values_masked(const double* x, const i64* loc, i64 n, double* out, cudaStream_t st) {
  if (n == 0) return;
  gather_values_masked_kernel<<<ceil_div(n, 256), 256, 0, st>>>(x, loc, n, out);
  CPB_LAUNCH_CHECK();
}

}  // namespace cpb
