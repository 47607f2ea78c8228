// Persistent per-iteration kernel: one cooperative launch runs a whole
// CPRAND / CPRAND-MIX outer iteration (every mode update, then the sampled
// fit and the stop rule; sampling.hpp:281-304, mixing.hpp:284-312).
//
// Per mode n, phases separated by grid barriers (all CTAs co-resident):
//   Z      Z_S rows, grid-strided                          (sampling.hpp:74-92)
//   B      CTAs [0, gparts): Gram partials, then GEMM tiles
//          last CTA: waits for the Gram partials, Gauss-Jordan inverse
//          (pivoted-Cholesky fallback when rank deficient)
//          others: split-K GEMM tiles on the fibers read in place
//   [MIX]  reduce the RHS partials; DCT-III + sign along I_n per column
//          (unmix_sampled_rhs, mixing.hpp:218-236, applied after the sum)
//   C      apply row blocks: A_un = RHS * Ginv, per-CTA column sums of
//          squares; the last CTA forms norms + lambda (kruskal.hpp:51-67)
//   [MIX]  mixed factor F_n D_n (A_un / norm)           (mixing.hpp:297-298)
// then the fit partials per virtual 256-entry block and, on the last CTA,
// fit + should_stop + trace. The phase bodies are the ones the standalone
// kernels use (phases.cuh, dct.cuh), with the same reduction orders.
#include "dct.cuh"
#include "phases.cuh"

namespace cpb {

namespace {

constexpr int kFusedThreads = 256;

// Sense-reversing grid barrier over bar[0] (arrivals) and bar[1]
// (generation). Requires every CTA co-resident (cooperative launch).
__device__ __forceinline__ void grid_sync(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* gen = bar + 1;
    const unsigned g = *gen;
    __threadfence();
    if (atomicAdd(bar, 1u) == gridDim.x - 1u) {
      bar[0] = 0u;
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (*gen == g) __nanosleep(40);
    }
    __threadfence();
  }
  __syncthreads();
}

__device__ __forceinline__ ModeWork work_of(const FusedIter& A, const FusedMode& M) {
  ModeWork w{};
  w.z = A.z;
  w.part_gram = A.part_gram;
  w.gram_parts = M.gparts;
  w.part_rhs = A.part_rhs;
  w.ginv = A.ginv;
  w.gfull = A.gfull;
  w.info = A.info;
  w.ticket = A.ticket;
  w.ssq = A.ssq;
  w.norms = M.norms;
  w.lambda = A.lambda;
  w.a = M.a;
  w.stop = nullptr;
  w.ks = M.ks;
  w.ks_len = M.ks_len;
  w.tol = M.tol;
  return w;
}

template <int RT, bool MIX>
__global__ void __launch_bounds__(kFusedThreads, 2) fused_iteration_kernel(const FusedIter* __restrict__ args) {
  const FusedIter& A = *args;
  if (A.stop && *A.stop) return;  // uniform: the flag only changes in a previous launch
  extern __shared__ __align__(16) double fsm[];
  __shared__ int perm[RT];
  __shared__ bool s_last;
  const unsigned G = gridDim.x, b = blockIdx.x;
  const int tid = threadIdx.x;
  const int r = A.r;
  auto stamp = [&](int n, int k) {
    if (A.phase_t && b == 0 && tid == 0) A.phase_t[n * 8 + k] = globaltimer();
  };
  for (int n = 0; n < A.order; ++n) {
    const FusedMode& M = A.mode[n];
    const ModeWork w = work_of(A, M);
    stamp(n, 0);
    // ---- Z_S
    ph::z_range<RT>(M.v, A.z, static_cast<i64>(b) * kFusedThreads + tid, static_cast<i64>(G) * kFusedThreads);
    stamp(n, 1);
    grid_sync(A.bar);
    stamp(n, 2);
    // ---- Gram + inverse (last CTA) beside the split-K GEMM (all others)
    if (b == G - 1) {
      if (tid == 0)
        while (*reinterpret_cast<volatile unsigned*>(A.gram_done) < static_cast<unsigned>(M.gparts)) __nanosleep(64);
      __syncthreads();
      __threadfence();
      const bool fail = ph::inverse_cta<RT, kFusedThreads>(A.part_gram, M.gparts, r, M.tol, A.ginv, A.gfull, A.info, fsm);
      if (fail) ph::pinv_fallback<RT>(A.gfull, r, M.tol, A.ginv, A.info, perm);
      if (tid == 0) *A.gram_done = 0u;
      if (A.phase_t && tid == 0) A.phase_t[n * 8 + 7] = globaltimer();  // inverse done
    } else {
      if (static_cast<int>(b) < M.gparts) {
        const int s0 = b * M.gklen;
        ph::gram_chunk<RT>(A.z, s0, min(M.v.s, s0 + M.gklen), A.part_gram + static_cast<i64>(b) * RT * RT, fsm);
        __threadfence();
        __syncthreads();
        if (tid == 0) atomicAdd(A.gram_done, 1u);
      }
      const int ntiles = M.mtiles * M.ks;
      for (int t = b; t < ntiles; t += G - 1) {
        if (M.vec16)
          ph::gemm_tile<RT, true>(M.v.x, 0, M.v.base, A.z, M.v.in, M.v.s, r, M.ks_len, A.part_rhs, t % M.mtiles,
                                  t / M.mtiles, fsm);
        else
          ph::gemm_tile<RT, false>(M.v.x, 0, M.v.base, A.z, M.v.in, M.v.s, r, M.ks_len, A.part_rhs, t % M.mtiles,
                                   t / M.mtiles, fsm);
      }
    }
    stamp(n, 3);
    grid_sync(A.bar);
    stamp(n, 4);
    const double* rhs = nullptr;
    if constexpr (MIX) {
      // unmix the summed RHS along I_n (linear, so equal to unmixing each fiber)
      const i64 tot = M.v.in * r;
      for (i64 e = static_cast<i64>(b) * kFusedThreads + tid; e < tot; e += static_cast<i64>(G) * kFusedThreads) {
        double s = 0.0;
        for (int k = 0; k < M.ks; ++k) s += A.part_rhs[static_cast<i64>(k) * tot + e];
        A.rhs_full[e] = s;
      }
      grid_sync(A.bar);
      for (int g = b; g * M.dctF < r; g += G)
        dct::transform_group(M.plan, A.rhs_full, A.rhs_full, r, r, static_cast<i64>(g) * M.dctF, M.dctF, M.sign, 0,
                             nullptr, reinterpret_cast<double2*>(fsm));
      grid_sync(A.bar);
      rhs = A.rhs_full;
    }
    // ---- apply + column norms
    {
      constexpr int BI = kFusedThreads / RT;
      double* gi = fsm;                    // RT x (RT+1)
      double* rh = fsm + RT * (RT + 1);    // BI x (RT+1)
      ph::load_ginv<RT, kFusedThreads>(A.ginv, r, gi);
      __syncthreads();
      const int nblk = static_cast<int>((M.v.in + BI - 1) / BI);
      double q = 0.0;
      for (int blk = b; blk < nblk; blk += G)
        q += ph::apply_block<RT, kFusedThreads>(M.v.in, r, w, rhs, static_cast<i64>(blk) * BI, gi, rh);
      ph::ssq_store<RT, kFusedThreads>(q, r, A.ssq + static_cast<i64>(b) * r, rh);
      __threadfence();
      __syncthreads();
      if (tid == 0) s_last = (atomicAdd(&A.ticket[0], 1u) == G - 1u);
      __syncthreads();
      if (s_last) {
        __threadfence();
        ph::norms_final<RT, kFusedThreads>(r, M.v.in, w, G, n == 0, A.rng, rh);
        if (tid == 0) A.ticket[0] = 0u;
      }
    }
    stamp(n, 5);
    grid_sync(A.bar);
    stamp(n, 6);
    if constexpr (MIX) {
      for (int g = b; g * M.dctF < r; g += G)
        dct::transform_group(M.plan, M.a, M.mixed, r, r, static_cast<i64>(g) * M.dctF, M.dctF, M.sign, 1, M.norms,
                             reinterpret_cast<double2*>(fsm));
      grid_sync(A.bar);
    }
  }
  // ---- sampled fit + stop rule (sampling.hpp:191-210, :237-251)
  if (A.has_fit) {
    const FitArgs& f = A.fit;
    const i64 nvb = (f.phat + 255) / 256;
    double* red = fsm;
    for (i64 vb = b; vb < nvb; vb += G) {
      const double part = ph::fit_block(f, vb, red);
      if (tid == 0) f.partials[vb] = part;
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = (atomicAdd(&A.ticket[1], 1u) == G - 1u);
    __syncthreads();
    if (s_last && tid == 0) {
      __threadfence();
      A.ticket[1] = 0u;
      ph::fit_final(f, nvb);
    }
  }
}

template <int RT, bool MIX>
void* fused_fn() {
  return reinterpret_cast<void*>(&fused_iteration_kernel<RT, MIX>);
}

void* pick(int rt, bool mix) {
  switch (rt) {
    case 16: return mix ? fused_fn<16, true>() : fused_fn<16, false>();
    case 32: return mix ? fused_fn<32, true>() : fused_fn<32, false>();
    default: return mix ? fused_fn<64, true>() : fused_fn<64, false>();
  }
}

}  // namespace

size_t fused_smem_bytes(int rt, bool mix, int max_dim) {
  size_t need = static_cast<size_t>(ph::GSTAGES * ph::GBK * (ph::GBM + rt)) * sizeof(double);
  need = std::max(need, static_cast<size_t>(ph::GS * rt) * sizeof(double));
  need = std::max(need, static_cast<size_t>(rt * (rt + 1) + (kFusedThreads / rt) * (rt + 1)) * sizeof(double));
  need = std::max(need, static_cast<size_t>(16 * rt + 40) * sizeof(double));
  need = std::max(need, static_cast<size_t>(256) * sizeof(double));
  if (mix) need = std::max(need, static_cast<size_t>(2) * 16 * static_cast<size_t>(max_dim));
  return need;
}

int fused_max_grid(int rt, bool mix, size_t smem, int device) {
  int coop = 0, sms = 0;
  CPB_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, device));
  CPB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  if (!coop) return 0;
  void* fn = pick(rt, mix);
  CPB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  int per_sm = 0;
  CPB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kFusedThreads, smem));
  return per_sm * sms;
}

void launch_fused_iteration(const FusedIter* dev_args, int rt, bool mix, int grid, size_t smem,
                            cudaStream_t st) {
  void* fn = pick(rt, mix);
  void* params[] = {const_cast<FusedIter**>(&dev_args)};
  CPB_CUDA(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kFusedThreads), params, smem, st));
}

}  // namespace cpb
