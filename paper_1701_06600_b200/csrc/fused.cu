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
#include "qr.cuh"
#include "tile.cuh"

namespace cpb {

namespace {

constexpr int kFusedThreads = 256;
static_assert(kFusedThreads == 256, "ph::inverse_la: warps 0-6 hold the matrix, warp 7 inverts the pivot blocks");

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

// Peer path: sys-scope polling with a time-out (a rank that never arrives
// must not hang the GPU: after 20 s the wait gives up and flags *err, which
// the host turns into an error).
__device__ __forceinline__ unsigned ld_relaxed_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.sys.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void peer_wait(const unsigned* p, unsigned target, int* err) {
  if (threadIdx.x == 0) {
    unsigned long long t0 = 0;
    while (ld_relaxed_sys(p) < target) {
      const unsigned long long now = globaltimer();
      if (!t0) t0 = now;
      if (now - t0 > 20000000000ull) {
        atomicExch(err, 1);
        break;
      }
    }
    asm volatile("fence.acq_rel.sys;\n" ::: "memory");
  }
  __syncthreads();
}
__device__ __forceinline__ void red_release_sys(unsigned* p, unsigned v) {
  asm volatile("red.release.sys.global.add.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}

// PEER: the slab-sharded CPRAND-MIX iteration (FusedIter::np ranks, peer
// memory as in rand_body): modes n < N-1 contract this rank's fibers (its
// owner-ordered sample range) and every apply block exchanges its rows' RHS
// sums with the same block of every rank (rank-order sum, so the mixed
// factors stay replicated); the last mode applies the slab's rows, stores
// them and the block's sums of squares into every rank's buffers, and CTA 0
// of every rank forms the norms once all ranks' partials are in.

template <int RT, bool MIX, bool PEER>
__device__ __forceinline__ void iter_body(const FusedIter* __restrict__ args, const unsigned G, const unsigned b) {
  const FusedIter& A = *args;
  if (A.stop && *A.stop) return;  // uniform: the flag only changes in a previous launch
  extern __shared__ __align__(16) double fsm[];
  __shared__ int perm[RT];
  __shared__ bool s_last;
  const int tid = threadIdx.x;
  const int r = A.r;
  const int np = PEER ? A.np : 1;
  const unsigned seq = A.seq;
  if (PEER && np > 1 && seq > 1)  // every rank's last-mode rows of the previous launch (Z_S of mode 0 reads them)
    peer_wait(A.mode[A.order - 1].adone + (b % kRep) * kCS, A.lastw * (seq - 1), A.perr);
  auto stamp = [&](int n, int k) {
    if (A.phase_t && b == 0 && tid == 0) A.phase_t[n * 16 + k] = globaltimer();
  };
  // grid barrier on this launch's own counter: arrive with a fire-and-forget
  // release add, wait for the k-th multiple of the grid (no returning atomic,
  // no reset: the counter is used by this launch only)
  unsigned kbar = 0;
  auto grid_bar = [&]() {
    ++kbar;
    __syncthreads();
    if (tid == 0) {
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;\n" ::"l"(A.lbar) : "memory");
      while (tl::ld_relaxed(A.lbar) < kbar * G) __nanosleep(32);
      asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
    }
    __syncthreads();
  };
  for (int n = 0; n < A.order; ++n) {
    const FusedMode& M = A.mode[n];
    const ModeWork w = work_of(A, M);
    stamp(n, 0);
    // ---- Z_S
    ph::z_range<RT>(M.v, A.z, static_cast<i64>(b) * kFusedThreads + tid, static_cast<i64>(G) * kFusedThreads);
    stamp(n, 1);
    grid_bar();
    stamp(n, 2);
    // ---- Gram + inverse (last CTA) beside the split-K GEMM (all others)
    if (b == G - 1) {
      if (tid == 0)
        while (*reinterpret_cast<volatile unsigned*>(A.gram_done) < static_cast<unsigned>(M.gparts)) __nanosleep(64);
      __syncthreads();
      __threadfence();
      bool fail;
      if constexpr (RT == 16) {
        // small Gram: the split partials summed in split order (one entry per
        // thread), then the CPRAND kernel's look-ahead block Gauss-Jordan
        // (measured: C3 10.3 k -> 10.7 k it/s; for RT >= 32 inverse_cta wins)
        double* gs = A.gfull + static_cast<i64>(r) * r;  // RT x RT scratch beyond the r x r Gram copy
        for (int e = tid; e < RT * RT; e += kFusedThreads) {
          double acc = 0.0;
          for (int k0 = 0; k0 < M.gparts; k0 += 8) {
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u)
              v[u] = (k0 + u < M.gparts) ? __ldcg(A.part_gram + static_cast<i64>(k0 + u) * RT * RT + e) : 0.0;
#pragma unroll
            for (int u = 0; u < 8; ++u)
              if (k0 + u < M.gparts) acc += v[u];
          }
          gs[e] = acc;
        }
        __syncthreads();
        fail = ph::inverse_la<RT>(gs, r, M.tol, A.ginv, A.gfull, A.info, fsm);
      } else {
        fail = ph::inverse_cta<RT, kFusedThreads>(A.part_gram, M.gparts, r, M.tol, A.ginv, A.gfull, A.info, fsm);
      }
      if (fail) {
        if (A.qrws)  // QR path (kr_linalg.hpp:105-118): the apply takes its rows from qr_rows
          ph::qr_factor<RT>(A.z, M.v.s, r, M.qtol, A.qrws, A.ginv, A.info, fsm);
        else
          ph::pinv_fallback<RT>(A.gfull, r, M.tol, A.ginv, A.info, perm);
      }
      if (tid == 0) *A.gram_done = 0u;
      if (A.phase_t && tid == 0) A.phase_t[n * 16 + 7] = globaltimer();  // inverse done
    } else {
      if (static_cast<int>(b) < M.gparts) {
        const int s0 = b * M.gklen;
        ph::gram_chunk<RT>(A.z, s0, min(M.v.s, s0 + M.gklen), A.part_gram + static_cast<i64>(b) * RT * RT, fsm);
        __threadfence();
        __syncthreads();
        if (tid == 0) atomicAdd(A.gram_done, 1u);
      }
      const int ntiles = M.mtiles * M.ks;
      // peer path, modes n < N-1: this rank's fibers, the owner-ordered range [loff, loff + lcnt)
      const bool loc = PEER && np > 1 && n < A.order - 1;
      const i64* gbase = loc ? M.v.base + M.loff : M.v.base;
      const double* gz = loc ? A.z + static_cast<i64>(M.loff) * RT : A.z;
      const int gs = loc ? M.lcnt : M.v.s;
      for (int t = b; t < ntiles; t += G - 1) {
        if (M.vec16)
          ph::gemm_tile<RT, true>(M.v.x, 0, gbase, gz, M.v.in, gs, r, M.ks_len, A.part_rhs, t % M.mtiles,
                                  t / M.mtiles, fsm);
        else
          ph::gemm_tile<RT, false>(M.v.x, 0, gbase, gz, M.v.in, gs, r, M.ks_len, A.part_rhs, t % M.mtiles,
                                   t / M.mtiles, fsm, M.est);
      }
    }
    stamp(n, 3);
    grid_bar();
    stamp(n, 4);
    // ---- the mode's solve in the mixed domain. The reference unmixes the
    // summed RHS (sign after DCT-III), solves, normalizes and mixes the
    // factor again (DCT-II after sign, mixing.hpp:284-312). The transforms
    // are orthonormal and act on the rows while G^-1 acts on the columns, so
    // mix(unmix(RHS) G^-1 / norms) = RHS G^-1 / norms with the same column
    // norms: the kernel keeps the mixed factor unnormalized (M.mixed, norms
    // applied lazily in Z_S like the CPRAND kernel) and unmixes each factor
    // once per iteration, for the fit and the result (below).
    // small modes (one CTA applies): sum the split-K partials over the grid
    // first; otherwise each apply block sums its rows' partials as it loads
    // them (same order, k = 0, 1, ...: the same bits), no extra barrier
    // QR mode (the inverse's pivot test failed): the rows come from qr_rows
    const bool qr = A.qrws && __ldcg(A.info + 2) != 0;
    const QrSrc qs{M.v.x, M.v.base, 0, M.est, M.v.s};
    if (M.tail1) {
      const i64 tot = M.v.in * r;
      if (qr) {
        constexpr int BQ = kFusedThreads / RT;
        for (i64 blk = b; blk * BQ < M.v.in; blk += G)
          ph::qr_rows<RT, kFusedThreads>(qs, A.qrws, r, M.v.in, blk * BQ, BQ, A.rhs_full + blk * BQ * r, r, fsm);
      } else {
        for (i64 e = static_cast<i64>(b) * kFusedThreads + tid; e < tot; e += static_cast<i64>(G) * kFusedThreads) {
          double s = 0.0;
          for (int k = 0; k < M.ks; ++k) s += A.part_rhs[static_cast<i64>(k) * tot + e];
          A.rhs_full[e] = s;
        }
      }
      grid_bar();
    }
    {
      ModeWork wm = w;
      wm.a = M.mixed;  // the apply writes the mixed, unnormalized factor
      const bool plast = PEER && np > 1 && n == A.order - 1;
      if (plast) wm.a = M.mixed + A.slab_off * r;  // this rank's slab rows of the last mode
      wm.q = qs;
      wm.qrws = A.qrws;
      constexpr int BI = kFusedThreads / RT;
      double* gi = fsm;                  // RT x (RT+1)
      double* rh = fsm + RT * (RT + 1);  // BI x (RT+1)
      const int nblk = static_cast<int>((M.v.in + BI - 1) / BI);
      // a zero column is refilled in the unmixed domain (norms_final writes
      // it to w.a = M.a); its mixed image replaces the mixed column
      auto remix = [&](unsigned long long zm) {
        for (int c = 0; c < r; ++c)
          if ((zm >> c) & 1ull) {
            __syncthreads();
            dct::transform_group(M.plan, M.a, M.mixed, r, c + 1, c, 2, M.sign, 1, nullptr,
                                 reinterpret_cast<double2*>(fsm));
          }
      };
      if (M.tail1) {  // small mode: one CTA, no ticket
        if (b == 0) {
          ph::load_ginv<RT, kFusedThreads>(A.ginv, r, gi);
          __syncthreads();
          double q = 0.0;
          for (int blk = 0; blk < nblk; ++blk)
            q += ph::apply_block<RT, kFusedThreads>(M.v.in, r, wm, A.rhs_full, static_cast<i64>(blk) * BI, gi, rh);
          ph::ssq_store<RT, kFusedThreads>(q, r, A.ssq, rh);
          remix(ph::norms_final<RT, kFusedThreads>(r, M.in_full, w, 1, n == 0, A.rng, rh));
        }
      } else if (PEER && np > 1) {
        // peer path: every CTA takes its row blocks (possibly none)
        ph::load_ginv<RT, kFusedThreads>(A.ginv, r, gi);
        __syncthreads();
        double q = 0.0;
        for (int blk = b; blk < nblk; blk += G) {
          const i64 i0 = static_cast<i64>(blk) * BI;
          if (!plast) {
            // this block's local RHS sums (split order) to block prank of
            // every rank's receive buffer; the same block of every rank then
            // sums the np blocks in rank order into rhs_full
            const i64 tot = M.v.in * r;
            for (int e = tid; e < BI * r; e += kFusedThreads) {
              const i64 i = i0 + e / r;
              if (i >= M.v.in) continue;
              const i64 o = i * r + e % r;
              double sum = 0.0;
              for (int k = 0; k < M.ks; ++k) sum += __ldcg(A.part_rhs + static_cast<i64>(k) * tot + o);
              for (int qq = 0; qq < np; ++qq) A.precv[qq][static_cast<i64>(A.prank) * A.rcv_ld + o] = sum;
            }
            __threadfence_system();
            __syncthreads();
            const i64 slot = (static_cast<i64>(n) * A.ptiles + blk) * kCS;
            if (tid < np) red_release_sys(A.prcnt[tid] + slot, 1u);
            peer_wait(A.prcnt[A.prank] + slot, static_cast<unsigned>(np) * seq, A.perr);
            for (int e = tid; e < BI * r; e += kFusedThreads) {
              const i64 i = i0 + e / r;
              if (i >= M.v.in) continue;
              const i64 o = i * r + e % r;
              double sum = 0.0;
              for (int qq = 0; qq < np; ++qq) sum += __ldcv(A.precv[A.prank] + static_cast<i64>(qq) * A.rcv_ld + o);
              A.rhs_full[o] = sum;
            }
            __syncthreads();
            q += ph::apply_block<RT, kFusedThreads>(M.v.in, r, wm, A.rhs_full, i0, gi, rh);
          } else {
            q += ph::apply_block<RT, kFusedThreads>(M.v.in, r, wm, nullptr, i0, gi, rh);
            // the block's rows into every other rank's mixed factor
            for (int e = tid; e < BI * r; e += kFusedThreads) {
              const i64 i = i0 + e / r;
              if (i >= M.v.in) continue;
              const i64 o = (A.slab_off + i) * r + e % r;
              const double v = __ldcg(M.mixed + o);
              for (int qq = 0; qq < np; ++qq)
                if (qq != A.prank) A.pfac[qq][o] = v;
            }
          }
        }
        if (plast) {
          // sums of squares into every rank's [np][G] partials, then every
          // rank's counter; CTA 0 of each rank forms the norms from all of them
          double* own = A.pssq[A.prank] + (static_cast<i64>(A.prank) * G + b) * r;
          ph::ssq_store<RT, kFusedThreads>(q, r, own, rh);
          if (tid < r)
            for (int qq = 0; qq < np; ++qq)
              if (qq != A.prank) A.pssq[qq][(static_cast<i64>(A.prank) * G + b) * r + tid] = own[tid];
          __threadfence_system();
          __syncthreads();
          if (tid < np * kRep) red_release_sys(A.pdone[tid / kRep] + (tid % kRep) * kCS, 1u);
          if (b == 0) {
            peer_wait(M.adone + (b % kRep) * kCS, A.lastw * seq, A.perr);
            ModeWork wq = w;
            wq.ssq = A.pssq[A.prank];
            remix(ph::norms_final<RT, kFusedThreads>(r, M.in_full, wq, np * static_cast<int>(G), n == 0, A.rng, rh));
          }
        } else {
          // replicated rows: the ticket-based norms below (every CTA took part)
          ph::ssq_store<RT, kFusedThreads>(q, r, A.ssq + static_cast<i64>(b) * r, rh);
          __threadfence();
          __syncthreads();
          if (tid == 0) s_last = (atomicAdd(&A.ticket[0], 1u) == G - 1u);
          __syncthreads();
          if (s_last) {
            __threadfence();
            remix(ph::norms_final<RT, kFusedThreads>(r, M.in_full, w, static_cast<int>(G), n == 0, A.rng, rh));
            if (tid == 0) A.ticket[0] = 0u;
          }
        }
      } else if (static_cast<int>(b) < min(static_cast<int>(G), nblk)) {
        // the CTAs that own row blocks: apply, column sums of squares, ticket;
        // the last of them forms the norms from their napp partials
        const unsigned napp = static_cast<unsigned>(min(static_cast<int>(G), nblk));
        ph::load_ginv<RT, kFusedThreads>(A.ginv, r, gi);
        __syncthreads();
        double q = 0.0;
        for (int blk = b; blk < nblk; blk += G)
          q += qr ? ph::apply_block_qr<RT, kFusedThreads>(M.v.in, r, wm, static_cast<i64>(blk) * BI, rh,
                                                           rh + BI * (RT + 1))
                  : ph::apply_block<RT, kFusedThreads>(M.v.in, r, wm, nullptr, static_cast<i64>(blk) * BI, gi, rh);
        ph::ssq_store<RT, kFusedThreads>(q, r, A.ssq + static_cast<i64>(b) * r, rh);
        __threadfence();
        __syncthreads();
        if (tid == 0) s_last = (atomicAdd(&A.ticket[0], 1u) == napp - 1u);
        __syncthreads();
        if (s_last) {
          __threadfence();
          remix(ph::norms_final<RT, kFusedThreads>(r, M.in_full, w, static_cast<int>(napp), n == 0, A.rng, rh));
          if (tid == 0) A.ticket[0] = 0u;
        }
      }
    }
    stamp(n, 5);
    grid_bar();
    stamp(n, 6);
  }
  // ---- the unmixed factors A_un = D DCT-III(mixed) of every mode (the fit
  // and the result read A_un / norms), one transform group per task; bench
  // mode (lazy_last) defers it to before the host reads the model
  if (A.has_fit || !A.lazy_last) {
    // groups of kUnmixF columns (one complex sequence): many small tasks over
    // the grid instead of one task of every column per mode (measured: C5,
    // R = 20, one 20-column task per mode took ~34 us of the iteration)
    constexpr int kUnmixF = 2;
    const int gm = (r + kUnmixF - 1) / kUnmixF;
    const int tasks = A.order * gm;
    for (int t = b; t < tasks; t += G) {
      const int m = t / gm, g = t - m * gm;
      const FusedMode& Q = A.mode[m];
      const int dFm = kUnmixF;
      __syncthreads();
      dct::transform_group(Q.plan, Q.mixed, Q.a, r, r, static_cast<i64>(g) * dFm, dFm, Q.sign, 0, nullptr,
                           reinterpret_cast<double2*>(fsm));
    }
    grid_bar();
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
    if (s_last) {  // the last CTA: every partial is written
      __threadfence();
      if (tid == 0) A.ticket[1] = 0u;
      ph::fit_final(f, nvb, red);
    }
  }
}

template <int RT, bool MIX>
__global__ void __launch_bounds__(kFusedThreads, 2) fused_iteration_kernel(const FusedIter* __restrict__ args) {
  iter_body<RT, MIX, false>(args, gridDim.x, blockIdx.x);
}
template <int RT>
__global__ void __launch_bounds__(kFusedThreads, 2) peer_mix_kernel(const FusedLaunch L) {
  const unsigned G = gridDim.x / static_cast<unsigned>(L.groups);
  const unsigned grp = blockIdx.x / G;
  const FusedIter* ap = L.a[0];
#pragma unroll
  for (int q = 1; q < kMaxPeer; ++q)
    if (static_cast<int>(grp) == q) ap = L.a[q];
  iter_body<RT, true, true>(ap, G, blockIdx.x - grp * G);
}

// ---------------------------------------------------------------------------
// CPRAND (no mixing): tile-owned mode updates, one grid-wide rendezvous per mode.
//
// CTAs [0, G-1) own (64-row block mt, sample split kb) tiles; CTA G-1 owns the
// Gram inverse. Per mode n, with no grid barrier between the phases:
//   tile CTA   Z_S rows of split kb -> shared memory (z_tile)
//              Gram blocks q = mt (mod tm) of split kb -> gpart; the last of
//              the tk splits to arrive sums block q into gsum (both triangles)
//              RHS partial (mt, kb) -> part_rhs, then arrive mt_cnt[mt]
//   inverse    waits for every Gram block, block Gauss-Jordan -> ginv, flag
//   tile CTA   waits mt_cnt[mt] == tk, sums its share of the rows of mt over
//              the splits, waits for ginv, A_un rows = RHS * Ginv, column
//              sums of squares
//   all        ticket; the last CTA forms norms + lambda (kruskal.hpp:51-67)
//              and releases the next mode (sense-reversing generation).
// Counters of mode n are reset by CTA 0 during mode n+1, when no CTA can
// still be waiting on them.
// sum_{k < n} p[k * step] in order k = 0, 1, ... (16 loads in flight per batch)
__device__ __forceinline__ double sum_strided(const double* __restrict__ p, i64 step, int n) {
  double sum = 0.0;
  int k = 0;
  for (; k + 16 <= n; k += 16) {
    double v[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) v[u] = __ldcg(p + (k + u) * step);
#pragma unroll
    for (int u = 0; u < 16; ++u) sum += v[u];
  }
  if (k < n) {
    double v[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) v[u] = (k + u < n) ? __ldcg(p + (k + u) * step) : 0.0;
#pragma unroll
    for (int u = 0; u < 16; ++u)
      if (k + u < n) sum += v[u];
  }
  return sum;
}

// the same sum with all (n <= 32) loads in flight at once: one L2 round trip
// for the row-block reducers on the Gram's critical path
__device__ __forceinline__ double sum_strided32(const double* __restrict__ p, i64 step, int n) {
  if (n > 32) return sum_strided(p, step, n);
  double v[32];
#pragma unroll
  for (int u = 0; u < 32; ++u) v[u] = (u < n) ? __ldcg(p + u * step) : 0.0;
  double sum = 0.0;
#pragma unroll
  for (int u = 0; u < 32; ++u)
    if (u < n) sum += v[u];
  return sum;
}

// L2 prefetch of one iteration's sample tables (all modes): global thread g
// prefetches 128-byte line g of the concatenated tables.
__device__ __forceinline__ void prefetch_tables(const FusedIter& A, unsigned b) {
  i64 line = static_cast<i64>(b) * blockDim.x + threadIdx.x;
  for (int n = 0; n < A.order; ++n) {
    const ModeView& v = A.mode[n].v;
    for (int c = 0; c <= v.kept; ++c) {
      const char* base = c < v.kept ? reinterpret_cast<const char*>(v.rows[c]) : reinterpret_cast<const char*>(v.base);
      const i64 nl = ((c < v.kept ? 4LL : 8LL) * v.s + 127) / 128;
      if (line < nl) {
        asm volatile("prefetch.global.L2 [%0];" ::"l"(base + line * 128));
        return;
      }
      line -= nl;
    }
  }
}

// Buffer of mode m's column sums of squares (one [G][r] block per buffer).
// Modes alternate between buffers 0 and 1: mode m's partials are read at the
// start of mode m + 1 and buffer m & 1 is next written in mode m + 2, behind
// that mode's start-of-mode wait. Under lazy_last the last mode's partials
// are read during mode 0 of the NEXT launch, which starts without such a
// wait: a CTA without a tile in mode 0 stores its (zero) partial at once, and
// where it had rows in the last mode (the modes' tilings differ) it could
// overwrite a partial the inverse CTA had not read yet. The last mode
// therefore has a buffer of its own, rewritten only in the next launch's last
// mode. (Found by tests/test_gpu_upload.py::test_repeated_solves_are_bitwise_
// equal: a lost partial only rescales the next Z_S's columns, which the
// normalization absorbs, so results moved by 1e-12, run to run.)
__device__ __forceinline__ int ssq_buf(const FusedIter& A, int m) {
  return (A.lazy_last && m == A.order - 1) ? 2 : (m & 1);
}

// GA: the Gram is summed with L2 fp64 atomics (FusedIter::gram_atomic).
// PEER: the slab-sharded path (FusedIter::np ranks exchanging through peer
// memory): modes n < N-1 contract this rank's fibers and exchange the RHS
// rows of every apply share with the counterpart CTAs of the other ranks
// (summed in rank order, so every rank applies the same rows); the last mode
// applies the slab's rows and stores them, with their column sums of
// squares, into every rank's factor.
// The CPRAND kernel's rarely taken LS paths (QR, pseudo-inverse fallback)
// stay out of line: inlined they sat between the phases every CTA runs each
// mode and cost the hot path instruction fetches (C4 9.06 k -> 9.25 k it/s on
// one box; the MIX kernel measured 1-2 % slower with them out of line, so it
// keeps them inline).
#ifdef CPB_NO_COLD
#define CPB_COLD_ATTR
#else
#define CPB_COLD_ATTR __noinline__
#endif
template <int RT>
__device__ CPB_COLD_ATTR void qr_factor_cold(const double* z, int s, int r, double qtol, double* ws, double* ginv,
                                            int* info, double* sh) {
  ph::qr_factor<RT>(z, s, r, qtol, ws, ginv, info, sh);
}
template <int RT>
__device__ CPB_COLD_ATTR void pinv_fallback_cold(double* gfull, int r, double tol, double* ginv, int* info, int* perm_sh) {
  ph::pinv_fallback<RT>(gfull, r, tol, ginv, info, perm_sh);
}
template <int RT>
__device__ CPB_COLD_ATTR void qr_rows_cold(const QrSrc& q, const double* ws, int r, i64 in, i64 i0, int nrow, double* out,
                                          int ldo, double* stage) {
  ph::qr_rows<RT, kFusedThreads>(q, ws, r, in, i0, nrow, out, ldo, stage);
}

template <int RT, bool GA, bool PEER>
__device__ __forceinline__ void rand_body(const FusedIter* __restrict__ args, const unsigned G, const unsigned b) {
  using namespace tl;
  const FusedIter& A = *args;
  if (A.stop && *A.stop) return;  // uniform: the flag only changes in a previous launch
  extern __shared__ __align__(16) double fsm[];
  __shared__ int perm[RT];
  __shared__ bool s_last;
  const int tid = threadIdx.x;
  const int np = PEER ? A.np : 1;
  if (A.census) {
    if (tid == 0) {
      unsigned sm;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
      A.census[b] = static_cast<int>(sm);
    }
    return;
  }
  // roles: CTA inv_cta inverts the Gram and reduces the norms; idle_cta (its
  // SM partner, if any) stays off the FP64 pipe; the rest own tiles in rank order
  const int inv = A.inv_cta >= 0 ? A.inv_cta : static_cast<int>(G) - 1;
  const int idle = A.idle_cta;
  const bool is_inv = static_cast<int>(b) == inv, is_idle = static_cast<int>(b) == idle;
  const unsigned Gw = G - 1 - (idle >= 0 ? 1u : 0u);
  const unsigned rank = b - (static_cast<int>(b) > inv ? 1u : 0u) - (idle >= 0 && static_cast<int>(b) > idle ? 1u : 0u);
  const int r = A.r;
  const int nfr = (r + 7) / 8;
  prefetch_tables(A, b);
  if (A.cta_t && tid == 0) {
    unsigned sm;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    A.cta_t[b * 16 + 14] = sm;
  }
  auto stamp = [&](int n, int k) {
    if (A.phase_t && rank == 0 && !is_inv && !is_idle && tid == 0) A.phase_t[n * 16 + k] = globaltimer();
    if (A.cta_t && n == 1 && tid == 0) A.cta_t[b * 16 + k] = globaltimer();
  };
  const unsigned seq = A.seq;
  // norms + lambda of mode m (inverse CTA), from the tile CTAs' column sums
  // of squares (buffer m & 1). Mode m >= 1 entered the next Z_S unnormalized,
  // so its solution carries mode m-1's norms as a column scale (lam_scale).
  auto form_norms = [&](int m) {
    const FusedMode& Q = A.mode[m];
    ModeWork wq = work_of(A, Q);
    wq.ssq = A.ssq + static_cast<i64>(ssq_buf(A, m)) * G * r;
    int nparts = static_cast<int>(Gw);
    if (PEER && np > 1 && m == A.order - 1) {  // every rank's slab partials, in (rank, CTA) order
      wq.ssq = A.pssq[A.prank];
      nparts = np * static_cast<int>(Gw);
    }
    // the column scale the solution carries: the norms of the factor that
    // entered this mode's Z_S unnormalized (mode m-1; for mode 0 under
    // lazy_last, the last mode)
    const double* lam_scale = m >= 1 ? A.mode[m - 1].norms : (A.lazy_last ? A.mode[A.order - 1].norms : nullptr);
    const unsigned long long zm =
        ph::norms_final<RT, kFusedThreads>(r, Q.in_full, wq, nparts, m == 0, A.rng, fsm, nullptr, lam_scale);
    signal_add_rep(Q.nready, 1u, kRep);
    return zm;
  };
  for (int n = 0; n < A.order; ++n) {
    const FusedMode& M = A.mode[n];
    const ModeWork w = work_of(A, M);
    const i64 in = M.v.in;
    const int ntiles = M.tm * M.tk;
    if (n >= 1 && !is_idle)  // the previous mode's factor rows are all written
      wait_geq(A.mode[n - 1].adone + (b % kRep) * kCS, seq * Gw);
    if (PEER && np > 1 && n == 0 && seq > 1 && !is_idle)  // every rank's last-mode rows of the previous launch
      peer_wait(A.mode[A.order - 1].adone + (b % kRep) * kCS, A.lastw * (seq - 1), A.perr);
    stamp(n, 0);
    if (b == 0) {  // reset the previous mode's counters: every wait on them is over
      const FusedMode& P = A.mode[(n + A.order - 1) % A.order];
      for (int e = tid; e < P.tm; e += kFusedThreads) P.mt_cnt[e * kCS] = 0u;
      for (int e = tid; e < P.tk; e += kFusedThreads) P.kb_cnt[e * kCS] = 0u;
      if (tid < 3) P.mcnt[tid * kCS] = 0u;
      if (tid < kRep) P.grdy[tid * kCS] = 0u;
      if (tid < kRep) P.gdone[tid * kCS] = 0u;
      for (int e = tid; e < P.tm; e += kFusedThreads) P.gm_cnt[e * kCS] = 0u;
    }
    if (is_inv) {
      // off the critical path: overlaps this mode's Z / Gram. A zero column
      // refilled here (kruskal.hpp:57-63) may race with the tile CTAs reading
      // the previous factor's rows for this mode's Z_S: the mode then takes
      // the QR path on a Z_S rebuilt below from the refilled factor.
      unsigned long long zmask = 0ull;
      if (n >= 1) {
        zmask = form_norms(n - 1);
      } else if (!PEER && A.lazy_last && seq > 1 && *reinterpret_cast<volatile int*>(A.npend)) {
        // the previous launch's last-mode norms (it ended without forming them)
        wait_geq(A.mode[A.order - 1].adone + (b % kRep) * kCS, (seq - 1) * Gw);
        zmask = form_norms(A.order - 1);
        if (tid == 0) *A.npend = 0;
      }
      if (A.phase_t && tid == 0) A.phase_t[n * 16 + 13] = globaltimer();
      // ---- Gram: the row-block reducers summed it (dist_gram), or sum the
      // split partials of every 8 x 8 block here (split order)
      if constexpr (GA) {
        // buffer (n-1) & 1 is next added to by mode n+1, whose tiles start
        // after this CTA's grdy(n): zero it now
        if (n >= 1)
          for (int e = tid; e < RT * RT; e += kFusedThreads) A.gsum[((n - 1) & 1) * RT * RT + e] = 0.0;
        wait_geq(M.gdone + (b % kRep) * kCS, static_cast<unsigned>(ntiles));
      } else if (M.dist_gram)
        wait_geq(M.gdone + (b % kRep) * kCS, static_cast<unsigned>(M.nblk));
      else
        wait_geq(M.mcnt, static_cast<unsigned>(ntiles));
      if (A.phase_t && tid == 0) A.phase_t[n * 16 + 8] = globaltimer();
      if (!M.dist_gram && !GA) {
        // every block's split partials, in split order (chunks of PER
        // elements per thread: r > 56 has more than 2048 block entries)
        constexpr int PER = 8, KC = 5;
        const int ne = M.nblk * 64;
        for (int e0 = 0; e0 < ne; e0 += PER * kFusedThreads) {
          double sum[PER];
#pragma unroll
          for (int u = 0; u < PER; ++u) sum[u] = 0.0;
          for (int k0 = 0; k0 < M.tk; k0 += KC) {
            double v[PER][KC];
#pragma unroll
            for (int u = 0; u < PER; ++u) {
              const int e = e0 + tid + u * kFusedThreads;
              const double* src = A.gpart + static_cast<i64>(e / 64) * M.tk * 64 + (e % 64);
#pragma unroll
              for (int k = 0; k < KC; ++k)
                v[u][k] = (e < ne && k0 + k < M.tk) ? __ldcg(src + (k0 + k) * 64) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < PER; ++u)
#pragma unroll
              for (int k = 0; k < KC; ++k)
                if (k0 + k < M.tk) sum[u] += v[u][k];
          }
#pragma unroll
          for (int u = 0; u < PER; ++u) {
            const int e = e0 + tid + u * kFusedThreads;
            if (e >= ne) continue;
            int bi, bj;
            gram_block_coords(e / 64, nfr, &bi, &bj);
            const int el = e % 64, gi = bi * 8 + el / 8, gj = bj * 8 + el % 8;
            A.gsum[gi * RT + gj] = sum[u];
            A.gsum[gj * RT + gi] = sum[u];
          }
        }
      }
      __syncthreads();
      if (A.phase_t && tid == 0) A.phase_t[n * 16 + 15] = globaltimer();
      // ---- inverse (pivoted-Cholesky min-norm fallback when rank deficient)
      const bool rebuild = zmask != 0ull && A.qrws;
      const bool fail = rebuild || ph::inverse_la<RT>(A.gsum + (GA ? (n & 1) * RT * RT : 0), r, M.tol, A.ginv,
                                                      A.gfull, A.info, fsm, A.phase_t ? A.phase_t + n * 16 + 11 : nullptr);
      if (fail) {
        if (A.qrws) {  // QR path (kr_linalg.hpp:105-118)
          const double* zq = A.z;
          if (rebuild) {  // Z_S from the refilled factor, into the workspace's V block
            ph::z_range<RT>(M.v, A.qrws, tid, kFusedThreads);
            __threadfence_block();
            __syncthreads();
            zq = A.qrws;
          }
          qr_factor_cold<RT>(zq, M.v.s, r, M.qtol, A.qrws, A.ginv, A.info, fsm);
        } else {
          pinv_fallback_cold<RT>(A.gfull, r, M.tol, A.ginv, A.info, perm);
        }
      }
      signal_add_rep(M.grdy, 1u, kRep);
      if (A.phase_t && tid == 0) A.phase_t[n * 16 + 7] = globaltimer();
    } else if (!is_idle) {
      const TileSmem t = tile_smem<RT>(fsm, M.zcap);
      if (n >= 2)  // Z_S divides by the norms of the modes before n-1
        wait_geq(A.mode[n - 2].nready + (b % kRep) * kCS, seq);
      if (!PEER && A.lazy_last && n == 1 && seq > 1 && A.order >= 3)  // ... and the previous launch's last mode
        wait_geq(A.mode[A.order - 1].nready + (b % kRep) * kCS, seq - 1);
      // this CTA's share of every one of its splits' Z rows, then signal
      // (no waiting here, so CTAs with several tiles cannot deadlock)
      for (int tt = rank; tt < ntiles; tt += Gw) {
        const int mt = tt % M.tm, kb = tt / M.tm;
        const int s0 = kb * M.tklen;
        const int cnt = min(M.v.s - s0, M.tklen);
        const int zr = (cnt + M.tm - 1) / M.tm;
        const int z0 = s0 + mt * zr, z1 = min(s0 + cnt, z0 + zr);
        if (z0 < z1) z_share<RT>(M.v, z0, z1, A.z);
        signal_add(M.kb_cnt + kb * kCS, 1u);
      }
      stamp(n, 9);
      for (int tt = rank; tt < ntiles; tt += Gw) {
        const int mt = tt % M.tm, kb = tt / M.tm;
        const int s0 = kb * M.tklen;
        const int cnt = min(M.v.s - s0, M.tklen);
        const int kpad = (cnt + BK - 1) / BK * BK;
        wait_geq(M.kb_cnt + kb * kCS, static_cast<unsigned>(M.tm));
        if (tt == static_cast<int>(rank)) stamp(n, 10);
        if (tt == static_cast<int>(rank) && A.cta_t && n == 1 && tid == 0)
          A.cta_t[b * 16 + 11] = (static_cast<unsigned long long>(mt) << 8) | static_cast<unsigned long long>(kb);
        z_load<RT>(M.v, A.z, s0, cnt, kpad, t);
        if (tt == static_cast<int>(rank)) stamp(n, 1);
        // Gram blocks q = mt, mt + tm, ... of this split (the inverse CTA sums them)
        if constexpr (GA) {
          gram_blocks_add<RT>(t, kpad, nfr, mt, M.tm, A.gsum + (n & 1) * RT * RT);
          signal_add(M.gdone + (inv % kRep) * kCS, 1u);
        } else {
          gram_blocks<RT>(t, kpad, nfr, mt, M.tm, kb, M.tk, A.gpart);
        }
        if constexpr (GA) {
        } else if (!M.dist_gram) {
          signal_add(M.mcnt, 1u);
        } else {
          signal_add(M.gm_cnt + mt * kCS, 1u);
          if (A.cta_t && n == 1 && tid == 0) A.cta_t[b * 16 + 12] = globaltimer();
          if (kb == M.tk - 1 && mt < M.nblk) {
            // row-block reducer: sum blocks q = mt, mt + tm, ... over the splits
            wait_geq(M.gm_cnt + mt * kCS, static_cast<unsigned>(M.tk));
            const int nq = (M.nblk - mt + M.tm - 1) / M.tm;
            for (int e = tid; e < nq * 64; e += kFusedThreads) {
              const int q = mt + (e / 64) * M.tm, el = e % 64;
              const double sum = sum_strided32(A.gpart + static_cast<i64>(q) * M.tk * 64 + el, 64, M.tk);
              int bi, bj;
              gram_block_coords(q, nfr, &bi, &bj);
              const int gi = bi * 8 + el / 8, gj = bj * 8 + el % 8;
              A.gsum[gi * RT + gj] = sum;
              A.gsum[gj * RT + gi] = sum;
            }
            signal_add_rep(M.gdone, static_cast<unsigned>(nq), kRep);
          }
        }
        // the RHS streams the fibers only after the Gram is summed, so the
        // Gram's round trips do not queue behind the fiber traffic (the RHS
        // has slack: it is consumed after the inverse)
        if (M.dist_gram && A.gram_first && !GA) wait_geq(M.gdone + (b % kRep) * kCS, static_cast<unsigned>(M.nblk));
        if (tt == static_cast<int>(rank)) stamp(n, 2);
        if (PEER && np > 1 && n < A.order - 1) {
          // this rank's fibers: local split kb of the owner-ordered range
          const int l0 = M.loff + kb * M.tkllen;
          const int cl = max(0, min(M.loff + M.lcnt, l0 + M.tkllen) - l0);
          const int kpl = (cl + BK - 1) / BK * BK;
          if (cl > 0) {
            for (int g = l0 / M.tklen; g <= (l0 + cl - 1) / M.tklen; ++g)
              wait_geq(M.kb_cnt + g * kCS, static_cast<unsigned>(M.tm));
            z_load<RT>(M.v, A.z, l0, cl, kpl, t);
          }
          gemm_tile<RT>(M.v.x, M.vec16 != 0, in, static_cast<i64>(mt) * BM, r, cl, kpl, t,
                        A.part_rhs + static_cast<i64>(kb) * in * r, M.v.xsize);
        } else {
          gemm_tile<RT>(M.v.x, M.vec16 != 0, in, static_cast<i64>(mt) * BM, r, cnt, kpad, t,
                        A.part_rhs + static_cast<i64>(kb) * in * r, M.v.xsize);
        }
        signal_add(M.mt_cnt + mt * kCS, 1u);
      }
      stamp(n, 3);
      // ---- apply: this CTA's share of the rows of each of its tiles
      double q2 = 0.0;  // thread c < r: column sum of squares over this CTA's rows
      constexpr int LD = RT + 1;
      double* gi = fsm;             // RT x LD
      double* rh = gi + RT * LD;    // rows_per x LD
      const int rows_per = (BM + M.tk - 1) / M.tk;
      double* ob = rh + rows_per * LD;
      bool have_ginv = false, qr = false;
      const QrSrc qs{M.v.x, M.v.base, 0, 1, M.v.s};
      // QR staging: after ob, or ob itself when it is large enough
      double* qstage = rows_per * LD >= ph::qr_rows_smem_doubles<RT, kFusedThreads>() ? ob : ob + rows_per * LD;
      for (int tt = rank; tt < ntiles; tt += Gw) {
        const int mt = tt % M.tm, kb = tt / M.tm;
        const i64 r0 = static_cast<i64>(mt) * BM + static_cast<i64>(kb) * rows_per;
        const i64 r1 = min(min(static_cast<i64>(mt) * BM + BM, in), r0 + rows_per);
        if (r0 >= r1) continue;
        const int nrow = static_cast<int>(r1 - r0);
        wait_geq(M.mt_cnt + mt * kCS, static_cast<unsigned>(M.tk));
        const i64 step = in * r;
        for (int e = tid; e < nrow * r; e += kFusedThreads) {
          const int il = e / r, c = e - il * r;
          const double* p = A.part_rhs + (r0 + il) * r + c;
          rh[il * LD + c] = sum_strided(p, step, M.tk);
        }
        if (PEER && np > 1 && n < A.order - 1) {
          // every rank gets these rows' local sums (block prank of its
          // receive buffer); the counterpart CTAs of the other ranks own the
          // same rows (same tiling), and all sum the np blocks in rank order
          __syncthreads();
          for (int q = 0; q < np; ++q) {
            double* dst = A.precv[q] + static_cast<i64>(A.prank) * A.rcv_ld + r0 * r;
            for (int e = tid; e < nrow * r; e += kFusedThreads) dst[e] = rh[(e / r) * LD + e % r];
          }
          __threadfence_system();
          __syncthreads();
          const i64 slot = (static_cast<i64>(n) * A.ptiles + tt) * kCS;
          if (tid < np) red_release_sys(A.prcnt[tid] + slot, 1u);
          peer_wait(A.prcnt[A.prank] + slot, static_cast<unsigned>(np) * seq, A.perr);
          const double* src = A.precv[A.prank] + r0 * r;
          for (int e = tid; e < nrow * r; e += kFusedThreads) {
            const int il = e / r, c = e - il * r;
            double sum = 0.0;
            for (int q = 0; q < np; ++q) sum += __ldcv(src + q * A.rcv_ld + e);
            rh[il * LD + c] = sum;
          }
        }
        if (!have_ginv) {
          wait_geq(M.grdy + (rank % kRep) * kCS, 1u);
          for (int e = tid; e < r * r; e += kFusedThreads) {
            const int x = e / r, y = e - x * r;
            gi[x * LD + y] = __ldcg(A.ginv + e);
          }
          have_ginv = true;
          qr = A.qrws && __ldcg(A.info + 2) != 0;
        }
        __syncthreads();
        if (qr) {  // QR mode: the rows from the sampled fibers (qr.cuh), times ginv = I
          constexpr int BQ = kFusedThreads / RT;
          for (int ch = 0; ch < nrow; ch += BQ)
            qr_rows_cold<RT>(qs, A.qrws, r, in, r0 + ch, min(BQ, nrow - ch), rh + ch * LD, LD, qstage);
        }
        for (int e = tid; e < nrow * r; e += kFusedThreads) {
          const int il = e / r, c = e - il * r;
          double o = 0.0;
          for (int cc = 0; cc < r; ++cc) o = fma(rh[il * LD + cc], gi[cc * LD + c], o);
          CPB_DCHECK(r0 + il < in && c < r, "apply: factor row");
          if (PEER && np > 1 && n == A.order - 1) {  // slab rows into every rank's factor
            for (int q = 0; q < np; ++q) A.pfac[q][(A.slab_off + r0 + il) * r + c] = o;
          } else {
            M.a[(r0 + il) * r + c] = o;
          }
          ob[il * LD + c] = o;
        }
        __syncthreads();
        if (tid < r)
          for (int il = 0; il < nrow; ++il) q2 += ob[il * LD + tid] * ob[il * LD + tid];
        __syncthreads();
      }
      stamp(n, 4);
      if (PEER && np > 1 && n == A.order - 1) {
        if (tid < r)
          for (int q = 0; q < np; ++q) A.pssq[q][(static_cast<i64>(A.prank) * Gw + rank) * r + tid] = q2;
        __threadfence_system();
        __syncthreads();
        if (tid < np * kRep) red_release_sys(A.pdone[tid / kRep] + (tid % kRep) * kCS, 1u);
      } else {
        if (tid < r) A.ssq[static_cast<i64>(ssq_buf(A, n)) * G * r + static_cast<i64>(rank) * r + tid] = q2;
        signal_add_rep(M.adone, 1u, kRep);
      }
      stamp(n, 5);
    }
    stamp(n, 6);
  }
  if (A.next) prefetch_tables(*A.next, b);
  {  // norms of the last mode (the next launch's Z_S and the fit need them)
    const FusedMode& Lm = A.mode[A.order - 1];
    if (is_inv && !PEER && A.lazy_last) {
      // the next launch (or fused_finish) forms them; this CTA need not wait
      if constexpr (GA)  // the last mode's buffer, for the next launch
        for (int e = tid; e < RT * RT; e += kFusedThreads) A.gsum[((A.order - 1) & 1) * RT * RT + e] = 0.0;
      if (tid == 0) *A.npend = 1;
    } else if (is_inv) {
      if (PEER && np > 1)
        peer_wait(Lm.adone + (b % kRep) * kCS, A.lastw * seq, A.perr);
      else
        wait_geq(Lm.adone + (b % kRep) * kCS, seq * Gw);
      if constexpr (GA)  // the last mode's buffer, for the next launch
        for (int e = tid; e < RT * RT; e += kFusedThreads) A.gsum[((A.order - 1) & 1) * RT * RT + e] = 0.0;
      form_norms(A.order - 1);
    }
    if (A.has_fit && !is_inv) wait_geq(Lm.nready + (b % kRep) * kCS, seq);
  }
  // debug stamps of the tail (slot 14 of modes 0..2: norms seen, fit block, fit final)
  if (A.phase_t && b == 0 && tid == 0) A.phase_t[14] = globaltimer();
  // ---- sampled fit + stop rule (sampling.hpp:191-210, :237-251)
  if (A.has_fit) {
    const FitArgs& f = A.fit;
    const i64 nvb = (f.phat + 255) / 256;
    double* red = fsm;
    for (i64 vb = b; vb < nvb; vb += G) {
      const double part = ph::fit_block(f, vb, red);
      if (tid == 0) f.partials[vb] = part;
    }
    if (A.phase_t && b == 0 && tid == 0 && A.order > 1) A.phase_t[16 + 14] = globaltimer();
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = (atomicAdd(&A.ticket[1], 1u) == G - 1u);
    __syncthreads();
    if (s_last) {  // the last CTA: every partial is written
      __threadfence();
      if (tid == 0) A.ticket[1] = 0u;
      ph::fit_final(f, nvb, red);
      if (A.phase_t && A.order > 2 && tid == 0) A.phase_t[32 + 14] = globaltimer();
    }
  }
}

template <int RT, bool GA>
__global__ void __launch_bounds__(kFusedThreads, 2) fused_rand_kernel(const FusedIter* __restrict__ args) {
  rand_body<RT, GA, false>(args, gridDim.x, blockIdx.x);
}
// the peer path: L.groups rank groups of gridDim.x / L.groups CTAs
template <int RT>
__global__ void __launch_bounds__(kFusedThreads, 2) peer_rand_kernel(const FusedLaunch L) {
  const unsigned G = gridDim.x / static_cast<unsigned>(L.groups);
  const unsigned grp = blockIdx.x / G;
  const FusedIter* ap = L.a[0];
#pragma unroll
  for (int q = 1; q < kMaxPeer; ++q)  // unrolled selects (a dynamic index would go through local memory)
    if (static_cast<int>(grp) == q) ap = L.a[q];
  rand_body<RT, false, true>(ap, G, blockIdx.x - grp * G);
}

// lazy_last: the last launch's last-mode norms, before the host reads the
// model (one CTA; the same norms_final call as the persistent kernel's)
template <int RT>
__global__ void __launch_bounds__(kFusedThreads) fused_finish_kernel(const FusedIter* __restrict__ args) {
  const FusedIter& A = *args;
  if (!*reinterpret_cast<volatile int*>(A.npend)) return;
  __shared__ double red[(kFusedThreads / RT) * (RT + 1)];
  const int m = A.order - 1;
  const FusedMode& Q = A.mode[m];
  const int gw = A.grid - 1 - (A.idle_cta >= 0 ? 1 : 0);
  ModeWork wq = work_of(A, Q);
  wq.ssq = A.ssq + static_cast<i64>(ssq_buf(A, m)) * A.grid * A.r;
  ph::norms_final<RT, kFusedThreads>(A.r, Q.in_full, wq, gw, m == 0, A.rng, red, nullptr, A.mode[m - 1].norms);
  tl::signal_add_rep(Q.nready, 1u, kRep);
  if (threadIdx.x == 0) *A.npend = 0;
}

template <int RT>
void* mix_fn(bool peer = false) {
  return peer ? reinterpret_cast<void*>(&peer_mix_kernel<RT>) : reinterpret_cast<void*>(&fused_iteration_kernel<RT, true>);
}
template <int RT>
void* rand_fn(bool ga, bool peer = false) {
  if (peer) return reinterpret_cast<void*>(&peer_rand_kernel<RT>);
  return ga ? reinterpret_cast<void*>(&fused_rand_kernel<RT, true>)
            : reinterpret_cast<void*>(&fused_rand_kernel<RT, false>);
}

void* pick(int rt, bool mix, bool ga = false, bool peer = false) {
  switch (rt) {
    case 16: return mix ? mix_fn<16>(peer) : rand_fn<16>(ga, peer);
    case 32: return mix ? mix_fn<32>(peer) : rand_fn<32>(ga, peer);
    default: return mix ? mix_fn<64>(peer) : rand_fn<64>(ga, peer);
  }
}

template <int RT>
size_t rand_smem_for(int zcap) {
  i64 need = tl::tile_smem_doubles<RT>(zcap);
  need = std::max<i64>(need, static_cast<i64>(RT) * (RT + 1) + 2 * static_cast<i64>(tl::BM) * (RT + 1));
  need = std::max<i64>(need, 48 * RT + 256);
  need = std::max<i64>(need, static_cast<i64>(kFusedThreads / RT) * (RT + 1));
  need = std::max<i64>(need, ph::kFitSmemDoubles);
  need = std::max<i64>(need, ph::qr_factor_smem_doubles<RT>());
  return static_cast<size_t>(need) * sizeof(double);
}

}  // namespace

int fused_rand_zcap(int rt) {
  // two CTAs per SM: keep the dynamic shared memory of one CTA near 110 KB
  const i64 budget = 110 * 1024 / 8;
  const i64 sb = rt + 8;
  const i64 fixed = static_cast<i64>(tl::STAGES) * tl::BK * tl::SA + 2 * kMaxOrder * rt + 1;
  const i64 per = sb + 1 + kMaxOrder / 2;
  i64 z = (budget - fixed) / per;
  z &= ~static_cast<i64>(tl::BK - 1);
  return static_cast<int>(std::max<i64>(z, tl::BK));
}

size_t fused_rand_smem(int rt, int zcap) {
  switch (rt) {
    case 16: return rand_smem_for<16>(zcap);
    case 32: return rand_smem_for<32>(zcap);
    default: return rand_smem_for<64>(zcap);
  }
}

void fused_rand_tiles(i64 in, int s, int gw, int zcap, int* tm, int* tk, int* tklen) {
  const int m = std::max(1, ceil_div(in, tl::BM));  // an empty slab still gets one (empty) row block
  int k = std::max(1, gw / m);
  k = std::max(k, ceil_div(s, zcap));
  int len = ceil_div(s, k);
  len = std::max(32, (len + 3) / 4 * 4);
  len = std::min(len, zcap);
  k = ceil_div(s, len);
  *tm = m;
  *tk = k;
  *tklen = len;
}

size_t fused_smem_bytes(int rt, bool mix, int max_dim) {
  size_t need = static_cast<size_t>(ph::GSTAGES * ph::GBK * (ph::GBM + rt)) * sizeof(double);
  need = std::max(need, static_cast<size_t>(ph::GS * rt) * sizeof(double));
  need = std::max(need, static_cast<size_t>(rt * (rt + 1) + (kFusedThreads / rt) * (rt + 1)) * sizeof(double));
  need = std::max(need, static_cast<size_t>(16 * rt + 40) * sizeof(double));
  need = std::max(need, static_cast<size_t>(ph::kFitSmemDoubles) * sizeof(double));
  if (mix) need = std::max(need, static_cast<size_t>(2) * 16 * static_cast<size_t>(max_dim));
  // QR path: the factorization (inverse CTA) and the apply's QR staging
  const size_t qf = rt == 16 ? ph::qr_factor_smem_doubles<16>() : rt == 32 ? ph::qr_factor_smem_doubles<32>()
                                                                          : ph::qr_factor_smem_doubles<64>();
  const size_t qa = static_cast<size_t>(rt * (rt + 1) + (kFusedThreads / rt) * (rt + 1)) +
                    (rt == 16 ? ph::qr_rows_smem_doubles<16, kFusedThreads>()
                              : rt == 32 ? ph::qr_rows_smem_doubles<32, kFusedThreads>()
                                         : ph::qr_rows_smem_doubles<64, kFusedThreads>());
  need = std::max(need, std::max(qf, qa) * sizeof(double));
  return need;
}

int fused_max_grid(int rt, bool mix, size_t smem, int device) {
  int coop = 0, sms = 0;
  CPB_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, device));
  CPB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  if (!coop) return 0;
  void* fn = pick(rt, mix);
  CPB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  if (!mix)
    CPB_CUDA(cudaFuncSetAttribute(pick(rt, false, true), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
  CPB_CUDA(cudaFuncSetAttribute(pick(rt, mix, false, true), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(smem)));
  int per_sm = 0;
  CPB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kFusedThreads, smem));
  return per_sm * sms;
}

void launch_fused_iteration(const FusedIter* dev_args, int rt, bool mix, int grid, size_t smem,
                            cudaStream_t st, bool gram_atomic) {
  void* fn = pick(rt, mix, gram_atomic);
  void* params[] = {const_cast<FusedIter**>(&dev_args)};
  CPB_CUDA(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kFusedThreads), params, smem, st));
}

void launch_fused_finish(const FusedIter* dev_args, int rt, cudaStream_t st) {
  switch (rt) {
    case 16: fused_finish_kernel<16><<<1, kFusedThreads, 0, st>>>(dev_args); break;
    case 32: fused_finish_kernel<32><<<1, kFusedThreads, 0, st>>>(dev_args); break;
    default: fused_finish_kernel<64><<<1, kFusedThreads, 0, st>>>(dev_args); break;
  }
  CPB_LAUNCH_CHECK();
}

void launch_fused_peer(const FusedLaunch& l, int rt, int grid, size_t smem, cudaStream_t st, bool mix) {
  void* fn = pick(rt, mix, false, true);
  FusedLaunch lc = l;
  void* params[] = {&lc};
  CPB_CUDA(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kFusedThreads), params, smem, st));
}

}  // namespace cpb
