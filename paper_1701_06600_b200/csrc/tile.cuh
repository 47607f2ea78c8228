// Tile-level device functions of the CPRAND (non-MIX) persistent kernel:
// one CTA owns a (64-row block, sample split) tile of the mode-n update.
//
//   z_tile        Z_S rows of the split into shared memory   sampling.hpp:74-92
//   gram_blocks   8 x 8 blocks of the split's Gram Z^T Z      kr_linalg.hpp:105 (normal eqs.)
//   gemm_tile     split-K RHS  X_(n)[rows, S_split] Z_split  (fibers read in place)
//
// The contractions use the FP64 MMA (mma.sync m8n8k4 .f64): one instruction
// is 256 FMAs, so the FP64 pipe stays fed with a few warps per SM and the
// shared-memory traffic per FMA is 4-8x lower than a DFMA register tile.
// Shared-memory rows are padded to 8 (mod 16) doubles so every fragment load
// is two conflict-free wavefronts.
#pragma once

#include "devutil.cuh"
#include "kernels.cuh"

namespace cpb {
namespace tl {

constexpr int NT = 256;      // threads per CTA
constexpr int BM = 64;       // tensor rows (mode-n indices) per tile
constexpr int BK = 16;       // samples per pipeline stage
constexpr int STAGES = 3;
constexpr int SA = BM + 8;   // A stage row stride (doubles)
template <int RT>
struct Cfg {
  static constexpr int SB = RT + 8;               // Z row stride (doubles)
  static constexpr int NFR = RT / 8;              // 8-wide column fragments
  static constexpr int WN = NFR >= 4 ? 4 : NFR;   // warps along the columns
  static constexpr int WM = 8 / WN;               // warps along the rows
  static constexpr int MF = BM / 8 / WM;          // row fragments per warp
  static constexpr int NFW = NFR / WN;            // column fragments per warp
};

// Shared-memory carve-up of one tile (doubles): A stages, Z rows, row
// offsets, per-kept-mode row indices, norms and their reciprocals.
struct TileSmem {
  double* as;
  double* zs;
  i64* roff;
  int* rows;
  double* nr;
  double* yr;
};
template <int RT>
__host__ __device__ constexpr i64 tile_smem_doubles(int zcap) {
  return static_cast<i64>(STAGES) * BK * SA + static_cast<i64>(zcap) * Cfg<RT>::SB + zcap +
         (static_cast<i64>(kMaxOrder) * zcap + 1) / 2 + 2 * kMaxOrder * RT;
}
template <int RT>
__device__ __forceinline__ TileSmem tile_smem(double* base, int zcap) {
  TileSmem t;
  t.as = base;
  t.zs = t.as + STAGES * BK * SA;
  t.roff = reinterpret_cast<i64*>(t.zs + zcap * Cfg<RT>::SB);
  t.rows = reinterpret_cast<int*>(t.roff + zcap);
  t.nr = reinterpret_cast<double*>(t.rows) + (kMaxOrder * zcap + 1) / 2;
  t.yr = t.nr + kMaxOrder * RT;
  return t;
}

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// a / n, correctly rounded, given y = RN(1/n): q = RN(a y), r = a - q n
// (exact by FMA), RN(q + r y) (Markstein). Outside the range where the
// correction step is proven (and for zeros, to keep the sign) it falls back
// to IEEE division, so the value is always the one `a / n` produces.
__device__ __forceinline__ double div_rn(double a, double n, double y) {
  const double q = a * y;
  const double aa = fabs(a), an = fabs(n);
  if (!(aa < 0x1p900 && aa > 0x1p-900 && an < 0x1p900 && an > 0x1p-900)) return a / n;
  const double r = fma(-q, n, a);
  return fma(r, y, q);
}

// Acquire load / release add for the flag protocol between CTAs.
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Whole CTA: returns after *p >= target was observed (thread 0 polls).
// Relaxed load for polling: an acquire load invalidates the SM's L1 on every
// poll (stalling the co-resident CTA's loads); poll relaxed, then one fence.
__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void wait_geq(const unsigned* p, unsigned target, unsigned sleep_ns = 0) {
  if (threadIdx.x == 0) {
    // sleep_ns == 0: spin (the hand-offs on the critical path; measured C4
    // 8.88 k -> 8.95 k it/s against a 32-64 ns nanosleep between polls);
    // otherwise back off between polls
    if (sleep_ns) {
      while (ld_relaxed(p) < target) __nanosleep(sleep_ns);
    } else {
#ifdef CPB_DEVICE_CHECKS
      const unsigned long long t0 = globaltimer();
      while (ld_relaxed(p) < target) CPB_DCHECK(globaltimer() - t0 < 5000000000ull, "flag wait > 5 s");
#else
      while (ld_relaxed(p) < target) {
      }
#endif
    }
    asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
  }
  __syncthreads();
}
// Whole CTA: publishes this CTA's prior writes (release), then adds v to *p
// without waiting for a reply.
__device__ __forceinline__ void signal_add(unsigned* p, unsigned v) {
  __syncthreads();
  if (threadIdx.x == 0) asm volatile("red.release.gpu.global.add.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
// Whole CTA: release-add v to nrep replicas p[0], p[kCS], ... (a flag that
// many CTAs poll is replicated over cache lines so the polling spreads over
// L2 slices); poll replica (CTA % nrep).
__device__ __forceinline__ void signal_add_rep(unsigned* p, unsigned v, int nrep) {
  __syncthreads();
  if (static_cast<int>(threadIdx.x) < nrep)
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;\n" ::"l"(p + threadIdx.x * kCS), "r"(v) : "memory");
}
// Whole CTA: publishes this CTA's prior writes, then adds v to *p.
__device__ __forceinline__ unsigned release_add(unsigned* p, unsigned v, unsigned* sh_old) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    *sh_old = atomicAdd(p, v);
  }
  __syncthreads();
  return *sh_old;
}

// Z_S rows [s0, s0 + cnt) of mode view v into t.zs (kpad rows, zero padded),
// the fibers' row offsets into t.roff. Factors and norms were written by
// other CTAs earlier in this launch: read through L2 (ld.global.cg). A warp
// forms whole Z rows (lanes over the R columns: coalesced factor-row reads),
// U rows per pass with every kept mode's loads in flight together.
template <int RT, int KEPT>
__device__ void z_rows(const ModeView& v, int cnt, int kpad, const TileSmem& t) {
  constexpr int SB = Cfg<RT>::SB;
  constexpr int CPL = RT >= 32 ? RT / 32 : 1;
  constexpr int U = KEPT <= 2 ? 8 : 4;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int r = v.r;
  for (int base = warp; base < kpad; base += 8 * U) {
    double av[KEPT][U][CPL];
#pragma unroll
    for (int c = 0; c < KEPT; ++c)
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int sl = base + 8 * u;
        const bool okr = sl < cnt;
        const i64 row = okr ? static_cast<i64>(t.rows[c * kpad + sl]) : 0;
        CPB_DCHECK(!okr || v.kdim[c] == 0 || (row >= 0 && row < v.kdim[c]), "z_rows: sampled row");
#pragma unroll
        for (int j = 0; j < CPL; ++j) {
          const int rr = lane + 32 * j;
          av[c][u][j] = (okr && rr < r) ? __ldcg(v.fac[c] + row * r + rr) : 0.0;
        }
      }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int sl = base + 8 * u;
      if (sl >= kpad) break;
#pragma unroll
      for (int j = 0; j < CPL; ++j) {
        const int rr = lane + 32 * j;
        if (rr >= RT) continue;
        double zv = 0.0;
        if (sl < cnt && rr < r) {
          zv = 1.0;
#pragma unroll
          for (int c = 0; c < KEPT; ++c) {
            double a = av[c][u][j];
            if (v.nrm[c]) a = div_rn(a, t.nr[c * RT + rr], t.yr[c * RT + rr]);
            zv = __dmul_rn(zv, a);
          }
        }
        t.zs[sl * SB + rr] = zv;
      }
    }
  }
}

template <int RT>
__device__ void z_tile(const ModeView& v, int s0, int cnt, int kpad, const TileSmem& t) {
  constexpr int SB = Cfg<RT>::SB;
  const int tid = threadIdx.x;
  for (int e = tid; e < cnt; e += NT) t.roff[e] = __ldg(v.base + s0 + e);
  for (int e = tid; e < v.kept * cnt; e += NT) {
    const int c = e / cnt, sl = e - c * cnt;
    t.rows[c * kpad + sl] = __ldg(v.rows[c] + s0 + sl);
  }
  for (int e = tid; e < v.kept * RT; e += NT) {
    const int c = e / RT, rr = e - c * RT;
    const double nv = (v.nrm[c] && rr < v.r) ? __ldcg(v.nrm[c] + rr) : 1.0;
    t.nr[e] = nv;
    t.yr[e] = __drcp_rn(nv);
  }
  __syncthreads();
  switch (v.kept) {
    case 1: z_rows<RT, 1>(v, cnt, kpad, t); break;
    case 2: z_rows<RT, 2>(v, cnt, kpad, t); break;
    case 3: z_rows<RT, 3>(v, cnt, kpad, t); break;
    default:
      for (int e = tid; e < kpad * RT; e += NT) {
        const int sl = e / RT, rr = e - sl * RT;
        double zv = 0.0;
        if (sl < cnt && rr < v.r) {
          zv = 1.0;
          for (int c = 0; c < v.kept; ++c) {
            double a = __ldcg(v.fac[c] + static_cast<i64>(t.rows[c * kpad + sl]) * v.r + rr);
            if (v.nrm[c]) a = div_rn(a, t.nr[c * RT + rr], t.yr[c * RT + rr]);
            zv = __dmul_rn(zv, a);
          }
        }
        t.zs[sl * SB + rr] = zv;
      }
  }
  __syncthreads();
}

// Z_S rows [z0, z1) of mode view v into z (global, [S][RT], zero-padded
// columns): one warp per row, lanes over the columns; the row indices and
// the norms are loaded together, then the factor rows. Each entry is the
// reference's left fold over the kept modes, factor entries divided by the
// column norm exactly as the reference stores A (col /= norm).
template <int RT, int KEPT>
__device__ void z_rows_global(const ModeView& v, int z0, int z1, double* __restrict__ z) {
  constexpr int CPL = RT >= 32 ? RT / 32 : 1;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int r = v.r;
  double nr[KEPT][CPL];
#pragma unroll
  for (int c = 0; c < KEPT; ++c)
#pragma unroll
    for (int j = 0; j < CPL; ++j) {
      const int rr = lane + 32 * j;
      nr[c][j] = (v.nrm[c] && rr < r) ? __ldcg(v.nrm[c] + rr) : 1.0;
    }
  for (int s = z0 + warp; s < z1; s += 8) {
    int row[KEPT];
#pragma unroll
    for (int c = 0; c < KEPT; ++c) {
      row[c] = __ldg(v.rows[c] + s);
      CPB_DCHECK(v.kdim[c] == 0 || (row[c] >= 0 && row[c] < v.kdim[c]), "z_rows_global: sampled row");
    }
    double av[KEPT][CPL];
#pragma unroll
    for (int c = 0; c < KEPT; ++c)
#pragma unroll
      for (int j = 0; j < CPL; ++j) {
        const int rr = lane + 32 * j;
        av[c][j] = rr < r ? __ldcg(v.fac[c] + static_cast<i64>(row[c]) * r + rr) : 0.0;
      }
#pragma unroll
    for (int j = 0; j < CPL; ++j) {
      const int rr = lane + 32 * j;
      if (rr >= RT) continue;
      double zv = 0.0;
      if (rr < r) {
        zv = 1.0;
#pragma unroll
        for (int c = 0; c < KEPT; ++c) zv = __dmul_rn(zv, v.nrm[c] ? av[c][j] / nr[c][j] : av[c][j]);
      }
      z[static_cast<i64>(s) * RT + rr] = zv;
    }
  }
}

template <int RT>
__device__ void z_share(const ModeView& v, int z0, int z1, double* __restrict__ z) {
  switch (v.kept) {
    case 1: z_rows_global<RT, 1>(v, z0, z1, z); break;
    case 2: z_rows_global<RT, 2>(v, z0, z1, z); break;
    case 3: z_rows_global<RT, 3>(v, z0, z1, z); break;
    case 4: z_rows_global<RT, 4>(v, z0, z1, z); break;
    case 5: z_rows_global<RT, 5>(v, z0, z1, z); break;
    case 6: z_rows_global<RT, 6>(v, z0, z1, z); break;
    default: z_rows_global<RT, 7>(v, z0, z1, z); break;
  }
}

// The split's Z rows [s0, s0 + cnt) from global into t.zs (kpad rows, zero
// padded) and the fibers' row offsets into t.roff.
template <int RT>
__device__ void z_load(const ModeView& v, const double* __restrict__ z, int s0, int cnt, int kpad,
                       const TileSmem& t) {
  constexpr int SB = Cfg<RT>::SB;
  const int tid = threadIdx.x;
  for (int e = tid; e < cnt; e += NT) t.roff[e] = __ldg(v.base + s0 + e);
  for (int e = tid; e < kpad * (RT / 2); e += NT) {
    const int sl = e / (RT / 2), c2 = (e - sl * (RT / 2)) * 2;
    double2 val = make_double2(0.0, 0.0);
    if (sl < cnt) val = __ldcg(reinterpret_cast<const double2*>(z + static_cast<i64>(s0 + sl) * RT + c2));
    *reinterpret_cast<double2*>(t.zs + sl * SB + c2) = val;
  }
  __syncthreads();
}

// Upper-triangular 8 x 8 block q of the Gram (bi <= bj) in row-major block order.
__device__ __forceinline__ void gram_block_coords(int q, int nfr, int* bi, int* bj) {
  int i = 0, rem = q;
  while (rem >= nfr - i) {
    rem -= nfr - i;
    ++i;
  }
  *bi = i;
  *bj = i + rem;
}

// Blocks q = first, first + step, ... of this split's Gram, one warp per
// block: gpart[(q * ks + kb) * 64 + 8 m + n] = sum_k Z(k, 8 bi + m) Z(k, 8 bj + n).
template <int RT>
__device__ void gram_blocks(const TileSmem& t, int kpad, int nfr, int first, int step, int kb, int ks,
                            double* __restrict__ gpart) {
  constexpr int SB = Cfg<RT>::SB;
  const int nblk = nfr * (nfr + 1) / 2;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int q = first + warp * step; q < nblk; q += 8 * step) {
    int bi, bj;
    gram_block_coords(q, nfr, &bi, &bj);
    // four independent accumulator chains (kpad is a multiple of BK = 16): a
    // dependent FP64 MMA issues only every ~100 cycles, and one warp owns
    // the whole k range of its block
    double acc[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
    const double* za = t.zs + (lane & 3) * SB + bi * 8 + (lane >> 2);
    const double* zb = t.zs + (lane & 3) * SB + bj * 8 + (lane >> 2);
    for (int k = 0; k < kpad; k += 16) {
#pragma unroll
      for (int u = 0; u < 4; ++u) dmma(acc[u], za[(k + 4 * u) * SB], zb[(k + 4 * u) * SB]);
    }
    double* o = gpart + (static_cast<i64>(q) * ks + kb) * 64 + (lane >> 2) * 8 + (lane & 3) * 2;
    o[0] = (acc[0][0] + acc[1][0]) + (acc[2][0] + acc[3][0]);
    o[1] = (acc[0][1] + acc[1][1]) + (acc[2][1] + acc[3][1]);
  }
}

// The same blocks added straight into the summed Gram g (both triangles,
// ld RT) with fire-and-forget L2 fp64 adds: no split partials, no reducer.
// The order of the adds is not fixed, so the Gram (and the run) is not
// bitwise reproducible; the two triangles may differ in the last bit.
template <int RT>
__device__ void gram_blocks_add(const TileSmem& t, int kpad, int nfr, int first, int step,
                                double* __restrict__ g) {
  constexpr int SB = Cfg<RT>::SB;
  const int nblk = nfr * (nfr + 1) / 2;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int q = first + warp * step; q < nblk; q += 8 * step) {
    int bi, bj;
    gram_block_coords(q, nfr, &bi, &bj);
    double acc[2] = {0.0, 0.0};
    const double* za = t.zs + (lane & 3) * SB + bi * 8 + (lane >> 2);
    const double* zb = t.zs + (lane & 3) * SB + bj * 8 + (lane >> 2);
#pragma unroll 4
    for (int k = 0; k < kpad; k += 4) dmma(acc, za[k * SB], zb[k * SB]);
    const int gi = bi * 8 + (lane >> 2), gj = bj * 8 + (lane & 3) * 2;
    atomicAdd(g + gi * RT + gj, acc[0]);
    atomicAdd(g + gi * RT + gj + 1, acc[1]);
    if (bi != bj) {  // and the mirrored block (the inverse reads whole rows)
      atomicAdd(g + gj * RT + gi, acc[0]);
      atomicAdd(g + (gj + 1) * RT + gi, acc[1]);
    }
  }
}

// Split-K RHS tile: out(i, c) = sum_{s < cnt} X(roff[s] + i) Z(s, c) for the
// 64 rows i0.. of a mode with `in` rows; out = part + kb * in * r, row-major
// (ld r). A (fibers) streams through a 3-stage cp.async pipeline; Z stays
// resident in shared memory.
template <int RT>
__device__ void gemm_tile(const double* __restrict__ x, bool vec16, i64 in, i64 i0, int r, int cnt,
                          int kpad, const TileSmem& t, double* __restrict__ out, i64 xsize = 0) {
#ifndef CPB_DEVICE_CHECKS
  (void)xsize;
#else
  if (xsize == 0) xsize = i64{1} << 62;
#endif
  using C = Cfg<RT>;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const int wm = warp / C::WN, wn = warp % C::WN;
  const int nstage = kpad / BK;
  auto load = [&](int st, int buf) {
    double* ab = t.as + buf * BK * SA;
    const int sb = st * BK;
    if (vec16) {
#pragma unroll
      for (int q = 0; q < BK * BM / 2 / NT; ++q) {
        const int c = tid + q * NT;
        const int sl = c / (BM / 2), ic = (c % (BM / 2)) * 2;
        const int s = sb + sl;
        const i64 i = i0 + ic;
        const bool ok = (s < cnt) && (i < in);
        const int bytes = !ok ? 0 : (i + 1 < in ? 16 : 8);
        CPB_DCHECK(!ok || (t.roff[s] >= 0 && t.roff[s] + i + bytes / 8 <= xsize), "gemm_tile: fiber read");
        cp_async16(ab + sl * SA + ic, ok ? x + t.roff[s] + i : x, bytes);
      }
    } else {
#pragma unroll
      for (int q = 0; q < BK * BM / NT; ++q) {
        const int c = tid + q * NT;
        const int sl = c / BM, ic = c % BM;
        const int s = sb + sl;
        const i64 i = i0 + ic;
        const bool ok = (s < cnt) && (i < in);
        CPB_DCHECK(!ok || (t.roff[s] >= 0 && t.roff[s] + i < xsize), "gemm_tile: fiber read");
        cp_async8(ab + sl * SA + ic, ok ? x + t.roff[s] + i : x, ok ? 8 : 0);
      }
    }
  };
  double acc[C::MF][C::NFW][2];
#pragma unroll
  for (int a = 0; a < C::MF; ++a)
#pragma unroll
    for (int b = 0; b < C::NFW; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  bool live[C::NFW];
#pragma unroll
  for (int b = 0; b < C::NFW; ++b) live[b] = (wn * C::NFW + b) * 8 < r;
#pragma unroll
  for (int st = 0; st < STAGES - 1; ++st) {
    if (st < nstage) load(st, st);
    cp_async_commit();
  }
  const int arow = wm * C::MF * 8 + (lane >> 2);
  const int bcol = wn * C::NFW * 8 + (lane >> 2);
  for (int st = 0; st < nstage; ++st) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    const int nx = st + STAGES - 1;
    if (nx < nstage) load(nx, nx % STAGES);
    cp_async_commit();
    const double* ab = t.as + (st % STAGES) * BK * SA + (lane & 3) * SA + arow;
    const double* zb = t.zs + (st * BK + (lane & 3)) * C::SB + bcol;
#pragma unroll
    for (int k = 0; k < BK; k += 4) {
      double af[C::MF], bf[C::NFW];
#pragma unroll
      for (int a = 0; a < C::MF; ++a) af[a] = ab[k * SA + a * 8];
#pragma unroll
      for (int b = 0; b < C::NFW; ++b) bf[b] = zb[k * C::SB + b * 8];
#pragma unroll
      for (int b = 0; b < C::NFW; ++b)
        if (live[b])
#pragma unroll
          for (int a = 0; a < C::MF; ++a) dmma(acc[a][b], af[a], bf[b]);
    }
  }
  cp_async_wait<0>();
  __syncthreads();
#pragma unroll
  for (int a = 0; a < C::MF; ++a) {
    const i64 i = i0 + arow + a * 8;
    if (i >= in) continue;
#pragma unroll
    for (int b = 0; b < C::NFW; ++b) {
      const int c = bcol - (lane >> 2) + b * 8 + (lane & 3) * 2;
      if (c < r) out[i * r + c] = acc[a][b][0];
      if (c + 1 < r) out[i * r + c + 1] = acc[a][b][1];
    }
  }
}

}  // namespace tl
}  // namespace cpb
