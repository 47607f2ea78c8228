// CPRAND-MIX preprocessing pass, v3: the whole-tensor forward transform
// along one mode (mix_tensor, mixing.hpp:130-156: sign, then orthonormal
// DCT-II of every mode-n fiber, in place) as a TMA-fed pipeline.
//
// A tile is W adjacent fibers (strided modes: W * 8 contiguous bytes per row,
// n rows `st` elements apart; mode 1: W whole fibers, one contiguous run).
// Each persistent CTA (one per SM, 512 threads) keeps three tile buffers in
// shared memory: while it transforms one, the tensor-memory accelerator
// loads the next two (cp.async.bulk.tensor 3D box / cp.async.bulk 1D,
// completion on an mbarrier) and writes the previous one back
// (cp.async.bulk ... bulk_group). The threads never issue a global load or
// store: HBM sees 16 B per element per mode and the SM's issue slots go to
// the FFT.
//
// The transform runs in place in the tile buffer. The W real fibers of a
// strided tile sit row-major ([row][fiber]), so fibers 2q and 2q+1 of a row
// are one double2: the buffer already is SEQ = W/2 complex sequences
// interleaved, sequence q at stride SEQ. The first Stockham pass reads with
// Makhoul's even/odd reorder and the sign folded into its addressing; every
// pass reads its butterfly inputs into registers, barrier, writes its
// outputs over the same buffer, barrier. The epilogue (quarter-wave phase
// and the orthonormal scales, unpacking the two real fibers of a sequence)
// writes each result where the output layout wants it. Butterflies, twiddle
// tables, radix order and epilogue formulas are those of mix_pass_fwd_kernel
// (mixpass.cu), so the two kernels agree bit for bit.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>

#include "dct.cuh"
#include "devutil.cuh"

namespace cpb {

namespace {

constexpr int kTmaThreads = 512;
constexpr size_t kTmaSmemCap = 225 * 1024;

using dct::PlanArgs;

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];\n" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, int c0, int c1, int c2, const void* src) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3}], [%4];\n" ::"l"(map),
               "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(src))
               : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_store(void* dst, const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

// j / d for j * d < 2^32 with M = floor((2^32 - 1) / d) + 1
__device__ __forceinline__ int udiv(int j, unsigned M) { return static_cast<int>(__umulhi(static_cast<unsigned>(j), M)); }
__host__ __device__ constexpr unsigned umagic(int d) { return 0xffffffffu / static_cast<unsigned>(d) + 1u; }

struct TmaArgs {
  PlanArgs p;
  double* x;            // tensor (mode 1: tile t at x + t * W * n)
  const double* sign;   // D_n (nullable: identity)
  i64 tiles;            // number of tiles
  i64 tiles_lo;         // strided: tiles per slab (st / W)
  int bw;               // strided: rows per TMA box
  int nbox;             // strided: boxes per tile (n / bw)
  int U[24];            // butterflies per thread in pass s (<= 4)
  unsigned Mm[24], Mns[24];  // magics of m and ns per pass
  int ns[24];
};

// What the passes read: scalars copied out of the kernel parameters once
// (a dynamically indexed __grid_constant__ struct is copied to local memory)
// and the per-pass constants in shared memory.
struct PassCtx {
  int n;
  const double2* tw;
  const double2* phase;
  const double* sign;
  double s0, sk;
  const int* ns;        // shared [nrad]
  const unsigned* Mns;  // shared [nrad]
};

// threadIdx.x through an opaque read: the index math of every inlined radix /
// U variant would otherwise be hoisted out of the tile loop (loop invariant)
// and spill
__device__ __forceinline__ int tid_x() {
  int t;
  asm volatile("mov.u32 %0, %%tid.x;" : "=r"(t));
  return t;
}

// Makhoul's reorder, inverted: sequence position d <- fiber element e
__device__ __forceinline__ int src_elem(int d, int n) { return (d < (n + 1) / 2) ? 2 * d : 2 * (n - 1 - d) + 1; }

// first pass (ns = 1, no twiddles): inputs of butterfly (q, j) are sequence
// positions j + r m, i.e. fiber elements src_elem(.) of fibers 2q, 2q + 1,
// times the sign; outputs at positions j R + r
template <int R, int U, int SEQ, bool CONTIG>
__device__ __forceinline__ void first_pass(const PassCtx& a, double* buf) {
  const int n = a.n, m = n / R, nb = SEQ * m;
  const unsigned Ms = umagic(SEQ);
  double2* cb = reinterpret_cast<double2*>(buf);
  // every thread computes U butterflies (the surplus ones on a clamped
  // index, not stored): no divergence around values held across the barrier
  double2 v[U][R];
  int dst[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int t = tid_x() + u * kTmaThreads;
    const int tc = min(t, nb - 1);
    const int j = udiv(tc, Ms), q = tc - j * SEQ;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int e = src_elem(j + r * m, n);
      const double sg = a.sign[e];
      double2 x;
      if constexpr (CONTIG) {
        x = make_double2(buf[(2 * q) * n + e], buf[(2 * q + 1) * n + e]);
      } else {
        x = cb[e * SEQ + q];
      }
      v[u][r] = make_double2(sg * x.x, sg * x.y);
    }
    dct::dft<R>(v[u], false);
    dst[u] = t < nb ? (j * R) * SEQ + q : -1;
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < U; ++u)
    if (dst[u] >= 0)
#pragma unroll
      for (int r = 0; r < R; ++r) cb[dst[u] + r * SEQ] = v[u][r];
  __syncthreads();
}

// Stockham pass s (radix R, ns > 1) in place over the SEQ interleaved sequences
template <int R, int U, int SEQ>
__device__ __forceinline__ void mid_pass(const PassCtx& a, int s, double* buf) {
  const int n = a.n, m = n / R, ns = a.ns[s], nb = SEQ * m;
  const int step = n / (ns * R);
  const unsigned Ms = umagic(SEQ), Mns = a.Mns[s];
  double2* cb = reinterpret_cast<double2*>(buf);
  double2 v[U][R];
  int dst[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int t = tid_x() + u * kTmaThreads;
    const int tc = min(t, nb - 1);
    const int j = udiv(tc, Ms), q = tc - j * SEQ;
    const int jj = udiv(j, Mns), k = j - jj * ns;
#pragma unroll
    for (int r = 0; r < R; ++r) v[u][r] = cb[(j + r * m) * SEQ + q];
#pragma unroll
    for (int r = 1; r < R; ++r) v[u][r] = dct::cmul(v[u][r], a.tw[r * k * step]);
    dct::dft<R>(v[u], false);
    dst[u] = t < nb ? (jj * ns * R + k) * SEQ + q : -1;
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < U; ++u)
    if (dst[u] >= 0)
#pragma unroll
      for (int r = 0; r < R; ++r) cb[dst[u] + r * ns * SEQ] = v[u][r];
  __syncthreads();
}

template <int SEQ, bool CONTIG, int R, int U>
__device__ __forceinline__ void pass_ru(const PassCtx& a, int s, double* buf) {
  if (s == 0)
    first_pass<R, U, SEQ, CONTIG>(a, buf);
  else
    mid_pass<R, U, SEQ>(a, s, buf);
}

// butterflies per thread a radix-R pass may hold in registers (R * U complex)
__host__ __device__ constexpr int umax_of(int R) { return R == 8 ? 2 : (R == 5 ? 3 : 4); }

template <int SEQ, bool CONTIG, int R>
__device__ __forceinline__ void pass_r(const PassCtx& a, int s, int u, double* buf) {
  constexpr int UM = umax_of(R);
  if (u <= 1)
    pass_ru<SEQ, CONTIG, R, 1>(a, s, buf);
  else if (u == 2 || UM == 2)
    pass_ru<SEQ, CONTIG, R, (UM < 2 ? UM : 2)>(a, s, buf);
  else if (u == 3 || UM == 3)
    pass_ru<SEQ, CONTIG, R, (UM < 3 ? UM : 3)>(a, s, buf);
  else
    pass_ru<SEQ, CONTIG, R, UM>(a, s, buf);
}

// epilogue (dct::transform_group's forward formulas): X_i of fibers 2q, 2q+1
// from V_i and conj V_{n-i}; the pair (k, n - k) belongs to one thread
template <int SEQ, bool CONTIG>
__device__ __forceinline__ void epilogue(const PassCtx& a, double* buf) {
  const int n = a.n, half = n / 2 + 1;  // k = 0 .. n/2
  const unsigned Ms = umagic(SEQ);
  double2* cb = reinterpret_cast<double2*>(buf);
  constexpr int UE = 4;
  double2 o[UE][2];
  int kk[UE], qq[UE];
  auto unpack = [&](double2 z, double2 zc, int i) {
    const double2 w = a.phase[i];
    const double sc = (i == 0) ? a.s0 : a.sk;
    const double vx0 = 0.5 * (z.x + zc.x), vy0 = 0.5 * (z.y - zc.y);
    const double vx1 = 0.5 * (z.y + zc.y), vy1 = -0.5 * (z.x - zc.x);
    return make_double2(sc * (w.x * vx0 - w.y * vy0), sc * (w.x * vx1 - w.y * vy1));
  };
  for (int t0 = 0; t0 < SEQ * half; t0 += UE * kTmaThreads) {
#pragma unroll
    for (int u = 0; u < UE; ++u) {
      const int t = t0 + tid_x() + u * kTmaThreads;
      kk[u] = -1;
      if (t < SEQ * half) {
        const int k = udiv(t, Ms), q = t - k * SEQ;
        const int kc = (k == 0) ? 0 : n - k;
        const double2 z = cb[k * SEQ + q], zc = cb[kc * SEQ + q];
        o[u][0] = unpack(z, zc, k);
        o[u][1] = unpack(zc, z, kc);
        kk[u] = k;
        qq[u] = q;
      }
    }
    if constexpr (CONTIG) __syncthreads();  // the outputs overwrite other threads' inputs
#pragma unroll
    for (int u = 0; u < UE; ++u) {
      const int k = kk[u];
      if (k < 0) continue;
      const int q = qq[u], kc = (k == 0) ? 0 : n - k;
      if constexpr (CONTIG) {
        buf[(2 * q) * n + k] = o[u][0].x;
        buf[(2 * q + 1) * n + k] = o[u][0].y;
        buf[(2 * q) * n + kc] = o[u][1].x;
        buf[(2 * q + 1) * n + kc] = o[u][1].y;
      } else {
        cb[k * SEQ + q] = o[u][0];
        cb[kc * SEQ + q] = o[u][1];
      }
    }
    if constexpr (CONTIG) __syncthreads();
  }
}

template <int SEQ, bool CONTIG, int kTmaStages>
__global__ void __launch_bounds__(kTmaThreads, 1)
    mix_tma_kernel(const __grid_constant__ CUtensorMap map, const __grid_constant__ TmaArgs a) {
  constexpr int W = 2 * SEQ;
  extern __shared__ __align__(128) double tsm[];
  __shared__ __align__(8) unsigned long long full[kTmaStages];
  __shared__ int s_rad[24], s_u[24], s_ns[24];
  __shared__ unsigned s_mns[24];
  const int n = a.p.n, nrad = a.p.nrad;
  if (threadIdx.x < 24) {
    const int i = threadIdx.x;
    s_rad[i] = a.p.radix[i];
    s_u[i] = a.U[i];
    s_ns[i] = a.ns[i];
    s_mns[i] = a.Mns[i];
  }
  // twiddles, phases and signs in shared memory after the tile buffers
  double2* s_tw = reinterpret_cast<double2*>(tsm + static_cast<size_t>(kTmaStages) * 2 * SEQ * n);
  double2* s_ph = s_tw + n;
  double* s_sg = reinterpret_cast<double*>(s_ph + n);
  for (int i = threadIdx.x; i < n; i += kTmaThreads) {
    s_tw[i] = a.p.tw[i];
    s_ph[i] = a.p.phase[i];
    s_sg[i] = a.sign ? a.sign[i] : 1.0;
  }
  PassCtx ctx;
  ctx.n = n;
  ctx.tw = s_tw;
  ctx.phase = s_ph;
  ctx.sign = s_sg;
  ctx.s0 = a.p.s0;
  ctx.sk = a.p.sk;
  ctx.ns = s_ns;
  ctx.Mns = s_mns;
  double* const x = a.x;
  const i64 tiles = a.tiles, tiles_lo = a.tiles_lo;
  const int bw = a.bw, nbox = a.nbox;
  const unsigned tile_bytes = static_cast<unsigned>(W) * n * 8u;
  double* bufs[kTmaStages];
#pragma unroll
  for (int s = 0; s < kTmaStages; ++s) bufs[s] = tsm + static_cast<size_t>(s) * W * n;
  auto coords = [&](i64 t, int* c0, int* c2) {
    const i64 hi = t / tiles_lo;
    *c0 = static_cast<int>((t - hi * tiles_lo) * W);
    *c2 = static_cast<int>(hi);
  };
  auto issue_load = [&](i64 t, int s) {  // thread 0
    mbar_expect_tx(&full[s], tile_bytes);
    if constexpr (CONTIG) {
      bulk_load(bufs[s], x + t * W * n, tile_bytes, &full[s]);
    } else {
      int c0, c2;
      coords(t, &c0, &c2);
      for (int bx = 0; bx < nbox; ++bx)
        tma_load_3d(bufs[s] + static_cast<size_t>(bx) * bw * W, &map, c0, bx * bw, c2, &full[s]);
    }
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < kTmaStages; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    for (int s = 0; s < kTmaStages - 1; ++s) {
      const i64 t = blockIdx.x + static_cast<i64>(s) * gridDim.x;
      if (t < tiles) issue_load(t, s);
    }
  }
  __syncthreads();
  int it = 0;
  for (i64 t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
    const int s = it % kTmaStages;
    if (threadIdx.x == 0) {
      // the buffer of iteration it - 1 is free once its store has read it
      const i64 tn = t + static_cast<i64>(kTmaStages - 1) * gridDim.x;
      bulk_wait_read0();
      if (tn < tiles) issue_load(tn, (it + kTmaStages - 1) % kTmaStages);
    }
    mbar_wait(&full[s], static_cast<unsigned>((it / kTmaStages) & 1));
    double* buf = bufs[s];
    for (int ps = 0; ps < nrad; ++ps) {
      const int u = s_u[ps];
      switch (s_rad[ps]) {
        case 2: pass_r<SEQ, CONTIG, 2>(ctx, ps, u, buf); break;
        case 3: pass_r<SEQ, CONTIG, 3>(ctx, ps, u, buf); break;
        case 4: pass_r<SEQ, CONTIG, 4>(ctx, ps, u, buf); break;
        case 5: pass_r<SEQ, CONTIG, 5>(ctx, ps, u, buf); break;
        default: pass_r<SEQ, CONTIG, 8>(ctx, ps, u, buf); break;
      }
    }
    epilogue<SEQ, CONTIG>(ctx, buf);
    fence_async_smem();  // this thread's shared-memory writes -> the async proxy
    __syncthreads();
    if (threadIdx.x == 0) {
      if constexpr (CONTIG) {
        bulk_store(x + t * W * n, buf, tile_bytes);
      } else {
        int c0, c2;
        coords(t, &c0, &c2);
        for (int bx = 0; bx < nbox; ++bx) tma_store_3d(&map, c0, bx * bw, c2, buf + static_cast<size_t>(bx) * bw * W);
      }
      bulk_commit();
    }
  }
  if (threadIdx.x == 0) bulk_wait0();
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    cudaDriverEntryPointQueryResult q{};
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// radices (8s first, then 4, 2, 5, 3; largest first), as fwd_radices in mixpass.cu
int tma_radices(int n, int* rad) {
  int k = 0, m = n;
  while (m % 8 == 0) { rad[k++] = 8; m /= 8; }
  while (m % 4 == 0) { rad[k++] = 4; m /= 4; }
  while (m % 2 == 0) { rad[k++] = 2; m /= 2; }
  while (m % 5 == 0) { rad[k++] = 5; m /= 5; }
  while (m % 3 == 0) { rad[k++] = 3; m /= 3; }
  if (m != 1 || k > 24) return 0;
  std::sort(rad, rad + k, [](int x, int y) { return x > y; });
  return k;
}

template <int SEQ, int ST>
void* tma_fn(bool contig) {
  return contig ? reinterpret_cast<void*>(&mix_tma_kernel<SEQ, true, ST>)
                : reinterpret_cast<void*>(&mix_tma_kernel<SEQ, false, ST>);
}

void* pick_fn(int seq, bool contig, int stages) {
  const bool three = stages == 3;
  switch (seq) {
    case 4: return three ? tma_fn<4, 3>(contig) : tma_fn<4, 2>(contig);
    case 8: return three ? tma_fn<8, 3>(contig) : tma_fn<8, 2>(contig);
    case 16: return three ? tma_fn<16, 3>(contig) : tma_fn<16, 2>(contig);
    default: return three ? tma_fn<32, 3>(contig) : tma_fn<32, 2>(contig);
  }
}

}  // namespace

// Forward pass along a mode of stride st with nfib fibers of length p.n, in
// place on x. Returns false (nothing launched) when the shape does not suit
// the kernel: then the caller uses mix_pass_fwd_kernel.
bool launch_mix_tma(const DctPlan& pl, double* x, i64 st, i64 nfib, const double* sign, cudaStream_t stream,
                    bool prepare_only) {
  if (std::getenv("CPRAND_MIX_V2")) return false;
  const int n = pl.n;
  // measured (tests/micro/mix_time.py): faster than mix_pass_fwd_kernel for
  // long fibers (n = 1000: 2.14-2.32 TB/s against 1.83-2.39); for n <= 320 a
  // tile holds too few butterflies per barrier and the v2 kernel wins
  // (CPRAND_MIX_TMA=1 forces this kernel, for tests)
  if (n < 512 && !std::getenv("CPRAND_MIX_TMA")) return false;
  if (n < 8) return false;
  TmaArgs a{};
  a.p = dct_args(pl);
  int rad[24];
  const int nr = tma_radices(n, rad);
  if (nr == 0) return false;
  a.p.nrad = nr;
  for (int i = 0; i < nr; ++i) a.p.radix[i] = rad[i];
  const bool contig = (st == 1);
  // fibers per tile: the widest W = 2 SEQ whose three buffers fit and whose
  // passes need <= 4 butterflies per thread
  // widest tile with >= 2 buffers beside the tables (40 B per element of n);
  // 3 buffers when they fit
  int seq = 0, stages = 0;
  const size_t tables = static_cast<size_t>(n) * 40;
  for (int cand : {32, 16, 8, 4}) {
    const int w = 2 * cand;
    const size_t tile = static_cast<size_t>(w) * n * 8;
    stages = (3 * tile + tables <= kTmaSmemCap) ? 3 : ((2 * tile + tables <= kTmaSmemCap) ? 2 : 0);
    if (stages == 0) continue;
    if (nfib % w != 0) continue;
    if (!contig && st % w != 0) continue;
    bool ok = true;
    for (int i = 0; i < nr; ++i) ok = ok && (cand * (n / rad[i]) <= umax_of(rad[i]) * kTmaThreads);
    // mode 1: the epilogue reads every (k, n - k) pair before any write, in one chunk
    if (contig) ok = ok && (cand * (n / 2 + 1) <= 4 * kTmaThreads);
    if (!ok) continue;
    seq = cand;
    break;
  }
  if (seq == 0) return false;
  const int w = 2 * seq;
  a.x = x;
  a.sign = sign;
  a.tiles = nfib / w;
  a.tiles_lo = contig ? 1 : st / w;
  int ns = 1;
  for (int i = 0; i < nr; ++i) {
    const int m = n / rad[i];
    a.U[i] = (seq * m + kTmaThreads - 1) / kTmaThreads;
    a.ns[i] = ns;
    a.Mm[i] = umagic(m);
    a.Mns[i] = umagic(ns);
    ns *= rad[i];
  }
  CUtensorMap map{};
  if (!contig) {
    int nb = (n + 255) / 256;
    while (nb <= n && n % nb != 0) ++nb;
    a.nbox = nb;
    a.bw = n / nb;
    if (a.bw < 8) return false;
    auto enc = encode_fn();
    if (!enc) return false;
    const i64 nhi = nfib / st;
    cuuint64_t gdim[3] = {static_cast<cuuint64_t>(st), static_cast<cuuint64_t>(n), static_cast<cuuint64_t>(nhi)};
    cuuint64_t gstr[2] = {static_cast<cuuint64_t>(st) * 8, static_cast<cuuint64_t>(st) * n * 8};
    cuuint32_t box[3] = {static_cast<cuuint32_t>(w), static_cast<cuuint32_t>(a.bw), 1};
    cuuint32_t es[3] = {1, 1, 1};
    if (st > 0x7fffffffLL || nhi > 0x7fffffffLL) return false;
    const CUresult rc = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, x, gdim, gstr, box, es,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (rc != CUDA_SUCCESS) return false;
  } else {
    if ((reinterpret_cast<uintptr_t>(x) & 15) != 0) return false;
  }
  void* fn = pick_fn(seq, contig, stages);
  const size_t smem = static_cast<size_t>(stages) * w * n * 8 + tables;
  CPB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  if (prepare_only) return true;
  int dev = 0, sms = 148;
  CPB_CUDA(cudaGetDevice(&dev));
  CPB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int grid = static_cast<int>(std::min<i64>(a.tiles, sms));
  void* args[] = {&map, &a};
  CPB_CUDA(cudaLaunchKernel(fn, dim3(grid), dim3(kTmaThreads), args, smem, stream));
  return true;
}

}  // namespace cpb
