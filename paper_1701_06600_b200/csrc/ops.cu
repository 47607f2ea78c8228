// Operator-level entry points: the reference's free functions (gather_fibers,
// skr, one sampled mode update, fit values / estimate, mixing transforms)
// run through the SAME device kernels the solver loop launches, with host
// buffers in and out. They exist for teacher-forced parity tests and for
// callers that use the reference's building blocks directly.
#include <cmath>
#include <cstring>
#include <memory>
#include <vector>

#include <functional>

#include "session.hpp"

namespace cpb {

namespace {

struct DBuf {
  void* p = nullptr;
  explicit DBuf(size_t bytes) { CPB_CUDA(cudaMalloc(&p, bytes ? bytes : 1)); }
  ~DBuf() {
    if (p) cudaFree(p);
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

template <class T>
void h2d(void* d, const T* h, size_t n) {
  CPB_CUDA(cudaMemcpy(d, h, n * sizeof(T), cudaMemcpyHostToDevice));
}
template <class T>
void d2h(T* h, const void* d, size_t n) {
  CPB_CUDA(cudaMemcpy(h, d, n * sizeof(T), cudaMemcpyDeviceToHost));
}

i64 prod(const std::vector<i64>& d) {
  i64 p = 1;
  for (i64 v : d) p *= v;
  return p;
}

std::vector<i64> strides_of(const std::vector<i64>& d) {
  std::vector<i64> s;
  i64 p = 1;
  for (i64 v : d) {
    s.push_back(p);
    p *= v;
  }
  return s;
}

void check_mode(int mode, size_t order) {
  if (mode < 0 || mode >= static_cast<int>(order)) throw InvalidArgument("mode out of range");
}

// Validated int32 row tables (c-major) + int64 base offsets for a sample table.
void build_rows(const i64* idxs, i64 s, const std::vector<i64>& dims, int mode, std::vector<int>& rows,
                std::vector<i64>& base) {
  const int n = static_cast<int>(dims.size());
  const auto st = strides_of(dims);
  rows.assign(static_cast<size_t>((n - 1) * s), 0);
  base.assign(static_cast<size_t>(s), 0);
  int c = 0;
  for (int k = 0; k < n; ++k) {
    if (k == mode) continue;
    for (i64 j = 0; j < s; ++j) {
      const i64 v = idxs[j + c * s];
      if (v < 0 || v >= dims[static_cast<size_t>(k)]) throw InvalidArgument("multiindex out of range");
      rows[static_cast<size_t>(c * s + j)] = static_cast<int>(v);
      base[static_cast<size_t>(j)] += v * st[static_cast<size_t>(k)];
    }
    ++c;
  }
}

std::vector<double> row_major(const double* cm, i64 rows, int r) {
  std::vector<double> out(static_cast<size_t>(rows * r));
  for (int c = 0; c < r; ++c)
    for (i64 i = 0; i < rows; ++i) out[static_cast<size_t>(i * r + c)] = cm[i + c * rows];
  return out;
}

void require_transform(int transform) {
  if (transform == 1 || transform == 2 || transform == 3) return;
  if (transform == 0) throw Unsupported("the operator-level FFT mixing entry points are complex; use cprand_solve");
  throw InvalidArgument("unknown transform kind");
}

}  // namespace

void op_gather(const double* x, const std::vector<i64>& dims, int mode, const i64* idxs, i64 s,
               double* out) {
  check_mode(mode, dims.size());
  if (s < 0) throw InvalidArgument("sample count must be >= 0");
  const i64 p = prod(dims);
  std::vector<int> rows;
  std::vector<i64> base;
  build_rows(idxs, s, dims, mode, rows, base);
  DBuf dx(p * sizeof(double)), db(s * sizeof(i64)), dout(s * dims[static_cast<size_t>(mode)] * sizeof(double));
  h2d(dx.p, x, static_cast<size_t>(p));
  h2d(db.p, base.data(), base.size());
  launch_gather_fibers(dx.as<double>(), dims[static_cast<size_t>(mode)], strides_of(dims)[static_cast<size_t>(mode)],
                       db.as<i64>(), static_cast<int>(s), dout.as<double>(), nullptr);
  d2h(out, dout.p, static_cast<size_t>(s * dims[static_cast<size_t>(mode)]));
}

void op_skr(const i64* idxs, i64 s, const std::vector<i64>& dims, int mode, int r,
            const double* const* factors, double* out) {
  check_mode(mode, dims.size());
  const int n = static_cast<int>(dims.size());
  std::vector<int> rows;
  std::vector<i64> base;
  build_rows(idxs, s, dims, mode, rows, base);
  std::vector<std::unique_ptr<DBuf>> facs;
  DBuf drows(rows.size() * sizeof(int)), dout(static_cast<size_t>(s * r) * sizeof(double));
  h2d(drows.p, rows.data(), rows.size());
  ModeView v{};
  v.s = static_cast<int>(s);
  v.r = r;
  v.kept = n - 1;
  int c = 0;
  for (int k = 0; k < n; ++k) {
    if (k == mode) continue;
    const i64 rr = dims[static_cast<size_t>(k)];
    auto rm = row_major(factors[k], rr, r);
    facs.push_back(std::make_unique<DBuf>(rm.size() * sizeof(double)));
    h2d(facs.back()->p, rm.data(), rm.size());
    v.fac[c] = facs.back()->as<double>();
    v.rows[c] = drows.as<int>() + static_cast<i64>(c) * s;
    ++c;
  }
  launch_skr(v, dout.as<double>(), nullptr);
  d2h(out, dout.p, static_cast<size_t>(s * r));
}

int op_mode_update(const double* x, const std::vector<i64>& dims, int mode, const i64* idxs, i64 s,
                   int r, const double* const* factors, double* lambda, int first, int transform,
                   std::uint64_t mix_seed, double* out_factor) {
  check_mode(mode, dims.size());
  if (s < r) throw InvalidArgument("sampled_update: need at least R samples");
  if (r < 1 || r > kMaxFusedRank) throw Unsupported("rank outside 1..64");
  const bool mix = transform == 1;
  if (transform >= 0) require_transform(transform);
  const int n = static_cast<int>(dims.size());
  const i64 p = prod(dims);
  const auto st = strides_of(dims);
  const i64 in = dims[static_cast<size_t>(mode)];
  std::vector<int> rows;
  std::vector<i64> base;
  build_rows(idxs, s, dims, mode, rows, base);
  cudaStream_t stream = nullptr;
  DBuf dx(p * sizeof(double)), drows(rows.size() * sizeof(int)), dbase(base.size() * sizeof(i64));
  h2d(dx.p, x, static_cast<size_t>(p));
  h2d(drows.p, rows.data(), rows.size());
  h2d(dbase.p, base.data(), base.size());
  int dev = 0, sms = 148;
  CPB_CUDA(cudaGetDevice(&dev));
  CPB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  std::vector<std::vector<double>> signs;
  std::vector<DctPlan> plans;
  std::vector<std::unique_ptr<DBuf>> facs, dsigns;
  if (mix) {
    signs = mixing_signs(dims, transform, mix_seed);
    for (int k = 0; k < n; ++k) {
      plans.push_back(make_mix_plan(transform, static_cast<int>(dims[static_cast<size_t>(k)])));
      dsigns.push_back(std::make_unique<DBuf>(signs[static_cast<size_t>(k)].size() * sizeof(double)));
      h2d(dsigns.back()->p, signs[static_cast<size_t>(k)].data(), signs[static_cast<size_t>(k)].size());
    }
  }
  ModeView v{};
  v.x = dx.as<double>();
  v.in = in;
  v.stride = st[static_cast<size_t>(mode)];
  v.s = static_cast<int>(s);
  v.r = r;
  v.kept = n - 1;
  v.base = dbase.as<i64>();
  int c = 0;
  for (int k = 0; k < n; ++k) {
    if (k == mode) continue;
    const i64 rr = dims[static_cast<size_t>(k)];
    auto rm = row_major(factors[k], rr, r);
    facs.push_back(std::make_unique<DBuf>(rm.size() * sizeof(double)));
    h2d(facs.back()->p, rm.data(), rm.size());
    if (mix)  // Z uses the mixed factors F D A (mixing.hpp:286-289)
      launch_mode_transform(plans[static_cast<size_t>(k)], facs.back()->as<double>(), facs.back()->as<double>(), r, r,
                            dsigns[static_cast<size_t>(k)]->as<double>(), 1, nullptr, stream);
    v.fac[c] = facs.back()->as<double>();
    v.rows[c] = drows.as<int>() + static_cast<i64>(c) * s;
    ++c;
  }
  int ks, len;
  const int rt = rank_bucket(r);
  mode_splits(in, static_cast<int>(s), rt, &ks, &len, sms);
  int gp, glen;
  gram_splits(static_cast<int>(s), &gp, &glen);
  const i64 ld = (in + 1) & ~i64{1};
  DBuf prhs(static_cast<size_t>(ks) * in * r * sizeof(double)), pgram(static_cast<size_t>(gp) * rt * rt * sizeof(double));
  DBuf ginv(static_cast<size_t>(r * r) * sizeof(double)), info(4 * sizeof(int)), tickets(8 * sizeof(unsigned));
  DBuf gfull(static_cast<size_t>(gram_scratch_doubles(r)) * sizeof(double));
  DBuf ssq(static_cast<size_t>(apply_grid(in, r)) * r * sizeof(double)), norms(r * sizeof(double));
  DBuf dlam(r * sizeof(double)), da(static_cast<size_t>(in * r) * sizeof(double)), rng(313 * sizeof(unsigned long long));
  DBuf rhs(static_cast<size_t>(in * r) * sizeof(double)), dz(static_cast<size_t>(s * rt) * sizeof(double));
  DBuf xs(static_cast<size_t>(s * ld + 2) * sizeof(double));
  CPB_CUDA(cudaMemset(tickets.p, 0, 8 * sizeof(unsigned)));
  h2d(dlam.p, lambda, static_cast<size_t>(r));
  launch_rng_seed(rng.as<unsigned long long>(), 0ULL, stream);
  ModeWork w{};
  w.z = dz.as<double>();
  w.part_gram = pgram.as<double>();
  w.gram_parts = gp;
  w.part_rhs = prhs.as<double>();
  w.ginv = ginv.as<double>();
  w.gfull = gfull.as<double>();
  w.info = info.as<int>();
  w.ticket = tickets.as<unsigned>();
  w.ssq = ssq.as<double>();
  w.norms = norms.as<double>();
  w.lambda = dlam.as<double>();
  w.a = da.as<double>();
  w.stop = nullptr;
  w.ks = ks;
  w.ks_len = len;
  // normal equations while every Gauss-Jordan pivot > kNeTol * d_max, else
  // the QR path with the reference's rank threshold (qr.cuh)
  DBuf qrws(static_cast<size_t>(qr_ws_doubles(static_cast<int>(s), rt)) * sizeof(double));
  w.qtol = static_cast<double>(std::max<i64>(s, r)) * 2.220446049250313e-16;
  w.tol = kNeTol;
  w.qrws = qrws.as<double>();
  w.q = QrSrc{xs.as<double>(), nullptr, ld, 1, static_cast<int>(s)};
  launch_gather_rows(v.x, in, v.stride, v.base, static_cast<int>(s), xs.as<double>(), ld, stream);
  launch_z(v, w.z, nullptr, stream);
  launch_gram(w.z, static_cast<int>(s), r, w.part_gram, nullptr, stream);
  launch_gram_inverse(w.part_gram, gp, r, w.tol, w.ginv, w.gfull, w.info, nullptr, stream, w.z,
                      static_cast<int>(s), w.qtol, w.qrws);
  launch_rhs_gemm(xs.as<double>(), ld, nullptr, true, w.z, in, static_cast<int>(s), r, ks, len, w.part_rhs, nullptr,
                  stream);
  const double* rhsp = nullptr;
  if (mix) {
    launch_reduce_rhs_qr(w, in, r, rhs.as<double>(), stream);
    launch_mode_transform(plans[static_cast<size_t>(mode)], rhs.as<double>(), rhs.as<double>(), r, r,
                          dsigns[static_cast<size_t>(mode)]->as<double>(), 0, nullptr, stream);
    rhsp = rhs.as<double>();
  }
  launch_mode_apply(in, r, w, rhsp, first, rng.as<unsigned long long>(), stream);
  CPB_CUDA(cudaDeviceSynchronize());
  std::vector<double> rm(static_cast<size_t>(in * r)), nv(static_cast<size_t>(r));
  d2h(rm.data(), da.p, rm.size());
  d2h(nv.data(), norms.p, nv.size());
  // normalized factor = A_un / norm (kruskal.hpp:65)
  for (int q = 0; q < r; ++q)
    for (i64 i = 0; i < in; ++i) out_factor[i + q * in] = rm[static_cast<size_t>(i * r + q)] / nv[static_cast<size_t>(q)];
  d2h(lambda, dlam.p, static_cast<size_t>(r));
  int k = 0;
  d2h(&k, info.p, 1);
  for (auto& pl : plans) free_dct_plan(pl);
  return k;
}

void op_fit_values(const double* x, i64 p, const i64* offsets, i64 n, double* out, double* norm) {
  for (i64 j = 0; j < n; ++j)
    if (offsets[j] < 0 || offsets[j] >= p) throw InvalidArgument("offset out of range");
  DBuf dx(p * sizeof(double)), doff(n * sizeof(i64)), dv(n * sizeof(double)), part(2048 * sizeof(double));
  h2d(dx.p, x, static_cast<size_t>(p));
  h2d(doff.p, offsets, static_cast<size_t>(n));
  launch_gather_values(dx.as<double>(), doff.as<i64>(), n, dv.as<double>(), nullptr);
  launch_sumsq(dx.as<double>(), p, part.as<double>(), 1024, part.as<double>() + 1024, nullptr);
  d2h(out, dv.p, static_cast<size_t>(n));
  double ss = 0.0;
  d2h(&ss, part.as<double>() + 1024, 1);
  if (norm) *norm = std::sqrt(ss);
}

double op_estimate_fit(const double* lambda, const double* const* factors,
                       const std::vector<i64>& dims, int r, const i64* idxs, const double* values,
                       i64 phat, double x_norm, i64 total) {
  const int n = static_cast<int>(dims.size());
  if (n > kMaxOrder) throw Unsupported("order > 8");
  if (phat < 1) throw InvalidArgument("fit sample count must be >= 1");
  std::vector<std::unique_ptr<DBuf>> facs, idx;
  FitArgs a{};
  a.order = n;
  a.r = r;
  a.phat = phat;
  for (int k = 0; k < n; ++k) {
    auto rm = row_major(factors[k], dims[static_cast<size_t>(k)], r);
    facs.push_back(std::make_unique<DBuf>(rm.size() * sizeof(double)));
    h2d(facs.back()->p, rm.data(), rm.size());
    std::vector<int> col(static_cast<size_t>(phat));
    for (i64 j = 0; j < phat; ++j) {
      const i64 v = idxs[j + k * phat];
      if (v < 0 || v >= dims[static_cast<size_t>(k)]) throw InvalidArgument("multiindex out of range");
      col[static_cast<size_t>(j)] = static_cast<int>(v);
    }
    idx.push_back(std::make_unique<DBuf>(col.size() * sizeof(int)));
    h2d(idx.back()->p, col.data(), col.size());
    a.fac[k] = facs.back()->as<double>();
    a.idx[k] = idx.back()->as<int>();
  }
  DBuf dl(r * sizeof(double)), dv(phat * sizeof(double)), part((phat / 256 + 2) * sizeof(double));
  DBuf tk(4 * sizeof(unsigned)), st(sizeof(FitState)), tr(sizeof(TraceRec));
  h2d(dl.p, lambda, static_cast<size_t>(r));
  h2d(dv.p, values, static_cast<size_t>(phat));
  CPB_CUDA(cudaMemset(tk.p, 0, 4 * sizeof(unsigned)));
  FitState fs{};
  fs.best_fit = -INFINITY;
  CPB_CUDA(cudaMemcpy(st.p, &fs, sizeof(fs), cudaMemcpyHostToDevice));
  a.lambda = dl.as<double>();
  a.values = dv.as<double>();
  a.x_norm = x_norm;
  a.total = static_cast<double>(total);
  a.partials = part.as<double>();
  a.ticket = tk.as<unsigned>();
  a.state = st.as<FitState>();
  a.trace = tr.as<TraceRec>();
  a.iteration = 1;
  a.max_iters = 1 << 30;
  a.stall_limit = 1 << 30;
  launch_estimate_fit(a, nullptr);
  TraceRec rec{};
  d2h(&rec, tr.p, 1);
  return rec.fit;
}

void op_transform_tensor(const double* x, const std::vector<i64>& dims, int transform,
                         std::uint64_t seed, double* out) {
  require_transform(transform);
  const i64 p = prod(dims);
  const auto st = strides_of(dims);
  if (transform == 3) {
    std::memcpy(out, x, sizeof(double) * p);
    return;
  }
  auto signs = mixing_signs(dims, transform, seed);
  DBuf dx(p * sizeof(double));
  h2d(dx.p, x, static_cast<size_t>(p));
  for (size_t m = 0; m < dims.size(); ++m) {
    DctPlan pl = make_mix_plan(transform, static_cast<int>(dims[m]));
    DBuf ds(signs[m].size() * sizeof(double));
    h2d(ds.p, signs[m].data(), signs[m].size());
    launch_mode_transform(pl, dx.as<double>(), dx.as<double>(), st[m], p / dims[m], ds.as<double>(), 1, nullptr,
                          nullptr);
    CPB_CUDA(cudaDeviceSynchronize());
    free_dct_plan(pl);
  }
  d2h(out, dx.p, static_cast<size_t>(p));
}

void op_transform_factor(const double* a, i64 rows, int r, const std::vector<i64>& dims,
                         int transform, std::uint64_t seed, int mode, int forward, double* out) {
  check_mode(mode, dims.size());
  require_transform(transform);
  if (rows != dims[static_cast<size_t>(mode)])
    throw InvalidArgument(forward ? "mix_factor: row mismatch" : "unmix_factor: row mismatch");
  if (transform == 3) {
    std::memcpy(out, a, sizeof(double) * rows * r);
    return;
  }
  auto signs = mixing_signs(dims, transform, seed);
  DctPlan pl = make_mix_plan(transform, static_cast<int>(rows));
  DBuf da(static_cast<size_t>(rows * r) * sizeof(double)), ds(rows * sizeof(double));
  h2d(da.p, a, static_cast<size_t>(rows * r));
  h2d(ds.p, signs[static_cast<size_t>(mode)].data(), static_cast<size_t>(rows));
  // column-major: column q is a contiguous fiber
  launch_mode_transform(pl, da.as<double>(), da.as<double>(), 1, r, ds.as<double>(), forward, nullptr, nullptr);
  CPB_CUDA(cudaDeviceSynchronize());
  free_dct_plan(pl);
  d2h(out, da.p, static_cast<size_t>(rows * r));
}

void op_unmix_rows(const double* g, i64 s, i64 in, const std::vector<i64>& dims, int transform,
                   std::uint64_t seed, int mode, double* out) {
  check_mode(mode, dims.size());
  require_transform(transform);
  if (in != dims[static_cast<size_t>(mode)])
    throw InvalidArgument("unmix_sampled_rhs: row-slice length mismatch");
  if (transform == 3) {
    std::memcpy(out, g, sizeof(double) * s * in);
    return;
  }
  auto signs = mixing_signs(dims, transform, seed);
  DctPlan pl = make_mix_plan(transform, static_cast<int>(in));
  DBuf dg(static_cast<size_t>(s * in) * sizeof(double)), ds(in * sizeof(double));
  h2d(dg.p, g, static_cast<size_t>(s * in));
  h2d(ds.p, signs[static_cast<size_t>(mode)].data(), static_cast<size_t>(in));
  // S x I_n column-major: row j is a fiber with stride S
  launch_mode_transform(pl, dg.as<double>(), dg.as<double>(), s, s, ds.as<double>(), 0, nullptr, nullptr);
  CPB_CUDA(cudaDeviceSynchronize());
  free_dct_plan(pl);
  d2h(out, dg.p, static_cast<size_t>(s * in));
}

// mix_tensor (mixing.hpp:130-156) in place on a device tensor: per mode,
// sign then orthonormal DCT-II; ms[mode] = CUDA-event time of that pass.
void op_tensor_mix(Tensor* t, int transform, std::uint64_t seed, double* ms, int mode_begin, int mode_end) {
  if (transform != 1 && transform != 2) throw Unsupported("in-place device mixing supports the dct and wht transforms");
  const int order = static_cast<int>(t->dims.size());
  if (mode_end < 0) mode_end = order;
  if (mode_begin < 0 || mode_begin > mode_end || mode_end > order) throw InvalidArgument("mode range out of bounds");
  CPB_CUDA(cudaSetDevice(t->device));
  // every mode's signs are drawn in order from one stream (mixing.hpp:34-40),
  // so a sub-range of the passes uses the same signs as the whole pass
  const auto signs = mixing_signs(t->dims, transform, seed);
  cudaEvent_t e0, e1;
  CPB_CUDA(cudaEventCreate(&e0));
  CPB_CUDA(cudaEventCreate(&e1));
  for (size_t n = static_cast<size_t>(mode_begin); n < static_cast<size_t>(mode_end); ++n) {
    DBuf sg(signs[n].size() * sizeof(double));
    h2d(sg.p, signs[n].data(), signs[n].size());
    DctPlan plan = make_mix_plan(transform, static_cast<int>(t->dims[n]));
    prepare_mode_transform(plan, t->strides[n], t->p / t->dims[n], 1);
    CPB_CUDA(cudaDeviceSynchronize());
    CPB_CUDA(cudaEventRecord(e0, nullptr));
    launch_mode_transform(plan, t->d, t->d, t->strides[n], t->p / t->dims[n], sg.as<double>(), 1, nullptr, nullptr);
    CPB_CUDA(cudaEventRecord(e1, nullptr));
    CPB_CUDA(cudaEventSynchronize(e1));
    float f = 0.f;
    CPB_CUDA(cudaEventElapsedTime(&f, e0, e1));
    if (ms) ms[n] = f;
    free_dct_plan(plan);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
}

void op_read_fibers(const Tensor* t, int mode, const i64* idxs, i64 s, double* out) {
  // plain strided copies (no kernel): an independent read path for checking
  // the device tensor against the oracle at sizes too large to download
  const int order = static_cast<int>(t->dims.size());
  if (mode < 0 || mode >= order) throw InvalidArgument("mode out of range");
  CPB_CUDA(cudaSetDevice(t->device));
  const i64 in = t->dims[static_cast<size_t>(mode)], st = t->strides[static_cast<size_t>(mode)];
  for (i64 j = 0; j < s; ++j) {
    i64 base = 0;
    for (int c = 0, k = 0; k < order; ++k) {
      if (k == mode) continue;
      const i64 v = idxs[j + static_cast<i64>(c) * s];
      if (v < 0 || v >= t->dims[static_cast<size_t>(k)]) throw InvalidArgument("sample index out of range");
      base += v * t->strides[static_cast<size_t>(k)];
      ++c;
    }
    CPB_CUDA(cudaMemcpy2D(out + j * in, sizeof(double), t->d + base, static_cast<size_t>(st) * sizeof(double),
                          sizeof(double), static_cast<size_t>(in), cudaMemcpyDeviceToHost));
  }
}

void op_debug_normals(std::uint64_t seed, int n, double* out) {
  DBuf st(313 * sizeof(unsigned long long)), d(static_cast<size_t>(n) * sizeof(double));
  launch_rng_seed(st.as<unsigned long long>(), seeded_engine_seed_value(seed, kInitStream + 7), nullptr);
  launch_rng_normals(st.as<unsigned long long>(), n, d.as<double>(), nullptr);
  d2h(out, d.p, static_cast<size_t>(n));
}

void op_synth(Tensor* t, int r, double c, double eta, std::uint64_t seed,
              double* const* out_factors, i64 last_off, i64 global_last,
              const std::function<void(double*)>& reduce_sums) {
  std::vector<i64> gdims = t->dims;
  if (global_last > 0) gdims.back() = global_last;
  std::vector<std::vector<double>> f;
  baseline_factors_host(gdims, r, c, seed, f);
  CPB_CUDA(cudaSetDevice(t->device));
  std::vector<std::unique_ptr<DBuf>> facs;
  std::vector<const double*> ptrs;
  for (size_t n = 0; n < t->dims.size(); ++n) {
    auto rm = row_major(f[n].data(), gdims[n], r);
    facs.push_back(std::make_unique<DBuf>(rm.size() * sizeof(double)));
    h2d(facs.back()->p, rm.data(), rm.size());
    ptrs.push_back(facs.back()->as<double>());
    if (out_factors) std::memcpy(out_factors[n], f[n].data(), f[n].size() * sizeof(double));
  }
  DBuf scratch((2 * 4096 + 8) * sizeof(double));
  launch_synth(t->d, static_cast<int>(t->dims.size()), t->dims.data(), r, ptrs.data(), eta, seed,
               scratch.as<double>(), nullptr, last_off, global_last, reduce_sums);
  CPB_CUDA(cudaDeviceSynchronize());
}

}  // namespace cpb
