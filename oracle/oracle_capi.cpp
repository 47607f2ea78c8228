// TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT.
// Flat C entry points over the oracle for tests/ (ctypes) and the bench's
// CPU-baseline legs. Matrices are column-major; factor lists are arrays of
// pointers. Status: 0 ok, 2 invalid_argument/out_of_range, 3
// numerical_consistency_error, 1 anything else (message: orc_last_error()).
#include <chrono>
#include <cstring>
#include <string>

#include "cprand_oracle.hpp"

using namespace orc;

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const numerical_consistency_error& e) {
    g_err = e.what();
    return 3;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 2;
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

Shape shape_of(const std::int64_t* dims, int order) { return Shape(dims, dims + order); }

TensorD tensor_of(const double* x, const std::int64_t* dims, int order) {
  Shape s = shape_of(dims, order);
  Index p = 1;
  for (Index d : s) p *= d;
  return make_tensor<double>(s, std::vector<double>(x, x + p));
}

Matd mat_of(const double* a, Index rows, Index cols) {
  Matd m(rows, cols);
  std::memcpy(m.v.data(), a, sizeof(double) * static_cast<std::size_t>(rows * cols));
  return m;
}

void put(const Matd& m, double* out) {
  std::memcpy(out, m.v.data(), sizeof(double) * m.v.size());
}

std::vector<Matd> factors_of(const double* const* f, const std::int64_t* dims, int order, Index r) {
  std::vector<Matd> out;
  for (int n = 0; n < order; ++n) out.push_back(mat_of(f[n], dims[n], r));
  return out;
}

struct Engine {
  std::mt19937_64 g;
};

}  // namespace

extern "C" {

struct orc_options {
  std::int32_t max_iters;
  double fit_tolerance;
  std::int32_t has_fit_threshold;
  double fit_threshold;
  std::uint64_t rng_seed;
  std::int32_t init;
  std::int64_t fit_sample_count;
  std::int32_t stall_limit;
  std::int32_t transform;  // -1 = unset
  std::int32_t bench_mode;
  std::int32_t exhaustive_samples;
  std::int32_t exact_fit_trace;
};

struct orc_trace {
  std::int32_t iteration;
  double elapsed_seconds;
  double fit;
  std::int32_t fit_is_estimate;
  double best_fit_so_far;
};

struct orc_result {
  std::int32_t iterations;
  std::int32_t reason;
  double setup_seconds;
  double total_seconds;
  std::int32_t trace_len;
};

const char* orc_last_error() { return g_err.c_str(); }

// ---- engines (rng.hpp) ----
void* orc_engine_new(std::uint64_t seed, std::uint64_t stream, int raw) {
  auto* e = new Engine;
  e->g = raw ? std::mt19937_64(seed) : seeded_engine(seed, stream);
  return e;
}
void orc_engine_free(void* e) { delete static_cast<Engine*>(e); }
void orc_engine_next(void* e, std::int64_t n, std::uint64_t* out) {
  for (std::int64_t i = 0; i < n; ++i) out[i] = static_cast<Engine*>(e)->g();
}
int orc_engine_uniform_int(void* e, std::int64_t a, std::int64_t b, std::int64_t n, std::int64_t* out) {
  return guarded([&] {
    std::uniform_int_distribution<Index> d(a, b);
    for (std::int64_t i = 0; i < n; ++i) out[i] = d(static_cast<Engine*>(e)->g);
  });
}
int orc_engine_uniform_real(void* e, double lo, double hi, std::int64_t n, double* out) {
  return guarded([&] {
    std::uniform_real_distribution<double> d(lo, hi);
    for (std::int64_t i = 0; i < n; ++i) out[i] = d(static_cast<Engine*>(e)->g);
  });
}
int orc_engine_normal(void* e, std::int64_t n, double* out) {
  return guarded([&] {
    std::normal_distribution<double> d(0.0, 1.0);
    for (std::int64_t i = 0; i < n; ++i) out[i] = d(static_cast<Engine*>(e)->g);
  });
}
int orc_engine_bernoulli(void* e, double p, std::int64_t n, std::int32_t* out) {
  return guarded([&] {
    std::bernoulli_distribution d(p);
    for (std::int64_t i = 0; i < n; ++i) out[i] = d(static_cast<Engine*>(e)->g) ? 1 : 0;
  });
}

// ---- tensor.hpp / sampling.hpp ----
std::int64_t orc_default_sample_count(std::int64_t r) {
  try {
    return default_sample_count(r);
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

int orc_unfold_column_index(std::int64_t mode, const std::int64_t* idx, const std::int64_t* dims,
                            int order, std::int64_t* out) {
  return guarded([&] { *out = unfold_column_index(mode, idx, shape_of(dims, order)); });
}

int orc_draw_samples(void* e, const std::int64_t* dims, int order, std::int64_t mode,
                     std::int64_t count, std::int64_t* out) {
  return guarded([&] {
    SampleSet s = draw_samples(shape_of(dims, order), mode, count, static_cast<Engine*>(e)->g);
    std::memcpy(out, s.idxs.v.data(), sizeof(Index) * s.idxs.v.size());
  });
}

int orc_exhaustive_samples(const std::int64_t* dims, int order, std::int64_t mode, std::int64_t* out) {
  return guarded([&] {
    SampleSet s = exhaustive_samples(shape_of(dims, order), mode);
    std::memcpy(out, s.idxs.v.data(), sizeof(Index) * s.idxs.v.size());
  });
}

int orc_gather_fibers(const double* x, const std::int64_t* dims, int order, std::int64_t mode,
                      const std::int64_t* idxs, std::int64_t s, std::int64_t ncols, double* out) {
  return guarded([&] {
    TensorD t = tensor_of(x, dims, order);
    IndexTable tab(s, ncols);
    std::memcpy(tab.v.data(), idxs, sizeof(Index) * tab.v.size());
    put(gather_fibers(t, mode, tab), out);
  });
}

int orc_skr(const std::int64_t* idxs, std::int64_t s, const std::int64_t* dims, int order,
            std::int64_t mode, std::int64_t r, const double* const* factors, double* out) {
  return guarded([&] {
    SampleSet ss;
    ss.mode = mode;
    ss.idxs = IndexTable(s, order - 1);
    std::memcpy(ss.idxs.v.data(), idxs, sizeof(Index) * ss.idxs.v.size());
    put(skr(ss, factors_of(factors, dims, order, r), mode), out);
  });
}

int orc_least_squares(const double* a, std::int64_t m, std::int64_t n, const double* b,
                      std::int64_t k, double* out, int* rank) {
  return guarded([&] { put(least_squares(mat_of(a, m, n), mat_of(b, m, k), rank), out); });
}

int orc_sampled_update(const double* zs, const double* xs, std::int64_t s, std::int64_t r,
                       std::int64_t in, std::int64_t xs_cols, double* out) {
  return guarded([&] { put(sampled_update(mat_of(zs, s, r), mat_of(xs, in, xs_cols)), out); });
}

int orc_normalize_columns(double* const* factors, const std::int64_t* dims, int order,
                          std::int64_t r, double* lambda, std::int64_t mode, int first, void* e) {
  return guarded([&] {
    KruskalModel m;
    m.lambda.assign(lambda, lambda + r);
    for (int n = 0; n < order; ++n) m.factors.push_back(mat_of(factors[n], dims[n], r));
    normalize_columns(m, mode, first != 0, static_cast<Engine*>(e)->g);
    put(m.factors[static_cast<std::size_t>(mode)], factors[mode]);
    std::memcpy(lambda, m.lambda.data(), sizeof(double) * static_cast<std::size_t>(r));
  });
}

double orc_stable_norm(const double* v, std::int64_t n) { return stable_norm(v, n); }

int orc_fit_offsets(std::int64_t total, std::int64_t want, void* e, std::int64_t* out,
                    std::int64_t* count) {
  return guarded([&] {
    auto offs = sample_offsets_without_replacement(total, want, static_cast<Engine*>(e)->g);
    std::memcpy(out, offs.data(), sizeof(Index) * offs.size());
    *count = static_cast<std::int64_t>(offs.size());
  });
}

int orc_make_fit_estimator(const double* x, const std::int64_t* dims, int order,
                           std::int64_t count, int stall, void* e, std::int64_t* idxs_out,
                           double* vals_out, std::int64_t* n_out, double* norm_out) {
  return guarded([&] {
    TensorD t = tensor_of(x, dims, order);
    FitEstimator est = make_fit_estimator(t, count, stall, static_cast<Engine*>(e)->g);
    std::memcpy(idxs_out, est.idxs.v.data(), sizeof(Index) * est.idxs.v.size());
    std::memcpy(vals_out, est.x_values.data(), sizeof(double) * est.x_values.size());
    *n_out = est.sample_count();
    *norm_out = est.x_norm;
  });
}

int orc_estimate_fit(const double* lambda, const double* const* factors, const std::int64_t* dims,
                     int order, std::int64_t r, const std::int64_t* idxs, const double* vals,
                     std::int64_t phat, double x_norm, std::int64_t total, double* out) {
  return guarded([&] {
    KruskalModel m;
    m.lambda.assign(lambda, lambda + r);
    m.factors = factors_of(factors, dims, order, r);
    FitEstimator est;
    est.idxs = IndexTable(phat, order);
    std::memcpy(est.idxs.v.data(), idxs, sizeof(Index) * est.idxs.v.size());
    est.x_values.assign(vals, vals + phat);
    est.x_norm = x_norm;
    est.total_count = total;
    *out = estimate_fit(m, est);
  });
}

int orc_exact_fit(const double* x, const std::int64_t* dims, int order, const double* lambda,
                  const double* const* factors, std::int64_t r, double* out) {
  return guarded([&] {
    KruskalModel m;
    m.lambda.assign(lambda, lambda + r);
    m.factors = factors_of(factors, dims, order, r);
    *out = exact_fit(tensor_of(x, dims, order), m);
  });
}

double orc_tensor_norm(const double* x, const std::int64_t* dims, int order) {
  return tensor_norm(tensor_of(x, dims, order));
}

// should_stop on a caller-held estimator state (best, stall).
int orc_should_stop(double* best_fit, int* stall_count, int stall_limit, double fit, int iteration,
                    int max_iters, int has_thr, double thr, int* stop, int* reason) {
  return guarded([&] {
    FitEstimator est;
    est.best_fit = *best_fit;
    est.stall_count = *stall_count;
    est.stall_limit = stall_limit;
    SolveOptions o;
    o.max_iters = max_iters;
    if (has_thr) o.fit_threshold = thr;
    StopDecision d = should_stop(est, fit, iteration, o);
    *best_fit = est.best_fit;
    *stall_count = est.stall_count;
    *stop = d.stop;
    *reason = static_cast<int>(d.reason);
  });
}

int orc_init_random(const std::int64_t* dims, int order, std::int64_t r, std::uint64_t seed,
                    double* lambda, double* const* factors) {
  return guarded([&] {
    KruskalModel m = init_random(shape_of(dims, order), r, seed);
    std::memcpy(lambda, m.lambda.data(), sizeof(double) * static_cast<std::size_t>(r));
    for (int n = 0; n < order; ++n) put(m.factors[static_cast<std::size_t>(n)], factors[n]);
  });
}

// ---- solvers ----
int orc_solve(int method, const double* x, const std::int64_t* dims, int order, std::int64_t r,
              std::int64_t s, const orc_options* o, const double* init_lambda,
              const double* const* init_factors, double* out_lambda, double* const* out_factors,
              orc_trace* trace, int trace_cap, orc_result* res) {
  return guarded([&] {
    SolveOptions opts;
    opts.max_iters = o->max_iters;
    opts.fit_tolerance = o->fit_tolerance;
    if (o->has_fit_threshold) opts.fit_threshold = o->fit_threshold;
    opts.rng_seed = o->rng_seed;
    opts.init = static_cast<InitKind>(o->init);
    opts.fit_sample_count = o->fit_sample_count;
    opts.stall_limit = o->stall_limit;
    if (o->transform >= 0) opts.transform = static_cast<TransformKind>(o->transform);
    opts.bench_mode = o->bench_mode != 0;
    opts.exhaustive_samples = o->exhaustive_samples != 0;
    opts.exact_fit_trace = o->exact_fit_trace != 0;
    if (init_factors) {
      KruskalModel m;
      m.lambda.assign(init_lambda, init_lambda + r);
      m.factors = factors_of(init_factors, dims, order, r);
      opts.init_model = m;
    }
    const TensorD t = tensor_of(x, dims, order);
    SolveResult sr;
    switch (method) {
      case 0: sr = cp_als(t, r, opts); break;
      case 1: sr = cprand(t, r, s, opts); break;
      case 2: sr = cprand_mix(t, r, s, opts); break;
      case 3: sr = cprand_premix(t, r, s, opts); break;
      default: throw std::invalid_argument("unknown method");
    }
    std::memcpy(out_lambda, sr.model.lambda.data(), sizeof(double) * static_cast<std::size_t>(r));
    for (int n = 0; n < order; ++n) put(sr.model.factors[static_cast<std::size_t>(n)], out_factors[n]);
    const int len = static_cast<int>(sr.trace.size());
    for (int i = 0; i < len && i < trace_cap; ++i)
      trace[i] = {sr.trace[static_cast<std::size_t>(i)].iteration, sr.trace[static_cast<std::size_t>(i)].elapsed_seconds,
                  sr.trace[static_cast<std::size_t>(i)].fit, sr.trace[static_cast<std::size_t>(i)].fit_is_estimate ? 1 : 0,
                  sr.trace[static_cast<std::size_t>(i)].best_fit_so_far};
    res->iterations = sr.iterations;
    res->reason = static_cast<int>(sr.reason);
    res->setup_seconds = sr.setup_seconds;
    res->total_seconds = sr.total_seconds;
    res->trace_len = len;
  });
}

// ---- mixing ----
int orc_mixing_signs(const std::int64_t* dims, int order, int kind, std::uint64_t seed, double* out) {
  return guarded([&] {
    MixingOperator op = make_mixing_operator(shape_of(dims, order), static_cast<TransformKind>(kind), seed);
    for (const auto& s : op.signs) {
      std::memcpy(out, s.data(), sizeof(double) * s.size());
      out += s.size();
    }
  });
}

int orc_mix_tensor(const double* x, const std::int64_t* dims, int order, int kind,
                   std::uint64_t seed, double* out_re, double* out_im) {
  return guarded([&] {
    const TensorD t = tensor_of(x, dims, order);
    MixingOperator op = make_mixing_operator(t.dims, static_cast<TransformKind>(kind), seed);
    if (out_im == nullptr) {
      TensorD y = mix_tensor_real(t, op);
      std::memcpy(out_re, y.values.data(), sizeof(double) * y.values.size());
    } else {
      TensorCd y = mix_tensor_complex(t, op);
      for (std::size_t i = 0; i < y.values.size(); ++i) {
        out_re[i] = y.values[i].real();
        out_im[i] = y.values[i].imag();
      }
    }
  });
}

int orc_mix_factor(const double* a, std::int64_t rows, std::int64_t r, const std::int64_t* dims,
                   int order, int kind, std::uint64_t seed, std::int64_t mode, double* out_re,
                   double* out_im) {
  return guarded([&] {
    MixingOperator op = make_mixing_operator(shape_of(dims, order), static_cast<TransformKind>(kind), seed);
    const Matd am = mat_of(a, rows, r);
    if (out_im == nullptr) {
      put(mix_factor<double>(am, op, mode), out_re);
    } else {
      Matcd y = mix_factor<Complex>(am, op, mode);
      for (std::size_t i = 0; i < y.v.size(); ++i) {
        out_re[i] = y.v[i].real();
        out_im[i] = y.v[i].imag();
      }
    }
  });
}

int orc_unmix_factor(const double* a_re, const double* a_im, std::int64_t rows, std::int64_t r,
                     const std::int64_t* dims, int order, int kind, std::uint64_t seed,
                     std::int64_t mode, double* out) {
  return guarded([&] {
    MixingOperator op = make_mixing_operator(shape_of(dims, order), static_cast<TransformKind>(kind), seed);
    if (a_im == nullptr) {
      put(unmix_factor<double>(mat_of(a_re, rows, r), op, mode), out);
    } else {
      Matcd c(rows, r);
      for (std::size_t i = 0; i < c.v.size(); ++i) c.v[i] = Complex(a_re[i], a_im[i]);
      put(unmix_factor<Complex>(c, op, mode), out);
    }
  });
}

int orc_unmix_sampled_rhs(const double* g_re, const double* g_im, std::int64_t s, std::int64_t in,
                          const std::int64_t* dims, int order, int kind, std::uint64_t seed,
                          std::int64_t mode, double* out_re, double* out_im) {
  return guarded([&] {
    MixingOperator op = make_mixing_operator(shape_of(dims, order), static_cast<TransformKind>(kind), seed);
    if (g_im == nullptr) {
      put(unmix_sampled_rhs<double>(mat_of(g_re, s, in), op, mode), out_re);
    } else {
      Matcd c(s, in);
      for (std::size_t i = 0; i < c.v.size(); ++i) c.v[i] = Complex(g_re[i], g_im[i]);
      Matcd y = unmix_sampled_rhs<Complex>(c, op, mode);
      for (std::size_t i = 0; i < y.v.size(); ++i) {
        out_re[i] = y.v[i].real();
        out_im[i] = y.v[i].imag();
      }
    }
  });
}

int orc_transform(int kind, int forward, double* re, double* im, std::int64_t n) {
  return guarded([&] {
    if (kind == 1) {
      forward ? dct_forward(re, n) : dct_adjoint(re, n);
    } else if (kind == 2) {
      wht_forward(re, n);
    } else if (kind == 0) {
      std::vector<Complex> z(static_cast<std::size_t>(n));
      for (Index i = 0; i < n; ++i) z[static_cast<std::size_t>(i)] = Complex(re[i], im[i]);
      forward ? fft_forward(z.data(), n) : fft_backward(z.data(), n);
      for (Index i = 0; i < n; ++i) {
        re[i] = z[static_cast<std::size_t>(i)].real();
        im[i] = z[static_cast<std::size_t>(i)].imag();
      }
    } else {
      throw std::invalid_argument("unknown transform kind");
    }
  });
}

// ---- synthetic inputs ----
int orc_gen_baseline(const std::int64_t* dims, int order, std::int64_t r, double c, double eta,
                     std::uint64_t seed, double* out_x, double* const* out_factors) {
  return guarded([&] {
    if (out_x == nullptr) {
      std::vector<Matd> f;
      baseline_factors(shape_of(dims, order), r, c, seed, f);
      for (int n = 0; n < order; ++n) put(f[static_cast<std::size_t>(n)], out_factors[n]);
      return;
    }
    BaselineSynth b = gen_baseline_problem(shape_of(dims, order), r, c, eta, seed);
    std::memcpy(out_x, b.tensor.values.data(), sizeof(double) * b.tensor.values.size());
    if (out_factors)
      for (int n = 0; n < order; ++n) put(b.truth.factors[static_cast<std::size_t>(n)], out_factors[n]);
  });
}

void orc_philox_gaussian(std::uint64_t seed, std::uint64_t counter0, std::int64_t n, double* out) {
  for (std::int64_t i = 0; i < n; ++i) out[i] = philox_gaussian(seed, counter0 + static_cast<std::uint64_t>(i));
}

int orc_gen_problem(const std::int64_t* dims, int order, std::int64_t rank, double c, double noise,
                    std::uint64_t seed, double* out_x, double* out_lambda, double* const* out_factors) {
  return guarded([&] {
    SynthProblem p = gen_problem(shape_of(dims, order), rank, c, noise, seed);
    std::memcpy(out_x, p.tensor.values.data(), sizeof(double) * p.tensor.values.size());
    std::memcpy(out_lambda, p.truth.lambda.data(), sizeof(double) * static_cast<std::size_t>(rank));
    for (int n = 0; n < order; ++n) put(p.truth.factors[static_cast<std::size_t>(n)], out_factors[n]);
  });
}

int orc_score(const double* const* fa, const double* const* fb, const std::int64_t* dims, int order,
              std::int64_t r, double* out) {
  return guarded([&] {
    KruskalModel a, b;
    a.lambda.assign(static_cast<std::size_t>(r), 1.0);
    b.lambda = a.lambda;
    a.factors = factors_of(fa, dims, order, r);
    b.factors = factors_of(fb, dims, order, r);
    *out = score(a, b);
  });
}

int orc_bench_mix_premixed(const double* x_hat, const std::int64_t* dims, int order, std::int64_t r,
                           std::int64_t s, int transform, std::uint64_t seed, int iters, double* out_seconds) {
  return guarded([&] {
    *out_seconds = bench_mix_premixed(x_hat, shape_of(dims, order), r, s, static_cast<TransformKind>(transform),
                                      seed, iters);
  });
}

}  // extern "C"
