// cprand_b200/cprand.hpp — C++ drop-in for the reference's randomized entry
// points, backed by the B200 C ABI (include/cprand_b200.h).
//
// Swap `#include <cprand/cprand.hpp>` for this header and link
// libcprand_b200.so: the calls below keep the reference's names, argument
// meaning and exception types (/root/reference/proj/include/cprand/):
//   cprand::cprand(x, r, s, opts)          sampling.hpp:257
//   cprand::cprand_mix(x, r, s, opts)      mixing.hpp:340
//   cprand::cprand_premix(x, r, s, opts)   mixing.hpp:372
//   cprand::default_sample_count(r)        sampling.hpp:18
//   SolveOptions / SolveResult / TraceRecord / StopReason  solver.hpp:40-90
// The value types are Eigen-free and layout-compatible with the reference's
// (column-major factors, generalized column-major tensors), so a caller that
// holds Eigen objects can map them without copies.
#pragma once

#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "../cprand_b200.h"

namespace cprand {

using Index = std::int64_t;
using Shape = std::vector<Index>;

class numerical_consistency_error : public std::runtime_error {  // types.hpp:37-41
 public:
  explicit numerical_consistency_error(const std::string& w) : std::runtime_error(w) {}
};
class device_error : public std::runtime_error {
 public:
  explicit device_error(const std::string& w) : std::runtime_error(w) {}
};

// Column-major matrix (Eigen's default storage).
struct Matd {
  Index rows = 0, cols = 0;
  std::vector<double> v;
  Matd() = default;
  Matd(Index r, Index c) : rows(r), cols(c), v(static_cast<size_t>(r * c), 0.0) {}
  double& operator()(Index i, Index j) { return v[static_cast<size_t>(i + j * rows)]; }
  double operator()(Index i, Index j) const { return v[static_cast<size_t>(i + j * rows)]; }
  const double* data() const { return v.data(); }
  double* data() { return v.data(); }
};

// DenseTensor<double> (tensor.hpp:17-78): mode-1 fastest storage.
struct TensorD {
  Shape dims;
  std::vector<double> values;
  TensorD(Shape d, std::vector<double> vals) : dims(std::move(d)), values(std::move(vals)) {
    if (dims.empty()) throw std::invalid_argument("tensor order must be >= 1");
    Index p = 1;
    for (Index x : dims) {
      if (x < 1) throw std::invalid_argument("tensor dims must be >= 1");
      p *= x;
    }
    if (p != static_cast<Index>(values.size())) throw std::invalid_argument("value count does not match dims");
  }
  Index order() const { return static_cast<Index>(dims.size()); }
  Index size() const { return static_cast<Index>(values.size()); }
};

struct KruskalModel {  // kruskal.hpp:16-34
  std::vector<double> lambda;
  std::vector<Matd> factors;
  Index order() const { return static_cast<Index>(factors.size()); }
  Index rank() const { return static_cast<Index>(lambda.size()); }
};

enum class InitKind { random = CPRAND_INIT_RANDOM, hosvd = CPRAND_INIT_HOSVD, given = CPRAND_INIT_GIVEN };
enum class TransformKind {
  fft = CPRAND_TRANSFORM_FFT, dct = CPRAND_TRANSFORM_DCT, wht = CPRAND_TRANSFORM_WHT,
  identity = CPRAND_TRANSFORM_IDENTITY
};
enum class StopReason {
  max_iterations, fit_stagnation, fit_threshold, best_fit_stall, zero_tensor, bench_complete
};

struct SolveOptions {  // solver.hpp:40-64
  int max_iters = 200;
  double fit_tolerance = 1e-4;
  std::optional<double> fit_threshold;
  std::uint64_t rng_seed = 0;
  InitKind init = InitKind::random;
  std::optional<KruskalModel> init_model;
  Index fit_sample_count = Index{1} << 14;
  int stall_limit = 10;
  std::optional<TransformKind> transform;
  bool bench_mode = false;
  bool exhaustive_samples = false;
  bool exact_fit_trace = false;
  int device = -1;  // B200 extension: CUDA ordinal (-1 = current)
};

struct TraceRecord {
  int iteration;
  double elapsed_seconds;
  double fit;
  bool fit_is_estimate;
  double best_fit_so_far;
};

struct SolveResult {
  KruskalModel model;
  std::vector<TraceRecord> trace;
  int iterations = 0;
  StopReason reason = StopReason::max_iterations;
  double setup_seconds = 0.0;
  double total_seconds = 0.0;
};

namespace detail {

inline void throw_status(int st) {
  if (st == CPRAND_OK) return;
  const std::string msg = cprand_last_error();
  switch (st) {
    case CPRAND_ERR_INVALID: throw std::invalid_argument(msg);
    case CPRAND_ERR_NUMERICAL: throw numerical_consistency_error(msg);
    default: throw device_error(msg);
  }
}

inline SolveResult run(int method, const TensorD& x, Index r, Index s, const SolveOptions& o) {
  cprand_options_t c;
  cprand_options_init(&c);
  c.max_iters = o.max_iters;
  c.fit_tolerance = o.fit_tolerance;
  c.has_fit_threshold = o.fit_threshold.has_value();
  c.fit_threshold = o.fit_threshold.value_or(0.0);
  c.rng_seed = o.rng_seed;
  c.init = static_cast<int32_t>(o.init);
  c.fit_sample_count = o.fit_sample_count;
  c.stall_limit = o.stall_limit;
  c.transform = o.transform ? static_cast<int32_t>(*o.transform) : CPRAND_TRANSFORM_UNSET;
  c.bench_mode = o.bench_mode;
  c.exhaustive_samples = o.exhaustive_samples;
  c.exact_fit_trace = o.exact_fit_trace;
  c.device = o.device;
  if (o.init == InitKind::given && !o.init_model)
    throw std::invalid_argument("init=given requires an init model");
  std::vector<const double*> init_f;
  if (o.init_model)
    for (const Matd& m : o.init_model->factors) init_f.push_back(m.data());
  SolveResult res;
  res.model.lambda.assign(static_cast<size_t>(r > 0 ? r : 0), 0.0);
  std::vector<double*> out_f;
  for (Index d : x.dims) {
    res.model.factors.emplace_back(d, r > 0 ? r : 0);
    out_f.push_back(res.model.factors.back().data());
  }
  std::vector<cprand_trace_record_t> trace(static_cast<size_t>(o.max_iters > 0 ? o.max_iters + 1 : 1));
  cprand_result_t cr{};
  throw_status(cprand_solve(method, x.values.data(), x.dims.data(), static_cast<int32_t>(x.order()), r, s, &c,
                            o.init_model ? o.init_model->lambda.data() : nullptr,
                            o.init_model ? init_f.data() : nullptr, res.model.lambda.data(), out_f.data(),
                            trace.data(), static_cast<int32_t>(trace.size()), &cr));
  for (int i = 0; i < cr.trace_len && i < static_cast<int>(trace.size()); ++i)
    res.trace.push_back({trace[static_cast<size_t>(i)].iteration, trace[static_cast<size_t>(i)].elapsed_seconds,
                         trace[static_cast<size_t>(i)].fit, trace[static_cast<size_t>(i)].fit_is_estimate != 0,
                         trace[static_cast<size_t>(i)].best_fit_so_far});
  res.iterations = cr.iterations;
  res.reason = static_cast<StopReason>(cr.reason);
  res.setup_seconds = cr.setup_seconds;
  res.total_seconds = cr.total_seconds;
  return res;
}

}  // namespace detail

inline Index default_sample_count(Index r) {
  const std::int64_t v = cprand_default_sample_count(r);
  if (v < 0) throw std::invalid_argument("rank must be >= 1");
  return v;
}

// exact_fit (solver.hpp:161-181) on the device: 1 - ||X - M|| / ||X||
inline double exact_fit(const TensorD& x, const KruskalModel& m, int device = -1) {
  if (m.order() != x.order()) throw std::invalid_argument("exact_fit: model dims do not match tensor");
  std::vector<const double*> f;
  for (Index n = 0; n < m.order(); ++n) {
    if (m.factors[static_cast<size_t>(n)].rows != x.dims[static_cast<size_t>(n)] ||
        m.factors[static_cast<size_t>(n)].cols != m.rank())
      throw std::invalid_argument("exact_fit: model dims do not match tensor");
    f.push_back(m.factors[static_cast<size_t>(n)].data());
  }
  double fit = 0.0;
  detail::throw_status(cprand_exact_fit(x.values.data(), x.dims.data(), static_cast<int32_t>(x.order()),
                                        m.lambda.data(), f.data(), m.rank(), device, &fit));
  return fit;
}

inline SolveResult cprand(const TensorD& x, Index r, Index s, const SolveOptions& opts) {
  return detail::run(CPRAND_METHOD_RAND, x, r, s, opts);
}
inline SolveResult cprand_mix(const TensorD& x, Index r, Index s, const SolveOptions& opts) {
  return detail::run(CPRAND_METHOD_MIX, x, r, s, opts);
}
inline SolveResult cprand_premix(const TensorD& x, Index r, Index s, const SolveOptions& opts) {
  return detail::run(CPRAND_METHOD_PREMIX, x, r, s, opts);
}

}  // namespace cprand
