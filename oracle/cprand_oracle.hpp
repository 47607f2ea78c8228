// TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT.
//
// CPU restatement ("oracle") of the reference CPRAND / CPRAND-MIX path
// (arXiv 1701.06600 artifact, /root/reference/proj/include/cprand/*.hpp).
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference legs may load it, and only as the checker or the CPU
// baseline. The product (paper_1701_06600_b200/) never links it.
//
// The reference itself cannot be compiled here: every header except rng.hpp
// includes <Eigen/Dense> (Eigen 3.4 is not installed, vendor/ is untracked).
// This file restates each function in plain C++20 + libstdc++ <random>, so
// every RNG draw (sample tables, fit offsets, init, signs, normalize) is
// bit-identical to the reference by construction (same libstdc++ code on the
// same mt19937_64 streams; pinned against the reference rng.hpp in
// tests/golden/). Linear algebra follows the Eigen algorithms the reference
// calls (ColPivHouseholderQR, CompleteOrthogonalDecomposition, LLT,
// stableNorm); agreement with an Eigen-built binary is at tolerance level
// (reduction order differs), never bit level.
#pragma once

#include <complex>
#include <cstdint>
#include <optional>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

namespace orc {

using Index = std::int64_t;
using Complex = std::complex<double>;
using Shape = std::vector<Index>;

// rng.hpp:11-15
inline constexpr std::uint64_t kInitStream = 1;
inline constexpr std::uint64_t kSamplingStream = 2;
inline constexpr std::uint64_t kFitStream = 3;
inline constexpr std::uint64_t kMixingStream = 4;
inline constexpr std::uint64_t kSynthStream = 5;

// types.hpp:37-41
class numerical_consistency_error : public std::runtime_error {
 public:
  explicit numerical_consistency_error(const std::string& w)
      : std::runtime_error(w) {}
};

// Column-major dense matrix (Eigen's default storage, types.hpp:21-30).
template <class T>
struct Mat {
  Index rows = 0, cols = 0;
  std::vector<T> v;
  Mat() = default;
  Mat(Index r, Index c, T init = T(0))
      : rows(r), cols(c), v(static_cast<std::size_t>(r * c), init) {}
  T& operator()(Index i, Index j) { return v[static_cast<std::size_t>(i + j * rows)]; }
  const T& operator()(Index i, Index j) const {
    return v[static_cast<std::size_t>(i + j * rows)];
  }
  T* col(Index j) { return v.data() + j * rows; }
  const T* col(Index j) const { return v.data() + j * rows; }
};
using Matd = Mat<double>;
using Matcd = Mat<Complex>;

// IndexTable (types.hpp:33): column-major Index matrix.
struct IndexTable {
  Index rows = 0, cols = 0;
  std::vector<Index> v;
  IndexTable() = default;
  IndexTable(Index r, Index c) : rows(r), cols(c), v(static_cast<std::size_t>(r * c), 0) {}
  Index& operator()(Index i, Index j) { return v[static_cast<std::size_t>(i + j * rows)]; }
  Index operator()(Index i, Index j) const { return v[static_cast<std::size_t>(i + j * rows)]; }
};

// DenseTensor<T> (tensor.hpp:17-78): generalized column-major, mode-1 fastest.
template <class T>
struct Tensor {
  Shape dims;
  std::vector<Index> strides;
  std::vector<T> values;
  Index order() const { return static_cast<Index>(dims.size()); }
  Index size() const { return static_cast<Index>(values.size()); }
  Index dim(Index m) const { return dims[static_cast<std::size_t>(m)]; }
  Index stride(Index m) const { return strides[static_cast<std::size_t>(m)]; }
};
using TensorD = Tensor<double>;
using TensorCd = Tensor<Complex>;

template <class T>
Tensor<T> make_tensor(Shape dims, std::vector<T> values);
Index shape_size(const Shape& dims);
double tensor_norm(const TensorD& x);

struct KruskalModel {
  std::vector<double> lambda;
  std::vector<Matd> factors;
  Index order() const { return static_cast<Index>(factors.size()); }
  Index rank() const { return static_cast<Index>(lambda.size()); }
  Shape dims() const {
    Shape d;
    for (const auto& a : factors) d.push_back(a.rows);
    return d;
  }
  void validate() const;
};

enum class InitKind { random = 0, hosvd = 1, given = 2 };
enum class TransformKind { fft = 0, dct = 1, wht = 2, identity = 3 };
enum class StopReason {
  max_iterations = 0, fit_stagnation, fit_threshold, best_fit_stall,
  zero_tensor, bench_complete
};

// SolveOptions (solver.hpp:40-64)
struct SolveOptions {
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
  void validate() const;
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

struct SampleSet {
  Index mode = 0;
  IndexTable idxs;
  Index count() const { return idxs.rows; }
};

struct FitEstimator {
  IndexTable idxs;
  std::vector<double> x_values;
  double x_norm = 0;
  Index total_count = 0;
  double best_fit = -std::numeric_limits<double>::infinity();
  int stall_count = 0;
  int stall_limit = 10;
  Index sample_count() const { return idxs.rows; }
};

struct StopDecision {
  bool stop = false;
  StopReason reason = StopReason::max_iterations;
};

struct MixingOperator {
  TransformKind kind = TransformKind::fft;
  Shape dims;
  std::vector<std::vector<double>> signs;
};

// --- API (each definition cites the reference lines it restates) ---------
std::mt19937_64 seeded_engine(std::uint64_t seed, std::uint64_t stream);
Index unfold_column_index(Index mode, const Index* idx, const Shape& dims);
void decode_column_index(Index mode, Index j, const Shape& dims, Index* idx);
template <class T>
Mat<T> gather_fibers(const Tensor<T>& x, Index mode, const IndexTable& idxs);
Index default_sample_count(Index r);
SampleSet draw_samples(const Shape& dims, Index mode, Index count, std::mt19937_64& rng);
SampleSet exhaustive_samples(const Shape& dims, Index mode);
template <class T>
Mat<T> skr(const SampleSet& s, const std::vector<Mat<T>>& factors, Index mode);
Matd least_squares(const Matd& a, const Matd& b, int* rank_out = nullptr);
Matd sampled_update(const Matd& zs, const Matd& xs);
double stable_norm(const double* v, Index n);
void normalize_columns(KruskalModel& m, Index mode, bool first_of_pass, std::mt19937_64& rng);
FitEstimator make_fit_estimator(const TensorD& x, Index sample_count, int stall_limit,
                                std::mt19937_64& rng);
FitEstimator exhaustive_fit_estimator(const TensorD& x, int stall_limit);
std::vector<Index> sample_offsets_without_replacement(Index total, Index want,
                                                      std::mt19937_64& rng);
double estimate_fit(const KruskalModel& m, const FitEstimator& est);
double model_entry(const KruskalModel& m, const Index* idx);
StopDecision should_stop(FitEstimator& est, double fit, int iteration, const SolveOptions& opts);
KruskalModel init_random(const Shape& dims, Index r, std::uint64_t seed);
double exact_fit(const TensorD& x, const KruskalModel& m);
Matd mttkrp(const TensorD& x, const std::vector<Matd>& factors, Index mode);
Matd gram_of_khatri_rao(const std::vector<Matd>& factors, Index skip);
Matd khatri_rao_seq(const std::vector<Matd>& factors, Index skip);
TensorD reconstruct_dense(const KruskalModel& m);
SolveResult cp_als(const TensorD& x, Index r, const SolveOptions& opts);
SolveResult cprand(const TensorD& x, Index r, Index s, const SolveOptions& opts);
MixingOperator make_mixing_operator(const Shape& dims, TransformKind kind, std::uint64_t seed);
TensorD mix_tensor_real(const TensorD& x, const MixingOperator& op);
TensorCd mix_tensor_complex(const TensorD& x, const MixingOperator& op);
template <class T>
Mat<T> mix_factor(const Matd& a, const MixingOperator& op, Index mode);
template <class T>
Matd unmix_factor(const Mat<T>& a_hat, const MixingOperator& op, Index mode);
template <class T>
Mat<T> unmix_sampled_rhs(const Mat<T>& g, const MixingOperator& op, Index mode);
Matd real_least_squares(const Matd& a, const Matd& b);
Matd real_least_squares(const Matcd& a, const Matcd& b);
SolveResult cprand_mix(const TensorD& x, Index r, Index s, const SolveOptions& opts,
                       const MixingOperator& op);
SolveResult cprand_mix(const TensorD& x, Index r, Index s, const SolveOptions& opts);
SolveResult cprand_premix(const TensorD& x, Index r, Index s, const SolveOptions& opts,
                          const MixingOperator& op);
SolveResult cprand_premix(const TensorD& x, Index r, Index s, const SolveOptions& opts);
// bench-iter of cprand_mix on an already-mixed tensor read in place (bench.py cpu_baseline for C5)
double bench_mix_premixed(const double* x_hat, const Shape& shape, Index r, Index s, TransformKind kind,
                          std::uint64_t seed, int iters);

// Dense transforms (test helpers).
void dct_forward(double* x, Index n);
void dct_adjoint(double* x, Index n);
void fft_forward(Complex* x, Index n);
void fft_backward(Complex* x, Index n);
void wht_forward(double* x, Index n);

// Synthetic inputs.
struct BaselineSynth {
  TensorD tensor;
  KruskalModel truth;
};
BaselineSynth gen_baseline_problem(const Shape& dims, Index r, double collinearity,
                                   double eta, std::uint64_t seed);
void baseline_factors(const Shape& dims, Index r, double collinearity, std::uint64_t seed,
                      std::vector<Matd>& out);
double philox_gaussian(std::uint64_t seed, std::uint64_t counter);
struct SynthProblem {
  TensorD tensor;
  KruskalModel truth;
};
SynthProblem gen_problem(const Shape& dims, Index rank, double collinearity, double noise,
                         std::uint64_t seed);
double score(const KruskalModel& a, const KruskalModel& b);

}  // namespace orc
