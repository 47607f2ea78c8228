// TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT. See cprand_oracle.hpp.
//
// Every function below restates one reference function; the comment above
// it names the file:line (paths relative to /root/reference/proj/include/
// cprand/). Restated, not copied: the reference depends on Eigen, which is
// absent, so each Eigen call is replaced by the published algorithm Eigen
// implements (ColPivHouseholderQR = LAPACK xGEQP3-style pivoted Householder
// QR with norm downdating; CompleteOrthogonalDecomposition = that QR plus an
// RZ reduction; LLT = unblocked Cholesky; stableNorm = scaled 2-norm).
#include "cprand_oracle.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <limits>
#include <numbers>
#include <numeric>
#include <thread>
#include <unordered_set>

namespace orc {

namespace {
constexpr double kPi = std::numbers::pi_v<double>;
using Clock = std::chrono::steady_clock;
double seconds_since(Clock::time_point t0) {
  return std::chrono::duration<double>(Clock::now() - t0).count();
}
}  // namespace

// ---------------------------------------------------------------- rng.hpp
// rng.hpp:19-34 — splitmix64-mixed (seed, stream) → mt19937_64.
static std::uint64_t splitmix_step(std::uint64_t& s) {
  std::uint64_t z = (s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

std::mt19937_64 seeded_engine(std::uint64_t seed, std::uint64_t stream) {
  std::uint64_t st = seed ^ (0xA0761D6478BD642Full * (stream + 1));
  splitmix_step(st);  // first output discarded (rng.hpp:32)
  return std::mt19937_64(splitmix_step(st));
}

// ---------------------------------------------------------- types.hpp
// types.hpp:47-59 — CPRAND_THREADS overrides hardware concurrency.
static int max_threads() {
  static const int cached = [] {
    int n = static_cast<int>(std::thread::hardware_concurrency());
    if (n <= 0) n = 1;
    if (const char* env = std::getenv("CPRAND_THREADS")) {
      char* end = nullptr;
      long v = std::strtol(env, &end, 10);
      if (end != env && v > 0) n = static_cast<int>(v);
    }
    return n;
  }();
  return cached;
}

// types.hpp:63-85 — contiguous chunks, one fresh std::thread per chunk.
template <class F>
static void parallel_for(Index begin, Index end, Index min_grain, F&& body) {
  const Index count = end - begin;
  int workers = max_threads();
  if (min_grain > 0 && count / min_grain < workers)
    workers = static_cast<int>(std::max<Index>(1, count / min_grain));
  if (workers <= 1) {
    for (Index i = begin; i < end; ++i) body(i);
    return;
  }
  std::vector<std::thread> pool;
  const Index chunk = (count + workers - 1) / workers;
  for (int w = 0; w < workers; ++w) {
    const Index lo = begin + chunk * w;
    const Index hi = std::min(end, lo + chunk);
    if (lo >= hi) break;
    pool.emplace_back([lo, hi, &body] {
      for (Index i = lo; i < hi; ++i) body(i);
    });
  }
  for (auto& t : pool) t.join();
}

// --------------------------------------------------------- tensor.hpp
// tensor.hpp:17-33 — validation + generalized column-major strides.
template <class T>
Tensor<T> make_tensor(Shape dims, std::vector<T> values) {
  if (dims.empty()) throw std::invalid_argument("tensor order must be >= 1");
  Tensor<T> t;
  t.strides.resize(dims.size());
  Index p = 1;
  for (std::size_t m = 0; m < dims.size(); ++m) {
    if (dims[m] < 1) throw std::invalid_argument("tensor dims must be >= 1");
    t.strides[m] = p;
    p *= dims[m];
  }
  if (p != static_cast<Index>(values.size()))
    throw std::invalid_argument("value count does not match dims");
  t.dims = std::move(dims);
  t.values = std::move(values);
  return t;
}
template Tensor<double> make_tensor(Shape, std::vector<double>);
template Tensor<Complex> make_tensor(Shape, std::vector<Complex>);

Index shape_size(const Shape& dims) {
  Index p = 1;
  for (Index d : dims) p *= d;
  return p;
}

// tensor.hpp:69 — Frobenius norm (Eigen redux order is not restated; this
// sums 4096-element blocks sequentially, then the block sums).
static double sq_sum(const double* v, Index n) {
  double total = 0.0;
  for (Index b = 0; b < n; b += 4096) {
    const Index e = std::min(n, b + 4096);
    double s = 0.0;
    for (Index i = b; i < e; ++i) s += v[i] * v[i];
    total += s;
  }
  return total;
}
double tensor_norm(const TensorD& x) { return std::sqrt(sq_sum(x.values.data(), x.size())); }

// tensor.hpp:92-106
Index unfold_column_index(Index mode, const Index* idx, const Shape& dims) {
  const Index n = static_cast<Index>(dims.size());
  if (mode < 0 || mode >= n) throw std::out_of_range("mode out of range");
  Index j = 0, jk = 1;
  for (Index k = 0; k < n; ++k) {
    if (k == mode) continue;
    if (idx[k] < 0 || idx[k] >= dims[static_cast<std::size_t>(k)])
      throw std::out_of_range("multiindex out of range");
    j += idx[k] * jk;
    jk *= dims[static_cast<std::size_t>(k)];
  }
  return j;
}

// tensor.hpp:110-118
void decode_column_index(Index mode, Index j, const Shape& dims, Index* idx) {
  const Index n = static_cast<Index>(dims.size());
  for (Index k = 0; k < n; ++k) {
    if (k == mode) continue;
    idx[k] = j % dims[static_cast<std::size_t>(k)];
    j /= dims[static_cast<std::size_t>(k)];
  }
}

// tensor.hpp:188-212 — column s = mode-`mode` fiber named by row s.
template <class T>
Mat<T> gather_fibers(const Tensor<T>& x, Index mode, const IndexTable& idxs) {
  const Index n = x.order();
  if (mode < 0 || mode >= n) throw std::out_of_range("mode out of range");
  if (idxs.cols != n - 1)
    throw std::invalid_argument("gather_fibers: table must have order-1 columns");
  const Index s = idxs.rows;
  const Index in = x.dim(mode);
  const Index stride = x.stride(mode);
  Mat<T> out(in, s);
  const T* v = x.values.data();
  parallel_for(Index{0}, s, Index{1 << 14} / std::max<Index>(in, 1), [&](Index col) {
    Index base = 0, c = 0;
    for (Index k = 0; k < n; ++k) {
      if (k == mode) continue;
      base += idxs(col, c++) * x.stride(k);
    }
    T* dst = out.col(col);
    for (Index i = 0; i < in; ++i) dst[i] = v[base + i * stride];
  });
  return out;
}
template Mat<double> gather_fibers(const Tensor<double>&, Index, const IndexTable&);
template Mat<Complex> gather_fibers(const Tensor<Complex>&, Index, const IndexTable&);

// -------------------------------------------------------- kruskal.hpp
void KruskalModel::validate() const {
  if (factors.empty()) throw std::invalid_argument("model has no factors");
  for (const Matd& a : factors)
    if (a.cols != static_cast<Index>(lambda.size()))
      throw std::invalid_argument("factor rank does not match lambda");
}

// kruskal.hpp:37-44
double model_entry(const KruskalModel& m, const Index* idx) {
  std::vector<double> p(m.lambda);
  for (Index n = 0; n < m.order(); ++n) {
    const Matd& a = m.factors[static_cast<std::size_t>(n)];
    for (Index r = 0; r < m.rank(); ++r) p[static_cast<std::size_t>(r)] *= a(idx[n], r);
  }
  double s = 0.0;
  for (double v : p) s += v;
  return s;
}

// Eigen stableNorm (kruskal.hpp:56,60): overflow/underflow-safe 2-norm,
// restated as the classic scaled sum of squares (LAPACK dnrm2 form).
double stable_norm(const double* v, Index n) {
  double scale = 0.0, ssq = 1.0;
  for (Index i = 0; i < n; ++i) {
    if (v[i] != 0.0) {
      const double a = std::abs(v[i]);
      if (scale < a) {
        ssq = 1.0 + ssq * (scale / a) * (scale / a);
        scale = a;
      } else {
        ssq += (a / scale) * (a / scale);
      }
    }
  }
  return scale * std::sqrt(ssq);
}

// kruskal.hpp:51-67 — the gauss distribution is local to the call, so its
// cached second polar variate dies with the call (stream consumption must
// match for the zero-column path).
void normalize_columns(KruskalModel& m, Index mode, bool first_of_pass, std::mt19937_64& rng) {
  Matd& a = m.factors[static_cast<std::size_t>(mode)];
  std::normal_distribution<double> gauss(0.0, 1.0);
  for (Index r = 0; r < a.cols; ++r) {
    const double norm = stable_norm(a.col(r), a.rows);
    if (norm == 0.0) {
      std::vector<double> fresh(static_cast<std::size_t>(a.rows));
      for (auto& f : fresh) f = gauss(rng);
      const double fn = stable_norm(fresh.data(), a.rows);
      for (Index i = 0; i < a.rows; ++i) a(i, r) = fresh[static_cast<std::size_t>(i)] / fn;
      m.lambda[static_cast<std::size_t>(r)] = 0.0;
      continue;
    }
    for (Index i = 0; i < a.rows; ++i) a(i, r) /= norm;
    m.lambda[static_cast<std::size_t>(r)] =
        first_of_pass ? m.lambda[static_cast<std::size_t>(r)] * norm : norm;
  }
}

// ------------------------------------------------------ kr_linalg.hpp
// kr_linalg.hpp:55-62 + :13-43 — explicit Khatri-Rao of the reversed-mode
// factor sequence (highest mode first, `skip` omitted). Test/oracle use only.
Matd khatri_rao_seq(const std::vector<Matd>& factors, Index skip) {
  std::vector<const Matd*> seq;
  for (Index m = static_cast<Index>(factors.size()) - 1; m >= 0; --m)
    if (m != skip) seq.push_back(&factors[static_cast<std::size_t>(m)]);
  if (seq.empty()) throw std::invalid_argument("khatri_rao: empty list");
  Matd out = *seq[0];
  for (std::size_t k = 1; k < seq.size(); ++k) {
    const Matd& b = *seq[k];
    Matd nxt(out.rows * b.rows, out.cols);
    for (Index r = 0; r < out.cols; ++r)
      for (Index i = 0; i < out.rows; ++i)
        for (Index j = 0; j < b.rows; ++j) nxt(i * b.rows + j, r) = out(i, r) * b(j, r);
    out = std::move(nxt);
  }
  return out;
}

// kr_linalg.hpp:65-77
Matd gram_of_khatri_rao(const std::vector<Matd>& factors, Index skip) {
  const Index r = factors[0].cols;
  Matd v(r, r, 1.0);
  for (Index m = 0; m < static_cast<Index>(factors.size()); ++m) {
    if (m == skip) continue;
    const Matd& a = factors[static_cast<std::size_t>(m)];
    for (Index j = 0; j < r; ++j)
      for (Index i = 0; i < r; ++i) {
        double s = 0.0;
        for (Index k = 0; k < a.rows; ++k) s += a(k, i) * a(k, j);
        v(i, j) *= s;
      }
  }
  return v;
}

// kr_linalg.hpp:80-89 — X_(n) · Z^(n), with the Khatri-Rao row of each
// unfolding column formed on the fly instead of materialized.
Matd mttkrp(const TensorD& x, const std::vector<Matd>& factors, Index mode) {
  if (static_cast<Index>(factors.size()) != x.order())
    throw std::invalid_argument("mttkrp: need one factor per mode");
  const Index r = factors[0].cols;
  const Index in = x.dim(mode);
  Matd w(in, r);
  const Index cols = x.size() / in;
  const Index n = x.order();
  std::vector<Index> idx(static_cast<std::size_t>(n), 0);
  std::vector<double> z(static_cast<std::size_t>(r));
  for (Index j = 0; j < cols; ++j) {
    decode_column_index(mode, j, x.dims, idx.data());
    std::fill(z.begin(), z.end(), 1.0);
    Index base = 0;
    for (Index m = n - 1; m >= 0; --m) {
      if (m == mode) continue;
      base += idx[static_cast<std::size_t>(m)] * x.stride(m);
      const Matd& a = factors[static_cast<std::size_t>(m)];
      for (Index c = 0; c < r; ++c) z[static_cast<std::size_t>(c)] *= a(idx[static_cast<std::size_t>(m)], c);
    }
    for (Index i = 0; i < in; ++i) {
      const double xv = x.values[static_cast<std::size_t>(base + i * x.stride(mode))];
      for (Index c = 0; c < r; ++c) w(i, c) += xv * z[static_cast<std::size_t>(c)];
    }
  }
  return w;
}

namespace {

// Eigen makeHouseholderInPlace on x[0..n): on return x[0] = beta, x[1..n)
// holds the essential part, tau the coefficient; H = I - tau v v^T, v0 = 1.
void make_householder(double* x, Index n, Index inc, double& tau, double& beta) {
  double tail = 0.0;
  for (Index i = 1; i < n; ++i) tail += x[i * inc] * x[i * inc];
  const double c0 = x[0];
  const double tol = std::numeric_limits<double>::min();
  if (tail <= tol) {
    tau = 0.0;
    beta = c0;
    for (Index i = 1; i < n; ++i) x[i * inc] = 0.0;
  } else {
    beta = std::sqrt(c0 * c0 + tail);
    if (c0 >= 0.0) beta = -beta;
    for (Index i = 1; i < n; ++i) x[i * inc] /= (c0 - beta);
    tau = (beta - c0) / beta;
  }
  x[0] = beta;
}

// Applies H = I - tau [1; ess][1; ess]^T from the left to rows [0, len) of
// the column-major block b (ld, ncols).
void apply_householder_left(const double* ess, Index ess_inc, double tau, Index len, double* b,
                            Index ld, Index ncols) {
  if (tau == 0.0) return;
  for (Index j = 0; j < ncols; ++j) {
    double* c = b + j * ld;
    double t = c[0];
    for (Index i = 1; i < len; ++i) t += ess[(i - 1) * ess_inc] * c[i];
    t *= tau;
    c[0] -= t;
    for (Index i = 1; i < len; ++i) c[i] -= t * ess[(i - 1) * ess_inc];
  }
}

// ColPivHouseholderQR (used at kr_linalg.hpp:110-113), restated.
struct PivQR {
  Matd qr;
  std::vector<double> hcoeffs;
  std::vector<Index> perm;  // perm[i] = original column at position i
  Index nonzero_pivots = 0;
  double maxpivot = 0.0;
  double threshold = 0.0;

  void compute(const Matd& a, double thr) {
    qr = a;
    threshold = thr;
    const Index rows = a.rows, cols = a.cols, size = std::min(rows, cols);
    hcoeffs.assign(static_cast<std::size_t>(size), 0.0);
    perm.resize(static_cast<std::size_t>(cols));
    std::iota(perm.begin(), perm.end(), Index{0});
    std::vector<double> upd(static_cast<std::size_t>(cols)), dir(static_cast<std::size_t>(cols));
    for (Index k = 0; k < cols; ++k) {
      dir[static_cast<std::size_t>(k)] = std::sqrt(sq_sum(qr.col(k), rows));
      upd[static_cast<std::size_t>(k)] = dir[static_cast<std::size_t>(k)];
    }
    double maxnorm = 0.0;
    for (double v : upd) maxnorm = std::max(maxnorm, v);
    const double eps = std::numeric_limits<double>::epsilon();
    const double threshold_helper = (maxnorm * eps) * (maxnorm * eps) / static_cast<double>(rows);
    const double downdate_thr = std::sqrt(eps);
    nonzero_pivots = size;
    maxpivot = 0.0;
    for (Index k = 0; k < size; ++k) {
      Index big = k;
      for (Index j = k + 1; j < cols; ++j)
        if (upd[static_cast<std::size_t>(j)] > upd[static_cast<std::size_t>(big)]) big = j;
      const double big_sq = upd[static_cast<std::size_t>(big)] * upd[static_cast<std::size_t>(big)];
      if (nonzero_pivots == size && big_sq < threshold_helper * static_cast<double>(rows - k))
        nonzero_pivots = k;
      if (big != k) {
        for (Index i = 0; i < rows; ++i) std::swap(qr(i, k), qr(i, big));
        std::swap(upd[static_cast<std::size_t>(k)], upd[static_cast<std::size_t>(big)]);
        std::swap(dir[static_cast<std::size_t>(k)], dir[static_cast<std::size_t>(big)]);
        std::swap(perm[static_cast<std::size_t>(k)], perm[static_cast<std::size_t>(big)]);
      }
      double tau, beta;
      make_householder(qr.col(k) + k, rows - k, 1, tau, beta);
      hcoeffs[static_cast<std::size_t>(k)] = tau;
      if (std::abs(beta) > maxpivot) maxpivot = std::abs(beta);
      apply_householder_left(qr.col(k) + k + 1, 1, tau, rows - k, qr.col(k + 1) + k, rows,
                             cols - k - 1);
      for (Index j = k + 1; j < cols; ++j) {
        double& u = upd[static_cast<std::size_t>(j)];
        if (u != 0.0) {
          double t = std::abs(qr(k, j)) / u;
          t = (1.0 + t) * (1.0 - t);
          t = t < 0.0 ? 0.0 : t;
          const double ratio = u / dir[static_cast<std::size_t>(j)];
          const double t2 = t * ratio * ratio;
          if (t2 <= downdate_thr) {
            dir[static_cast<std::size_t>(j)] = std::sqrt(sq_sum(qr.col(j) + k + 1, rows - k - 1));
            u = dir[static_cast<std::size_t>(j)];
          } else {
            u *= std::sqrt(t);
          }
        }
      }
    }
  }

  Index rank() const {
    const double pre = std::abs(maxpivot) * threshold;
    Index r = 0;
    for (Index i = 0; i < nonzero_pivots; ++i) r += std::abs(qr(i, i)) > pre;
    return r;
  }

  // c <- H_{len-1} ... H_0 c  (i.e. Q^T c restricted to the first len reflectors)
  void apply_qt(Matd& c, Index len) const {
    for (Index k = 0; k < len; ++k)
      apply_householder_left(qr.col(k) + k + 1, 1, hcoeffs[static_cast<std::size_t>(k)],
                             qr.rows - k, c.v.data() + k, c.rows, c.cols);
  }

  Matd solve(const Matd& b) const {
    const Index cols = qr.cols;
    Matd dst(cols, b.cols);
    const Index nz = nonzero_pivots;
    if (nz == 0) return dst;
    Matd c = b;
    apply_qt(c, nz);
    for (Index j = 0; j < c.cols; ++j)
      for (Index i = nz - 1; i >= 0; --i) {
        double s = c(i, j);
        for (Index k = i + 1; k < nz; ++k) s -= qr(i, k) * c(k, j);
        c(i, j) = s / qr(i, i);
      }
    for (Index i = 0; i < nz; ++i)
      for (Index j = 0; j < c.cols; ++j) dst(perm[static_cast<std::size_t>(i)], j) = c(i, j);
    return dst;
  }
};

// CompleteOrthogonalDecomposition (kr_linalg.hpp:114-117), restated: the
// pivoted QR above, then an RZ reduction of the leading rank rows.
struct COD {
  PivQR cp;
  std::vector<double> zcoeffs;
  Index rk = 0;

  void compute(const Matd& a, double thr) {
    cp.compute(a, thr);
    rk = cp.rank();
    const Index cols = a.cols;
    zcoeffs.assign(static_cast<std::size_t>(cols), 0.0);
    if (rk >= cols) return;
    Matd& q = cp.qr;
    for (Index k = rk - 1; k >= 0; --k) {
      if (k != rk - 1)
        for (Index i = 0; i <= k; ++i) std::swap(q(i, k), q(i, rk - 1));
      // reflector over [X(k, rk-1), X(k, rk:cols)] (row k, stride rows)
      double tau, beta;
      make_householder(&q(k, rk - 1), cols - rk + 1, q.rows, tau, beta);
      zcoeffs[static_cast<std::size_t>(k)] = tau;
      q(k, rk - 1) = beta;
      if (k > 0 && tau != 0.0) {
        // apply from the right to rows [0,k) of columns {rk-1, rk..cols)
        for (Index i = 0; i < k; ++i) {
          double t = q(i, rk - 1);
          for (Index j = rk; j < cols; ++j) t += q(i, j) * q(k, j);
          t *= tau;
          q(i, rk - 1) -= t;
          for (Index j = rk; j < cols; ++j) q(i, j) -= t * q(k, j);
        }
      }
      if (k != rk - 1)
        for (Index i = 0; i <= k; ++i) std::swap(q(i, k), q(i, rk - 1));
    }
  }

  Matd solve(const Matd& b) const {
    const Index cols = cp.qr.cols;
    Matd dst(cols, b.cols);
    if (rk == 0) return dst;
    Matd c = b;
    cp.apply_qt(c, rk);
    const Matd& q = cp.qr;
    for (Index j = 0; j < b.cols; ++j)
      for (Index i = rk - 1; i >= 0; --i) {
        double s = c(i, j);
        for (Index k = i + 1; k < rk; ++k) s -= q(i, k) * dst(k, j);
        dst(i, j) = s / q(i, i);
      }
    if (rk < cols) {
      // y = Z^T [z; 0]: apply Z(k) for k = 0..rk-1 on rows {k} ∪ [rk, cols)
      for (Index k = 0; k < rk; ++k) {
        const double tau = zcoeffs[static_cast<std::size_t>(k)];
        if (tau == 0.0) continue;
        for (Index j = 0; j < dst.cols; ++j) {
          double t = dst(k, j);
          for (Index i = rk; i < cols; ++i) t += q(k, i) * dst(i, j);
          t *= tau;
          dst(k, j) -= t;
          for (Index i = rk; i < cols; ++i) dst(i, j) -= t * q(k, i);
        }
      }
    }
    Matd out(cols, b.cols);
    for (Index i = 0; i < cols; ++i)
      for (Index j = 0; j < b.cols; ++j) out(cp.perm[static_cast<std::size_t>(i)], j) = dst(i, j);
    return out;
  }
};

double rank_threshold(const Matd& a) {  // kr_linalg.hpp:88-92
  return static_cast<double>(std::max(a.rows, a.cols)) * std::numeric_limits<double>::epsilon();
}

Matd transpose(const Matd& a) {
  Matd t(a.cols, a.rows);
  for (Index j = 0; j < a.cols; ++j)
    for (Index i = 0; i < a.rows; ++i) t(j, i) = a(i, j);
  return t;
}

}  // namespace

// kr_linalg.hpp:99-113 — pivoted QR solve; rank deficiency → COD min-norm.
Matd least_squares(const Matd& a, const Matd& b, int* rank_out) {
  if (a.rows < a.cols) throw std::invalid_argument("least_squares: system is underdetermined");
  if (b.rows != a.rows) throw std::invalid_argument("least_squares: rhs row count mismatch");
  PivQR qr;
  qr.compute(a, rank_threshold(a));
  const Index rk = qr.rank();
  if (rank_out) *rank_out = static_cast<int>(rk);
  if (rk == a.cols) return qr.solve(b);
  COD cod;
  cod.compute(a, rank_threshold(a));
  return cod.solve(b);
}

// ------------------------------------------------------- sampling.hpp
// sampling.hpp:18-23
Index default_sample_count(Index r) {
  if (r < 1) throw std::invalid_argument("rank must be >= 1");
  if (r == 1) return 10;
  return static_cast<Index>(
      std::lround(10.0 * static_cast<double>(r) * std::log(static_cast<double>(r))));
}

// sampling.hpp:35-51 — one uniform_int_distribution per kept mode, consumed
// row by row, low mode first.
SampleSet draw_samples(const Shape& dims, Index mode, Index count, std::mt19937_64& rng) {
  const Index n = static_cast<Index>(dims.size());
  if (mode < 0 || mode >= n) throw std::out_of_range("mode out of range");
  if (count < 1) throw std::invalid_argument("sample count must be >= 1");
  SampleSet s;
  s.mode = mode;
  s.idxs = IndexTable(count, n - 1);
  std::vector<std::uniform_int_distribution<Index>> dist;
  for (Index k = 0; k < n; ++k)
    if (k != mode) dist.emplace_back(Index{0}, dims[static_cast<std::size_t>(k)] - 1);
  for (Index j = 0; j < count; ++j)
    for (Index c = 0; c < n - 1; ++c) s.idxs(j, c) = dist[static_cast<std::size_t>(c)](rng);
  return s;
}

// sampling.hpp:54-69
SampleSet exhaustive_samples(const Shape& dims, Index mode) {
  const Index n = static_cast<Index>(dims.size());
  if (mode < 0 || mode >= n) throw std::out_of_range("mode out of range");
  const Index rows = shape_size(dims) / dims[static_cast<std::size_t>(mode)];
  SampleSet s;
  s.mode = mode;
  s.idxs = IndexTable(rows, n - 1);
  std::vector<Index> idx(static_cast<std::size_t>(n), 0);
  for (Index j = 0; j < rows; ++j) {
    decode_column_index(mode, j, dims, idx.data());
    Index c = 0;
    for (Index k = 0; k < n; ++k)
      if (k != mode) s.idxs(j, c++) = idx[static_cast<std::size_t>(k)];
  }
  return s;
}

// sampling.hpp:74-92 — Z = ones, then *= factor rows in ascending mode.
template <class T>
Mat<T> skr(const SampleSet& s, const std::vector<Mat<T>>& factors, Index mode) {
  const Index n = static_cast<Index>(factors.size());
  if (mode != s.mode) throw std::invalid_argument("skr: sample set mode mismatch");
  if (s.idxs.cols != n - 1) throw std::invalid_argument("skr: sample table width mismatch");
  const Index r = factors[0].cols;
  Mat<T> z(s.count(), r, T(1.0));
  Index c = 0;
  for (Index m = 0; m < n; ++m) {
    if (m == mode) continue;
    const Mat<T>& a = factors[static_cast<std::size_t>(m)];
    for (Index j = 0; j < s.count(); ++j) {
      const Index row = s.idxs(j, c);
      for (Index q = 0; q < r; ++q) z(j, q) *= a(row, q);
    }
    ++c;
  }
  return z;
}
template Mat<double> skr(const SampleSet&, const std::vector<Mat<double>>&, Index);
template Mat<Complex> skr(const SampleSet&, const std::vector<Mat<Complex>>&, Index);

// sampling.hpp:96-102
Matd sampled_update(const Matd& zs, const Matd& xs) {
  if (zs.rows < zs.cols) throw std::invalid_argument("sampled_update: need at least R samples");
  if (xs.cols != zs.rows) throw std::invalid_argument("sampled_update: fiber count mismatch");
  return transpose(least_squares(zs, transpose(xs)));
}

// sampling.hpp:121-149
std::vector<Index> sample_offsets_without_replacement(Index total, Index want,
                                                      std::mt19937_64& rng) {
  std::vector<Index> out;
  if (want >= total) {
    out.resize(static_cast<std::size_t>(total));
    std::iota(out.begin(), out.end(), Index{0});
    return out;
  }
  if (total <= 4 * want) {
    std::vector<Index> pool(static_cast<std::size_t>(total));
    std::iota(pool.begin(), pool.end(), Index{0});
    for (Index i = 0; i < want; ++i) {
      std::uniform_int_distribution<Index> pick(i, total - 1);
      std::swap(pool[static_cast<std::size_t>(i)], pool[static_cast<std::size_t>(pick(rng))]);
    }
    out.assign(pool.begin(), pool.begin() + want);
  } else {
    std::unordered_set<Index> seen;
    std::uniform_int_distribution<Index> pick(Index{0}, total - 1);
    out.reserve(static_cast<std::size_t>(want));
    while (static_cast<Index>(out.size()) < want) {
      const Index cand = pick(rng);
      if (seen.insert(cand).second) out.push_back(cand);
    }
  }
  std::sort(out.begin(), out.end());
  return out;
}

// sampling.hpp:155-179
FitEstimator make_fit_estimator(const TensorD& x, Index sample_count, int stall_limit,
                                std::mt19937_64& rng) {
  if (sample_count < 1) throw std::invalid_argument("fit sample count must be >= 1");
  if (stall_limit < 1) throw std::invalid_argument("stall limit must be >= 1");
  FitEstimator est;
  est.stall_limit = stall_limit;
  est.total_count = x.size();
  est.x_norm = tensor_norm(x);
  const auto offsets = sample_offsets_without_replacement(x.size(), sample_count, rng);
  const Index n = x.order();
  const Index p = static_cast<Index>(offsets.size());
  est.idxs = IndexTable(p, n);
  est.x_values.resize(static_cast<std::size_t>(p));
  for (Index j = 0; j < p; ++j) {
    Index rem = offsets[static_cast<std::size_t>(j)];
    for (Index k = 0; k < n; ++k) {
      est.idxs(j, k) = rem % x.dim(k);
      rem /= x.dim(k);
    }
    est.x_values[static_cast<std::size_t>(j)] = x.values[static_cast<std::size_t>(offsets[static_cast<std::size_t>(j)])];
  }
  return est;
}

// sampling.hpp:182-186
FitEstimator exhaustive_fit_estimator(const TensorD& x, int stall_limit) {
  auto rng = seeded_engine(0, kFitStream);
  return make_fit_estimator(x, x.size(), stall_limit, rng);
}

// sampling.hpp:191-210
double estimate_fit(const KruskalModel& m, const FitEstimator& est) {
  if (est.x_norm == 0.0) return 1.0;
  if (est.idxs.cols != m.order()) throw std::invalid_argument("estimate_fit: estimator order mismatch");
  const Index p_hat = est.sample_count();
  const Index r = m.rank();
  std::vector<double> prod(static_cast<std::size_t>(r));
  double sq_sum_v = 0.0;
  for (Index j = 0; j < p_hat; ++j) {
    for (Index q = 0; q < r; ++q) prod[static_cast<std::size_t>(q)] = m.lambda[static_cast<std::size_t>(q)];
    for (Index n = 0; n < m.order(); ++n) {
      const Matd& a = m.factors[static_cast<std::size_t>(n)];
      const Index row = est.idxs(j, n);
      for (Index q = 0; q < r; ++q) prod[static_cast<std::size_t>(q)] *= a(row, q);
    }
    double s = 0.0;
    for (double v : prod) s += v;
    const double e = est.x_values[static_cast<std::size_t>(j)] - s;
    sq_sum_v += e * e;
  }
  const double mu = sq_sum_v / static_cast<double>(p_hat);
  return 1.0 - std::sqrt(static_cast<double>(est.total_count) * mu) / est.x_norm;
}

// sampling.hpp:237-251
StopDecision should_stop(FitEstimator& est, double fit, int iteration, const SolveOptions& opts) {
  if (fit > est.best_fit) {
    est.best_fit = fit;
    est.stall_count = 0;
  } else {
    ++est.stall_count;
  }
  if (opts.fit_threshold && fit >= *opts.fit_threshold) return {true, StopReason::fit_threshold};
  if (est.stall_count >= est.stall_limit) return {true, StopReason::best_fit_stall};
  if (iteration >= opts.max_iters) return {true, StopReason::max_iterations};
  return {false, StopReason::max_iterations};
}

// --------------------------------------------------------- solver.hpp
// solver.hpp:54-63
void SolveOptions::validate() const {
  if (max_iters < 1) throw std::invalid_argument("max_iters must be >= 1");
  if (!(fit_tolerance > 0.0)) throw std::invalid_argument("fit_tolerance must be > 0");
  if (fit_sample_count < 1) throw std::invalid_argument("fit_sample_count must be >= 1");
  if (stall_limit < 1) throw std::invalid_argument("stall_limit must be >= 1");
  if (init == InitKind::given && !init_model)
    throw std::invalid_argument("init=given requires an init model");
}

// solver.hpp:104-123
KruskalModel init_random(const Shape& dims, Index r, std::uint64_t seed) {
  if (r < 1) throw std::invalid_argument("rank must be >= 1");
  KruskalModel m;
  m.lambda.assign(static_cast<std::size_t>(r), 1.0);
  auto rng = seeded_engine(seed, kInitStream);
  std::uniform_real_distribution<double> unif(0.0, 1.0);
  for (std::size_t n = 0; n < dims.size(); ++n) {
    Matd a(dims[n], r);
    if (n != 0)
      for (Index j = 0; j < r; ++j)
        for (Index i = 0; i < dims[n]; ++i) a(i, j) = unif(rng);
    m.factors.push_back(std::move(a));
  }
  return m;
}

// solver.hpp:166-181 — exact fit via the mode-1 MTTKRP Gram expansion.
double exact_fit(const TensorD& x, const KruskalModel& m) {
  m.validate();
  if (m.dims() != x.dims) throw std::invalid_argument("exact_fit: model dims do not match tensor");
  const double xnorm = tensor_norm(x);
  if (xnorm == 0.0) return 1.0;
  const Matd w = mttkrp(x, m.factors, 0);
  const Matd& a0 = m.factors[0];
  const Matd v = gram_of_khatri_rao(m.factors, 0);
  const Index r = m.rank();
  double cross = 0.0;
  for (Index j = 0; j < r; ++j)
    for (Index i = 0; i < a0.rows; ++i) cross += a0(i, j) * w(i, j) * m.lambda[static_cast<std::size_t>(j)];
  double model_sq = 0.0;
  for (Index i = 0; i < r; ++i) {
    double row = 0.0;
    for (Index j = 0; j < r; ++j) {
      double g = 0.0;
      for (Index k = 0; k < a0.rows; ++k) g += a0(k, i) * a0(k, j);
      row += v(i, j) * g * m.lambda[static_cast<std::size_t>(j)];
    }
    model_sq += m.lambda[static_cast<std::size_t>(i)] * row;
  }
  const double resid_sq = std::max(0.0, xnorm * xnorm - 2.0 * cross + model_sq);
  return 1.0 - std::sqrt(resid_sq) / xnorm;
}

namespace {

// solver.hpp:185-201
KruskalModel make_init(const TensorD& x, Index r, const SolveOptions& opts) {
  switch (opts.init) {
    case InitKind::random:
      return init_random(x.dims, r, opts.rng_seed);
    case InitKind::hosvd:
      throw std::invalid_argument("hosvd init is outside the restated path");
    case InitKind::given: {
      KruskalModel m = *opts.init_model;
      m.validate();
      if (m.dims() != x.dims || m.rank() != r)
        throw std::invalid_argument("init model does not match problem");
      return m;
    }
  }
  throw std::invalid_argument("unknown init kind");
}

// solver.hpp:204-216
SolveResult zero_tensor_result(const TensorD& x, Index r, const SolveOptions& opts) {
  SolveResult res;
  res.model = init_random(x.dims, r, opts.rng_seed);
  auto rng = seeded_engine(opts.rng_seed, kInitStream);
  for (Index n = 0; n < x.order(); ++n) normalize_columns(res.model, n, false, rng);
  std::fill(res.model.lambda.begin(), res.model.lambda.end(), 0.0);
  res.trace.push_back({0, 0.0, 1.0, false, 1.0});
  res.iterations = 0;
  res.reason = StopReason::zero_tensor;
  return res;
}

// Eigen LLT (solver.hpp:244): lower Cholesky; false when not positive definite.
bool llt_solve(const Matd& v, const Matd& b, Matd& out) {
  const Index n = v.rows;
  Matd l(n, n);
  for (Index j = 0; j < n; ++j) {
    double d = v(j, j);
    for (Index k = 0; k < j; ++k) d -= l(j, k) * l(j, k);
    if (!(d > 0.0)) return false;
    l(j, j) = std::sqrt(d);
    for (Index i = j + 1; i < n; ++i) {
      double s = v(i, j);
      for (Index k = 0; k < j; ++k) s -= l(i, k) * l(j, k);
      l(i, j) = s / l(j, j);
    }
  }
  out = b;
  for (Index c = 0; c < b.cols; ++c) {
    for (Index i = 0; i < n; ++i) {
      double s = out(i, c);
      for (Index k = 0; k < i; ++k) s -= l(i, k) * out(k, c);
      out(i, c) = s / l(i, i);
    }
    for (Index i = n - 1; i >= 0; --i) {
      double s = out(i, c);
      for (Index k = i + 1; k < n; ++k) s -= l(k, i) * out(k, c);
      out(i, c) = s / l(i, i);
    }
  }
  return true;
}

}  // namespace

// solver.hpp:225-277 — classical CP-ALS (exhaustive-degeneracy oracle).
SolveResult cp_als(const TensorD& x, Index r, const SolveOptions& opts) {
  opts.validate();
  if (r < 1) throw std::invalid_argument("rank must be >= 1");
  if (tensor_norm(x) == 0.0 && !opts.bench_mode) return zero_tensor_result(x, r, opts);
  const auto t0 = Clock::now();
  SolveResult res;
  res.model = make_init(x, r, opts);
  auto norm_rng = seeded_engine(opts.rng_seed, kInitStream + 7);
  res.setup_seconds = seconds_since(t0);
  const Index n_modes = x.order();
  double prev_fit = std::numeric_limits<double>::quiet_NaN();
  double best = -std::numeric_limits<double>::infinity();
  for (int it = 1; it <= opts.max_iters; ++it) {
    for (Index n = 0; n < n_modes; ++n) {
      const Matd v = gram_of_khatri_rao(res.model.factors, n);
      const Matd w = mttkrp(x, res.model.factors, n);
      Matd sol;
      if (llt_solve(v, transpose(w), sol)) {
        res.model.factors[static_cast<std::size_t>(n)] = transpose(sol);
      } else {
        COD cod;
        cod.compute(v, std::numeric_limits<double>::epsilon() * static_cast<double>(v.rows));
        res.model.factors[static_cast<std::size_t>(n)] = transpose(cod.solve(transpose(w)));
      }
      normalize_columns(res.model, n, n == 0, norm_rng);
    }
    res.iterations = it;
    if (opts.bench_mode) continue;
    const double fit = exact_fit(x, res.model);
    best = std::max(best, fit);
    res.trace.push_back({it, seconds_since(t0), fit, false, best});
    if (opts.fit_threshold && fit >= *opts.fit_threshold) {
      res.reason = StopReason::fit_threshold;
      res.total_seconds = seconds_since(t0);
      return res;
    }
    if (it > 1 && std::abs(fit - prev_fit) <= opts.fit_tolerance) {
      res.reason = StopReason::fit_stagnation;
      res.total_seconds = seconds_since(t0);
      return res;
    }
    prev_fit = fit;
  }
  res.reason = opts.bench_mode ? StopReason::bench_complete : StopReason::max_iterations;
  res.total_seconds = seconds_since(t0);
  return res;
}

// sampling.hpp:257-310 — CPRAND.
SolveResult cprand(const TensorD& x, Index r, Index s, const SolveOptions& opts) {
  opts.validate();
  if (r < 1) throw std::invalid_argument("rank must be >= 1");
  if (s < r) throw std::invalid_argument("sample count must be at least the rank");
  if (tensor_norm(x) == 0.0 && !opts.bench_mode) return zero_tensor_result(x, r, opts);
  const auto t0 = Clock::now();
  SolveResult res;
  res.model = make_init(x, r, opts);
  auto sample_rng = seeded_engine(opts.rng_seed, kSamplingStream);
  auto fit_rng = seeded_engine(opts.rng_seed, kFitStream);
  auto norm_rng = seeded_engine(opts.rng_seed, kInitStream + 7);
  FitEstimator est;
  if (!opts.bench_mode)
    est = opts.exhaustive_samples
              ? exhaustive_fit_estimator(x, opts.stall_limit)
              : make_fit_estimator(x, opts.fit_sample_count, opts.stall_limit, fit_rng);
  res.setup_seconds = seconds_since(t0);
  const Index n_modes = x.order();
  for (int it = 1; it <= opts.max_iters; ++it) {
    for (Index n = 0; n < n_modes; ++n) {
      const SampleSet samples = opts.exhaustive_samples ? exhaustive_samples(x.dims, n)
                                                        : draw_samples(x.dims, n, s, sample_rng);
      const Matd zs = skr(samples, res.model.factors, n);
      const Matd xs = gather_fibers(x, n, samples.idxs);
      res.model.factors[static_cast<std::size_t>(n)] = sampled_update(zs, xs);
      normalize_columns(res.model, n, n == 0, norm_rng);
    }
    res.iterations = it;
    if (opts.bench_mode) continue;
    const double fit = opts.exact_fit_trace ? exact_fit(x, res.model) : estimate_fit(res.model, est);
    const StopDecision d = should_stop(est, fit, it, opts);
    res.trace.push_back({it, seconds_since(t0), fit, !opts.exact_fit_trace, est.best_fit});
    if (d.stop) {
      res.reason = d.reason;
      res.total_seconds = seconds_since(t0);
      return res;
    }
  }
  res.reason = opts.bench_mode ? StopReason::bench_complete : StopReason::max_iterations;
  res.total_seconds = seconds_since(t0);
  return res;
}

// ----------------------------------------------------- transforms.hpp
namespace {

bool is_pow2(Index n) { return n >= 1 && (n & (n - 1)) == 0; }
Index next_pow2(Index n) {
  Index p = 1;
  while (p < n) p <<= 1;
  return p;
}

// transforms.hpp:27-118 — radix-2 with a direct-trig twiddle table for
// powers of two; Bluestein (chirp-z) over the next power of two >= 2n-1
// otherwise. Unnormalized; backward = conj ∘ forward ∘ conj.
class Fft {
 public:
  explicit Fft(Index n) : n_(n) {
    if (n < 1) throw std::invalid_argument("fft length must be >= 1");
    if (is_pow2(n_)) {
      tables(n_);
      return;
    }
    m_ = next_pow2(2 * n_ - 1);
    tables(m_);
    chirp_.resize(static_cast<std::size_t>(n_));
    for (Index j = 0; j < n_; ++j) {
      const Index q = (j * j) % (2 * n_);
      const double ang = -kPi * static_cast<double>(q) / static_cast<double>(n_);
      chirp_[static_cast<std::size_t>(j)] = Complex(std::cos(ang), std::sin(ang));
    }
    spec_.assign(static_cast<std::size_t>(m_), Complex(0.0));
    spec_[0] = Complex(1.0);
    for (Index j = 1; j < n_; ++j) {
      const Complex b = std::conj(chirp_[static_cast<std::size_t>(j)]);
      spec_[static_cast<std::size_t>(j)] = b;
      spec_[static_cast<std::size_t>(m_ - j)] = b;
    }
    radix2(spec_.data(), m_);
  }

  void forward(Complex* d) const {
    if (is_pow2(n_)) {
      radix2(d, n_);
      return;
    }
    std::vector<Complex> a(static_cast<std::size_t>(m_), Complex(0.0));
    for (Index j = 0; j < n_; ++j) a[static_cast<std::size_t>(j)] = d[j] * chirp_[static_cast<std::size_t>(j)];
    radix2(a.data(), m_);
    for (Index k = 0; k < m_; ++k) a[static_cast<std::size_t>(k)] *= spec_[static_cast<std::size_t>(k)];
    for (auto& z : a) z = std::conj(z);
    radix2(a.data(), m_);
    const double inv_m = 1.0 / static_cast<double>(m_);
    for (Index k = 0; k < n_; ++k)
      d[k] = std::conj(a[static_cast<std::size_t>(k)]) * inv_m * chirp_[static_cast<std::size_t>(k)];
  }

  void backward(Complex* d) const {
    for (Index j = 0; j < n_; ++j) d[j] = std::conj(d[j]);
    forward(d);
    for (Index j = 0; j < n_; ++j) d[j] = std::conj(d[j]);
  }

 private:
  void tables(Index n) {
    tw_.resize(static_cast<std::size_t>(std::max<Index>(n / 2, 1)));
    for (Index k = 0; k < static_cast<Index>(tw_.size()); ++k) {
      const double ang = -2.0 * kPi * static_cast<double>(k) / static_cast<double>(n);
      tw_[static_cast<std::size_t>(k)] = Complex(std::cos(ang), std::sin(ang));
    }
  }

  void radix2(Complex* a, Index n) const {
    for (Index i = 1, j = 0; i < n; ++i) {  // bit reversal
      Index bit = n >> 1;
      for (; j & bit; bit >>= 1) j ^= bit;
      j ^= bit;
      if (i < j) std::swap(a[i], a[j]);
    }
    for (Index len = 2; len <= n; len <<= 1) {
      const Index half = len >> 1, step = n / len;
      for (Index i = 0; i < n; i += len)
        for (Index k = 0; k < half; ++k) {
          const Complex w = tw_[static_cast<std::size_t>(k * step)];
          const Complex u = a[i + k];
          const Complex v = a[i + k + half] * w;
          a[i + k] = u + v;
          a[i + k + half] = u - v;
        }
    }
  }

  Index n_ = 0, m_ = 0;
  std::vector<Complex> tw_, chirp_, spec_;
};

// transforms.hpp:124-166 — orthonormal DCT-II / DCT-III via a length-2n FFT.
class Dct {
 public:
  explicit Dct(Index n) : n_(n), fft_(2 * n) {
    phase_.resize(static_cast<std::size_t>(n_));
    for (Index k = 0; k < n_; ++k) {
      const double ang = -kPi * static_cast<double>(k) / (2.0 * static_cast<double>(n_));
      phase_[static_cast<std::size_t>(k)] = Complex(std::cos(ang), std::sin(ang));
    }
    s0_ = std::sqrt(1.0 / static_cast<double>(n_));
    sk_ = std::sqrt(2.0 / static_cast<double>(n_));
  }
  void forward(double* x) const {
    std::vector<Complex> y(static_cast<std::size_t>(2 * n_), Complex(0.0));
    for (Index j = 0; j < n_; ++j) y[static_cast<std::size_t>(j)] = Complex(x[j]);
    fft_.forward(y.data());
    for (Index k = 0; k < n_; ++k) {
      const double c = (phase_[static_cast<std::size_t>(k)] * y[static_cast<std::size_t>(k)]).real();
      x[k] = (k == 0 ? s0_ : sk_) * c;
    }
  }
  void adjoint(double* x) const {
    std::vector<Complex> h(static_cast<std::size_t>(2 * n_), Complex(0.0));
    for (Index k = 0; k < n_; ++k) {
      const double g = (k == 0 ? s0_ : sk_) * x[k];
      h[static_cast<std::size_t>(k)] = g * std::conj(phase_[static_cast<std::size_t>(k)]);
    }
    fft_.backward(h.data());
    for (Index j = 0; j < n_; ++j) x[j] = h[static_cast<std::size_t>(j)].real();
  }

 private:
  Index n_;
  Fft fft_;
  std::vector<Complex> phase_;
  double s0_, sk_;
};

// transforms.hpp:170-197
void wht(double* x, Index n) {
  for (Index len = 1; len < n; len <<= 1)
    for (Index i = 0; i < n; i += 2 * len)
      for (Index k = 0; k < len; ++k) {
        const double u = x[i + k], v = x[i + k + len];
        x[i + k] = u + v;
        x[i + k + len] = u - v;
      }
  const double scale = 1.0 / std::sqrt(static_cast<double>(n));
  for (Index j = 0; j < n; ++j) x[j] *= scale;
}

// mixing.hpp:55-111 — one mode's orthonormal/unitary transform.
template <class T>
class ModeTransform {
 public:
  ModeTransform(TransformKind kind, Index n) : kind_(kind), n_(n) {
    if constexpr (std::is_same_v<T, Complex>) {
      if (kind != TransformKind::fft && kind != TransformKind::identity)
        throw std::invalid_argument("real transform applied on complex path");
      if (kind == TransformKind::fft) {
        fft_ = std::make_unique<Fft>(n);
        scale_ = 1.0 / std::sqrt(static_cast<double>(n));
      }
    } else {
      if (kind == TransformKind::dct) dct_ = std::make_unique<Dct>(n);
      else if (kind == TransformKind::fft) throw std::invalid_argument("fft requires the complex path");
    }
  }
  void forward(T* v) const {
    if constexpr (std::is_same_v<T, Complex>) {
      if (!fft_) return;
      fft_->forward(v);
      for (Index i = 0; i < n_; ++i) v[i] *= scale_;
    } else {
      if (dct_) dct_->forward(v);
      else if (kind_ == TransformKind::wht) wht(v, n_);
    }
  }
  void adjoint(T* v) const {
    if constexpr (std::is_same_v<T, Complex>) {
      if (!fft_) return;
      fft_->backward(v);
      for (Index i = 0; i < n_; ++i) v[i] *= scale_;
    } else {
      if (dct_) dct_->adjoint(v);
      else if (kind_ == TransformKind::wht) wht(v, n_);
    }
  }

 private:
  TransformKind kind_;
  Index n_;
  double scale_ = 1.0;
  std::unique_ptr<Fft> fft_;
  std::unique_ptr<Dct> dct_;
};

template <class T>
void require_mix_scalar(TransformKind kind) {  // mixing.hpp:113-122
  if constexpr (std::is_same_v<T, Complex>) {
    if (kind != TransformKind::fft && kind != TransformKind::identity)
      throw std::invalid_argument("real transforms mix on the real path");
  } else {
    if (kind == TransformKind::fft) throw std::invalid_argument("fft mixing produces a complex tensor");
  }
}

}  // namespace

void dct_forward(double* x, Index n) { Dct(n).forward(x); }
void dct_adjoint(double* x, Index n) { Dct(n).adjoint(x); }
void fft_forward(Complex* x, Index n) { Fft(n).forward(x); }
void fft_backward(Complex* x, Index n) { Fft(n).backward(x); }
void wht_forward(double* x, Index n) {
  if (!is_pow2(n)) throw std::invalid_argument("wht length must be a power of two");
  wht(x, n);
}

// ------------------------------------------------------- mixing.hpp
// mixing.hpp:25-49
MixingOperator make_mixing_operator(const Shape& dims, TransformKind kind, std::uint64_t seed) {
  if (dims.empty()) throw std::invalid_argument("mixing: empty shape");
  if (kind == TransformKind::wht)
    for (Index d : dims)
      if (!is_pow2(d)) throw std::invalid_argument("wht requires power-of-two mode lengths");
  MixingOperator op;
  op.kind = kind;
  op.dims = dims;
  auto rng = seeded_engine(seed, kMixingStream);
  std::bernoulli_distribution coin(0.5);
  for (Index d : dims) {
    std::vector<double> s(static_cast<std::size_t>(d), 1.0);
    if (kind != TransformKind::identity)
      for (auto& v : s) v = coin(rng) ? 1.0 : -1.0;
    op.signs.push_back(std::move(s));
  }
  return op;
}

// mixing.hpp:130-156 — per mode, per fiber: sign, then forward transform.
template <class T>
static Tensor<T> mix_tensor_impl(const TensorD& x, const MixingOperator& op) {
  require_mix_scalar<T>(op.kind);
  if (x.dims != op.dims) throw std::invalid_argument("mix_tensor: operator shape mismatch");
  std::vector<T> buf(x.values.begin(), x.values.end());
  std::vector<T> fb;
  for (Index m = 0; m < x.order(); ++m) {
    const Index in = x.dim(m), stride = x.stride(m), blocks = x.size() / (stride * in);
    const auto& d = op.signs[static_cast<std::size_t>(m)];
    ModeTransform<T> t(op.kind, in);
    fb.resize(static_cast<std::size_t>(in));
    for (Index hi = 0; hi < blocks; ++hi)
      for (Index lo = 0; lo < stride; ++lo) {
        T* base = buf.data() + hi * stride * in + lo;
        for (Index i = 0; i < in; ++i) fb[static_cast<std::size_t>(i)] = base[i * stride] * d[static_cast<std::size_t>(i)];
        t.forward(fb.data());
        for (Index i = 0; i < in; ++i) base[i * stride] = fb[static_cast<std::size_t>(i)];
      }
  }
  return make_tensor<T>(x.dims, std::move(buf));
}
TensorD mix_tensor_real(const TensorD& x, const MixingOperator& op) { return mix_tensor_impl<double>(x, op); }
TensorCd mix_tensor_complex(const TensorD& x, const MixingOperator& op) { return mix_tensor_impl<Complex>(x, op); }

// mixing.hpp:159-174
template <class T>
Mat<T> mix_factor(const Matd& a, const MixingOperator& op, Index mode) {
  require_mix_scalar<T>(op.kind);
  const Index in = op.dims[static_cast<std::size_t>(mode)];
  if (a.rows != in) throw std::invalid_argument("mix_factor: row mismatch");
  const auto& d = op.signs[static_cast<std::size_t>(mode)];
  ModeTransform<T> t(op.kind, in);
  Mat<T> out(in, a.cols);
  for (Index r = 0; r < a.cols; ++r) {
    for (Index i = 0; i < in; ++i) out(i, r) = T(a(i, r) * d[static_cast<std::size_t>(i)]);
    t.forward(out.col(r));
  }
  return out;
}
template Mat<double> mix_factor(const Matd&, const MixingOperator&, Index);
template Mat<Complex> mix_factor(const Matd&, const MixingOperator&, Index);

// mixing.hpp:190-212
template <class T>
Matd unmix_factor(const Mat<T>& a_hat, const MixingOperator& op, Index mode) {
  const Index in = op.dims[static_cast<std::size_t>(mode)];
  if (a_hat.rows != in) throw std::invalid_argument("unmix_factor: row mismatch");
  const auto& d = op.signs[static_cast<std::size_t>(mode)];
  ModeTransform<T> t(op.kind, in);
  Mat<T> out(in, a_hat.cols);
  for (Index r = 0; r < a_hat.cols; ++r) {
    for (Index i = 0; i < in; ++i) out(i, r) = a_hat(i, r);
    t.adjoint(out.col(r));
    for (Index i = 0; i < in; ++i) out(i, r) *= d[static_cast<std::size_t>(i)];
  }
  Matd re(in, a_hat.cols);
  double mag2 = 0.0, im2 = 0.0;
  for (std::size_t k = 0; k < out.v.size(); ++k) {
    if constexpr (std::is_same_v<T, Complex>) {
      mag2 += std::norm(out.v[k]);
      im2 += out.v[k].imag() * out.v[k].imag();
      re.v[k] = out.v[k].real();
    } else {
      mag2 += out.v[k] * out.v[k];
      re.v[k] = out.v[k];
    }
  }
  const double mag = std::sqrt(mag2), residue = std::sqrt(im2);
  if (mag > 0 && residue > 1e-8 * mag)
    throw numerical_consistency_error("unmix_factor: imaginary residue exceeds tolerance");
  return re;
}
template Matd unmix_factor(const Mat<double>&, const MixingOperator&, Index);
template Matd unmix_factor(const Mat<Complex>&, const MixingOperator&, Index);

// mixing.hpp:218-236 — adjoint then sign along each length-I_n row.
template <class T>
Mat<T> unmix_sampled_rhs(const Mat<T>& g, const MixingOperator& op, Index mode) {
  require_mix_scalar<T>(op.kind);
  const Index in = op.dims[static_cast<std::size_t>(mode)];
  if (g.cols != in) throw std::invalid_argument("unmix_sampled_rhs: row-slice length mismatch");
  const auto& d = op.signs[static_cast<std::size_t>(mode)];
  ModeTransform<T> t(op.kind, in);
  Mat<T> out(g.rows, in);
  std::vector<T> row(static_cast<std::size_t>(in));
  for (Index j = 0; j < g.rows; ++j) {
    for (Index i = 0; i < in; ++i) row[static_cast<std::size_t>(i)] = g(j, i);
    t.adjoint(row.data());
    for (Index i = 0; i < in; ++i) out(j, i) = row[static_cast<std::size_t>(i)] * d[static_cast<std::size_t>(i)];
  }
  return out;
}
template Mat<double> unmix_sampled_rhs(const Mat<double>&, const MixingOperator&, Index);
template Mat<Complex> unmix_sampled_rhs(const Mat<Complex>&, const MixingOperator&, Index);

// mixing.hpp:242-254
Matd real_least_squares(const Matd& a, const Matd& b) { return least_squares(a, b); }
Matd real_least_squares(const Matcd& a, const Matcd& b) {
  if (a.rows != b.rows) throw std::invalid_argument("real_least_squares: row mismatch");
  Matd as(2 * a.rows, a.cols), bs(2 * b.rows, b.cols);
  for (Index j = 0; j < a.cols; ++j)
    for (Index i = 0; i < a.rows; ++i) {
      as(i, j) = a(i, j).real();
      as(i + a.rows, j) = a(i, j).imag();
    }
  for (Index j = 0; j < b.cols; ++j)
    for (Index i = 0; i < b.rows; ++i) {
      bs(i, j) = b(i, j).real();
      bs(i + b.rows, j) = b(i, j).imag();
    }
  return least_squares(as, bs);
}

namespace {

template <class T>
Mat<T> transpose_t(const Mat<T>& a) {
  Mat<T> t(a.cols, a.rows);
  for (Index j = 0; j < a.cols; ++j)
    for (Index i = 0; i < a.rows; ++i) t(j, i) = a(i, j);
  return t;
}

// mixing.hpp:258-318 — estimator on the ORIGINAL tensor, solve on the mixed
// one, fit on the unmixed model.
template <class T>
SolveResult cprand_mix_impl(const TensorD& x, Index r, Index s, const SolveOptions& opts,
                            const MixingOperator& op) {
  const auto t0 = Clock::now();
  SolveResult res;
  res.model = make_init(x, r, opts);
  auto sample_rng = seeded_engine(opts.rng_seed, kSamplingStream);
  auto fit_rng = seeded_engine(opts.rng_seed, kFitStream);
  auto norm_rng = seeded_engine(opts.rng_seed, kInitStream + 7);
  FitEstimator est;
  if (!opts.bench_mode)
    est = opts.exhaustive_samples
              ? exhaustive_fit_estimator(x, opts.stall_limit)
              : make_fit_estimator(x, opts.fit_sample_count, opts.stall_limit, fit_rng);
  const Tensor<T> x_hat = mix_tensor_impl<T>(x, op);
  const Index n_modes = x.order();
  std::vector<Mat<T>> mixed(static_cast<std::size_t>(n_modes));
  for (Index n = 0; n < n_modes; ++n)
    mixed[static_cast<std::size_t>(n)] = mix_factor<T>(res.model.factors[static_cast<std::size_t>(n)], op, n);
  res.setup_seconds = seconds_since(t0);
  for (int it = 1; it <= opts.max_iters; ++it) {
    for (Index n = 0; n < n_modes; ++n) {
      const SampleSet samples = opts.exhaustive_samples ? exhaustive_samples(x.dims, n)
                                                        : draw_samples(x.dims, n, s, sample_rng);
      const Mat<T> zs = skr(samples, mixed, n);
      const Mat<T> gathered = gather_fibers(x_hat, n, samples.idxs);
      const Mat<T> rhs = unmix_sampled_rhs<T>(transpose_t(gathered), op, n);
      res.model.factors[static_cast<std::size_t>(n)] = transpose(real_least_squares(zs, rhs));
      normalize_columns(res.model, n, n == 0, norm_rng);
      mixed[static_cast<std::size_t>(n)] = mix_factor<T>(res.model.factors[static_cast<std::size_t>(n)], op, n);
    }
    res.iterations = it;
    if (opts.bench_mode) continue;
    const double fit = opts.exact_fit_trace ? exact_fit(x, res.model) : estimate_fit(res.model, est);
    const StopDecision d = should_stop(est, fit, it, opts);
    res.trace.push_back({it, seconds_since(t0), fit, !opts.exact_fit_trace, est.best_fit});
    if (d.stop) {
      res.reason = d.reason;
      res.total_seconds = seconds_since(t0);
      return res;
    }
  }
  res.reason = opts.bench_mode ? StopReason::bench_complete : StopReason::max_iterations;
  res.total_seconds = seconds_since(t0);
  return res;
}

}  // namespace

// mixing.hpp:326-338
SolveResult cprand_mix(const TensorD& x, Index r, Index s, const SolveOptions& opts,
                       const MixingOperator& op) {
  opts.validate();
  if (r < 1) throw std::invalid_argument("rank must be >= 1");
  if (s < r) throw std::invalid_argument("sample count must be at least the rank");
  if (tensor_norm(x) == 0.0 && !opts.bench_mode) return zero_tensor_result(x, r, opts);
  if (op.kind == TransformKind::fft) return cprand_mix_impl<Complex>(x, r, s, opts, op);
  return cprand_mix_impl<double>(x, r, s, opts, op);
}

// mixing.hpp:340-345 — default transform is the FFT.
SolveResult cprand_mix(const TensorD& x, Index r, Index s, const SolveOptions& opts) {
  const TransformKind kind = opts.transform.value_or(TransformKind::fft);
  return cprand_mix(x, r, s, opts, make_mixing_operator(x.dims, kind, opts.rng_seed));
}

// mixing.hpp:351-370
SolveResult cprand_premix(const TensorD& x, Index r, Index s, const SolveOptions& opts,
                          const MixingOperator& op) {
  opts.validate();
  if (op.kind == TransformKind::fft) throw std::invalid_argument("premix requires a real orthogonal transform");
  if (tensor_norm(x) == 0.0 && !opts.bench_mode) return zero_tensor_result(x, r, opts);
  const auto t0 = Clock::now();
  const TensorD x_hat = mix_tensor_real(x, op);
  const double mix_seconds = seconds_since(t0);
  SolveResult res = cprand(x_hat, r, s, opts);
  for (Index n = 0; n < x.order(); ++n)
    res.model.factors[static_cast<std::size_t>(n)] =
        unmix_factor<double>(res.model.factors[static_cast<std::size_t>(n)], op, n);
  res.setup_seconds += mix_seconds;
  res.total_seconds += mix_seconds;
  for (TraceRecord& t : res.trace) t.elapsed_seconds += mix_seconds;
  return res;
}

// mixing.hpp:372-377 — default transform is DCT-II.
SolveResult cprand_premix(const TensorD& x, Index r, Index s, const SolveOptions& opts) {
  const TransformKind kind = opts.transform.value_or(TransformKind::dct);
  return cprand_premix(x, r, s, opts, make_mixing_operator(x.dims, kind, opts.rng_seed));
}

// kruskal.hpp:70-81 — dense reconstruction (tests only).
TensorD reconstruct_dense(const KruskalModel& m) {
  m.validate();
  const Shape dims = m.dims();
  const Index p = shape_size(dims), n = m.order(), r = m.rank();
  std::vector<double> v(static_cast<std::size_t>(p), 0.0);
  std::vector<Index> idx(static_cast<std::size_t>(n), 0);
  for (Index off = 0; off < p; ++off) {
    Index rem = off;
    for (Index k = 0; k < n; ++k) {
      idx[static_cast<std::size_t>(k)] = rem % dims[static_cast<std::size_t>(k)];
      rem /= dims[static_cast<std::size_t>(k)];
    }
    v[static_cast<std::size_t>(off)] = model_entry(m, idx.data());
  }
  (void)r;
  return make_tensor<double>(dims, std::move(v));
}

// ----------------------------------------------------- synthetic inputs
// BASELINE.json generator: A_n = G_n L^T, G_n iid N(0,1) from
// seeded_engine(seed, kSynthStream) (one normal_distribution across modes,
// column-major fill), L = chol((1-C) I + C 11^T); lambda = 1; noise from a
// counter-based Philox4x32-10 + Box-Muller so the GPU generator can produce
// the same stream entry by entry; X = X_true + eta ||X_true|| / ||N|| * N
// (noise scaling as synth.hpp:76-84).
void baseline_factors(const Shape& dims, Index r, double c, std::uint64_t seed,
                      std::vector<Matd>& out) {
  if (!(c >= 0.0 && c < 1.0)) throw std::invalid_argument("collinearity must be in [0, 1)");
  Matd l(r, r);
  for (Index j = 0; j < r; ++j) {
    double d = 1.0;
    for (Index k = 0; k < j; ++k) d -= l(j, k) * l(j, k);
    l(j, j) = std::sqrt(d);
    for (Index i = j + 1; i < r; ++i) {
      double s = c;
      for (Index k = 0; k < j; ++k) s -= l(i, k) * l(j, k);
      l(i, j) = s / l(j, j);
    }
  }
  auto rng = seeded_engine(seed, kSynthStream);
  std::normal_distribution<double> gauss(0.0, 1.0);
  out.clear();
  for (Index d : dims) {
    Matd g(d, r);
    for (Index j = 0; j < r; ++j)
      for (Index i = 0; i < d; ++i) g(i, j) = gauss(rng);
    Matd a(d, r);
    for (Index j = 0; j < r; ++j)
      for (Index i = 0; i < d; ++i) {
        double s = 0.0;
        for (Index k = 0; k <= j; ++k) s += g(i, k) * l(j, k);
        a(i, j) = s;
      }
    out.push_back(std::move(a));
  }
}

static void philox4x32_10(std::uint32_t ctr[4], std::uint32_t k0, std::uint32_t k1) {
  for (int round = 0; round < 10; ++round) {
    const std::uint64_t p0 = static_cast<std::uint64_t>(0xD2511F53u) * ctr[0];
    const std::uint64_t p1 = static_cast<std::uint64_t>(0xCD9E8D57u) * ctr[2];
    const std::uint32_t hi0 = static_cast<std::uint32_t>(p0 >> 32), lo0 = static_cast<std::uint32_t>(p0);
    const std::uint32_t hi1 = static_cast<std::uint32_t>(p1 >> 32), lo1 = static_cast<std::uint32_t>(p1);
    const std::uint32_t n0 = hi1 ^ ctr[1] ^ k0, n2 = hi0 ^ ctr[3] ^ k1;
    ctr[0] = n0;
    ctr[1] = lo1;
    ctr[2] = n2;
    ctr[3] = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

double philox_gaussian(std::uint64_t seed, std::uint64_t counter) {
  std::uint32_t c[4] = {static_cast<std::uint32_t>(counter), static_cast<std::uint32_t>(counter >> 32),
                        0x6E6F6973u, 0u};
  philox4x32_10(c, static_cast<std::uint32_t>(seed), static_cast<std::uint32_t>(seed >> 32) ^ 0x5EEDu);
  const std::uint64_t w1 = ((static_cast<std::uint64_t>(c[0]) << 32) | c[1]) >> 11;
  const std::uint64_t w2 = ((static_cast<std::uint64_t>(c[2]) << 32) | c[3]) >> 11;
  const double u1 = static_cast<double>(w1 + 1) * 0x1.0p-53;  // (0, 1]
  const double u2 = static_cast<double>(w2) * 0x1.0p-53;      // [0, 1)
  return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * kPi * u2);
}

BaselineSynth gen_baseline_problem(const Shape& dims, Index r, double c, double eta,
                                   std::uint64_t seed) {
  BaselineSynth out;
  baseline_factors(dims, r, c, seed, out.truth.factors);
  out.truth.lambda.assign(static_cast<std::size_t>(r), 1.0);
  const Index p = shape_size(dims), n = static_cast<Index>(dims.size());
  std::vector<double> xt(static_cast<std::size_t>(p));
  const int nt = max_threads();
  const Index chunk = (p + nt - 1) / nt;
  std::vector<std::thread> pool;
  std::vector<double> part_s(static_cast<std::size_t>(nt), 0.0), part_n(static_cast<std::size_t>(nt), 0.0);
  for (int t = 0; t < nt; ++t)
    pool.emplace_back([&, t] {
      const Index lo = t * chunk, hi = std::min(p, lo + chunk);
      std::vector<Index> idx(static_cast<std::size_t>(n));
      for (Index off = lo; off < hi; ++off) {
        Index rem = off;
        for (Index k = 0; k < n; ++k) {
          idx[static_cast<std::size_t>(k)] = rem % dims[static_cast<std::size_t>(k)];
          rem /= dims[static_cast<std::size_t>(k)];
        }
        double sum = 0.0;
        for (Index q = 0; q < r; ++q) {
          double prod = out.truth.factors[0](idx[0], q);
          for (Index k = 1; k < n; ++k) prod *= out.truth.factors[static_cast<std::size_t>(k)](idx[static_cast<std::size_t>(k)], q);
          sum += prod;
        }
        xt[static_cast<std::size_t>(off)] = sum;
      }
    });
  for (auto& th : pool) th.join();
  pool.clear();
  if (eta > 0.0) {
    std::vector<double> noise(static_cast<std::size_t>(p));
    for (int t = 0; t < nt; ++t)
      pool.emplace_back([&, t] {
        const Index lo = t * chunk, hi = std::min(p, lo + chunk);
        for (Index off = lo; off < hi; ++off) noise[static_cast<std::size_t>(off)] = philox_gaussian(seed, static_cast<std::uint64_t>(off));
      });
    for (auto& th : pool) th.join();
    const double signal = std::sqrt(sq_sum(xt.data(), p));
    const double nn = std::sqrt(sq_sum(noise.data(), p));
    const double scale = eta * signal / nn;
    for (Index i = 0; i < p; ++i) xt[static_cast<std::size_t>(i)] += scale * noise[static_cast<std::size_t>(i)];
  }
  (void)part_s;
  (void)part_n;
  out.tensor = make_tensor<double>(dims, std::move(xt));
  return out;
}

// synth.hpp:23-41 — Q L^T with Q the thin Householder Q of a Gaussian matrix.
static Matd gen_collinear_factor(Index i_dim, Index r, double c, std::mt19937_64& rng) {
  if (r < 1 || i_dim < r) throw std::invalid_argument("collinear factor needs 1 <= R <= I");
  if (!(c >= 0.0 && c < 1.0)) throw std::invalid_argument("collinearity must be in [0, 1)");
  std::normal_distribution<double> gauss(0.0, 1.0);
  Matd g(i_dim, r);
  for (Index col = 0; col < r; ++col)
    for (Index row = 0; row < i_dim; ++row) g(row, col) = gauss(rng);
  std::vector<double> tau(static_cast<std::size_t>(r));
  for (Index k = 0; k < r; ++k) {
    double t, beta;
    make_householder(g.col(k) + k, i_dim - k, 1, t, beta);
    tau[static_cast<std::size_t>(k)] = t;
    apply_householder_left(g.col(k) + k + 1, 1, t, i_dim - k, g.col(k + 1) + k, i_dim, r - k - 1);
  }
  Matd q(i_dim, r);
  for (Index j = 0; j < r; ++j) q(j, j) = 1.0;
  for (Index k = r - 1; k >= 0; --k)
    apply_householder_left(g.col(k) + k + 1, 1, tau[static_cast<std::size_t>(k)], i_dim - k,
                           q.v.data() + k, i_dim, r);
  Matd l(r, r);
  for (Index j = 0; j < r; ++j) {
    double d = 1.0;
    for (Index k = 0; k < j; ++k) d -= l(j, k) * l(j, k);
    l(j, j) = std::sqrt(d);
    for (Index i = j + 1; i < r; ++i) {
      double s = c;
      for (Index k = 0; k < j; ++k) s -= l(i, k) * l(j, k);
      l(i, j) = s / l(j, j);
    }
  }
  Matd a(i_dim, r);
  for (Index j = 0; j < r; ++j)
    for (Index i = 0; i < i_dim; ++i) {
      double s = 0.0;
      for (Index k = 0; k <= j; ++k) s += q(i, k) * l(j, k);
      a(i, j) = s;
    }
  return a;
}

// synth.hpp:60-85
SynthProblem gen_problem(const Shape& dims, Index rank, double c, double noise, std::uint64_t seed) {
  if (dims.empty()) throw std::invalid_argument("gen_problem: empty shape");
  if (noise < 0.0) throw std::invalid_argument("noise must be >= 0");
  auto rng = seeded_engine(seed, kSynthStream);
  SynthProblem p;
  for (Index d : dims) p.truth.factors.push_back(gen_collinear_factor(d, rank, c, rng));
  std::uniform_real_distribution<double> unif(0.2, 0.8);
  for (Index r = 0; r < rank; ++r) p.truth.lambda.push_back(unif(rng));
  TensorD xt = reconstruct_dense(p.truth);
  if (noise == 0.0) {
    p.tensor = std::move(xt);
    return p;
  }
  std::normal_distribution<double> gauss(0.0, 1.0);
  std::vector<double> nv(static_cast<std::size_t>(xt.size()));
  for (auto& v : nv) v = gauss(rng);
  const double signal = tensor_norm(xt);
  const double nn = std::sqrt(sq_sum(nv.data(), static_cast<Index>(nv.size())));
  if (signal > 0.0 && nn > 0.0) {
    const double sc = noise * signal / nn;
    for (std::size_t i = 0; i < nv.size(); ++i) xt.values[i] += sc * nv[i];
  }
  p.tensor = std::move(xt);
  return p;
}

// synth.hpp:146-185 — best matching of per-component cosine products.
double score(const KruskalModel& a, const KruskalModel& b) {
  const Index r = a.rank();
  Matd pair(r, r, 1.0);
  for (Index n = 0; n < a.order(); ++n) {
    const Matd& fa = a.factors[static_cast<std::size_t>(n)];
    const Matd& fb = b.factors[static_cast<std::size_t>(n)];
    for (Index i = 0; i < r; ++i) {
      const double na = stable_norm(fa.col(i), fa.rows);
      for (Index j = 0; j < r; ++j) {
        const double nb = stable_norm(fb.col(j), fb.rows);
        double dot = 0.0;
        for (Index k = 0; k < fa.rows; ++k) dot += fa(k, i) * fb(k, j);
        pair(i, j) *= (na > 0 && nb > 0) ? dot / (na * nb) : 0.0;
      }
    }
  }
  std::vector<Index> perm(static_cast<std::size_t>(r));
  std::iota(perm.begin(), perm.end(), Index{0});
  if (r <= 8) {
    double best = -std::numeric_limits<double>::infinity();
    do {
      double tot = 0.0;
      for (Index i = 0; i < r; ++i) tot += pair(i, perm[static_cast<std::size_t>(i)]);
      best = std::max(best, tot);
    } while (std::next_permutation(perm.begin(), perm.end()));
    return best / static_cast<double>(r);
  }
  // Hungarian (min-cost on -pair) with potentials.
  const Index nn = r;
  const double inf = std::numeric_limits<double>::infinity();
  std::vector<double> u(static_cast<std::size_t>(nn + 1)), v(static_cast<std::size_t>(nn + 1));
  std::vector<Index> p(static_cast<std::size_t>(nn + 1)), way(static_cast<std::size_t>(nn + 1));
  for (Index i = 1; i <= nn; ++i) {
    p[0] = i;
    Index j0 = 0;
    std::vector<double> minv(static_cast<std::size_t>(nn + 1), inf);
    std::vector<char> used(static_cast<std::size_t>(nn + 1), 0);
    do {
      used[static_cast<std::size_t>(j0)] = 1;
      const Index i0 = p[static_cast<std::size_t>(j0)];
      double delta = inf;
      Index j1 = 0;
      for (Index j = 1; j <= nn; ++j)
        if (!used[static_cast<std::size_t>(j)]) {
          const double cur = -pair(i0 - 1, j - 1) - u[static_cast<std::size_t>(i0)] - v[static_cast<std::size_t>(j)];
          if (cur < minv[static_cast<std::size_t>(j)]) {
            minv[static_cast<std::size_t>(j)] = cur;
            way[static_cast<std::size_t>(j)] = j0;
          }
          if (minv[static_cast<std::size_t>(j)] < delta) {
            delta = minv[static_cast<std::size_t>(j)];
            j1 = j;
          }
        }
      for (Index j = 0; j <= nn; ++j) {
        if (used[static_cast<std::size_t>(j)]) {
          u[static_cast<std::size_t>(p[static_cast<std::size_t>(j)])] += delta;
          v[static_cast<std::size_t>(j)] -= delta;
        } else {
          minv[static_cast<std::size_t>(j)] -= delta;
        }
      }
      j0 = j1;
    } while (p[static_cast<std::size_t>(j0)] != 0);
    do {
      const Index j1 = way[static_cast<std::size_t>(j0)];
      p[static_cast<std::size_t>(j0)] = p[static_cast<std::size_t>(j1)];
      j0 = j1;
    } while (j0);
  }
  double tot = 0.0;
  for (Index j = 1; j <= nn; ++j) tot += pair(p[static_cast<std::size_t>(j)] - 1, j - 1);
  return tot / static_cast<double>(r);
}

// bench-iter (tools/cprand_main.cpp:179-206, setup excluded from the rate)
// of cprand_mix_impl (mixing.hpp:258-318) on a tensor that is ALREADY mixed
// (the device-mixed C5 tensor, 84 GB: the reference's own setup would mix it
// again on the host for hours, and bench-iter does not time setup). The loop
// body is cprand_mix_impl's, bench mode (no estimator); the fibers are read
// in place from x_hat (no copy of the tensor). Real kinds (dct, wht) only.
// Returns the wall seconds of `iters` iterations. Test infrastructure (the
// cpu_baseline leg of bench.py), not part of the reference.
double bench_mix_premixed(const double* x_hat, const Shape& shape, Index r, Index s, TransformKind kind,
                          std::uint64_t seed, int iters) {
  {
    if (kind == TransformKind::fft) throw std::invalid_argument("real transforms only");
    const MixingOperator op = make_mixing_operator(shape, kind, seed);
    KruskalModel model = init_random(shape, r, seed);
    auto sample_rng = seeded_engine(seed, 2);
    auto norm_rng = seeded_engine(seed, 1 + 7);
    std::vector<Index> strides(shape.size());
    Index st = 1;
    for (std::size_t k = 0; k < shape.size(); ++k) {
      strides[k] = st;
      st *= shape[k];
    }
    std::vector<Matd> mixed(shape.size());
    for (std::size_t n = 0; n < shape.size(); ++n) mixed[n] = mix_factor<double>(model.factors[n], op, static_cast<Index>(n));
    const auto t0 = std::chrono::steady_clock::now();
    for (int it = 0; it < iters; ++it)
      for (Index n = 0; n < static_cast<Index>(shape.size()); ++n) {
        const SampleSet samples = draw_samples(shape, n, s, sample_rng);
        const Matd zs = skr(samples, mixed, n);
        // gather_fibers (tensor.hpp:188-212) from the caller's buffer
        const Index in = shape[static_cast<std::size_t>(n)], stn = strides[static_cast<std::size_t>(n)];
        Matd gathered(in, s);
        parallel_for(Index{0}, s, Index{1 << 14} / std::max<Index>(in, 1), [&](Index col) {
          Index base = 0, c = 0;
          for (Index k = 0; k < static_cast<Index>(shape.size()); ++k) {
            if (k == n) continue;
            base += samples.idxs(col, c++) * strides[static_cast<std::size_t>(k)];
          }
          double* dst = gathered.col(col);
          for (Index i = 0; i < in; ++i) dst[i] = x_hat[base + i * stn];
        });
        const Matd rhs = unmix_sampled_rhs<double>(transpose(gathered), op, n);
        model.factors[static_cast<std::size_t>(n)] = transpose(real_least_squares(zs, rhs));
        normalize_columns(model, n, n == 0, norm_rng);
        mixed[static_cast<std::size_t>(n)] = mix_factor<double>(model.factors[static_cast<std::size_t>(n)], op, n);
      }
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }
}


}  // namespace orc
