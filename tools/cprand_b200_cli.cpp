// cprand_b200: the reference's command-line front end (tools/cprand_main.cpp)
// for the B200 path. Same subcommands, options, file formats and output
// lines for the solve commands; the solve runs on the GPU through the C ABI
// (include/cprand_b200/cprand.hpp -> libcprand_b200.so).
//
//   cprand_b200 decompose --in X.dnt --rank R [--method rand|mix|premix]
//                [--samples S] [--fit-samples P] [--stall N] [--max-iters N]
//                [--fit-tol T] [--fit-threshold F] [--init random|hosvd]
//                [--transform fft|dct|wht] [--seed N] --out model.json
//                [--trace trace.csv] [--device D]
//   cprand_b200 bench-iter --in X.dnt --rank R [--method M]... [--samples S]
//                [--iters N] [--transform fft|dct|wht] [--seed N] [--out f.csv]
//   cprand_b200 eval --model M.json --in X.dnt [--truth T.json]
//                (exact fit on the GPU: mode-1 MTTKRP + Gram expansion;
//                 score: synth.hpp:146-185 on the host)
//
// Exit codes as the reference (cprand_main.cpp:365-386): 0 ok, 2 usage /
// invalid input / any other error, 3 numerical consistency error.
// `gen` and `bench-fitcheck` are not on the B200 path: use the
// reference's tool for them; the DNT1 files are the same.
#include <cprand_b200/cprand.hpp>
#include <cprand_b200/io.hpp>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <limits>
#include <iostream>
#include <map>
#include <optional>
#include <sstream>
#include <string>
#include <vector>

namespace {

using cprand::Index;

struct Args {
  std::map<std::string, std::vector<std::string>> kv;
  bool has(const std::string& k) const { return kv.count(k) > 0; }
  const std::string& one(const std::string& k) const {
    auto it = kv.find(k);
    if (it == kv.end() || it->second.empty()) throw std::invalid_argument("missing value for --" + k);
    return it->second.back();
  }
};

Args parse(int argc, char** argv, int first, const std::vector<std::string>& known) {
  Args a;
  for (int i = first; i < argc; ++i) {
    std::string s = argv[i];
    if (s.rfind("--", 0) != 0) throw std::invalid_argument("unexpected argument: " + s);
    s = s.substr(2);
    std::string val;
    const auto eq = s.find('=');
    if (eq != std::string::npos) {
      val = s.substr(eq + 1);
      s = s.substr(0, eq);
    } else {
      if (i + 1 >= argc) throw std::invalid_argument("missing value for --" + s);
      val = argv[++i];
    }
    if (std::find(known.begin(), known.end(), s) == known.end()) throw std::invalid_argument("unknown option --" + s);
    a.kv[s].push_back(val);
  }
  return a;
}

long long to_int(const std::string& v, const std::string& k) {
  char* end = nullptr;
  const long long x = std::strtoll(v.c_str(), &end, 10);
  if (!end || *end) throw std::invalid_argument("--" + k + " expects an integer, got " + v);
  return x;
}
double to_real(const std::string& v, const std::string& k) {
  char* end = nullptr;
  const double x = std::strtod(v.c_str(), &end);
  if (!end || *end) throw std::invalid_argument("--" + k + " expects a number, got " + v);
  return x;
}

enum class Method { als, rand, mix, premix };
Method method_of(const std::string& s) {
  if (s == "als") return Method::als;
  if (s == "rand") return Method::rand;
  if (s == "mix") return Method::mix;
  if (s == "premix") return Method::premix;
  throw std::invalid_argument("--method must be als | rand | mix | premix");
}
const char* method_name(Method m) {
  switch (m) {
    case Method::als: return "als";
    case Method::rand: return "rand";
    case Method::mix: return "mix";
    default: return "premix";
  }
}
cprand::TransformKind transform_of(const std::string& s) {
  if (s == "fft") return cprand::TransformKind::fft;
  if (s == "dct") return cprand::TransformKind::dct;
  if (s == "wht") return cprand::TransformKind::wht;
  throw std::invalid_argument("--transform must be fft | dct | wht");
}
const char* stop_name(cprand::StopReason r) {
  switch (r) {
    case cprand::StopReason::max_iterations: return "max_iterations";
    case cprand::StopReason::fit_stagnation: return "fit_stagnation";
    case cprand::StopReason::fit_threshold: return "fit_threshold";
    case cprand::StopReason::best_fit_stall: return "best_fit_stall";
    case cprand::StopReason::zero_tensor: return "zero_tensor";
    default: return "bench_complete";
  }
}

cprand::SolveResult dispatch(Method m, const cprand::TensorD& x, Index r, Index s, const cprand::SolveOptions& o) {
  switch (m) {
    case Method::rand: return cprand::cprand(x, r, s, o);
    case Method::mix: return cprand::cprand_mix(x, r, s, o);
    case Method::premix: return cprand::cprand_premix(x, r, s, o);
    default:
      throw std::invalid_argument("--method als (exact CP-ALS) is outside the B200 path; use rand, mix or premix");
  }
}

int run_decompose(const Args& a) {
  const Method m = a.has("method") ? method_of(a.one("method")) : Method::als;
  const Index r = to_int(a.one("rank"), "rank");
  if (r < 1) throw std::invalid_argument("--rank must be positive");
  const bool transform_given = a.has("transform");
  if (m == Method::rand && transform_given) std::cerr << "warning: --transform has no effect with --method rand\n";
  cprand::SolveOptions o;
  if (a.has("max-iters")) o.max_iters = static_cast<int>(to_int(a.one("max-iters"), "max-iters"));
  if (a.has("fit-tol")) o.fit_tolerance = to_real(a.one("fit-tol"), "fit-tol");
  if (a.has("fit-threshold")) o.fit_threshold = to_real(a.one("fit-threshold"), "fit-threshold");
  if (a.has("seed")) o.rng_seed = static_cast<std::uint64_t>(to_int(a.one("seed"), "seed"));
  if (a.has("init")) {
    const std::string& v = a.one("init");
    if (v == "hosvd") o.init = cprand::InitKind::hosvd;
    else if (v != "random") throw std::invalid_argument("--init must be random | hosvd");
  }
  if (a.has("fit-samples")) o.fit_sample_count = to_int(a.one("fit-samples"), "fit-samples");
  if (a.has("stall")) o.stall_limit = static_cast<int>(to_int(a.one("stall"), "stall"));
  if (transform_given) o.transform = transform_of(a.one("transform"));
  if (a.has("device")) o.device = static_cast<int>(to_int(a.one("device"), "device"));
  const Index s = a.has("samples") && to_int(a.one("samples"), "samples") > 0 ? to_int(a.one("samples"), "samples")
                                                                                : cprand::default_sample_count(r);
  const cprand::TensorD x = cprand::read_tensor_file(a.one("in"));
  const cprand::SolveResult res = dispatch(m, x, r, s, o);
  cprand::write_model_file(a.one("out"), res.model);
  if (a.has("trace")) {
    std::ofstream os(a.one("trace"));
    if (!os) throw std::invalid_argument("cannot open for write: " + a.one("trace"));
    cprand::write_trace_csv(os, res.trace);
  }
  std::cout << std::setprecision(17);
  std::cout << "method=" << method_name(m) << " iters=" << res.iterations << " fit=";
  // the reference reports the exact fit when there is no trace (cprand_main.cpp:157-160)
  std::cout << (res.trace.empty() ? cprand::exact_fit(x, res.model) : res.trace.back().fit);
  std::cout << " time_s=" << res.total_seconds << " stop=" << stop_name(res.reason) << '\n';
  return 0;
}

int run_bench_iter(const Args& a) {
  std::vector<Method> methods;
  if (a.has("method"))
    for (const auto& v : a.kv.at("method")) methods.push_back(method_of(v));
  else
    methods = {Method::rand};  // the reference's default pair is (als, rand); als is not on this path
  const Index r = to_int(a.one("rank"), "rank");
  if (r < 1) throw std::invalid_argument("--rank must be positive");
  const int iters = a.has("iters") ? static_cast<int>(to_int(a.one("iters"), "iters")) : 100;
  if (iters < 1) throw std::invalid_argument("--iters must be positive");
  const Index s = a.has("samples") && to_int(a.one("samples"), "samples") > 0 ? to_int(a.one("samples"), "samples")
                                                                                : cprand::default_sample_count(r);
  const cprand::TensorD x = cprand::read_tensor_file(a.one("in"));
  std::ostringstream csv;
  csv << std::setprecision(17) << "method,iters,setup_s,mean_iter_s\n";
  for (Method m : methods) {
    cprand::SolveOptions o;
    o.max_iters = iters;
    o.bench_mode = true;
    if (a.has("seed")) o.rng_seed = static_cast<std::uint64_t>(to_int(a.one("seed"), "seed"));
    if (a.has("transform")) o.transform = transform_of(a.one("transform"));
    const cprand::SolveResult res = dispatch(m, x, r, s, o);
    const double iter_total = res.total_seconds - res.setup_seconds;
    csv << method_name(m) << ',' << res.iterations << ',' << res.setup_seconds << ','
        << iter_total / std::max(res.iterations, 1) << '\n';
  }
  if (a.has("out")) {
    std::ofstream os(a.one("out"));
    if (!os) throw std::invalid_argument("cannot open for write: " + a.one("out"));
    os << csv.str();
  } else {
    std::cout << csv.str();
  }
  return 0;
}

// score (synth.hpp:146-185): best matching of the per-component products of
// column cosines over the modes; exhaustive for R <= 8, Hungarian beyond
std::vector<int> hungarian_min(const std::vector<double>& cost, int n) {
  const double inf = std::numeric_limits<double>::infinity();
  std::vector<double> u(n + 1, 0.0), v(n + 1, 0.0), minv(n + 1);
  std::vector<int> p(n + 1, 0), way(n + 1, 0);
  std::vector<char> used(n + 1);
  for (int i = 1; i <= n; ++i) {
    p[0] = i;
    int j0 = 0;
    std::fill(minv.begin(), minv.end(), inf);
    std::fill(used.begin(), used.end(), 0);
    do {
      used[j0] = 1;
      const int i0 = p[j0];
      double delta = inf;
      int j1 = 0;
      for (int j = 1; j <= n; ++j)
        if (!used[j]) {
          const double cur = cost[static_cast<size_t>((i0 - 1) * n + (j - 1))] - u[i0] - v[j];
          if (cur < minv[j]) {
            minv[j] = cur;
            way[j] = j0;
          }
          if (minv[j] < delta) {
            delta = minv[j];
            j1 = j;
          }
        }
      for (int j = 0; j <= n; ++j)
        if (used[j]) {
          u[p[j]] += delta;
          v[j] -= delta;
        } else {
          minv[j] -= delta;
        }
      j0 = j1;
    } while (p[j0] != 0);
    do {
      const int j1 = way[j0];
      p[j0] = p[j1];
      j0 = j1;
    } while (j0);
  }
  std::vector<int> match(n);
  for (int j = 1; j <= n; ++j) match[p[j] - 1] = j - 1;
  return match;
}

double score(const cprand::KruskalModel& a, const cprand::KruskalModel& b) {
  if (a.order() != b.order() || a.rank() != b.rank()) throw std::invalid_argument("score: models must share dims and rank");
  const int r = static_cast<int>(a.rank());
  std::vector<double> ps(static_cast<size_t>(r * r), 1.0);
  for (Index n = 0; n < a.order(); ++n) {
    const cprand::Matd& fa = a.factors[static_cast<size_t>(n)];
    const cprand::Matd& fb = b.factors[static_cast<size_t>(n)];
    if (fa.rows != fb.rows) throw std::invalid_argument("score: models must share dims and rank");
    auto norm = [](const cprand::Matd& f, int c) {
      double s2 = 0.0;
      for (Index i = 0; i < f.rows; ++i) s2 += f(i, c) * f(i, c);
      return std::sqrt(s2);
    };
    for (int i = 0; i < r; ++i)
      for (int j = 0; j < r; ++j) {
        const double na = norm(fa, i), nb = norm(fb, j);
        double dot = 0.0;
        for (Index k = 0; k < fa.rows; ++k) dot += fa(k, i) * fb(k, j);
        ps[static_cast<size_t>(i * r + j)] *= (na > 0 && nb > 0) ? dot / (na * nb) : 0.0;
      }
  }
  double total = 0.0;
  if (r <= 8) {
    std::vector<int> perm(static_cast<size_t>(r));
    for (int i = 0; i < r; ++i) perm[static_cast<size_t>(i)] = i;
    double best = -std::numeric_limits<double>::infinity();
    do {
      double t = 0.0;
      for (int i = 0; i < r; ++i) t += ps[static_cast<size_t>(i * r + perm[static_cast<size_t>(i)])];
      best = std::max(best, t);
    } while (std::next_permutation(perm.begin(), perm.end()));
    total = best;
  } else {
    std::vector<double> neg(ps.size());
    for (size_t e = 0; e < ps.size(); ++e) neg[e] = -ps[e];
    const auto m = hungarian_min(neg, r);
    for (int i = 0; i < r; ++i) total += ps[static_cast<size_t>(i * r + m[static_cast<size_t>(i)])];
  }
  return total / r;
}

int run_eval(const Args& a) {
  const cprand::KruskalModel m = cprand::read_model_file(a.one("model"));
  const cprand::TensorD x = cprand::read_tensor_file(a.one("in"));
  std::cout << std::setprecision(17);
  std::cout << "fit," << cprand::exact_fit(x, m) << '\n';
  if (a.has("truth")) std::cout << "score," << score(m, cprand::read_model_file(a.one("truth"))) << '\n';
  return 0;
}

void usage(std::ostream& os) {
  os << "usage: cprand_b200 decompose --in X.dnt --rank R --method rand|mix|premix --out model.json [options]\n"
        "       cprand_b200 bench-iter --in X.dnt --rank R [--method M]... [--iters N] [options]\n"
        "       cprand_b200 eval --model M.json --in X.dnt [--truth T.json]\n";
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2 || std::string(argv[1]) == "--help" || std::string(argv[1]) == "-h") {
    usage(argc < 2 ? std::cerr : std::cout);
    return argc < 2 ? 2 : 0;
  }
  const std::string cmd = argv[1];
  try {
    if (cmd == "decompose") {
      const Args a = parse(argc, argv, 2,
                           {"in", "method", "rank", "samples", "fit-samples", "stall", "max-iters", "fit-tol",
                            "fit-threshold", "init", "transform", "seed", "out", "trace", "device"});
      for (const char* req : {"in", "rank", "out"})
        if (!a.has(req)) throw std::invalid_argument(std::string("--") + req + " is required");
      return run_decompose(a);
    }
    if (cmd == "bench-iter") {
      const Args a = parse(argc, argv, 2, {"in", "method", "rank", "samples", "iters", "transform", "seed", "out"});
      for (const char* req : {"in", "rank"})
        if (!a.has(req)) throw std::invalid_argument(std::string("--") + req + " is required");
      return run_bench_iter(a);
    }
    if (cmd == "eval") {
      const Args a = parse(argc, argv, 2, {"model", "truth", "in"});
      for (const char* req : {"model", "in"})
        if (!a.has(req)) throw std::invalid_argument(std::string("--") + req + " is required");
      return run_eval(a);
    }
    if (cmd == "gen" || cmd == "bench-fitcheck") {
      std::cerr << "error: '" << cmd << "' is not on the B200 path; use the reference's tool (same DNT1 files)\n";
      return 2;
    }
    usage(std::cerr);
    return 2;
  } catch (const cprand::numerical_consistency_error& e) {
    std::cerr << "numerical consistency error: " << e.what() << '\n';
    return 3;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << '\n';
    return 2;
  }
}
