// Drop-in check: the reference's own call sequence (README "Library use",
// proj/README.md:96-104) compiled against include/cprand_b200/cprand.hpp
// and linked to libcprand_b200.so. Prints one CSV line for the pytest side.
#include <cprand_b200/cprand.hpp>

#include <cmath>
#include <cstdio>
#include <random>

int main() {
  using namespace cprand;
  const Shape dims{12, 11, 10};
  // rank-2 positive factors, as test_sampling.cpp:273-288
  std::mt19937_64 g(837);
  std::uniform_real_distribution<double> u(0.1, 1.0);
  std::vector<std::vector<double>> f(3);
  for (int n = 0; n < 3; ++n) {
    f[n].resize(static_cast<size_t>(dims[n] * 2));
    for (auto& v : f[n]) v = u(g);
  }
  std::vector<double> vals(12 * 11 * 10);
  for (Index k = 0; k < 10; ++k)
    for (Index j = 0; j < 11; ++j)
      for (Index i = 0; i < 12; ++i) {
        double s = 0;
        for (int r = 0; r < 2; ++r) s += f[0][i + 12 * r] * f[1][j + 11 * r] * f[2][k + 10 * r];
        vals[static_cast<size_t>(i + 12 * (j + 11 * k))] = s;
      }
  TensorD x(dims, vals);
  SolveOptions opts;
  opts.rng_seed = 7;
  opts.max_iters = 100;
  opts.stall_limit = 30;
  SolveResult res = cprand::cprand(x, 2, 60, opts);
  int bad = 0;
  try {
    cprand::cprand(x, 3, 2, opts);
  } catch (const std::invalid_argument&) {
    bad = 1;
  }
  std::printf("iters=%d,reason=%d,fit=%.17g,trace=%zu,invalid_caught=%d,dsc5=%lld\n", res.iterations,
              static_cast<int>(res.reason), res.trace.empty() ? -1.0 : res.trace.back().fit, res.trace.size(),
              bad, static_cast<long long>(default_sample_count(5)));
  return 0;
}
