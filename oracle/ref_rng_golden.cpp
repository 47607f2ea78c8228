// TEST INFRASTRUCTURE. Golden-vector generator built FROM THE REFERENCE
// SOURCE: includes /root/reference/proj/include/cprand/rng.hpp (the only
// reference header that compiles without Eigen) and prints, as JSON, the
// raw seeded_engine streams plus the libstdc++ distribution draws the
// reference path consumes (uniform_int for draw_samples / fit offsets,
// uniform_real for init_random, bernoulli for mixing signs, normal for the
// normalize zero-column path). Built by oracle/Makefile into oracle/_ref/;
// output committed as tests/golden/rng_golden.json by oracle/make_golden.py.
#include <cstdio>
#include <random>

#include "cprand/rng.hpp"

static void raw(std::uint64_t seed, std::uint64_t stream, int n, bool comma) {
  auto g = cprand::seeded_engine(seed, stream);
  std::printf("  {\"seed\": %llu, \"stream\": %llu, \"raw\": [", (unsigned long long)seed,
              (unsigned long long)stream);
  for (int i = 0; i < n; ++i) std::printf("%s\"%llu\"", i ? ", " : "", (unsigned long long)g());
  // uniform_int over [0, 99], [0, 79], [0, 999] — one distribution per range
  // consumed round-robin, as draw_samples does for three kept modes.
  std::uniform_int_distribution<long> d0(0, 99), d1(0, 79), d2(0, 999);
  std::printf("], \"uint_rr\": [");
  for (int i = 0; i < 3 * n; ++i) {
    long v = (i % 3 == 0) ? d0(g) : (i % 3 == 1) ? d1(g) : d2(g);
    std::printf("%s%ld", i ? ", " : "", v);
  }
  std::uniform_real_distribution<double> u(0.0, 1.0);
  std::printf("], \"ureal\": [");
  for (int i = 0; i < n; ++i) std::printf("%s%.17g", i ? ", " : "", u(g));
  std::bernoulli_distribution b(0.5);
  std::printf("], \"bern\": [");
  for (int i = 0; i < n; ++i) std::printf("%s%d", i ? ", " : "", b(g) ? 1 : 0);
  std::normal_distribution<double> nd(0.0, 1.0);
  std::printf("], \"normal\": [");
  for (int i = 0; i < n; ++i) std::printf("%s%.17g", i ? ", " : "", nd(g));
  std::printf("]}%s\n", comma ? "," : "");
}

int main() {
  std::printf("{\"source\": \"/root/reference/proj/include/cprand/rng.hpp\",\n \"streams\": [\n");
  const std::uint64_t seeds[] = {0, 1, 3, 17, 0xDEADBEEFull};
  const std::uint64_t streams[] = {cprand::kInitStream, cprand::kSamplingStream, cprand::kFitStream,
                                   cprand::kMixingStream, cprand::kSynthStream,
                                   cprand::kInitStream + 7};
  const int ns = 5, nt = 6;
  for (int i = 0; i < ns; ++i)
    for (int j = 0; j < nt; ++j) raw(seeds[i], streams[j], 24, !(i == ns - 1 && j == nt - 1));
  std::printf("]}\n");
  return 0;
}
