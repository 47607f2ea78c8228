// CPU check of include/cprand_b200/io.hpp (no GPU calls): DNT1 tensor and
// model JSON round trips, and the reader's rejections. Prints "ok" or the
// first failure.
#include <cprand_b200/io.hpp>

#include <cstdio>
#include <sstream>

int main() {
  using namespace cprand;
  std::vector<double> vals(2 * 3 * 4);
  for (size_t i = 0; i < vals.size(); ++i) vals[i] = 0.1 * static_cast<double>(i) - 1.0 / 3.0;
  TensorD x(Shape{2, 3, 4}, vals);
  std::stringstream ts;
  write_tensor(ts, x);
  const TensorD y = read_tensor(ts);
  if (y.dims != x.dims || y.values != x.values) { std::puts("tensor round trip"); return 1; }
  KruskalModel m;
  m.lambda = {1.5, -2.25e-7};
  for (Index d : x.dims) {
    Matd a(d, 2);
    for (Index i = 0; i < d; ++i)
      for (Index q = 0; q < 2; ++q) a(i, q) = 1.0 / (1.0 + static_cast<double>(i + 7 * q)) - 0.3;
    m.factors.push_back(a);
  }
  std::stringstream ms;
  write_model(ms, m);
  const KruskalModel n = read_model(ms.str());
  if (n.lambda != m.lambda || n.factors.size() != m.factors.size()) { std::puts("model round trip"); return 1; }
  for (size_t k = 0; k < m.factors.size(); ++k)
    if (n.factors[k].v != m.factors[k].v || n.factors[k].rows != m.factors[k].rows) { std::puts("factor"); return 1; }
  int rejected = 0;
  for (const char* bad : {"{\"lambda\": [1], \"factors\": [[[1, 2]]]}", "{\"factors\": [[[1]]]}", "[1]"}) {
    try {
      read_model(bad);
    } catch (const std::invalid_argument&) {
      ++rejected;
    }
  }
  std::stringstream bad_t("DNT2");
  try {
    read_tensor(bad_t);
  } catch (const std::invalid_argument&) {
    ++rejected;
  }
  if (rejected != 4) { std::printf("rejected %d of 4\n", rejected); return 1; }
  std::puts("ok");
  return 0;
}
