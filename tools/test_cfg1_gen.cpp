// Checks tools/cfg1_gen.c against <random> (std::mt19937_64 +
// std::uniform_real_distribution<double>): prints "ok" when the first systems
// are identical. Built and run by tests/test_cfg1_gen.py.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <random>
#include <vector>

extern "C" void cfg1_generate(double* a, double* b, double* c, double* d, int64_t n,
                              int64_t batch, uint64_t seed);

int main() {
  const int64_t n = 1024, batch = 64;
  std::vector<double> a(n * batch), b(n * batch), c(n * batch), d(n * batch);
  cfg1_generate(a.data(), b.data(), c.data(), d.data(), n, batch, 2024);
  std::mt19937_64 rng(2024);
  std::uniform_real_distribution<double> neg(-1.0, 0.0), sym(-1.0, 1.0);
  long bad = 0;
  for (int64_t s = 0; s < batch; ++s)
    for (int64_t k = 0; k < n; ++k) {
      const double lo = k > 0 ? neg(rng) : 0.0;
      const double up = k < n - 1 ? neg(rng) : 0.0;
      const double rhs = sym(rng);
      const double diag = 2.05 + std::fabs(lo) + std::fabs(up);
      const int64_t o = s * n + k;
      if (a[o] != lo || c[o] != up || d[o] != rhs || b[o] != diag) ++bad;
    }
  std::printf(bad ? "mismatch %ld\n" : "ok\n", bad);
  return bad ? 1 : 0;
}
