/* cfg1_gen.c -- configs[1]'s input data exactly as SURVEY 8(d) specifies it:
 * std::mt19937_64(2024); for each system s, then each row k:
 *   a = U[-1, 0] (k > 0), c = U[-1, 0] (k < n-1), rhs = U[-1, 1],
 *   b = 2.05 + |a| + |c|;  a[0] = c[n-1] = 0,
 * with std::uniform_real_distribution<double>'s libstdc++ arithmetic
 * (generate_canonical<double, 53> over one 64-bit draw: x / 2^64, clamped
 * below 1; then lo + (hi - lo) * u). Bench data generation (not the product,
 * not the oracle). Line-contiguous layout: system s, row k at s*n + k.
 * tools/test_cfg1_gen.cpp checks the stream against <random> itself. */
#include <stdint.h>

#define NN 312
#define MM 156

typedef struct {
  uint64_t mt[NN];
  int i;
} mt64;

static void mt64_seed(mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < NN; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->i = NN;
}

static uint64_t mt64_next(mt64* g) {
  static const uint64_t mag[2] = {0ULL, 0xB5026F5AA96619E9ULL};
  const uint64_t um = 0xFFFFFFFF80000000ULL, lm = 0x7FFFFFFFULL;
  if (g->i >= NN) {
    int k;
    uint64_t x;
    for (k = 0; k < NN - MM; ++k) {
      x = (g->mt[k] & um) | (g->mt[k + 1] & lm);
      g->mt[k] = g->mt[k + MM] ^ (x >> 1) ^ mag[x & 1ULL];
    }
    for (; k < NN - 1; ++k) {
      x = (g->mt[k] & um) | (g->mt[k + 1] & lm);
      g->mt[k] = g->mt[k + (MM - NN)] ^ (x >> 1) ^ mag[x & 1ULL];
    }
    x = (g->mt[NN - 1] & um) | (g->mt[0] & lm);
    g->mt[NN - 1] = g->mt[MM - 1] ^ (x >> 1) ^ mag[x & 1ULL];
    g->i = 0;
  }
  uint64_t x = g->mt[g->i++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}

static double uniform(mt64* g, double lo, double hi) {
  const double r = 18446744073709551616.0; /* 2^64 */
  double u = (double)mt64_next(g) / r;
  if (u >= 1.0) u = 0x1.fffffffffffffp-1; /* nextafter(1, 0) */
  return lo + (hi - lo) * u;
}

void cfg1_generate(double* a, double* b, double* c, double* d, int64_t n, int64_t batch,
                   uint64_t seed) {
  mt64 g;
  mt64_seed(&g, seed);
  for (int64_t s = 0; s < batch; ++s)
    for (int64_t k = 0; k < n; ++k) {
      const int64_t o = s * n + k;
      const double lo = k > 0 ? uniform(&g, -1.0, 0.0) : 0.0;
      const double up = k < n - 1 ? uniform(&g, -1.0, 0.0) : 0.0;
      const double rhs = uniform(&g, -1.0, 1.0);
      a[o] = lo;
      c[o] = up;
      d[o] = rhs;
      b[o] = 2.05 + (lo < 0 ? -lo : lo) + (up < 0 ? -up : up);
    }
}
