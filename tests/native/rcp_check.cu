// rcp_check: the branch-free reciprocal rcp_rn_nb (adi_device.cuh) against
// __drcp_rn, bit for bit, on random doubles over the range rcp_rn_nb accepts
// (and the flag on the ones it rejects), plus the per-row cost of the exact
// Thomas forward recurrence with each reciprocal (one warp, data in smem).
// built by tests/native/Makefile (target rcp_check); run by tests/test_divcheck.py
#include <cstdio>
#include <cstdlib>

#include "../../paper_1912_03744_b200/csrc/adi_device.cuh"

using pcgpu::rcp_rn_nb;

__device__ __forceinline__ unsigned long long mix(unsigned long long x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

// random double: sign and mantissa from the hash, biased exponent in [elo, ehi];
// every 4th value gets an extreme mantissa (all ones / all zeros / one bit)
__device__ __forceinline__ double rnd(unsigned long long h, int elo, int ehi) {
  unsigned long long mant = h & 0xfffffffffffffull;
  const int sel = static_cast<int>((h >> 60) & 7);
  if (sel == 0) mant = 0xfffffffffffffull ^ ((h >> 20) & 0xff);
  if (sel == 1) mant = (h >> 20) & 0xff;
  const int e = elo + static_cast<int>((h >> 52) % (ehi - elo + 1));
  const unsigned long long bits =
      (static_cast<unsigned long long>(e) << 52) | mant | ((h >> 63) << 63);
  return __longlong_as_double(static_cast<long long>(bits));
}

__global__ void check(unsigned long long seed, long long n, int elo, int ehi,
                      unsigned long long* cnt, double* example) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long k = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; k < n;
       k += stride) {
    const double x = rnd(mix(seed ^ k), elo, ehi);
    bool bad = false;
    const double r = rcp_rn_nb(x, bad);
    if (bad) {
      atomicAdd(cnt + 1, 1ull);
    } else if (__double_as_longlong(r) != __double_as_longlong(__drcp_rn(x))) {
      if (atomicAdd(cnt, 1ull) == 0) example[0] = x;
    }
  }
}

// specials: all must be flagged (zero, subnormal, huge, inf, nan)
__global__ void specials(unsigned long long* cnt) {
  const double v[] = {0.0, -0.0, 1e-310, -1e-310, 0x1p-1022, 0x1p1023, -0x1p1023,
                      __longlong_as_double(0x7ff0000000000000ll),
                      __longlong_as_double(static_cast<long long>(0xfff0000000000000ull)),
                      __longlong_as_double(0x7ff8000000000000ll)};
  for (int i = threadIdx.x; i < static_cast<int>(sizeof(v) / sizeof(v[0])); i += blockDim.x) {
    bool bad = false;
    (void)rcp_rn_nb(v[i], bad);
    if (!bad) atomicAdd(cnt + 2, 1ull);
  }
}

template <bool kNb>
__global__ void thomas(double* out, long long* cyc, int rows) {
  __shared__ double s[4][32][32];
  const int lane = threadIdx.x;
  for (int r = 0; r < 32; ++r) {
    s[0][r][lane] = -0.25 - 0.001 * lane;
    s[1][r][lane] = 2.0 + 0.01 * r;
    s[2][r][lane] = -0.5;
    s[3][r][lane] = 1.0 + r;
  }
  __syncwarp();
  double w = 0, x = 0;
  bool bad = false;
  long long t0 = clock64();
  for (int r = 0; r < rows; ++r) {
    const int q = r & 31;
    const double a = s[0][q][lane], b = s[1][q][lane], c = s[2][q][lane], d = s[3][q][lane];
    const double piv = b - a * w;
    const double inv = kNb ? rcp_rn_nb(piv, bad) : __drcp_rn(piv);
    w = c * inv;
    x = (d - a * x) * inv;
  }
  long long t1 = clock64();
  out[lane] = w + x + (bad ? 1.0 : 0.0);
  if (lane == 0) cyc[0] = t1 - t0;
}

int main(int argc, char** argv) {
  const long long n = argc > 1 ? atoll(argv[1]) : (1ll << 32);
  unsigned long long* cnt;
  double *ex, *d;
  long long* cyc;
  cudaMalloc(&cnt, 24);
  cudaMalloc(&ex, 8);
  cudaMalloc(&d, 32 * 8);
  cudaMalloc(&cyc, 8);
  cudaMemset(cnt, 0, 24);
  // biased exponent ranges: the physical range, the whole accepted range and
  // beyond it (flagged values are not compared)
  const int ranges[][2] = {{1023 - 60, 1023 + 60}, {1, 2046}, {0x018, 0x7e6}};
  for (int r = 0; r < 3; ++r)
    check<<<148 * 16, 256>>>(0x51ed27ull + r, n / 3, ranges[r][0], ranges[r][1], cnt, ex);
  specials<<<1, 32>>>(cnt);
  unsigned long long h[3];
  double e = 0;
  cudaMemcpy(h, cnt, 24, cudaMemcpyDeviceToHost);
  cudaMemcpy(&e, ex, 8, cudaMemcpyDeviceToHost);
  const cudaError_t err = cudaDeviceSynchronize();
  printf("values %lld mismatches %llu flagged %llu unflagged-specials %llu%s", n, h[0], h[1],
         h[2], h[0] ? "" : "\n");
  if (h[0]) printf(" (e.g. x = %a)\n", e);
  long long c0 = 0, c1 = 0;
  const int rows = 16384;
  thomas<false><<<1, 32>>>(d, cyc, rows);
  thomas<false><<<1, 32>>>(d, cyc, rows);
  cudaMemcpy(&c0, cyc, 8, cudaMemcpyDeviceToHost);
  thomas<true><<<1, 32>>>(d, cyc, rows);
  thomas<true><<<1, 32>>>(d, cyc, rows);
  cudaMemcpy(&c1, cyc, 8, cudaMemcpyDeviceToHost);
  printf("thomas forward cycles/row: __drcp_rn %.1f  rcp_rn_nb %.1f\n", c0 / (double)rows,
         c1 / (double)rows);
  return (err != cudaSuccess || h[0] || h[2]) ? 1 : 0;
}
