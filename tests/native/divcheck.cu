// divcheck: div_rn(a, b, RN(1/b)) (adi_device.cuh) against the IEEE division
// a / b, bit for bit, on random pairs spanning wide exponent ranges plus the
// special values. Prints "pairs mismatches" and exits 1 on any mismatch.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 divcheck.cu -o divcheck
#include <cstdio>
#include <cstdlib>

#include "../../paper_1912_03744_b200/csrc/adi_device.cuh"

using pcgpu::div_rn;

__device__ __forceinline__ unsigned long long mix(unsigned long long x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

// random double: sign, mantissa from the hash, exponent in [-emax, emax]
__device__ __forceinline__ double rnd(unsigned long long h, int emax) {
  const unsigned long long mant = h & 0xfffffffffffffull;
  const int e = static_cast<int>((h >> 52) % (2 * emax + 1)) - emax;
  const unsigned long long bits =
      (static_cast<unsigned long long>(e + 1023) << 52) | mant | ((h >> 63) << 63);
  return __longlong_as_double(static_cast<long long>(bits));
}

__global__ void check(unsigned long long seed, long long n, int emax_a, int emax_b,
                      unsigned long long* bad, double* example) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long k = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; k < n;
       k += stride) {
    const unsigned long long h1 = mix(seed ^ (2 * k)), h2 = mix(seed ^ (2 * k + 1));
    const double a = rnd(h1, emax_a);
    const double b = rnd(h2, emax_b);
    const double rb = __drcp_rn(b);
    const double q = div_rn(a, b, rb, true);
    const double r = a / b;
    if (__double_as_longlong(q) != __double_as_longlong(r)) {
      if (atomicAdd(bad, 1ull) == 0) {
        example[0] = a;
        example[1] = b;
      }
    }
  }
}

__global__ void specials(unsigned long long* bad) {
  // a: anything; b: the precondition's range [2^-100, 2^100] (both signs)
  const double va[] = {0.0, -0.0, 1.0, -1.0, 3.0, 1e-310, -1e-310, 1e308, -1e308,
                       __longlong_as_double(0x7ff0000000000000ll),
                       __longlong_as_double(static_cast<long long>(0xfff0000000000000ull)),
                       __longlong_as_double(0x7ff8000000000000ll), 0x1p-1022, 0x1p1023,
                       0x1p-800, 0x1p800, -0x1p-800, 0x1.fffffffffffffp-801, 7.0, 1.0 / 3.0};
  const double vb[] = {1.0, -1.0, 3.0, 0x1p-100, -0x1p-100, 0x1p100, 0x1.fffffffffffffp99,
                       7.0, 1.0 / 3.0, 1e-7, 1e3};
  const int na = sizeof(va) / sizeof(va[0]), nb = sizeof(vb) / sizeof(vb[0]);
  for (int i = threadIdx.x; i < na * nb; i += blockDim.x) {
    const double a = va[i / nb], b = vb[i % nb];
    const double q = div_rn(a, b, __drcp_rn(b), true), r = a / b;
    const bool both_nan = q != q && r != r;
    if (!both_nan && __double_as_longlong(q) != __double_as_longlong(r)) atomicAdd(bad, 1ull);
  }
}

int main(int argc, char** argv) {
  const long long n = argc > 1 ? atoll(argv[1]) : (1ll << 32);
  unsigned long long* bad;
  double* ex;
  cudaMalloc(&bad, 8);
  cudaMalloc(&ex, 16);
  cudaMemset(bad, 0, 8);
  // exponent ranges (a, b): physical values, and a up to the double range with
  // b within the precondition's [2^-100, 2^100]
  const int ranges[][2] = {{40, 40}, {200, 100}, {1000, 100}, {20, 8}};
  unsigned long long total_bad = 0, h;
  for (int r = 0; r < 4; ++r) {
    check<<<148 * 16, 256>>>(0x1234567ull + r, n / 4, ranges[r][0], ranges[r][1], bad, ex);
  }
  specials<<<1, 256>>>(bad);
  if (cudaDeviceSynchronize() != cudaSuccess) {
    printf("cuda error\n");
    return 2;
  }
  cudaMemcpy(&h, bad, 8, cudaMemcpyDeviceToHost);
  total_bad = h;
  double e[2];
  cudaMemcpy(e, ex, 16, cudaMemcpyDeviceToHost);
  printf("%lld %llu\n", n, total_bad);
  if (total_bad) printf("example a=%a b=%a\n", e[0], e[1]);
  return total_bad ? 1 : 0;
}
