// clock64 vs %globaltimer over a dependent FP64 chain (one warp, and with all
// SMs busy): the SM-cycle rate clock64 counts at, against wall time.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 clock_check.cu -o clock_check
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void chain(double* out, long long* res, double a, int n) {
  double x = a;
  const unsigned long long g0 = gt();
  const long long c0 = clock64();
  for (int i = 0; i < n; ++i) x = x * a + 1e-9;
  const long long c1 = clock64();
  const unsigned long long g1 = gt();
  out[blockIdx.x * blockDim.x + threadIdx.x] = x;
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    res[0] = c1 - c0;
    res[1] = static_cast<long long>(g1 - g0);
  }
}

int main() {
  double* d;
  long long* r;
  long long h[2];
  cudaMalloc(&d, sizeof(double) * 148 * 1024);
  cudaMalloc(&r, 16);
  for (int blocks : {1, 148}) {
    for (int rep = 0; rep < 3; ++rep) {
      chain<<<blocks, 32>>>(d, r, 0.999999, 2000000);
      cudaMemcpy(h, r, 16, cudaMemcpyDeviceToHost);
    }
    std::printf("%d CTA(s): clock64 %lld ticks over %lld ns -> %.1f MHz; %.2f ticks per DFMA-chain step\n",
                blocks, h[0], h[1], 1e3 * h[0] / h[1], h[0] / 2e6);
  }
  return 0;
}
