// Micro-benchmark: FP64 dependent-chain latencies on the current GPU and the
// per-row cost of the exact Thomas recurrence (one warp, data in smem).
// nvcc -gencode arch=compute_100a,code=sm_100a --fmad=false -O3 fp64_lat.cu -o fp64_lat
#include <cstdio>
#include <cuda_runtime.h>

__global__ void chain(double* out, long long* cyc, double a, double b, int n) {
  double x = a, y = b;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = x * y;  // DMUL chain
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) x = x + y;  // DADD chain
  long long t2 = clock64();
  for (int i = 0; i < n; ++i) x = __fma_rn(x, y, a);  // DFMA chain
  long long t3 = clock64();
  for (int i = 0; i < n; ++i) x = __drcp_rn(x + 1.0);  // rcp chain
  long long t4 = clock64();
  for (int i = 0; i < n; ++i) x = a / x;  // div chain
  long long t5 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4;
  }
}

// Thomas forward/backward recurrences over rows held in smem, one warp.
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
  long long t0 = clock64();
  for (int r = 0; r < rows; ++r) {
    const int q = r & 31;
    const double a = s[0][q][lane], b = s[1][q][lane], c = s[2][q][lane], d = s[3][q][lane];
    const double piv = b - a * w;
    const double inv = __drcp_rn(piv);
    w = c * inv;
    x = (d - a * x) * inv;
  }
  long long t1 = clock64();
  double xn = 0, m = 0;
  for (int r = 0; r < rows; ++r) {
    const int q = r & 31;
    const double wv = s[0][q][lane], xv = s[1][q][lane];
    xn = xv - wv * xn;
    const double o = s[2][q][lane] + xn;
    m = fmax(m, fabs(o - s[3][q][lane]));
  }
  long long t2 = clock64();
  out[lane] = w + x + m + xn;
  if (lane == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; }
}

int main() {
  double* d; long long* c; long long h[8];
  cudaMalloc(&d, 1024 * 8); cudaMalloc(&c, 64);
  const int n = 4096;
  chain<<<1, 32>>>(d, c, 1.0000001, 0.9999999, n);
  chain<<<1, 32>>>(d, c, 1.0000001, 0.9999999, n);
  cudaMemcpy(h, c, 40, cudaMemcpyDeviceToHost);
  printf("cycles/op: DMUL %.1f DADD %.1f DFMA %.1f drcp_rn(x+1) %.1f div %.1f\n", h[0] / (double)n,
         h[1] / (double)n, h[2] / (double)n, h[3] / (double)n, h[4] / (double)n);
  const int rows = 16384;
  thomas<<<1, 32>>>(d, c, rows);
  thomas<<<1, 32>>>(d, c, rows);
  cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost);
  printf("thomas cycles/row: forward %.1f backward %.1f\n", h[0] / (double)rows, h[1] / (double)rows);
  return 0;
}
