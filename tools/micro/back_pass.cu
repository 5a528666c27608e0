// Micro-benchmark: the exact back substitution (x[i] -= w[i] x[i+1],
// out = base + x, NaN-ignoring line max) over rows held in shared memory, one
// warp, in the variants the short-line kernel can use.
// nvcc -gencode arch=compute_100a,code=sm_100a --fmad=false -O3 back_pass.cu -o back_pass
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double ref_max(double a, double b) { return a < b ? b : a; }

constexpr int kRows = 200;

template <int kVariant>
__global__ void back(double* __restrict__ out, long long* cyc, int ld) {
  extern __shared__ double s[];  // 4 arrays [kRows][32]
  const int lane = threadIdx.x;
  double* sw = s;
  double* sx = s + kRows * 32;
  double* sb = s + 2 * kRows * 32;
  double* st = s + 3 * kRows * 32;
  for (int r = 0; r < kRows; ++r) {
    sw[r * 32 + lane] = 0.25 + 0.001 * lane;
    sx[r * 32 + lane] = 1.0 + r;
    sb[r * 32 + lane] = 4.2;
    st[r * 32 + lane] = 5.0;
  }
  __syncwarp();
  double x_next = 0.0, dmax = 0.0;
  double* po = out + lane + static_cast<long long>(kRows - 1) * ld;
  const long long t0 = clock64();
  if (kVariant == 0) {  // as the kernel: loads, chain, global store, running max
#pragma unroll 4
    for (int i = kRows - 1; i >= 0; --i) {
      const double wv = sw[i * 32 + lane], xv = sx[i * 32 + lane];
      const double bv = sb[i * 32 + lane], tv = st[i * 32 + lane];
      const double xi = xv - wv * x_next;
      const double o = bv + xi;
      *po = o;
      po -= ld;
      dmax = ref_max(dmax, fabs(o - tv));
      x_next = xi;
    }
  } else if (kVariant == 1) {  // no global store
#pragma unroll 4
    for (int i = kRows - 1; i >= 0; --i) {
      const double wv = sw[i * 32 + lane], xv = sx[i * 32 + lane];
      const double bv = sb[i * 32 + lane], tv = st[i * 32 + lane];
      const double xi = xv - wv * x_next;
      const double o = bv + xi;
      dmax = ref_max(dmax, fabs(o - tv));
      x_next = xi;
    }
    *po = dmax;
  } else if (kVariant == 2) {  // chain only
#pragma unroll 4
    for (int i = kRows - 1; i >= 0; --i) {
      const double wv = sw[i * 32 + lane], xv = sx[i * 32 + lane];
      x_next = xv - wv * x_next;
    }
    *po = x_next;
  } else {  // loads of the next 4 rows ahead of the current 4 (software pipelined)
    double w[4], x[4], b[4], t[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      w[k] = sw[(kRows - 1 - k) * 32 + lane];
      x[k] = sx[(kRows - 1 - k) * 32 + lane];
      b[k] = sb[(kRows - 1 - k) * 32 + lane];
      t[k] = st[(kRows - 1 - k) * 32 + lane];
    }
    for (int i = kRows - 1; i >= 3; i -= 4) {
      double w2[4], x2[4], b2[4], t2[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int r = i - 4 - k >= 0 ? i - 4 - k : 0;
        w2[k] = sw[r * 32 + lane];
        x2[k] = sx[r * 32 + lane];
        b2[k] = sb[r * 32 + lane];
        t2[k] = st[r * 32 + lane];
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const double xi = x[k] - w[k] * x_next;
        const double o = b[k] + xi;
        *po = o;
        po -= ld;
        dmax = ref_max(dmax, fabs(o - t[k]));
        x_next = xi;
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        w[k] = w2[k];
        x[k] = x2[k];
        b[k] = b2[k];
        t[k] = t2[k];
      }
    }
  }
  const long long t1 = clock64();
  if (lane == 0) cyc[kVariant] = t1 - t0;
  out[lane] += dmax + x_next;
}

int main() {
  double* d;
  long long* c;
  long long h[8] = {};
  const int ld = 256;
  cudaMalloc(&d, sizeof(double) * ld * kRows);
  cudaMalloc(&c, 64);
  const int smem = 4 * kRows * 32 * 8;
  cudaFuncSetAttribute(back<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(back<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(back<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(back<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int rep = 0; rep < 2; ++rep) {
    back<0><<<1, 32, smem>>>(d, c, ld);
    back<1><<<1, 32, smem>>>(d, c, ld);
    back<2><<<1, 32, smem>>>(d, c, ld);
    back<3><<<1, 32, smem>>>(d, c, ld);
  }
  cudaMemcpy(h, c, 32, cudaMemcpyDeviceToHost);
  std::printf("back pass cycles/row: kernel form %.1f, no store %.1f, chain only %.1f, "
              "pipelined %.1f (%s)\n",
              h[0] / (double)kRows, h[1] / (double)kRows, h[2] / (double)kRows,
              h[3] / (double)kRows, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
