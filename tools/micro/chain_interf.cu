// Micro-benchmark: the exact Thomas forward recurrence (warp 0: b - a*w,
// reciprocal as in the kernels' fast path, w = c*inv, x = (d - a*x)*inv, rows
// from shared memory) while the other 8 warps of the CTA run one kind of work:
// 0 nothing, 1 DFMA chains, 2 FP64<->int conversions (F2I.F64.CEIL / I2F.F64),
// 3 LDG.128 from a small L1-resident table, 4 shared-memory loads/stores,
// 5 MUFU.RCP64H, 6 DADD/DMUL mix. One CTA per SM on every SM.
// nvcc -gencode arch=compute_100a,code=sm_100a --fmad=false -O3 chain_interf.cu -o chain_interf
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double rcp_seed(double x) {
  double r;
  asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  return r;
}

__global__ void __launch_bounds__(288, 1) k(double* out, long long* cyc, const double2* tab, int rows, int mode) {
  __shared__ double s[4][32][32];
  __shared__ double junk[8][32][4];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int r = warp; r < 32; r += 9) {
    s[0][r][lane] = -0.25 - 0.001 * lane;
    s[1][r][lane] = 2.0 + 0.01 * r;
    s[2][r][lane] = -0.5;
    s[3][r][lane] = 1.0 + r;
  }
  __shared__ volatile int done;
  if (threadIdx.x == 0) done = 0;
  __syncthreads();
  if (warp == 0) {
    double w = 0, x = 0;
    const long long t0 = clock64();
    for (int r = 0; r < rows; ++r) {
      const int q = r & 31;
      const double a = s[0][q][lane], b = s[1][q][lane], c = s[2][q][lane], d = s[3][q][lane];
      const double piv = b - a * w;
      const double inv = __drcp_rn(piv);
      w = c * inv;
      x = (d - a * x) * inv;
    }
    const long long t1 = clock64();
    done = 1;
    out[blockIdx.x * 32 + lane] = w + x;
    if (lane == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
    return;
  }
  double v = 1.0 + 1e-3 * threadIdx.x, u = 0.5;
  double h8[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) h8[q] = v + q;
  long long it = 0;
  while (!done) {
#pragma unroll 16
    for (int i = 0; i < 64; ++i) {
      switch (mode) {
        case 1: v = fma(v, 0.999, 1e-9); break;
        case 2: { const int kk = static_cast<int>(ceil(v * 3.7)); v = v - static_cast<double>(kk - 1) * 1e-9; } break;
        case 3: { const double2 p = tab[(static_cast<unsigned>(it * 7 + i * 13 + lane * 5)) & 511]; v += p.x * 1e-12; } break;
        case 4: junk[warp - 1][lane][i & 3] = v; v += junk[warp - 1][(lane + 3) & 31][(i + 1) & 3] * 1e-12; break;
        case 5: v = v + rcp_seed(v + 2.0) * 1e-9; break;
        case 6: v = v * 0.999 + u; u = u * 1.0001; break;
        case 7: {  // 8 independent DFMA chains per thread (high ILP)
#pragma unroll
          for (int q = 0; q < 8; ++q) h8[q] = fma(h8[q], 0.999, 1e-9);
        } break;
        case 8: {  // 8 independent conversion chains per thread
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int kk = static_cast<int>(ceil(h8[q] * 3.7));
            h8[q] = h8[q] - static_cast<double>(kk - 1) * 1e-9;
          }
        } break;
        case 9: {  // 8 independent DADD/DMUL chains
#pragma unroll
          for (int q = 0; q < 8; ++q) h8[q] = h8[q] * 0.999 + 1e-9;
        } break;
        default: break;
      }
    }
    ++it;
  }
#pragma unroll
  for (int q = 0; q < 8; ++q) v += h8[q];
  out[148 * 32 + blockIdx.x * 288 + threadIdx.x] = v;
}

int main() {
  double* d;
  long long* c;
  double2* tab;
  cudaMalloc(&d, sizeof(double) * 148 * 400);
  cudaMalloc(&c, 64);
  cudaMalloc(&tab, sizeof(double2) * 512);
  cudaMemset(tab, 0, sizeof(double2) * 512);
  const char* names[] = {"idle", "DFMA", "F2I/I2F", "LDG.128 L1", "LDS/STS", "MUFU.RCP64H", "DADD/DMUL",
                         "8x DFMA", "8x F2I/I2F", "8x DMUL+DADD"};
  const int rows = 20000;
  for (int mode = 0; mode < 10; ++mode) {
    long long h = 0;
    for (int rep = 0; rep < 2; ++rep) {
      k<<<148, 288>>>(d, c, tab, rows, mode);
      cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    }
    std::printf("producers %-12s: chain %.1f cycles/row (%s)\n", names[mode], h / (double)rows,
                cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
