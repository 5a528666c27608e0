// tridiag_batch.cu -- batched tridiagonal solves (BASELINE configs[1]).
//
// The reference's line solver is thomas_solve_inplace (tridiagonal.hpp:25-42):
//   inv = 1/b0; w0 = c0*inv; x0 = d0*inv
//   k>=1: piv = b[k] - a[k]*w[k-1]; inv = 1/piv; w[k] = c[k]*inv;
//         x[k] = (d[k] - a[k]*x[k-1])*inv
//   back: x[k] -= w[k]*x[k+1]
// Exact variants keep that operation order per system (thread per system,
// compiled with FMA contraction disabled via __dmul_rn/__dadd_rn-free code in
// this TU: see the Makefile --fmad=false rule for this file).
//
//   strided layout    (row k of system s at k*batch + s): lanes own adjacent
//                     systems, every row access is a coalesced 256-B warp load.
//   contiguous layout (row k of system s at s*n + k): each warp stages 32x32
//                     tiles (32 systems x 32 rows) through shared memory so
//                     global accesses stay coalesced while each thread walks
//                     its own system row by row.
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/pcgpu.h"
#include "adi_device.cuh"

namespace pcgpu {
extern unsigned long long g_launches;

namespace {

constexpr int kT = 32;
constexpr int kP = kT + 1;

// Strided layout, thread per system, rows software-pipelined in blocks of
// kB: the next block's bands are loaded while the current block's recurrence
// runs, so each thread keeps 4*kB independent loads in flight.
constexpr int kB = 8;
__global__ void __launch_bounds__(128)
    k_thomas_strided(const double* __restrict__ a, const double* __restrict__ b,
                     const double* __restrict__ c, const double* __restrict__ d,
                     double* __restrict__ x, double* __restrict__ w, int64_t n, int64_t batch,
                     unsigned long long* fail) {
  const int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s >= batch) return;
  double w_prev = 0.0, x_prev = 0.0;
  bool bad = false;
  double na[kB], nb[kB], nc[kB], nd[kB];
  auto load = [&](int64_t k0) {
#pragma unroll
    for (int q = 0; q < kB; ++q) {
      const int64_t k = k0 + q;
      if (k < n) {
        const int64_t o = k * batch + s;
        na[q] = __ldg(a + o);
        nb[q] = __ldg(b + o);
        nc[q] = __ldg(c + o);
        nd[q] = __ldg(d + o);
      }
    }
  };
  load(0);
  for (int64_t k0 = 0; k0 < n; k0 += kB) {
    double ca[kB], cb[kB], cc[kB], cd[kB];
#pragma unroll
    for (int q = 0; q < kB; ++q) { ca[q] = na[q]; cb[q] = nb[q]; cc[q] = nc[q]; cd[q] = nd[q]; }
    load(k0 + kB);
#pragma unroll
    for (int q = 0; q < kB; ++q) {
      const int64_t k = k0 + q;
      if (k < n) {
        const int64_t o = k * batch + s;
        double piv, xv;
        if (k == 0) {
          piv = cb[q];
          const double inv = 1.0 / piv;
          w_prev = cc[q] * inv;
          xv = cd[q] * inv;
        } else {
          piv = cb[q] - ca[q] * w_prev;
          const double inv = 1.0 / piv;
          w_prev = cc[q] * inv;
          xv = (cd[q] - ca[q] * x_prev) * inv;
        }
        bad |= piv == 0.0;
        w[o] = w_prev;
        x[o] = xv;
        x_prev = xv;
      }
    }
  }
  // back substitution, pipelined in reverse
  double nw[kB], nx[kB];
  auto loadb = [&](int64_t k0) {  // rows k0-kB+1 .. k0
#pragma unroll
    for (int q = 0; q < kB; ++q) {
      const int64_t k = k0 - q;
      if (k >= 0) {
        const int64_t o = k * batch + s;
        nw[q] = w[o];
        nx[q] = x[o];
      }
    }
  };
  loadb(n - 2);
  for (int64_t k0 = n - 2; k0 >= 0; k0 -= kB) {
    double cw[kB], cx[kB];
#pragma unroll
    for (int q = 0; q < kB; ++q) { cw[q] = nw[q]; cx[q] = nx[q]; }
    loadb(k0 - kB);
#pragma unroll
    for (int q = 0; q < kB; ++q) {
      const int64_t k = k0 - q;
      if (k >= 0) {
        x_prev = cx[q] - cw[q] * x_prev;
        x[k * batch + s] = x_prev;
      }
    }
  }
  if (bad) atomicMin(fail, static_cast<unsigned long long>(s));
}

// Contiguous layout: one warp = 32 systems; rows processed in 32-row tiles.
__global__ void __launch_bounds__(32)
    k_thomas_contig(const double* __restrict__ a, const double* __restrict__ b,
                    const double* __restrict__ c, const double* __restrict__ d,
                    double* __restrict__ x, double* __restrict__ w, int64_t n, int64_t batch,
                    unsigned long long* fail) {
  __shared__ double ta[kT][kP], tb[kT][kP], tc[kT][kP], td[kT][kP];
  const int lane = threadIdx.x;
  const int64_t s0 = static_cast<int64_t>(blockIdx.x) * kT;
  const int64_t s = s0 + lane;
  double w_prev = 0.0, x_prev = 0.0;
  bool bad = false;
  for (int64_t k0 = 0; k0 < n; k0 += kT) {
    // Coalesced tile load: lane = row within the tile.
    for (int q = 0; q < kT; ++q) {
      const int64_t sq = s0 + q, k = k0 + lane;
      if (sq < batch && k < n) {
        const int64_t o = sq * n + k;
        ta[q][lane] = a[o];
        tb[q][lane] = b[o];
        tc[q][lane] = c[o];
        td[q][lane] = d[o];
      }
    }
    __syncwarp();
    if (s < batch) {
      const int kend = static_cast<int>(n - k0 < kT ? n - k0 : kT);
      for (int kk = 0; kk < kend; ++kk) {
        const double bk = tb[lane][kk], ck = tc[lane][kk], dk = td[lane][kk];
        double piv, xv;
        if (k0 + kk == 0) {
          piv = bk;
          const double inv = 1.0 / piv;
          w_prev = ck * inv;
          xv = dk * inv;
        } else {
          const double ak = ta[lane][kk];
          piv = bk - ak * w_prev;
          const double inv = 1.0 / piv;
          w_prev = ck * inv;
          xv = (dk - ak * x_prev) * inv;
        }
        bad |= piv == 0.0;
        tb[lane][kk] = w_prev;  // reuse tiles as the w/x staging buffers
        td[lane][kk] = xv;
        x_prev = xv;
      }
    }
    __syncwarp();
    for (int q = 0; q < kT; ++q) {
      const int64_t sq = s0 + q, k = k0 + lane;
      if (sq < batch && k < n) {
        const int64_t o = sq * n + k;
        w[o] = tb[q][lane];
        x[o] = td[q][lane];
      }
    }
    __syncwarp();
  }
  // Back substitution, tiles in reverse.
  const int64_t last_tile = ((n - 1) / kT) * kT;
  for (int64_t k0 = last_tile; k0 >= 0; k0 -= kT) {
    for (int q = 0; q < kT; ++q) {
      const int64_t sq = s0 + q, k = k0 + lane;
      if (sq < batch && k < n) {
        const int64_t o = sq * n + k;
        tb[q][lane] = w[o];
        td[q][lane] = x[o];
      }
    }
    __syncwarp();
    if (s < batch) {
      const int kend = static_cast<int>(n - k0 < kT ? n - k0 : kT);
      for (int kk = kend - 1; kk >= 0; --kk) {
        if (k0 + kk == n - 1) continue;  // x[n-1] is final
        x_prev = td[lane][kk] - tb[lane][kk] * x_prev;
        td[lane][kk] = x_prev;
      }
    }
    __syncwarp();
    for (int q = 0; q < kT; ++q) {
      const int64_t sq = s0 + q, k = k0 + lane;
      if (sq < batch && k < n) x[sq * n + k] = td[q][lane];
    }
    __syncwarp();
  }
  if (s < batch && bad) atomicMin(fail, static_cast<unsigned long long>(s));
}

// dst[c * rows + r] = src[r * cols + c] (rows x cols -> cols x rows)
__global__ void k_tr(const double* __restrict__ src, int64_t rows, int64_t cols,
                     double* __restrict__ dst) {
  __shared__ double t[32][33];
  const int64_t c0 = static_cast<int64_t>(blockIdx.x) * 32, r0 = static_cast<int64_t>(blockIdx.y) * 32;
  const int lx = threadIdx.x & 31, ly = threadIdx.x >> 5;
  for (int rr = ly; rr < 32; rr += 8) {
    const int64_t r = r0 + rr, c = c0 + lx;
    if (r < rows && c < cols) t[rr][lx] = src[r * cols + c];
  }
  __syncthreads();
  for (int cc = ly; cc < 32; cc += 8) {
    const int64_t c = c0 + cc, r = r0 + lx;
    if (r < rows && c < cols) dst[c * rows + r] = t[lx][cc];
  }
}

void tr(const double* src, int64_t rows, int64_t cols, double* dst, cudaStream_t s) {
  dim3 grid(static_cast<unsigned>((cols + 31) / 32), static_cast<unsigned>((rows + 31) / 32));
  k_tr<<<grid, 256, 0, s>>>(src, rows, cols, dst);
  ++g_launches;
}

}  // namespace
}  // namespace pcgpu

extern "C" int pcgpu_tridiag_batch(const double* lower, const double* diag, const double* upper,
                                   const double* rhs, double* x, int64_t n, int64_t batch,
                                   int32_t layout, int32_t exact, void* stream,
                                   int64_t* failed_system) {
  using namespace pcgpu;
  (void)exact;  // the exact kernels are also the current fast path
  if (failed_system) *failed_system = -1;
  if (n < 1 || batch < 1 || !lower || !diag || !upper || !rhs || !x) return PCGPU_ERR_ARG;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  {
    // keep the stream-ordered pool's memory mapped between calls (the
    // scratch is ~1-6 GB for configs[1]; re-mapping it per call costs ms)
    static bool pool_set = false;
    int dev = 0;
    cudaMemPool_t pool;
    if (!pool_set && cudaGetDevice(&dev) == cudaSuccess &&
        cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
      pool_set = true;
    }
  }
  double* w = nullptr;
  unsigned long long* fail = nullptr;
  if (cudaMallocAsync(&w, sizeof(double) * static_cast<size_t>(n * batch), s) != cudaSuccess)
    return PCGPU_ERR_CUDA;
  if (cudaMallocAsync(&fail, sizeof(unsigned long long), s) != cudaSuccess) return PCGPU_ERR_CUDA;
  cudaMemsetAsync(fail, 0xff, sizeof(unsigned long long), s);
  if (layout == PCGPU_LAYOUT_STRIDED) {
    const int th = 128;
    k_thomas_strided<<<static_cast<unsigned>((batch + th - 1) / th), th, 0, s>>>(
        lower, diag, upper, rhs, x, w, n, batch, fail);
  } else if (exact == 2) {
    // legacy warp-tiled contiguous kernel (kept for comparison)
    k_thomas_contig<<<static_cast<unsigned>((batch + 31) / 32), 32, 0, s>>>(
        lower, diag, upper, rhs, x, w, n, batch, fail);
  } else {
    // Contiguous layout: transpose the bands to the strided layout (coalesced
    // 32x32 tiles), run the pipelined thread-per-system solve, transpose x
    // back. Same per-system arithmetic, so still bit-identical.
    double* tmp = nullptr;
    const size_t cells = static_cast<size_t>(n * batch);
    if (cudaMallocAsync(&tmp, sizeof(double) * cells * 5, s) != cudaSuccess) return PCGPU_ERR_CUDA;
    double* ta = tmp;
    double* tb = tmp + cells;
    double* tc = tmp + 2 * cells;
    double* td = tmp + 3 * cells;
    double* tx = tmp + 4 * cells;
    tr(lower, batch, n, ta, s);
    tr(diag, batch, n, tb, s);
    tr(upper, batch, n, tc, s);
    tr(rhs, batch, n, td, s);
    const int th = 128;
    k_thomas_strided<<<static_cast<unsigned>((batch + th - 1) / th), th, 0, s>>>(
        ta, tb, tc, td, tx, w, n, batch, fail);
    tr(tx, n, batch, x, s);
    cudaFreeAsync(tmp, s);
  }
  ++g_launches;
  unsigned long long hfail = ~0ull;
  cudaMemcpyAsync(&hfail, fail, sizeof hfail, cudaMemcpyDeviceToHost, s);
  cudaFreeAsync(w, s);
  cudaFreeAsync(fail, s);
  if (cudaStreamSynchronize(s) != cudaSuccess) return PCGPU_ERR_CUDA;
  if (hfail != ~0ull) {
    if (failed_system) *failed_system = static_cast<int64_t>(hfail);
    return PCGPU_ERR_ZERO_PIVOT;
  }
  return PCGPU_OK;
}
