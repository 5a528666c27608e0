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
//   contiguous layout (row k of system s at s*n + k): k_thomas_contig_tma --
//                     TMA boxes of 16 rows x 32 systems (128-B swizzle) feed a
//                     thread per system; the (work, x') scratch is private and
//                     strided; x leaves through swizzled tiles and TMA stores.
//                     Odd n (no 16-B row stride) and exact = 3 take the
//                     transpose path (strided kernel between 32x32 transposes).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

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

// ---------------------------------------------------------------------------
// Contiguous layout, fused (no transposes). A CTA is one warp = 32 systems,
// lane = system; 4 CTAs per SM. The bands arrive as TMA boxes of 16 rows x 32
// systems with the 128-B swizzle: a system's 16 rows are one 128-B smem row,
// its 16-B chunks XOR-ed with (system & 7), so the 32 lanes reading row k hit
// 8 distinct chunks (4-way instead of 32-way bank conflicts). Three stages of
// the four bands (48 KB) are in flight per warp. The forward elimination keeps
// the reference's order per row and writes (work, x') to a private scratch in
// the strided layout (row k of system s at k*batch + s: 256-B coalesced warp
// stores and loads). The back substitution streams the scratch in reverse
// (register-prefetched one tile ahead) and stages x in swizzled tiles that a
// TMA store writes back as contiguous rows (double-buffered, bulk groups).
// Traffic per row: 32 B bands + 16 B scratch out + 16 B scratch in + 8 B x.
constexpr int kCR = 16;                 // rows per tile (128 B per system)
constexpr int kCS = 3;                  // forward stages
constexpr int kBS = 4;                  // back-substitution stages
constexpr int kTileB = 32 * kCR * 8;    // bytes of one [32 systems][16 rows] tile
constexpr int kContigSmem = kCS * 4 * kTileB + 1024 + 64;

struct ContigMaps {
  CUtensorMap a, b, c, d, x, ws, xs;
};
static_assert(2 + 2 * kBS <= 4 * kCS, "back-substitution stages fit the forward stages");

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y,
                                            unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int x,
                                             int y) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                   map),
               "r"(x), "r"(y), "r"(smem_u32(src))
               : "memory");
}
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// byte offset of (system s, row k) in a swizzled [32][16] tile
__device__ __forceinline__ int swz(int s, int k) {
  return s * 128 + ((((k >> 1) ^ (s & 7)) << 4) | ((k & 1) << 3));
}

__global__ void __launch_bounds__(32)
    k_thomas_contig_tma(const __grid_constant__ ContigMaps maps, double* __restrict__ xs,
                        double* __restrict__ ws, int n, int64_t batch, int64_t ld,
                        unsigned long long* fail) {
  extern __shared__ unsigned char sm_raw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(sm + kCS * 4 * kTileB);
  unsigned long long* bbar = bar + kCS;
  const int lane = threadIdx.x;
  const int s0 = blockIdx.x * 32;
  const int64_t s = s0 + lane;
  const bool live = s < batch;
  const int ntiles = (n + kCR - 1) / kCR;
  if (lane == 0) {
    for (int i = 0; i < kCS + kBS; ++i) mbar_init(&bar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  auto issue = [&](int t) {
    const int st = t % kCS;
    unsigned char* dst = sm + st * 4 * kTileB;
    mbar_expect_tx(&bar[st], 4 * kTileB);
    tma_load_2d(dst, &maps.a, t * kCR, s0, &bar[st]);
    tma_load_2d(dst + kTileB, &maps.b, t * kCR, s0, &bar[st]);
    tma_load_2d(dst + 2 * kTileB, &maps.c, t * kCR, s0, &bar[st]);
    tma_load_2d(dst + 3 * kTileB, &maps.d, t * kCR, s0, &bar[st]);
  };
  if (lane == 0)
    for (int t = 0; t < kCS && t < ntiles; ++t) issue(t);
  double w_prev = 0.0, x_prev = 0.0;
  bool bad = false;
  for (int t = 0; t < ntiles; ++t) {
    const int st = t % kCS;
    mbar_wait(&bar[st], (t / kCS) & 1);
    const unsigned char* tile = sm + st * 4 * kTileB;
    const int k0 = t * kCR;
#pragma unroll
    for (int kk = 0; kk < kCR; ++kk) {
      const int k = k0 + kk;
      if (k < n) {
        const int off = swz(lane, kk);
        const double bk = *reinterpret_cast<const double*>(tile + kTileB + off);
        const double ck = *reinterpret_cast<const double*>(tile + 2 * kTileB + off);
        const double dk = *reinterpret_cast<const double*>(tile + 3 * kTileB + off);
        double piv, xv;
        if (k == 0) {  // tridiagonal.hpp:26-30
          piv = bk;
          const double inv = 1.0 / piv;
          w_prev = ck * inv;
          xv = dk * inv;
        } else {  // :31-37
          const double ak = *reinterpret_cast<const double*>(tile + off);
          piv = bk - ak * w_prev;
          const double inv = 1.0 / piv;
          w_prev = ck * inv;
          xv = (dk - ak * x_prev) * inv;
        }
        bad |= piv == 0.0;
        x_prev = xv;
        if (live) {
          const int64_t o = static_cast<int64_t>(k) * ld + s;
          ws[o] = w_prev;
          xs[o] = xv;
        }
      }
    }
    __syncwarp();
    if (lane == 0 && t + kCS < ntiles) {
      fence_async_smem();
      issue(t + kCS);
    }
  }
  // Back substitution (:39): x[k] -= work[k] * x[k+1], tiles in reverse. The
  // forward stages are free now (every issued load was waited for). The
  // scratch tiles [16 rows][32 systems] come back by TMA through kBS stages
  // (after a proxy fence: they were written by generic stores); two more
  // tiles stage x for the TMA stores.
  asm volatile("fence.proxy.async.global;" ::: "memory");
  __syncwarp();
  unsigned char* xstage = sm;                  // 2 x-output tiles
  unsigned char* bstage = sm + 2 * kTileB;     // kBS stages of (work, x') tiles
  auto issue_b = [&](int i) {                  // i-th tile from the end
    const int st = i % kBS, t = ntiles - 1 - i;
    unsigned char* dst = bstage + st * 2 * kTileB;
    mbar_expect_tx(&bbar[st], 2 * kTileB);
    tma_load_2d(dst, &maps.ws, s0, t * kCR, &bbar[st]);
    tma_load_2d(dst + kTileB, &maps.xs, s0, t * kCR, &bbar[st]);
  };
  if (lane == 0)
    for (int i = 0; i < kBS && i < ntiles; ++i) issue_b(i);
  for (int i = 0; i < ntiles; ++i) {
    const int t = ntiles - 1 - i, st = i % kBS;
    mbar_wait(&bbar[st], (i / kBS) & 1);
    const double* tw = reinterpret_cast<const double*>(bstage + st * 2 * kTileB);
    const double* tx = tw + 32 * kCR;
    unsigned char* out = xstage + (i & 1) * kTileB;
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    __syncwarp();
#pragma unroll
    for (int kk = kCR - 1; kk >= 0; --kk) {
      const int k = t * kCR + kk;
      if (k < n) {
        const double xk = tx[kk * 32 + lane];
        if (k < n - 1) x_prev = xk - tw[kk * 32 + lane] * x_prev;
        else x_prev = xk;
        *reinterpret_cast<double*>(out + swz(lane, kk)) = x_prev;
      }
    }
    fence_async_smem();
    __syncwarp();
    if (lane == 0) {
      tma_store_2d(&maps.x, out, t * kCR, s0);
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      if (i + kBS < ntiles) issue_b(i + kBS);
    }
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  if (live && bad) atomicMin(fail, static_cast<unsigned long long>(s));
}

// ---- host: tensor maps of the fused contiguous kernel ----------------------
static PFN_cuTensorMapEncodeTiled_v12000 tma_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// [batch][n] contiguous systems, boxes of 16 rows x 32 systems, 128-B swizzle
static bool encode_contig(CUtensorMap* m, const double* base, int64_t n, int64_t batch) {
  auto enc = tma_encoder();
  if (!enc || !base) return false;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(n), static_cast<cuuint64_t>(batch)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(n) * sizeof(double)};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(kCR), 32u};
  cuuint32_t es[2] = {1u, 1u};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box,
             es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

// [n][ld] scratch rows, boxes of 32 systems x 16 rows, no swizzle
static bool encode_scratch(CUtensorMap* m, const double* base, int64_t n, int64_t ld) {
  auto enc = tma_encoder();
  if (!enc || !base) return false;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(ld), static_cast<cuuint64_t>(n)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * sizeof(double)};
  cuuint32_t box[2] = {32u, static_cast<cuuint32_t>(kCR)};
  cuuint32_t es[2] = {1u, 1u};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box,
             es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

// The fused contiguous kernel needs 16-B aligned bands and row strides (TMA)
// and every tensor map to encode; PCGPU_TRIDIAG_NO_TMA=1 forces the
// transpose path (A/B switch).
static bool contig_tma_ok(const double* a, const double* b, const double* c, const double* d,
                          const double* x, int64_t n, int64_t batch) {
  static const bool off = std::getenv("PCGPU_TRIDIAG_NO_TMA") != nullptr;
  if (off || n % 2 != 0 || n > (1ll << 30) || batch > (1ll << 31) || !tma_encoder()) return false;
  for (const double* p : {a, b, c, d, static_cast<const double*>(x)})
    if (reinterpret_cast<uintptr_t>(p) % 16 != 0) return false;
  CUtensorMap m;
  return encode_contig(&m, a, n, batch);
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
  // the fused contiguous kernel keeps its own (padded) scratch; the other
  // kernels take `work` from w
  const bool fused = layout != PCGPU_LAYOUT_STRIDED && exact != 2 && exact != 3 &&
                     contig_tma_ok(lower, diag, upper, rhs, x, n, batch);
  double* w = nullptr;
  unsigned long long* fail = nullptr;
  if (!fused &&
      cudaMallocAsync(&w, sizeof(double) * static_cast<size_t>(n * batch), s) != cudaSuccess)
    return PCGPU_ERR_CUDA;
  if (cudaMallocAsync(&fail, sizeof(unsigned long long), s) != cudaSuccess) return PCGPU_ERR_CUDA;
  cudaMemsetAsync(fail, 0xff, sizeof(unsigned long long), s);
  if (layout == PCGPU_LAYOUT_STRIDED) {
    const int th = 128;
    k_thomas_strided<<<static_cast<unsigned>((batch + th - 1) / th), th, 0, s>>>(
        lower, diag, upper, rhs, x, w, n, batch, fail);
  } else if (fused) {
    ContigMaps maps{};
    encode_contig(&maps.a, lower, n, batch);
    encode_contig(&maps.b, diag, n, batch);
    encode_contig(&maps.c, upper, n, batch);
    encode_contig(&maps.d, rhs, n, batch);
    encode_contig(&maps.x, x, n, batch);
    // private (work, x') scratch in the strided layout, row stride padded to
    // 32 systems so that its TMA boxes are aligned
    const int64_t ld = (batch + 31) / 32 * 32;
    double* scr = nullptr;
    if (cudaMallocAsync(&scr, sizeof(double) * static_cast<size_t>(2 * n * ld), s) != cudaSuccess)
      return PCGPU_ERR_CUDA;
    double* xs = scr + n * ld;
    encode_scratch(&maps.ws, scr, n, ld);
    encode_scratch(&maps.xs, xs, n, ld);
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(k_thomas_contig_tma, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           kContigSmem);
      attr = true;
    }
    k_thomas_contig_tma<<<static_cast<unsigned>((batch + 31) / 32), 32, kContigSmem, s>>>(
        maps, xs, scr, static_cast<int>(n), batch, ld, fail);
    cudaFreeAsync(scr, s);
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
  if (w) cudaFreeAsync(w, s);
  cudaFreeAsync(fail, s);
  if (cudaStreamSynchronize(s) != cudaSuccess) return PCGPU_ERR_CUDA;
  if (hfail != ~0ull) {
    if (failed_system) *failed_system = static_cast<int64_t>(hfail);
    return PCGPU_ERR_ZERO_PIVOT;
  }
  return PCGPU_OK;
}
