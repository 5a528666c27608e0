// adi_kernels.h -- host-side launcher declarations for the ADI kernels.
#pragma once

#include <cuda_runtime.h>

#include "adi_device.cuh"

namespace pcgpu {

// Field layouts (both nr x nz FP64):
//   N ("natural", the reference's Array2): (i, j) at j*nr + i -- r-lines contiguous.
//   T ("transposed"):                      (i, j) at i*nz + j -- z-lines contiguous.

// ---- exact mode (bit-identical to the reference; adi_exact.cu, --fmad=false) ----

// K3 explicit_axial_pass (solver.cpp:162-189): explT = Lambda_z[srcN]; also
// writes srcT = transpose(srcN) (the anchor for the T-layout radial sweep).
void launch_explicit_axial_exact(const DevProblem& P, const double* srcN, double* explT,
                                 double* srcT, DevStatus* st, cudaStream_t s);
// K1 one Picard iteration of the radial sweep (solver.cpp:191-233, :245-248),
// T layout, thread per radial line. Early-exits when iteration it-1 converged.
void launch_radial_exact(const DevProblem& P, int it, double eps, double half_k, double pulse,
                         const double* TsT, const double* TcT, const double* explT,
                         const double* powT, double* outT, double* wT, double* xT,
                         DevStatus* st, cudaStream_t s);
// K4 axial_fixed_rhs_pass (solver.cpp:259-284) from the T-layout half field:
// kbarN, explN and halfN (transposed copy) in N layout. kbarN == nullptr: no
// K-bar field (the c_V lookups are still made, for their clamp events / range
// errors); the axial sweep then computes K-bar itself (kbar_on_the_fly).
void launch_axial_rhs_exact(const DevProblem& P, double half_k, double pulse,
                            const double* halfT, const double* powN, double* kbarN,
                            double* explN, double* halfN, DevStatus* st, cudaStream_t s);
// K2 one Picard iteration of the axial sweep (solver.cpp:286-332, :343-345),
// N layout, thread per axial line. kbarN == nullptr (only when
// kbar_on_the_fly(P)): K-bar = rho * c_V(ThN) * half_k inside the sweep.
bool kbar_on_the_fly(const DevProblem& P);
void launch_axial_exact(const DevProblem& P, int it, double eps, double half_k, const double* TsN,
                        const double* ThN, const double* kbarN, const double* explN,
                        double* outN, double* wN, double* xN, DevStatus* st, cudaStream_t s);

// ---- partitioned (multi-GPU) slabs, exact mode (adi_exact.cu) ----
// z-slab: radial lines j0..j0+nj-1, T layout [i][j-j0] (ld nj);
// r-slab: axial lines i0..i0+ni-1, N layout [j][i-i0] (ld ni).
// K3 over the row tiles covering [j_begin, j_end) (multiples of 64 rows except
// at nz): the exact t3 kernel, for a field that arrives in row blocks.
constexpr int kK3RowTile = 64;
void launch_explicit_axial_exact_rows(const DevProblem& P, const double* srcN, double* explT,
                                      double* srcT, DevStatus* st, int j_begin, int j_end,
                                      cudaStream_t s);
// ld: row stride of the line arrays (0: dense slab, ld = nj); the arrays may
// then be a line range of a wider field (pointers offset to its first line).
void launch_radial_exact_slab(const DevProblem& P, int it, double eps, double half_k,
                              double pulse, int j0, int nj, const double* TsT, const double* TcT,
                              const double* explT, const double* powT, double* outT, double* wT,
                              double* xT, DevStatus* st, cudaStream_t s, long long ld = 0);
void launch_axial_exact_slab(const DevProblem& P, int it, double eps, double half_k, int i0,
                             int ni, const double* TsN, const double* ThN, const double* kbarN,
                             const double* explN, double* outN, double* wN, double* xN,
                             DevStatus* st, cudaStream_t s);
// K3 on an r-slab: explR = Lambda_z[TR]
void launch_expl_rslab_exact(const DevProblem& P, int i0, int ni, const double* TR,
                             double* explR, DevStatus* st, cudaStream_t s);
// K4 without K-bar on a z-slab: explZ = Lambda_r[halfZ] + X(halfZ)
void launch_rhs_zslab_exact(const DevProblem& P, double pulse, int j0, int nj,
                            const double* halfZ, double* explZ, DevStatus* st, cudaStream_t s);
// K-bar on an r-slab (kbarR == nullptr: the clamp events / range errors only)
void launch_kbar_rslab_exact(const DevProblem& P, double half_k, int i0, int ni,
                             const double* halfR, double* kbarR, DevStatus* st, cudaStream_t s);

// Fused compute + all-to-all (peer transport): destination slabs of every rank.
constexpr int kMaxPeers = 16;
struct PeerSlabs {
  double* zTc[kMaxPeers];    // rank q's z-slab anchor, T layout [i][j - zb[q]]
  double* zExpl[kMaxPeers];  // rank q's Lambda_z, same layout
  double* rHalf[kMaxPeers];  // rank q's r-slab T_half, N layout [j][i - rb[q]]
  double* rExpl[kMaxPeers];  // rank q's Lambda_r + X, same layout
  int zb[kMaxPeers + 1], rb[kMaxPeers + 1];
  int nranks;
};
// K3 on an r-slab, (Lambda_z, T_cur) stored into the owners' z-slabs
void launch_expl_rslab_scatter(const DevProblem& P, int i0, int ni, const double* TR,
                               const PeerSlabs& ps, DevStatus* st, cudaStream_t s);
// K4 without K-bar on a z-slab, (T_half, Lambda_r + X) stored into the owners' r-slabs
void launch_rhs_zslab_scatter(const DevProblem& P, double pulse, int j0, int nj,
                              const double* halfZ, const PeerSlabs& ps, DevStatus* st,
                              cudaStream_t s);

// ---- layout helpers (masked: only in-mask cells are written) ----
void launch_transpose_N2T(const DevProblem& P, const double* srcN, double* dstT, cudaStream_t s);
void launch_transpose_T2N(const DevProblem& P, const double* srcT, double* dstN, cudaStream_t s);

// ---- fast mode (adi_fast.cu): partitioned line solves on contiguous lines ----
bool fast_supported(const DevProblem& P);
// K3: explN = Lambda_z[field] and TcN = field (from the T-layout field).
void launch_explicit_axial_fast(const DevProblem& P, const double* fieldT, double* explN,
                                double* TcN, DevStatus* st, cudaStream_t s);
// K1: radial Picard iteration on N-layout lines.
void launch_radial_fast(const DevProblem& P, int it, double eps, double half_k, double pulse,
                        const double* TsN, const double* TcN, const double* explN,
                        const double* powN, double* outN, DevStatus* st, cudaStream_t s);
// K4: explT = Lambda_r[half] + X(half) and halfT = half (from the N-layout half field).
void launch_axial_rhs_fast(const DevProblem& P, double pulse, const double* halfN,
                           const double* powN, double* explT, double* halfT, DevStatus* st,
                           cudaStream_t s);
// K2: axial Picard iteration on T-layout lines (K-bar recomputed from the anchor).
void launch_axial_fast(const DevProblem& P, int it, double eps, double half_k, const double* TsT,
                       const double* ThT, const double* explT, double* outT, DevStatus* st,
                       cudaStream_t s);

// ---- partitioned (multi-GPU) slabs, fast mode (adi_fast.cu) ----
void launch_radial_fast_slab(const DevProblem& P, int it, double eps, double half_k, double pulse,
                             int j0, int nj, const double* TsN, const double* TcN,
                             const double* explN, double* outN, DevStatus* st, cudaStream_t s);
void launch_axial_fast_slab(const DevProblem& P, int it, double eps, double half_k, int i0,
                            int ni, const double* TsT, const double* ThT, const double* explT,
                            double* outT, DevStatus* st, cudaStream_t s);
void launch_rhs_zslab(const DevProblem& P, double pulse, int j0, int nj, const double* hN,
                      double* eN, DevStatus* st, cudaStream_t s);
void launch_expl_rslab(const DevProblem& P, int i0, int ni, const double* fT, double* eT,
                       DevStatus* st, cudaStream_t s);

// Kernel launch counter (for the bench's gpu_launches claim).
extern unsigned long long g_launches;

}  // namespace pcgpu
