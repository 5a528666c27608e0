// adi_kernels.h -- host-side launcher declarations for the ADI kernels.
#pragma once

#include <cuda_runtime.h>

#include "adi_device.cuh"

namespace pcgpu {

// Field layouts (both nr x nz FP64):
//   N ("natural", the reference's Array2): (i, j) at j*nr + i -- r-lines contiguous.
//   T ("transposed"):                      (i, j) at i*nz + j -- z-lines contiguous.

// ---- exact mode (bit-identical to the reference; adi_exact.cu, --fmad=false) ----

// Speculative batches (pcgpu.cu host_run): K3's / K4's source is the result
// of the previous sweep, picked on the device by that sweep's convergence
// count (odd / even iterate buffer); a half-step whose status carries
// kSpecAbort is skipped whole. st == nullptr: the source pointer as given.
struct SpecPick {
  const DevStatus* st = nullptr;  // the sweep that produced the source
  const double* odd = nullptr;    // its result after an odd count
  const double* even = nullptr;   // ... after an even count
  double eps = 0.0;
};

// K3 explicit_axial_pass (solver.cpp:162-189): explT = Lambda_z[srcN]; also
// writes srcT = transpose(srcN) (the anchor for the T-layout radial sweep).
void launch_explicit_axial_exact(const DevProblem& P, const double* srcN, double* explT,
                                 double* srcT, DevStatus* st, cudaStream_t s,
                                 const SpecPick& pick = SpecPick{});
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
                            double* explN, double* halfN, DevStatus* st, cudaStream_t s,
                            const SpecPick& pick = SpecPick{});
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

// ---- resident stepper: a batch of whole steps in one cooperative launch ----
// The tau controller, the Picard loops and their max-norm convergence tests,
// the accept-or-halve decision and the field-buffer rotation all run on the
// device; phases (K3, Picard iterations, K4) are separated by grid-wide
// barriers. The host supplies a schedule -- per step t, the first attempt's
// tau and pulse_value(t + tau_h / 2) for h = 0..kResHalv halvings, computed
// by the host functions the reference uses -- that assumes no halvings; a
// batch therefore ends after the first step that halved (its successors'
// times change) and the host resumes from the device state.
constexpr int kResHalv = 8;     // halvings with a precomputed pulse per step
constexpr int kResProbes = 16;  // probe values gathered per step (evolve)
constexpr int kResThreads = 384;
struct ResSched {
  double tau0;
  double pulse[kResHalv + 1];
};
struct ResLog {
  pcgpu_step_result r;
  double updates;  // active cells x Picard iterations over every attempt
  double probes[kResProbes];
};
enum ResStop { kResRan = 0, kResHalved = 1, kResError = 2, kResFloor = 3, kResNeedHost = 4 };
struct ResCtl {
  int steps;  // accepted steps of the batch
  int stop;   // ResStop
  int state;  // index of the field buffer after the last accepted step
  int pad;
  unsigned long long err;  // kResError: the line error word (line << 3 | code)
  double tau;              // kResFloor: the attempt's tau below the floor
  double updates;          // kResError / kResFloor / kResNeedHost: the failed step's work
  unsigned long long clamp_save[kMaxLayers];
  // phase profile (lead thread, %globaltimer ns; ResArgs::profile): time and
  // count per phase -- 0 status reset, 1 K3, 2 radial iteration, 3 K4,
  // 4 axial iteration, 5 step epilogue
  unsigned long long prof_ns[8], prof_n[8];
  // ... and per phase the busiest CTA's time from its exit of the previous
  // barrier to its arrival at the next one (busy_max: the current phase)
  unsigned long long prof_busy[8], busy_max[8];
  unsigned long long prof_cyc;  // lead thread: clock64 over the profiled phases (SM clock)
};
struct ResArgs {
  double* X[3];  // N-layout field rotation: X[state] is the field
  double *TcT, *ExplT, *HalfT;  // radial anchor / explicit term / iterate (T); K4 -> HalfN, ExplN
  double* kbarN;                // nullptr: K-bar computed in the axial sweep
  double *W, *Xs;               // Thomas scratch
  DevStatus* st2;               // [2] status, alternating per half-step
  const ResSched* sched;
  ResLog* log;
  ResCtl* ctl;
  const int* probe_off;  // [n_probes] N-layout offsets
  int n_probes;
  int nsteps, state0;
  int max_iter, max_halv;  // max_halv <= kResHalv (lower: tests of the host redo)
  int profile;             // record ResCtl::prof_*
  int short_r, short_a;    // the sweep's lines fit the shared-memory (w, x) variant
  double eps, tau_floor, active;
};
// Whether the resident stepper applies (exact-x / exact-lean lookups, no FIELD
// source, <= kResProbes probes) and its grid size (0: not co-resident).
int resident_grid(const DevProblem& P);
// Whether that grid runs as a single thread-block cluster (<= 16 CTAs).
bool resident_cluster(const DevProblem& P, int grid);
void launch_resident(const DevProblem& P, const ResArgs& A, int grid, bool cluster,
                     cudaStream_t s);

// Selects `dev` for the scope of an entry point and restores the caller's
// current device afterwards (the library never leaves the current device
// changed; every entry point works on its stepper's own device).
struct DeviceGuard {
  int prev = -1;
  bool ok = true, changed = false;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) {
      ok = cudaSetDevice(dev) == cudaSuccess;
      changed = ok && prev >= 0;
    }
  }
  ~DeviceGuard() {
    if (changed) cudaSetDevice(prev);
  }
  DeviceGuard(const DeviceGuard&) = delete;
  DeviceGuard& operator=(const DeviceGuard&) = delete;
};

// Kernel launch counter (for the bench's gpu_launches claim).
extern unsigned long long g_launches;

}  // namespace pcgpu
