// pcgpu_dist.cu -- partitioned ADI stepper for one node of B200s.
//
// The reference is shared-memory only (SPEC.md:389 lists distributed memory as
// a non-goal); this is the B200-native scale-out of the same step:
//
//   z-slabs: rank p owns the radial lines j in Z_p (N layout, contiguous), so
//            the radial Picard sweep is local;
//   r-slabs: rank p owns the axial lines i in R_p (T layout, contiguous), so
//            the axial Picard sweep is local;
//   between the sweeps an all-to-all transpose moves the half-step field and
//   its explicit term (Lambda_r[T_half] + X, computed on the z-slab where the
//   radial stencil is local) from z-slabs to r-slabs; after an accepted step
//   the new field and Lambda_z[T_new] (computed on the r-slab) move back;
//   each Picard iteration's max-norm is an allreduce(max) of one uint64 (the
//   bit pattern of a non-negative double), so every rank takes the same
//   convergence / tau-halving decisions without host round trips.
//
// The per-cell and per-line arithmetic is exactly the single-GPU exact
// path's (adi_exact.cu slab kernels), so a partitioned run is bit-identical to
// a single-GPU run (and so to the reference): tests run P "virtual ranks" in
// one process on one GPU (Comm::Local) and compare bit-for-bit. Real ranks (one process per GPU)
// use NCCL (grouped ncclSend/ncclRecv for the all-to-all, ncclAllReduce for
// the norm), loaded with dlopen so the single-GPU library has no NCCL
// dependency.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/pcgpu.h"
#include "adi_kernels.h"
#include "extents.h"

using namespace pcgpu;

// shared with pcgpu.cu
void build_dev_problem(const pcgpu_desc* d, DevProblem& P, std::vector<void*>& allocs);
std::string pcgpu_validate_desc(const pcgpu_desc* d);
double pcgpu_host_initial_tau(const pcgpu_desc& d, double t);
double pcgpu_host_pulse_value(const pcgpu_desc& d, double t);

namespace {

struct DistError {
  int code;
  std::string what;
};

#define DCK(x)                                                                       \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess)                                                           \
      throw DistError{PCGPU_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)}; \
  } while (0)

// ---- NCCL via dlopen --------------------------------------------------------
struct Nccl {
  void* h = nullptr;
  decltype(&ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&ncclCommInitRank) commInitRank = nullptr;
  decltype(&ncclCommDestroy) commDestroy = nullptr;
  decltype(&ncclAllReduce) allReduce = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGroupStart) groupStart = nullptr;
  decltype(&ncclGroupEnd) groupEnd = nullptr;
  decltype(&ncclGetErrorString) errorString = nullptr;

  bool load(std::string& err) {
    if (h) return true;
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* n : names)
      if ((h = dlopen(n, RTLD_NOW | RTLD_GLOBAL))) break;
    if (!h) {
      err = "pcgpu_dist: cannot dlopen libnccl.so.2";
      return false;
    }
#define SYM(f, n) f = reinterpret_cast<decltype(f)>(dlsym(h, n))
    SYM(getUniqueId, "ncclGetUniqueId");
    SYM(commInitRank, "ncclCommInitRank");
    SYM(commDestroy, "ncclCommDestroy");
    SYM(allReduce, "ncclAllReduce");
    SYM(send, "ncclSend");
    SYM(recv, "ncclRecv");
    SYM(groupStart, "ncclGroupStart");
    SYM(groupEnd, "ncclGroupEnd");
    SYM(errorString, "ncclGetErrorString");
#undef SYM
    if (!getUniqueId || !commInitRank || !allReduce || !send || !recv || !groupStart ||
        !groupEnd) {
      err = "pcgpu_dist: libnccl is missing symbols";
      return false;
    }
    return true;
  }
} g_nccl;

#define NCK(x)                                                                           \
  do {                                                                                   \
    ncclResult_t r_ = (x);                                                               \
    if (r_ != ncclSuccess)                                                               \
      throw DistError{PCGPU_ERR_CUDA, std::string(#x) + ": " +                           \
                                          (g_nccl.errorString ? g_nccl.errorString(r_)   \
                                                              : "nccl error")};          \
  } while (0)

// ---- small kernels ------------------------------------------------------------
// dst[c * dst_ld + r] = src[r * src_ld + c] for r < rows, c < cols.
__global__ void k_transpose_block(const double* __restrict__ src, long long src_ld, int rows,
                                  int cols, double* __restrict__ dst, long long dst_ld) {
  __shared__ double t[32][33];
  const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  const int lx = threadIdx.x & 31, ly = threadIdx.x >> 5;
  for (int rr = ly; rr < 32; rr += 8) {
    const int r = r0 + rr, c = c0 + lx;
    if (r < rows && c < cols) t[rr][lx] = src[static_cast<long long>(r) * src_ld + c];
  }
  __syncthreads();
  for (int cc = ly; cc < 32; cc += 8) {
    const int c = c0 + cc, r = r0 + lx;
    if (r < rows && c < cols) dst[static_cast<long long>(c) * dst_ld + r] = t[lx][cc];
  }
}

void transpose_block(const double* src, long long src_ld, int rows, int cols, double* dst,
                     long long dst_ld, cudaStream_t s) {
  if (rows <= 0 || cols <= 0) return;
  dim3 grid((cols + 31) / 32, (rows + 31) / 32);
  k_transpose_block<<<grid, 256, 0, s>>>(src, src_ld, rows, cols, dst, dst_ld);
  ++g_launches;
}

// Local emulation of allreduce(max) of delta[it] and allreduce(min) of err
// over P virtual ranks' status blocks.
__global__ void k_reduce_status(DevStatus** st, int nranks, int it) {
  if (threadIdx.x != 0) return;
  unsigned long long dmax = 0, emin = kNoError;
  for (int r = 0; r < nranks; ++r) {
    dmax = max(dmax, st[r]->delta[it]);
    emin = min(emin, st[r]->err);
  }
  for (int r = 0; r < nranks; ++r) {
    st[r]->delta[it] = dmax;
    st[r]->err = emin;
  }
}

// Balanced contiguous split of n lines with per-line cell counts ext(l).
template <typename F>
std::vector<int> split_lines(int n, int parts, F ext) {
  std::vector<double> pre(n + 1, 0.0);
  for (int l = 0; l < n; ++l) pre[l + 1] = pre[l] + ext(l);
  std::vector<int> b(parts + 1, 0);
  b[parts] = n;
  for (int p = 1; p < parts; ++p) {
    const double target = pre[n] * p / parts;
    int l = static_cast<int>(std::lower_bound(pre.begin(), pre.end(), target) - pre.begin());
    b[p] = std::max(b[p - 1], std::min(l, n));
  }
  return b;
}

}  // namespace

// One rank's slabs and buffers.
struct RankState {
  int rank = 0;
  int j0 = 0, nj = 0;  // z-slab lines
  int i0 = 0, ni = 0;  // r-slab lines
  double *zTc = nullptr, *zExpl = nullptr, *zHalf = nullptr, *zIter = nullptr, *zR = nullptr;
  double *rHalf = nullptr, *rExpl = nullptr, *rOut = nullptr, *rIter = nullptr;
  double* recv = nullptr;
  // exact mode: Thomas scratch on both slabs, K-bar and the r-slab copy of
  // the step's anchor (Lambda_z is recomputed from it every attempt, like the
  // single-GPU stepper)
  double *zW = nullptr, *zX = nullptr, *rW = nullptr, *rX = nullptr;
  double *rKbar = nullptr, *rTc = nullptr;
  DevStatus* st = nullptr;
};

struct pcgpu_dist {
  pcgpu_desc d{};
  DevProblem P{};
  std::vector<void*> allocs;
  cudaStream_t stream = nullptr;
  int nranks = 1;
  bool local = true;  // P virtual ranks in this process
  ncclComm_t comm = nullptr;
  std::vector<int> zb, rb;  // slab boundaries (lines)
  std::vector<RankState> ranks;  // local ranks (all of them in local mode)
  DevStatus** st_dev_list = nullptr;
  DevStatus* st_host = nullptr;
  int64_t active = 0;
  double tau_floor = 0;
  std::string err;
  int64_t err_line = -1;
  int pred_r = 1, pred_a = 1;
  // exact mode transport: peer stores from the fused slab passes (emulated
  // ranks, or IPC-mapped peer slabs after pcgpu_dist_ipc_import), else NCCL
  // all-to-all transposes
  bool peer = false;
  PeerSlabs ps{};
  std::vector<void*> ipc_opened;
  unsigned long long* d_barrier = nullptr;
  // timing
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  double transpose_ms = 0;
  int64_t transposes = 0, allreduces = 0;
  double radial_ms = 0, axial_ms = 0;
  int64_t radial_launches = 0, axial_launches = 0;
  bool timing = false;

  ~pcgpu_dist() {
    if (stream) cudaStreamSynchronize(stream);
    for (void* p : ipc_opened) cudaIpcCloseMemHandle(p);
    if (comm && g_nccl.commDestroy) g_nccl.commDestroy(comm);
    for (void* p : allocs) cudaFree(p);
    if (st_host) cudaFreeHost(st_host);
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    if (stream) cudaStreamDestroy(stream);
  }

  double* alloc(size_t n) {
    double* p = nullptr;
    DCK(cudaMalloc(&p, sizeof(double) * std::max<size_t>(n, 1)));
    allocs.push_back(p);
    return p;
  }

  int zcount(int p) const { return zb[p + 1] - zb[p]; }
  int rcount(int p) const { return rb[p + 1] - rb[p]; }

  // ---- collectives ----
  // Cross-rank ordering point after peer stores (multi-process peer
  // transport): every rank's scatter kernel has completed before any rank
  // reads its slabs. Emulated ranks share one stream and need none.
  void barrier() {
    if (local) return;
    NCK(g_nccl.allReduce(d_barrier, d_barrier, 1, ncclUint64, ncclMax, comm, stream));
  }

  void build_peer_table_local() {
    ps = PeerSlabs{};
    ps.nranks = nranks;
    for (int q = 0; q <= nranks; ++q) {
      ps.zb[q] = zb[q];
      ps.rb[q] = rb[q];
    }
    for (RankState& R : ranks) {
      ps.zTc[R.rank] = R.zTc;
      ps.zExpl[R.rank] = R.zExpl;
      ps.rHalf[R.rank] = R.rHalf;
      ps.rExpl[R.rank] = R.rExpl;
    }
  }

  void allreduce_status(int it) {
    ++allreduces;
    if (local) {
      k_reduce_status<<<1, 32, 0, stream>>>(st_dev_list, nranks, it);
      ++g_launches;
      return;
    }
    RankState& R = ranks[0];
    NCK(g_nccl.groupStart());
    NCK(g_nccl.allReduce(&R.st->delta[it], &R.st->delta[it], 1, ncclUint64, ncclMax, comm,
                         stream));
    NCK(g_nccl.allReduce(&R.st->err, &R.st->err, 1, ncclUint64, ncclMin, comm, stream));
    NCK(g_nccl.groupEnd());
  }

  void reset_status(bool clear_err = true) {
    for (RankState& R : ranks) {
      DCK(cudaMemsetAsync(R.st->delta, 0, sizeof(R.st->delta), stream));
      if (clear_err) DCK(cudaMemsetAsync(&R.st->err, 0xff, sizeof(R.st->err), stream));
    }
  }

  // Exact-mode all-to-all of k fields between the dense slabs.
  // z2r: z-slab T layout [i][j - j0] (ld nj) -> r-slab N layout [j][i - i0] (ld ni);
  // r2z: the reverse. The block a rank sends to q is a contiguous row range of
  // its slab (rows i in R_q, resp. j in Z_q), so it is sent straight from the
  // field; the receiver transposes each block into place.
  void transpose_exact(bool z2r, int k, double* const* const* src, double* const* const* dst) {
    if (timing) DCK(cudaEventRecord(ev0, stream));
    // exchange into recv staging: per field f, blocks ordered by source rank
    auto blk_rows = [&](int q) { return z2r ? rcount(q) : zcount(q); };  // rows sent to q
    auto src_cols = [&](int p) { return z2r ? zcount(p) : rcount(p); };  // ld of p's slab
    auto row0 = [&](int q) { return z2r ? rb[q] : zb[q]; };
    if (local) {
      for (int f = 0; f < k; ++f)
        for (int q = 0; q < nranks; ++q) {
          size_t roff = static_cast<size_t>(f) * (z2r ? static_cast<size_t>(rcount(q)) * d.nz
                                                      : static_cast<size_t>(zcount(q)) * d.nr);
          for (int p = 0; p < nranks; ++p) {
            const size_t n = static_cast<size_t>(blk_rows(q)) * src_cols(p);
            if (n)
              DCK(cudaMemcpyAsync(ranks[q].recv + roff,
                                  src[f][p] + static_cast<size_t>(row0(q)) * src_cols(p),
                                  sizeof(double) * n, cudaMemcpyDeviceToDevice, stream));
            roff += n;
          }
        }
    } else {
      RankState& R = ranks[0];
      const int me = R.rank;
      NCK(g_nccl.groupStart());
      for (int f = 0; f < k; ++f) {
        size_t roff = static_cast<size_t>(f) * (z2r ? static_cast<size_t>(R.ni) * d.nz
                                                    : static_cast<size_t>(R.nj) * d.nr);
        for (int q = 0; q < nranks; ++q) {
          const size_t sn = static_cast<size_t>(blk_rows(q)) * src_cols(me);
          const size_t rn = static_cast<size_t>(blk_rows(me)) * src_cols(q);
          if (sn)
            NCK(g_nccl.send(src[f][0] + static_cast<size_t>(row0(q)) * src_cols(me), sn,
                            ncclDouble, q, comm, stream));
          if (rn) NCK(g_nccl.recv(R.recv + roff, rn, ncclDouble, q, comm, stream));
          roff += rn;
        }
      }
      NCK(g_nccl.groupEnd());
    }
    // unpack: block from p is [rows of mine][cols of p] -> transpose into place
    for (size_t lr = 0; lr < ranks.size(); ++lr) {
      RankState& R = ranks[lr];
      const int me = R.rank;
      for (int f = 0; f < k; ++f) {
        size_t off = static_cast<size_t>(f) * (z2r ? static_cast<size_t>(R.ni) * d.nz
                                                   : static_cast<size_t>(R.nj) * d.nr);
        for (int p = 0; p < nranks; ++p) {
          const int rows = blk_rows(me), cols = src_cols(p);
          // z2r: block [i - i0][j - zb[p]] -> dst[j * ni + (i - i0)], j = zb[p] + c
          // r2z: block [j - j0][i - rb[p]] -> dst[i * nj + (j - j0)], i = rb[p] + c
          const int c0 = z2r ? zb[p] : rb[p];
          const long long dld = z2r ? R.ni : R.nj;
          transpose_block(R.recv + off, cols, rows, cols, dst[f][lr] + c0 * dld, dld, stream);
          off += static_cast<size_t>(rows) * cols;
        }
      }
    }
    ++transposes;
    if (timing) {
      DCK(cudaEventRecord(ev1, stream));
      DCK(cudaEventSynchronize(ev1));
      float ms = 0;
      DCK(cudaEventElapsedTime(&ms, ev0, ev1));
      transpose_ms += ms;
    }
  }

  // One exact ADI step (solver.cpp:356-373) on the partitioned state: z-slab
  // anchor zTc (T layout) and its r-slab copy rTc (N layout).
  int step_exact(double t, pcgpu_step_result* r, double* updates) {
    double tau = pcgpu_host_initial_tau(d, t);
    *r = pcgpu_step_result{};
    const size_t nl = ranks.size();
    std::vector<double*> a(nl), b(nl), c(nl), e(nl);
    for (;;) {
      const double pulse = d.source_kind == PCGPU_SOURCE_JOULE
                               ? pcgpu_host_pulse_value(d, t + 0.5 * tau) : 0.0;
      const double hk = 2.0 / tau;
      // ---- radial half-step: Lambda_z[T_cur] on the r-slabs -> z-slabs ----
      reset_status();
      if (peer) {
        // fused: Lambda_z and T_cur stored straight into the owners' z-slabs
        for (RankState& R : ranks)
          launch_expl_rslab_scatter(P, R.i0, R.ni, R.rTc, ps, R.st, stream);
        barrier();
      } else {
        for (size_t lr = 0; lr < nl; ++lr) {
          RankState& R = ranks[lr];
          launch_expl_rslab_exact(P, R.i0, R.ni, R.rTc, R.rExpl, R.st, stream);
          a[lr] = R.rExpl;
          b[lr] = R.zExpl;
        }
        double* const* s1[1] = {a.data()};
        double* const* d1[1] = {b.data()};
        transpose_exact(false, 1, s1, d1);
      }
      auto zsrc = [&](RankState& R, int it) -> const double* {
        return it == 1 ? R.zTc : (it % 2 == 0 ? R.zHalf : R.zIter);
      };
      auto zdst = [&](RankState& R, int it) -> double* { return it % 2 == 1 ? R.zHalf : R.zIter; };
      int conv = picard(pred_r, [&](size_t lr, int it) {
        RankState& R = ranks[lr];
        launch_radial_exact_slab(P, it, d.epsilon, hk, pulse, R.j0, R.nj, zsrc(R, it), R.zTc,
                                 R.zExpl, nullptr, zdst(R, it), R.zW, R.zX, R.st, stream);
      }, &r->radial, true);
      if (conv < 0) return -conv;
      *updates += static_cast<double>(active) * r->radial.iterations;
      if (conv > 0) {
        // ---- axial half-step: Lambda_r + X on the z-slabs, -> r-slabs, K-bar ----
        reset_status();
        if (peer) {
          // fused: T_half and Lambda_r + X stored straight into the owners' r-slabs
          for (RankState& R : ranks)
            launch_rhs_zslab_scatter(P, pulse, R.j0, R.nj, zdst(R, conv), ps, R.st, stream);
          barrier();
        } else {
          for (size_t lr = 0; lr < nl; ++lr) {
            RankState& R = ranks[lr];
            a[lr] = zdst(R, conv);
            launch_rhs_zslab_exact(P, pulse, R.j0, R.nj, a[lr], R.zR, R.st, stream);
            b[lr] = R.zR;
            c[lr] = R.rHalf;
            e[lr] = R.rExpl;
          }
          double* const* s2[2] = {a.data(), b.data()};
          double* const* d2[2] = {c.data(), e.data()};
          transpose_exact(true, 2, s2, d2);
        }
        // K-bar: a field, or (exact lookups) computed by the axial sweep itself and
        // only its c_V lookups' clamp events / range errors taken here
        const bool fly = kbar_on_the_fly(P);
        for (RankState& R : ranks)
          launch_kbar_rslab_exact(P, hk, R.i0, R.ni, R.rHalf, fly ? nullptr : R.rKbar, R.st,
                                  stream);
        reset_status(false);  // keep errors of the K4 passes
        auto rsrc = [&](RankState& R, int it) -> const double* {
          return it == 1 ? R.rHalf : (it % 2 == 0 ? R.rOut : R.rIter);
        };
        auto rdst = [&](RankState& R, int it) -> double* { return it % 2 == 1 ? R.rOut : R.rIter; };
        const int aconv = picard(pred_a, [&](size_t lr, int it) {
          RankState& R = ranks[lr];
          launch_axial_exact_slab(P, it, d.epsilon, hk, R.i0, R.ni, rsrc(R, it), R.rHalf,
                                  fly ? nullptr : R.rKbar, R.rExpl, rdst(R, it), R.rW, R.rX,
                                  R.st, stream);
        }, &r->axial, false);
        if (aconv < 0) return -aconv;
        *updates += static_cast<double>(active) * r->axial.iterations;
        if (aconv > 0) {
          // accept: the r-slab result becomes the anchor (the next attempt's
          // K3 moves it to the z-slabs: fused with the peer transport, here
          // with the NCCL transport)
          for (size_t lr = 0; lr < nl; ++lr) {
            RankState& R = ranks[lr];
            double* res = rdst(R, aconv);
            if (res == R.rOut) std::swap(R.rOut, R.rTc); else std::swap(R.rIter, R.rTc);
            a[lr] = R.rTc;
            b[lr] = R.zTc;
          }
          if (!peer) {
            double* const* s1[1] = {a.data()};
            double* const* d1[1] = {b.data()};
            transpose_exact(false, 1, s1, d1);
          }
          r->tau_used = tau;
          return PCGPU_OK;
        }
      }
      tau *= 0.5;
      ++r->halvings;
      if (tau < tau_floor) {
        err = "time step fell below floor";
        return PCGPU_ERR_TAU_FLOOR;
      }
      r->axial = pcgpu_outcome{};
    }
  }

  void fetch_status(int n) {
    DevStatus* s0 = ranks[0].st;
    DCK(cudaMemcpyAsync(st_host->delta, s0->delta, sizeof(unsigned long long) * (n + 1),
                        cudaMemcpyDeviceToHost, stream));
    DCK(cudaMemcpyAsync(&st_host->err, &s0->err, sizeof(s0->err), cudaMemcpyDeviceToHost,
                        stream));
    DCK(cudaStreamSynchronize(stream));
  }

  double delta_of(int it) const {
    double v;
    std::memcpy(&v, &st_host->delta[it], sizeof v);
    return v;
  }

  // Picard loop over all local ranks with the norm allreduce after each
  // iteration. Returns converged iteration, 0, or -error.
  template <typename Launch>
  int picard(int& pred, Launch&& launch, pcgpu_outcome* o, bool radial) {
    const int max_iter = d.max_iter;
    int launched = 0, batch = std::min(max_iter, std::max(1, pred) + 1);
    *o = pcgpu_outcome{};
    while (launched < max_iter) {
      const int upto = std::min(max_iter, launched + batch);
      for (int it = launched + 1; it <= upto; ++it) {
        if (timing) DCK(cudaEventRecord(ev0, stream));
        for (size_t lr = 0; lr < ranks.size(); ++lr) launch(lr, it);
        if (timing) {
          DCK(cudaEventRecord(ev1, stream));
          DCK(cudaEventSynchronize(ev1));
          float ms = 0;
          DCK(cudaEventElapsedTime(&ms, ev0, ev1));
          (radial ? radial_ms : axial_ms) += ms;
          ++(radial ? radial_launches : axial_launches);
        }
        allreduce_status(it);
      }
      launched = upto;
      fetch_status(launched);
      if (st_host->err != kNoError) {
        const int code = static_cast<int>(st_host->err & 7ull);
        err_line = static_cast<int64_t>(st_host->err >> 3);
        err = "line " + std::to_string(err_line) + " failed";
        return -code;
      }
      for (int it = 1; it <= launched; ++it) {
        const double dl = delta_of(it);
        if (dl < d.epsilon) {
          o->converged = 1;
          o->iterations = it;
          o->last_delta = dl;
          pred = it;
          return it;
        }
      }
      batch = 2;
    }
    o->iterations = max_iter;
    o->last_delta = delta_of(max_iter);
    return 0;
  }

  // One ADI step (solver.cpp:356-373) on the partitioned state
  // (z-slab anchor zTc + zExpl = Lambda_z[zTc]).
  int step(double t, pcgpu_step_result* r, double* updates) {
    return step_exact(t, r, updates);
  }
};

extern "C" {

int pcgpu_nccl_unique_id(void* id128) {
  std::string e;
  if (!g_nccl.load(e)) return PCGPU_ERR_CUDA;
  ncclUniqueId id;
  if (g_nccl.getUniqueId(&id) != ncclSuccess) return PCGPU_ERR_CUDA;
  std::memcpy(id128, &id, sizeof id);
  return PCGPU_OK;
}

thread_local std::string g_dist_create_error;

int pcgpu_dist_create(const pcgpu_desc* d, int32_t rank, int32_t nranks, const void* nccl_id,
                      pcgpu_dist** out) {
  if (!d || !out || nranks < 1) return PCGPU_ERR_ARG;
  *out = nullptr;
  std::string v = pcgpu_validate_desc(d);
  if (v.empty() && d->source_kind == PCGPU_SOURCE_FIELD)
    v = "pcgpu_dist: the partitioned stepper supports Null and Joule sources";
  if (!v.empty()) {
    g_dist_create_error = v;
    return PCGPU_ERR_CONFIG;
  }
  DeviceGuard dg(d->device);
  if (!dg.ok) {
    g_dist_create_error = "pcgpu_dist_create: cannot select device";
    return PCGPU_ERR_CUDA;
  }
  auto h = std::make_unique<pcgpu_dist>();
  try {
    h->d = *d;
    h->nranks = nranks;
    h->local = nccl_id == nullptr;
    DCK(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
    DCK(cudaEventCreate(&h->ev0));
    DCK(cudaEventCreate(&h->ev1));
    build_dev_problem(d, h->P, h->allocs);
    h->d.row_extent = h->d.col_extent = nullptr;  // copied; no pointer kept
    const int nr = d->nr, nz = d->nz;
    h->tau_floor = d->tau_min > 0 ? d->tau_min : 1e-12 * d->t_per;
    const std::vector<int> re = desc_row_extent(d), ce = desc_col_extent(d);
    for (int i = 0; i < nr; ++i) h->active += ce[i];
    h->zb = split_lines(nz, nranks, [&](int j) { return re[j]; });
    h->rb = split_lines(nr, nranks, [&](int i) { return ce[i]; });
    std::vector<int> mine;
    if (h->local) {
      for (int p = 0; p < nranks; ++p) mine.push_back(p);
    } else {
      if (rank < 0 || rank >= nranks) throw DistError{PCGPU_ERR_ARG, "pcgpu_dist: bad rank"};
      mine.push_back(rank);
      std::string e;
      if (!g_nccl.load(e)) throw DistError{PCGPU_ERR_CUDA, e};
      ncclUniqueId id;
      std::memcpy(&id, nccl_id, sizeof id);
      NCK(g_nccl.commInitRank(&h->comm, nranks, id, rank));
    }
    std::vector<DevStatus*> sts;
    for (int p : mine) {
      RankState R;
      R.rank = p;
      R.j0 = h->zb[p];
      R.nj = h->zcount(p);
      R.i0 = h->rb[p];
      R.ni = h->rcount(p);
      const size_t zc = static_cast<size_t>(R.nj) * nr, rc = static_cast<size_t>(R.ni) * nz;
      R.zTc = h->alloc(zc);
      R.zExpl = h->alloc(zc);
      R.zHalf = h->alloc(zc);
      R.zIter = h->alloc(zc);
      R.zR = h->alloc(zc);
      R.rHalf = h->alloc(rc);
      R.rExpl = h->alloc(rc);
      R.rOut = h->alloc(rc);
      R.rIter = h->alloc(rc);
      // staging: z->r sends 2*zc, receives 2*rc; r->z the reverse
      R.zW = h->alloc(zc);
      R.zX = h->alloc(zc);
      R.rW = h->alloc(rc);
      R.rX = h->alloc(rc);
      R.rKbar = h->alloc(rc);
      R.rTc = h->alloc(rc);
      R.recv = h->alloc(2 * std::max(zc, rc));  // sends go straight from the fields
      DevStatus* st = nullptr;
      DCK(cudaMalloc(&st, sizeof(DevStatus)));
      h->allocs.push_back(st);
      R.st = st;
      sts.push_back(st);
      h->ranks.push_back(R);
    }
    DCK(cudaMalloc(&h->st_dev_list, sizeof(DevStatus*) * sts.size()));
    h->allocs.push_back(h->st_dev_list);
    DCK(cudaMemcpy(h->st_dev_list, sts.data(), sizeof(DevStatus*) * sts.size(),
                   cudaMemcpyHostToDevice));
    DCK(cudaMallocHost(&h->st_host, sizeof(DevStatus)));
    DCK(cudaMalloc(&h->d_barrier, sizeof(unsigned long long)));
    h->allocs.push_back(h->d_barrier);
    DCK(cudaMemset(h->d_barrier, 0, sizeof(unsigned long long)));
    if (nranks > kMaxPeers && d->mode == PCGPU_MODE_EXACT)
      throw DistError{PCGPU_ERR_CONFIG, "pcgpu_dist: at most 16 ranks"};
    if (h->local && d->mode == PCGPU_MODE_EXACT) {
      const char* tr = std::getenv("PCGPU_DIST_TRANSPORT");
      h->peer = !(tr && std::string(tr) == "nccl");
      h->build_peer_table_local();
    }
    DCK(cudaDeviceSynchronize());
  } catch (const DistError& e) {
    g_dist_create_error = e.what;
    return e.code;
  }
  *out = h.release();
  return PCGPU_OK;
}

void pcgpu_dist_destroy(pcgpu_dist* h) {
  if (!h) return;
  DeviceGuard dg_(h->d.device);
  delete h;
}

const char* pcgpu_dist_last_error(const pcgpu_dist* h) {
  return h ? h->err.c_str() : g_dist_create_error.c_str();
}

int pcgpu_dist_slabs(const pcgpu_dist* h, int32_t* z0, int32_t* z1, int32_t* r0, int32_t* r1) {
  // first local rank's slabs (the only one in NCCL mode)
  const RankState& R = h->ranks[0];
  *z0 = R.j0;
  *z1 = R.j0 + R.nj;
  *r0 = R.i0;
  *r1 = R.i0 + R.ni;
  return PCGPU_OK;
}

// Every rank passes the full initial field (device, N layout). Each rank
// keeps its z-slab lines and Lambda_z on them (computed on the full field).
int pcgpu_dist_set_field(pcgpu_dist* h, const double* fieldN) {
  if (!h) return PCGPU_ERR_ARG;
  DeviceGuard dg_(h->d.device);
  try {
    const int nr = h->d.nr;
    for (RankState& R : h->ranks) {
      // z-slab T layout [i][j - j0] <- N rows j0 .. j0+nj-1
      transpose_block(fieldN + static_cast<size_t>(R.j0) * nr, nr, R.nj, nr, R.zTc, R.nj,
                      h->stream);
      // r-slab N layout [j][i - i0] <- columns i0 .. i0+ni-1
      if (R.ni)
        DCK(cudaMemcpy2DAsync(R.rTc, sizeof(double) * R.ni, fieldN + R.i0, sizeof(double) * nr,
                              sizeof(double) * R.ni, h->d.nz, cudaMemcpyDeviceToDevice,
                              h->stream));
    }
    DCK(cudaStreamSynchronize(h->stream));
  } catch (const DistError& e) {
    h->err = e.what;
    return e.code;
  }
  return PCGPU_OK;
}

// Writes each local rank's z-slab lines into the full-size N-layout buffer.
int pcgpu_dist_get_field(pcgpu_dist* h, double* fieldN) {
  if (!h) return PCGPU_ERR_ARG;
  DeviceGuard dg_(h->d.device);
  try {
    const int nr = h->d.nr;
    for (RankState& R : h->ranks)  // r-slab N layout [j][i - i0] -> columns i0 .. i0+ni-1
      if (R.ni)
        DCK(cudaMemcpy2DAsync(fieldN + R.i0, sizeof(double) * nr, R.rTc, sizeof(double) * R.ni,
                              sizeof(double) * R.ni, h->d.nz, cudaMemcpyDeviceToDevice,
                              h->stream));
    DCK(cudaStreamSynchronize(h->stream));
  } catch (const DistError& e) {
    h->err = e.what;
    return e.code;
  }
  return PCGPU_OK;
}

int pcgpu_dist_set_field_host(pcgpu_dist* h, const double* host) {
  if (!h) return PCGPU_ERR_ARG;
  DeviceGuard dg_(h->d.device);
  try {
    const int nr = h->d.nr;
    std::vector<double*> a, b;
    for (RankState& R : h->ranks) {
      // r-slab N layout [j][i - i0] <- host columns i0 .. i0+ni-1
      if (R.ni)
        DCK(cudaMemcpy2DAsync(R.rTc, sizeof(double) * R.ni, host + R.i0, sizeof(double) * nr,
                              sizeof(double) * R.ni, h->d.nz, cudaMemcpyHostToDevice,
                              h->stream));
      a.push_back(R.rTc);
      b.push_back(R.zTc);
    }
    // the peer transport rebuilds the z-slab anchor from rTc in every attempt's
    // fused K3; the NCCL transport keeps it, so refresh it like an acceptance
    if (!h->peer) {
      double* const* s1[1] = {a.data()};
      double* const* d1[1] = {b.data()};
      h->transpose_exact(false, 1, s1, d1);
    }
    DCK(cudaStreamSynchronize(h->stream));
  } catch (const DistError& e) {
    h->err = e.what;
    return e.code;
  }
  return PCGPU_OK;
}

int pcgpu_dist_get_field_host(pcgpu_dist* h, double* host) {
  if (!h) return PCGPU_ERR_ARG;
  DeviceGuard dg_(h->d.device);
  try {
    const int nr = h->d.nr;
    for (RankState& R : h->ranks)
      if (R.ni)
        DCK(cudaMemcpy2DAsync(host + R.i0, sizeof(double) * nr, R.rTc, sizeof(double) * R.ni,
                              sizeof(double) * R.ni, h->d.nz, cudaMemcpyDeviceToHost,
                              h->stream));
    DCK(cudaStreamSynchronize(h->stream));
  } catch (const DistError& e) {
    h->err = e.what;
    return e.code;
  }
  return PCGPU_OK;
}

int pcgpu_dist_run(pcgpu_dist* h, double t0, int32_t nsteps, pcgpu_step_result* results,
                   pcgpu_run_stats* stats) {
  if (!h) return PCGPU_ERR_ARG;
  DeviceGuard dg_(h->d.device);
  pcgpu_run_stats s{};
  double t = t0;
  int rc = PCGPU_OK;
  try {
    for (int32_t k = 0; k < nsteps; ++k) {
      pcgpu_step_result r;
      double upd = 0;
      rc = h->step(t, &r, &upd);
      if (rc) break;
      t += r.tau_used;
      if (results) results[k] = r;
      s.steps += 1;
      s.halvings += r.halvings;
      s.radial_iterations += r.radial.iterations;
      s.axial_iterations += r.axial.iterations;
      s.cell_updates += upd;
      s.cell_updates_accepted +=
          static_cast<double>(h->active) * (r.radial.iterations + r.axial.iterations);
      s.attempt_cells += 2.0 * static_cast<double>(h->active) * (r.halvings + 1);
    }
    DCK(cudaStreamSynchronize(h->stream));
  } catch (const DistError& e) {
    h->err = e.what;
    return e.code;
  }
  s.t_end = t;
  if (stats) *stats = s;
  return rc;
}

int32_t pcgpu_dist_transport(const pcgpu_dist* h) { return h->peer ? 1 : 0; }

int pcgpu_dist_ipc_export(pcgpu_dist* h, void* handles) {
  if (!h) return PCGPU_ERR_ARG;
  DeviceGuard dg_(h->d.device);
  if (!h || !handles || h->local) return PCGPU_ERR_ARG;
  try {
    RankState& R = h->ranks[0];
    double* bufs[4] = {R.zTc, R.zExpl, R.rHalf, R.rExpl};
    auto* out = static_cast<unsigned char*>(handles);
    for (int k = 0; k < 4; ++k) {
      cudaIpcMemHandle_t m;
      DCK(cudaIpcGetMemHandle(&m, bufs[k]));
      std::memcpy(out + k * sizeof m, &m, sizeof m);
    }
  } catch (const DistError& e) {
    h->err = e.what;
    return e.code;
  }
  return PCGPU_OK;
}

int pcgpu_dist_ipc_import(pcgpu_dist* h, const void* all_handles) {
  if (!h) return PCGPU_ERR_ARG;
  DeviceGuard dg_(h->d.device);
  if (!h || !all_handles || h->local) return PCGPU_ERR_ARG;
  try {
    const auto* in = static_cast<const unsigned char*>(all_handles);
    PeerSlabs ps{};
    ps.nranks = h->nranks;
    for (int q = 0; q <= h->nranks; ++q) {
      ps.zb[q] = h->zb[q];
      ps.rb[q] = h->rb[q];
    }
    const int me = h->ranks[0].rank;
    for (int q = 0; q < h->nranks; ++q) {
      double** dst[4] = {&ps.zTc[q], &ps.zExpl[q], &ps.rHalf[q], &ps.rExpl[q]};
      if (q == me) {
        RankState& R = h->ranks[0];
        *dst[0] = R.zTc;
        *dst[1] = R.zExpl;
        *dst[2] = R.rHalf;
        *dst[3] = R.rExpl;
        continue;
      }
      for (int k = 0; k < 4; ++k) {
        cudaIpcMemHandle_t m;
        std::memcpy(&m, in + (static_cast<size_t>(q) * 4 + k) * sizeof m, sizeof m);
        void* p = nullptr;
        const cudaError_t ce = cudaIpcOpenMemHandle(&p, m, cudaIpcMemLazyEnablePeerAccess);
        if (ce != cudaSuccess) {
          (void)cudaGetLastError();
          for (void* o : h->ipc_opened) cudaIpcCloseMemHandle(o);
          h->ipc_opened.clear();
          DCK(ce);
        }
        h->ipc_opened.push_back(p);
        *dst[k] = static_cast<double*>(p);
      }
    }
    h->ps = ps;
    h->peer = true;
  } catch (const DistError& e) {
    h->err = e.what;
    return e.code;
  }
  return PCGPU_OK;
}

int pcgpu_dist_peer_off(pcgpu_dist* h) {
  if (!h) return PCGPU_ERR_ARG;
  DeviceGuard dg_(h->d.device);
  if (!h) return PCGPU_ERR_ARG;
  if (h->local) return PCGPU_OK;  // emulated ranks: peer stores into local slabs
  cudaStreamSynchronize(h->stream);
  for (void* p : h->ipc_opened) cudaIpcCloseMemHandle(p);
  h->ipc_opened.clear();
  h->peer = false;
  return PCGPU_OK;
}

void* pcgpu_dist_stream(const pcgpu_dist* h) { return h->stream; }

int64_t pcgpu_dist_launch_count(const pcgpu_dist* h) {
  (void)h;
  return static_cast<int64_t>(g_launches);
}

int pcgpu_dist_plan(const pcgpu_desc* d, int32_t nranks, int32_t* zb, int32_t* rb) {
  if (!d || nranks < 1 || !zb || !rb) return PCGPU_ERR_ARG;
  const int nr = d->nr, nz = d->nz;
  const std::vector<int> re = desc_row_extent(d), ce = desc_col_extent(d);
  const auto z = split_lines(nz, nranks, [&](int j) { return re[j]; });
  const auto r = split_lines(nr, nranks, [&](int i) { return ce[i]; });
  for (int p = 0; p <= nranks; ++p) {
    zb[p] = z[p];
    rb[p] = r[p];
  }
  return PCGPU_OK;
}

int pcgpu_dist_enable_timing(pcgpu_dist* h, int32_t on) {
  h->timing = on != 0;
  h->transpose_ms = h->radial_ms = h->axial_ms = 0;
  h->transposes = h->allreduces = h->radial_launches = h->axial_launches = 0;
  return PCGPU_OK;
}

int pcgpu_dist_timing(const pcgpu_dist* h, double* transpose_ms, int64_t* transposes,
                      int64_t* allreduces, double* radial_ms, double* axial_ms) {
  *transpose_ms = h->transpose_ms;
  *transposes = h->transposes;
  *allreduces = h->allreduces;
  *radial_ms = h->radial_ms;
  *axial_ms = h->axial_ms;
  return PCGPU_OK;
}

}  // extern "C"
