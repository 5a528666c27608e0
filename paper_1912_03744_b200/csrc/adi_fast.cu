// adi_fast.cu -- throughput-mode ADI kernels (sm_100a, FP64).
//
// Same discrete equations as the reference (solver.cpp:162-332), solved with a
// partitioned line solver instead of one sequential Thomas recurrence per
// line, so that a long line is spread over many threads and a cluster of CTAs:
//
//  * Each line lives in the layout where it is CONTIGUOUS: radial lines in the
//    natural layout N (j*nr + i), axial lines in the transposed layout T
//    (i*nz + j). The explicit passes (K3/K4) write the layout the next sweep
//    needs, so the transposes cost no extra pass.
//  * A cluster of CL CTAs owns one line (CL = ceil(n / 2048)); a CTA owns a
//    2048-row segment, a thread owns R = 16 consecutive rows. Rows are staged
//    into shared memory with coalesced cp.async (16-B) into an XOR-swizzled
//    tile (conflict-free 128-bit reads of a thread's own 16 rows).
//  * Per thread: assemble the 16 rows' coefficients (face conductivities,
//    capacities, Joule power -- the reference's formulas) fused with the
//    forward elimination of the chunk interior (rows 0..14), carrying two
//    extra right-hand sides for the coupling to the neighbouring chunks'
//    last unknowns (a "lasts-only" partition: one reduced unknown per chunk).
//  * Reduced system (one unknown per chunk, 128 per CTA): parallel cyclic
//    reduction in shared memory with three right-hand sides (the particular
//    solution and the two spikes towards the neighbouring CTAs).
//  * Cluster level: every CTA publishes its first/last reduced unknowns'
//    affine form to all CTAs of the cluster through distributed shared memory;
//    each CTA solves the 2*CL boundary system (block Thomas, O(CL)) itself.
//  * Back-substitution per chunk, out = anchor + x, line max |out - T_iter|,
//    swizzled tile -> coalesced store; one atomicMax per warp for the delta.
// DRAM traffic per Picard iteration = read iterate, anchor, explicit term,
// write the new iterate: 32 B per cell; K-bar is recomputed
// from the anchor in the axial sweep instead of being stored.
#include <cooperative_groups.h>

#include <cstdint>
#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "adi_kernels.h"

namespace cg = cooperative_groups;

namespace pcgpu {

namespace {

constexpr int R = 16;          // rows per thread
constexpr int NT = 128;        // threads per CTA
constexpr int SEG = NT * R;    // rows per CTA
constexpr int kMaxCluster = 8; // portable cluster size -> lines up to 16384 rows

__device__ __forceinline__ int row_extent(const DevProblem& P, int j) {
  return __ldg(P.row_ext + j);
}
__device__ __forceinline__ int col_extent(const DevProblem& P, int i) {
  return __ldg(P.col_ext + i);
}

__device__ __forceinline__ bool skip_iteration(const DevStatus* st, int it, double eps) {
  if (st->err != kNoError) return true;
  if (it <= 1) return false;
  return __longlong_as_double(static_cast<long long>(st->delta[it - 1])) < eps;
}

// Byte offset of element e of a 2048-row tile: thread chunk t = e/16 occupies
// 128 B; its 16-B quad q is stored at quad slot q ^ (t & 7).
__device__ __forceinline__ uint32_t swz(int e) {
  const int t = e >> 4, o = e & 15, q = o >> 1;
  return static_cast<uint32_t>(t * 128 + ((q ^ (t & 7)) << 4) + ((o & 1) << 3));
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void cp_async16(uint32_t saddr, const void* g, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(saddr), "l"(g),
               "r"(src_bytes));
}
__device__ __forceinline__ void cp_async8(uint32_t saddr, const void* g, int src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(saddr), "l"(g),
               "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}

struct alignas(16) Tile {
  double v[SEG];
};

struct FastSmem {
  // small per-CTA state first (low shared-memory offsets)
  double halo[4];              // ts[seg0-1], ta[seg0-1], ts[seg0+SEG], ta[seg0+SEG]
  double bnd[kMaxCluster][6];  // per-CTA boundary forms (y0,p0,r0,yL,pL,rL)
  double EF[2];                // E_{rank-1}, F_{rank+1}
  double bs[4][kMaxCluster + 1];  // boundary-system scratch (ph, ps, ea, eb)
  double fu[NT + 1], fv[NT + 1], fw[NT + 1];  // first-interior-row affine forms
  double q[NT];                // reduced unknowns (last row of each chunk)
  double pL[2][NT], pD[2][NT], pU[2][NT], pY[2][NT], pP[2][NT], pR[2][NT];  // PCR
  Tile ts, ta, ex;             // iterate, anchor, explicit term (swizzled, 16-B aligned)
};

// Lean-variant table lookup (all tables of a property share an exactly
// uniform power-of-two knot grid): clamp by selects, bracket by arithmetic,
// interval start recomputed exactly (t0 + (k-1) h), one 16-B load {v, slope}.
// Returns the value and counts an out-of-range evaluation in *oor.
// Reciprocal without the IEEE slow path: MUFU seed + two Newton steps
// (relative error ~1 ulp for the normal, positive pivots of these M-matrices).
__device__ __forceinline__ double rcp_nr(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = __fma_rn(-x, r, 1.0);
  r = __fma_rn(r, e, r);
  e = __fma_rn(-x, r, 1.0);
  return __fma_rn(r, e, r);
}

// Register-resident per-layer table data for the lean lookup.
struct LeanTab {
  int off;
  double v0, vK;
};

// Lean-variant lookup. Tables of one property share an exactly uniform
// power-of-two knot grid across layers (P.lean_*); entry (prop, layer, k) of
// P.lean_tab holds {v[k-1], slope_k}. T is clamped to the knot range first;
// at the clamp points the interpolation reproduces the end values up to one
// rounding. Out-of-range evaluations (clamp_events) are counted in `oor`.
__device__ __forceinline__ double lean_lookup2(const DevProblem& P, int prop, int L, double T,
                                               int& oor, bool valid) {
  const double t0 = P.lean_t0[prop], tK = P.lean_tK[prop];
  const double Tc = fmin(fmax(T, t0), tK);
  int k = static_cast<int>(__dmul_rn(Tc - t0, P.lean_inv_h[prop])) + 1;
  k = min(k, P.lean_kmax[prop]);
  const double2 vs =
      __ldg(reinterpret_cast<const double2*>(P.lean_tab) + P.lean_base[prop] +
            L * P.lean_stride[prop] + k);
  const double tlo = __dadd_rn(t0, __dmul_rn(static_cast<double>(k - 1), P.lean_h[prop]));
  oor += (valid && !(T >= t0 && T <= tK)) ? 1 : 0;
  return __dadd_rn(vs.x, __dmul_rn(Tc - tlo, vs.y));
}

// Lean v2 lookup: value = a_k + s_k * T on the interval located by
// x = T / h - t0 / h (one FMA, one conversion, one 16-B load, one FMA).
// Out-of-range temperatures are rare: a warp vote sends them to the clamp
// (materials.hpp:40-41) and the clamp_events count (materials.cpp:68).
__device__ __forceinline__ double lean_v(const DevProblem& P, int prop, int L, double T,
                                         bool valid) {
  const double x = fma(T, P.lean_ih[prop], -P.lean_x0[prop]);
  int k = __double2int_rz(x);
  k = min(max(k, 0), P.lean_kmax[prop] - 1);
  const double2 ab = __ldg(reinterpret_cast<const double2*>(P.lean_ab) + P.lean_base[prop] +
                           L * P.lean_stride[prop] + k + 1);
  double v = fma(ab.y, T, ab.x);
  const bool o = !(x >= 0.0 && x <= P.lean_kmaxd[prop]);
  if (__any_sync(0xffffffffu, o)) {
    if (o) {
      const double t0 = P.lean_t0[prop], tK = P.lean_tK[prop];
      const double Tc = T < t0 ? t0 : (T > tK ? tK : T);
      v = fma(ab.y, Tc, ab.x);
      if (valid) atomicAdd(P.clamp + L, 1ull);
    }
  }
  return v;
}

__device__ __forceinline__ double tile_get(const Tile& t, int e) {
  return *reinterpret_cast<const double*>(reinterpret_cast<const char*>(t.v) + swz(e));
}
__device__ __forceinline__ void tile_put(Tile& t, int e, double v) {
  *reinterpret_cast<double*>(reinterpret_cast<char*>(t.v) + swz(e)) = v;
}

struct LineArgs {
  const double* Ts;  // Picard iterate
  const double* Ta;  // anchor (T_cur for the radial sweep, T_half for the axial)
  const double* ex;  // explicit term (Lambda_z[T_cur] / Lambda_r[T_half] + X(T_half))
  const double* pw;  // bound power field (N layout) for PCGPU_SOURCE_FIELD, or null
  double* out;
  long long ld;      // line stride in elements
  int nlines;        // lines in this launch
  int line0;         // global index of the first line (slab offset)
  int it;
  double eps, hk, pulse;
  DevStatus* st;
};

// ---------------------------------------------------------------------------
// One Picard iteration of a sweep over contiguous lines.
// kLean: 0 = generic (any rule / policy / table / source); 1 = lean, no
// source term in the sweep; 2 = lean with the Joule source (radial sweep).
// Lean requires: MeanTemperature faces, Clamp policy, every table exactly
// uniform (power-of-two step) with one knot grid per property across layers.
template <bool kAxial, bool kU2, int kLean, bool kDirect = false>
__global__ void __launch_bounds__(NT, kDirect ? 4 : 3) k_line_fast(DevProblem P, LineArgs A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  FastSmem& S = *reinterpret_cast<FastSmem*>(smem_raw);
  if (skip_iteration(A.st, A.it, A.eps)) return;

  cg::cluster_group cluster = cg::this_cluster();
  const int CL = static_cast<int>(cluster.num_blocks());
  const int rank = static_cast<int>(cluster.block_rank());
  const int lline = blockIdx.x / CL;    // line within this launch's slab
  const int line = A.line0 + lline;     // global line index (masks, layers, errors)
  const int tid = threadIdx.x;
  const int n = kAxial ? col_extent(P, line) : row_extent(P, line);
  const int seg0 = rank * SEG;
  const size_t lbase = static_cast<size_t>(lline) * static_cast<size_t>(A.ld);
  const double* gTs = A.Ts + lbase;
  const double* gTa = A.Ta + lbase;
  const double* gEx = A.ex + lbase;

  // ---- stage the segment's rows (coalesced cp.async, zero-filled past n) ----
  const int nseg = max(0, min(SEG, n - seg0));
  if (kDirect) {
    // rows are read straight into registers below (no shared-memory tiles)
  } else if ((A.ld & 1) == 0) {
    for (int e = 2 * tid; e < SEG; e += 2 * NT) {
      const int valid = max(0, min(2, nseg - e));
      const int r = seg0 + (valid ? e : 0);
      const uint32_t o = swz(e);
      cp_async16(smem_u32(S.ts.v) + o, gTs + r, valid * 8);
      cp_async16(smem_u32(S.ta.v) + o, gTa + r, valid * 8);
      cp_async16(smem_u32(S.ex.v) + o, gEx + r, valid * 8);
    }
  } else {
    for (int e = tid; e < SEG; e += NT) {
      const int valid = e < nseg ? 1 : 0;
      const int r = seg0 + (valid ? e : 0);
      const uint32_t o = swz(e);
      cp_async8(smem_u32(S.ts.v) + o, gTs + r, valid * 8);
      cp_async8(smem_u32(S.ta.v) + o, gTa + r, valid * 8);
      cp_async8(smem_u32(S.ex.v) + o, gEx + r, valid * 8);
    }
  }
  if (!kDirect && tid == 0) {
    const bool lo = seg0 >= 1 && seg0 - 1 < n;
    const bool hi = seg0 + SEG < n;
    S.halo[0] = lo ? gTs[seg0 - 1] : 0.0;
    S.halo[1] = lo ? gTa[seg0 - 1] : 0.0;
    S.halo[2] = hi ? gTs[seg0 + SEG] : 0.0;
    S.halo[3] = hi ? gTa[seg0 + SEG] : 0.0;
  }
  cp_async_wait_all();
  __syncthreads();

  // ---- per-line constants ----
  int Lline = 0;
  double rho_hk = 0.0, face_top = 0.0;
  bool dirichlet = false;
  if (kAxial) {
    Lline = P.layer[line];
    rho_hk = P.mats[Lline].rho * A.hk;
    dirichlet = Lline == 0 && !P.all_neumann;
    if (dirichlet && n - 1 >= seg0 + tid * R && n - 1 < seg0 + (tid + 1) * R) {
      // lambda(T0) / (0.5 * width_z(m-1)) at the terminal Dirichlet face (solver.cpp:315-320)
      face_top = mat_eval_fast(P, Lline, kLambda, P.T0, A.st, line) * __drcp_rn(0.5 * P.width_z[n - 1]);
    }
  }

  // ---- this thread's rows, streamed from the tile with a rolling window ----
  // Row index k in [-1, R] of the chunk <-> global row s + k.
  const int s = seg0 + tid * R;
  const int e0 = tid * R;
  // Direct variant: the chunk's rows (and one halo row each side) are loaded
  // with 16-B vector loads straight into registers; no shared-memory tiles.
  double rts[R + 2], rta[R + 2], rex[R];
  if (kDirect) {
    const bool full = s + R <= n;
    if (full) {
#pragma unroll
      for (int q = 0; q < R / 2; ++q) {
        const double2 a = __ldg(reinterpret_cast<const double2*>(gTs + s) + q);
        const double2 b = __ldg(reinterpret_cast<const double2*>(gTa + s) + q);
        const double2 c = __ldg(reinterpret_cast<const double2*>(gEx + s) + q);
        rts[2 * q + 1] = a.x; rts[2 * q + 2] = a.y;
        rta[2 * q + 1] = b.x; rta[2 * q + 2] = b.y;
        rex[2 * q] = c.x; rex[2 * q + 1] = c.y;
      }
    } else {
#pragma unroll
      for (int k = 0; k < R; ++k) {
        const bool v = s + k < n;
        const int r = v ? s + k : 0;
        rts[k + 1] = v ? __ldg(gTs + r) : 0.0;
        rta[k + 1] = v ? __ldg(gTa + r) : 0.0;
        rex[k] = v ? __ldg(gEx + r) : 0.0;
      }
    }
    const bool lo = s >= 1 && s - 1 < n;
    const bool hi = s + R < n;
    rts[0] = lo ? __ldg(gTs + s - 1) : 0.0;
    rta[0] = lo ? __ldg(gTa + s - 1) : 0.0;
    rts[R + 1] = hi ? __ldg(gTs + s + R) : 0.0;
    rta[R + 1] = hi ? __ldg(gTa + s + R) : 0.0;
  }
  auto ld_ts = [&](int k) -> double {
    if (kDirect) return rts[k + 1];
    if (k < 0) return tid > 0 ? tile_get(S.ts, e0 - 1) : S.halo[0];
    if (k >= R) return tid < NT - 1 ? tile_get(S.ts, e0 + R) : S.halo[2];
    return tile_get(S.ts, e0 + k);
  };
  auto ld_ta = [&](int k) -> double {
    if (kDirect) return rta[k + 1];
    if (k < 0) return tid > 0 ? tile_get(S.ta, e0 - 1) : S.halo[1];
    if (k >= R) return tid < NT - 1 ? tile_get(S.ta, e0 + R) : S.halo[3];
    return tile_get(S.ta, e0 + k);
  };
  auto ld_ex = [&](int k) -> double { return kDirect ? rex[k] : tile_get(S.ex, e0 + k); };
  // final update: re-read (L1/L2-resident) so the row registers die after assembly
  auto fin_ts = [&](int k) -> double { return kDirect ? __ldg(gTs + min(s + k, n - 1)) : ld_ts(k); };
  auto fin_ta = [&](int k) -> double { return kDirect ? __ldg(gTa + min(s + k, n - 1)) : ld_ta(k); };
  // Face f = s + k (between rows f-1 and f): conductance and anchor flux.
  auto face = [&](int k, double ts_lo, double ts_hi, double ta_lo, double ta_hi, double& c,
                  double& flux) {
    const int f = s + k;
    c = 0.0;
    if (f >= 1 && f <= n - 1) {
      if (kAxial) {
        const double lam = k == 0 ? face_lambda_fast<false, kU2>(P, Lline, Lline, ts_lo, ts_hi, A.st, line)
                                  : face_lambda_fast<true, kU2>(P, Lline, Lline, ts_lo, ts_hi, A.st, line);
        c = lam * P.inv_gap_z[f];
      } else {
        const int lo = P.layer[f - 1], hi = P.layer[f];
        const double lam = k == 0 ? face_lambda_fast<false, kU2>(P, lo, hi, ts_lo, ts_hi, A.st, line)
                                  : face_lambda_fast<true, kU2>(P, lo, hi, ts_lo, ts_hi, A.st, line);
        c = P.face_r_lo[f] * lam * P.inv_gap_r[f];
      }
    }
    flux = c * (ta_hi - ta_lo);
  };

  // ---- rows: assembly fused with the forward elimination of the interior ----
  double cp[R - 1], up[R - 1], vp[R - 1];
  double wp = 0.0;
  double AL = 0.0, CL_ = 0.0, bL = 1.0, dL = 0.0;
  if (kLean) {
    // Branch-free assembly: invalid faces/rows are neutralised by selects;
    // table data comes from the property-grouped lean table (one 16-B load
    // per lookup, no per-row parameter indexing).
    const int nm1 = n - 1;
    const int Lax = kAxial ? P.layer[line] : 0;
    const double rho_hk_ax = kAxial ? P.mats[Lax].rho * A.hk : 0.0;
    const double src_amp = (kLean == 2 && A.pulse != 0.0) ? P.amplitude * A.pulse : 0.0;
    int oor = 0;  // out-of-range evaluations (clamp_events), axial sweep
    double ts_c = ld_ts(0), ta_c = ld_ta(0);
    double fc_lo, fl_lo;
    int Lc = kAxial ? Lax : __ldg(P.layer + min(s, P.nr - 1));
    {
      // face s (lower face of the chunk): owned by the previous chunk's count
      const int f = s;
      const bool vf = f >= 1 && f <= nm1;
      const double tp = ld_ts(-1), tpa = ld_ta(-1);
      int dummy = 0;
      double c;
      if (kAxial) {
        c = lean_v(P, kLambda, Lax, 0.5 * (tp + ts_c), false) * __ldg(P.inv_gap_z + min(f, P.nz));
      } else {
        const int Lp = __ldg(P.layer + min(max(f - 1, 0), P.nr - 1));
        c = lean_v(P, kLambda, Lp, 0.5 * (tp + ts_c), false) * __ldg(P.gfac_r + min(f, P.nr));
      }
      fc_lo = vf ? c : 0.0;
      fl_lo = fc_lo * (ta_c - tpa);
    }
    double cp_prev = 0.0, up_prev = 0.0, vp_prev = 0.0;
    const double2* met = reinterpret_cast<const double2*>(kAxial ? P.zmet : P.rmet);
    const int nmet = kAxial ? P.nz : P.nr;
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const int i = s + k;
      const double ts_n = ld_ts(k + 1), ta_n = ld_ta(k + 1);
      const int f = i + 1;  // face between rows i and i+1
      const bool vf = f <= nm1;
      const bool vi = i < n;
      // per-row metrics {face conductance factor of face i+1, 1/control volume of row i}
      const double2 mt = __ldg(met + min(i, nmet - 1));
      int Ln = Lc;
      double lam;
      if (kAxial) {
        lam = lean_v(P, kLambda, Lax, 0.5 * (ts_c + ts_n), vf);
      } else {
        Ln = __ldg(P.layer + min(f, P.nr - 1));
        lam = lean_v(P, kLambda, Lc, 0.5 * (ts_c + ts_n), vf);
      }
      const double fc_hi = vf ? lam * mt.x : 0.0;
      const double fl_hi = fc_hi * (ta_n - ta_c);
      const double exk = ld_ex(k);
      const double inv = mt.y;  // inv_eta (axial) / inv_vol (radial)
      double Ak = fc_lo * inv, Ck = fc_hi * inv, bk, dk;
      if (kAxial) {
        const double K = A.hk * lean_v(P, kCv, Lax, ta_c, vi);  // rho folded in
        bk = K + Ak + Ck;
        const bool top = i == nm1;  // terminal Dirichlet face (face_top = 0 elsewhere)
        bk += top ? face_top * inv : 0.0;
        const double fh = fl_hi + (top ? face_top * (P.T0 - ta_c) : 0.0);
        dk = exk + (fh - fl_lo) * inv;
      } else {
        const double K = A.hk * lean_v(P, kCv, Lc, ts_c, vi);  // rho folded in
        double src = 0.0;
        if (kLean == 2) {
          // JouleSource::power: chi(T) * amplitude * pulse in the source layer
          const bool on = Lc == P.source_layer;
          src = (on ? src_amp : 0.0) *
                lean_v(P, kChi, P.source_layer, ts_c, vi && on && src_amp != 0.0);
        }
        bk = K + Ak + Ck;
        dk = (fl_hi - fl_lo) * inv + exk + src;
      }
      Ak = vi ? Ak : 0.0;
      Ck = vi ? Ck : 0.0;
      bk = vi ? bk : 1.0;
      dk = vi ? dk : 0.0;
      if (k < R - 1) {
        const double piv = k == 0 ? bk : bk + Ak * cp_prev;
        const double ip = rcp_nr(piv);
        const double cc = k < R - 2 ? -Ck * ip : 0.0;
        if (k == R - 2) wp = Ck * ip;
        const double u = k == 0 ? dk * ip : (dk + Ak * up_prev) * ip;
        const double v = k == 0 ? Ak * ip : Ak * vp_prev * ip;
        cp[k] = cc;
        up[k] = u;
        vp[k] = v;
        cp_prev = cc;
        up_prev = u;
        vp_prev = v;
      } else {
        AL = Ak;
        CL_ = Ck;
        bL = bk;
        dL = dk;
      }
      ts_c = ts_n;
      ta_c = ta_n;
      fc_lo = fc_hi;
      fl_lo = fl_hi;
      Lc = Ln;
    }
    if (kAxial && oor) atomicAdd(P.clamp + Lax, static_cast<unsigned long long>(oor));
  } else {
    double ts_c = ld_ts(0), ta_c = ld_ta(0);
    double fc_lo, fl_lo;
    face(0, ld_ts(-1), ts_c, ld_ta(-1), ta_c, fc_lo, fl_lo);
    double cp_prev = 0.0, up_prev = 0.0, vp_prev = 0.0;
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const double ts_n = ld_ts(k + 1), ta_n = ld_ta(k + 1);
      double fc_hi, fl_hi;
      face(k + 1, ts_c, ts_n, ta_c, ta_n, fc_hi, fl_hi);
      const int i = s + k;
      double Ak = 0.0, Ck = 0.0, bk = 1.0, dk = 0.0;
      if (i < n) {
        const double exk = ld_ex(k);
        if (kAxial) {
          const double inv_eta = P.inv_eta[i];
          Ak = fc_lo * inv_eta;
          Ck = fc_hi * inv_eta;
          const double K = rho_hk * mat_eval_fast<true, kU2>(P, Lline, kCv, ta_c, A.st, line);
          bk = K + Ak + Ck;
          double fh = fl_hi;
          if (i == n - 1 && dirichlet) {
            bk += face_top * inv_eta;
            fh += face_top * (P.T0 - ta_c);
          }
          dk = exk + (fh - fl_lo) * inv_eta;
        } else {
          const int L = P.layer[i];
          const double inv_vol = P.inv_vol_r[i];
          Ak = fc_lo * inv_vol;
          Ck = fc_hi * inv_vol;
          const double K = P.mats[L].rho * A.hk * mat_eval_fast<true, kU2>(P, L, kCv, ts_c, A.st, line);
          bk = K + Ak + Ck;
          const double fp = P.source_kind == PCGPU_SOURCE_FIELD
                                ? A.pw[static_cast<size_t>(line) * P.nr + i] : 0.0;
          dk = (fl_hi - fl_lo) * inv_vol + exk +
               source_power_fast<kU2>(P, A.pulse, L, ts_c, fp, A.st, line);
        }
      }
      if (k < R - 1) {
        // interior row: a_k = -A_k, c_k = -C_k (the last interior row's c
        // couples to the chunk's last unknown and goes to the w spike)
        const double piv = k == 0 ? bk : bk + Ak * cp_prev;
        if (piv == 0.0) report_error(A.st, line, PCGPU_ERR_ZERO_PIVOT);
        const double ip = __drcp_rn(piv);
        const double c = k < R - 2 ? -Ck * ip : 0.0;
        if (k == R - 2) wp = Ck * ip;  // rhs +C_{R-2} * Q (row R-2's coupling moved right)
        const double u = k == 0 ? dk * ip : (dk + Ak * up_prev) * ip;
        const double v = k == 0 ? Ak * ip : Ak * vp_prev * ip;
        cp[k] = c;
        up[k] = u;
        vp[k] = v;
        cp_prev = c;
        up_prev = u;
        vp_prev = v;
      } else {
        AL = Ak;
        CL_ = Ck;
        bL = bk;
        dL = dk;
      }
      ts_c = ts_n;
      ta_c = ta_n;
      fc_lo = fc_hi;
      fl_lo = fl_hi;
    }
  }
  // Interior solution as an affine form of (Q_prev, Q_own): x_k = u + Qp v + Qo w.
  double uL = up[R - 2], vL = vp[R - 2], wL = wp;
  {
    double u = uL, v = vL, w = wL;
#pragma unroll
    for (int k = R - 3; k >= 0; --k) {
      u = up[k] - cp[k] * u;
      v = vp[k] - cp[k] * v;
      w = -cp[k] * w;
    }
    S.fu[tid] = u;
    S.fv[tid] = v;
    S.fw[tid] = w;
  }
  if (CL > 1) cluster.sync(); else __syncthreads();
  double nu = 0.0, nv = 0.0, nw = 0.0;
  if (tid < NT - 1) {
    nu = S.fu[tid + 1]; nv = S.fv[tid + 1]; nw = S.fw[tid + 1];
  } else if (rank + 1 < CL) {
    FastSmem* R1 = cluster.map_shared_rank(&S, rank + 1);
    nu = R1->fu[0]; nv = R1->fv[0]; nw = R1->fw[0];
  }
  // Reduced row of this chunk's last unknown (row R-1):
  //   a_L x_{R-2} + b_L Q + c_L x_{next first} = d_L
  {
    double Lr = -AL * vL;
    double Dr = bL - AL * wL - CL_ * nv;
    double Ur = -CL_ * nw;
    double Yr = dL + AL * uL + CL_ * nu;
    double Pp = 0.0, Rr = 0.0;
    if (tid == 0) { Pp = -Lr; Lr = 0.0; }          // spike towards the previous CTA
    if (tid == NT - 1) { Rr = -Ur; Ur = 0.0; }     // spike towards the next CTA
    S.pL[0][tid] = Lr; S.pD[0][tid] = Dr; S.pU[0][tid] = Ur;
    S.pY[0][tid] = Yr; S.pP[0][tid] = Pp; S.pR[0][tid] = Rr;
  }
  __syncthreads();
  // ---- parallel cyclic reduction on the CTA's reduced system (3 rhs) ----
  int cur = 0;
#pragma unroll 1
  for (int d = 1; d < NT; d <<= 1) {
    const double Lr = S.pL[cur][tid], Dr = S.pD[cur][tid], Ur = S.pU[cur][tid];
    double Y = S.pY[cur][tid], Pp = S.pP[cur][tid], Rr = S.pR[cur][tid];
    double nL = 0.0, nD = Dr, nU = 0.0;
    if (tid - d >= 0) {
      const int m = tid - d;
      const double k1 = Lr * __drcp_rn(S.pD[cur][m]);
      nL = -S.pL[cur][m] * k1;
      nD -= S.pU[cur][m] * k1;
      Y -= S.pY[cur][m] * k1;
      Pp -= S.pP[cur][m] * k1;
      Rr -= S.pR[cur][m] * k1;
    }
    if (tid + d < NT) {
      const int p = tid + d;
      const double k2 = Ur * __drcp_rn(S.pD[cur][p]);
      nU = -S.pU[cur][p] * k2;
      nD -= S.pL[cur][p] * k2;
      Y -= S.pY[cur][p] * k2;
      Pp -= S.pP[cur][p] * k2;
      Rr -= S.pR[cur][p] * k2;
    }
    const int nx = cur ^ 1;
    S.pL[nx][tid] = nL; S.pD[nx][tid] = nD; S.pU[nx][tid] = nU;
    S.pY[nx][tid] = Y; S.pP[nx][tid] = Pp; S.pR[nx][tid] = Rr;
    cur = nx;
    __syncthreads();
  }
  const double invD = __drcp_rn(S.pD[cur][tid]);
  const double qy = S.pY[cur][tid] * invD, qp = S.pP[cur][tid] * invD, qr = S.pR[cur][tid] * invD;
  double Eprev = 0.0, Fnext = 0.0;
  if (CL > 1) {
    // publish (y, p, r) of the first and last reduced unknowns to every CTA
    if (tid == 0 || tid == NT - 1) {
      const int o = tid == 0 ? 0 : 3;
      for (int c = 0; c < CL; ++c) {
        FastSmem* Rc = cluster.map_shared_rank(&S, c);
        Rc->bnd[rank][o] = qy;
        Rc->bnd[rank][o + 1] = qp;
        Rc->bnd[rank][o + 2] = qr;
      }
    }
    cluster.sync();
    if (tid == 0) {
      // Boundary system over CTAs c: F_c = y0 + p0 E_{c-1} + r0 F_{c+1},
      //                              E_c = yL + pL E_{c-1} + rL F_{c+1}.
      // Forward: E_{c-1} = al + be F_c; back: F_c = ph_c + ps_c F_{c+1}.
      double al = 0.0, be = 0.0;
      double* ph = S.bs[0];
      double* ps = S.bs[1];
      double* ea = S.bs[2];
      double* eb = S.bs[3];
      for (int c = 0; c < CL; ++c) {
        const double* b = S.bnd[c];
        const double den = __drcp_rn(1.0 - b[1] * be);
        ph[c] = (b[0] + b[1] * al) * den;
        ps[c] = b[2] * den;
        ea[c] = b[3] + b[4] * (al + be * ph[c]);
        eb[c] = b[4] * be * ps[c] + b[5];
        al = ea[c];
        be = eb[c];
      }
      // Back substitution: F_c = ph_c + ps_c F_{c+1}, E_c = ea_c + eb_c F_{c+1}.
      double F = 0.0, Eprev_ = 0.0, Fnext_ = 0.0;
      for (int c = CL - 1; c >= 0; --c) {
        if (c == rank) Fnext_ = F;
        if (c == rank - 1) Eprev_ = ea[c] + eb[c] * F;
        F = ph[c] + ps[c] * F;
      }
      S.EF[0] = Eprev_;
      S.EF[1] = Fnext_;
    }
    __syncthreads();
    Eprev = S.EF[0];
    Fnext = S.EF[1];
  }
  const double Q = qy + Eprev * qp + Fnext * qr;
  S.q[tid] = Q;
  __syncthreads();
  const double Qprev = tid > 0 ? S.q[tid - 1] : Eprev;

  // ---- back substitution, update, delta, staged store ----
  double dmax = 0.0;
  double* gOut = A.out + lbase;
  if (kDirect) {
    double ro[R];
    double xn = Q;
    ro[R - 1] = xn;
    double x = up[R - 2] + Qprev * vp[R - 2] + wp * Q;
#pragma unroll
    for (int k = R - 2; k >= 0; --k) {
      if (k < R - 2) x = up[k] + Qprev * vp[k] - cp[k] * xn;
      ro[k] = x;
      xn = x;
    }
    const bool full = s + R <= n;
#pragma unroll
    for (int q = 0; q < R / 2; ++q) {
      double o0 = 0.0, o1 = 0.0;
      if (full) {
        const double2 a = __ldg(reinterpret_cast<const double2*>(gTa + s) + q);
        const double2 t = __ldg(reinterpret_cast<const double2*>(gTs + s) + q);
        o0 = a.x + ro[2 * q];
        o1 = a.y + ro[2 * q + 1];
        dmax = ref_max(dmax, fabs(o0 - t.x));
        dmax = ref_max(dmax, fabs(o1 - t.y));
        reinterpret_cast<double2*>(gOut + s)[q] = make_double2(o0, o1);
      } else {
        for (int h = 0; h < 2; ++h) {
          const int k = 2 * q + h;
          if (s + k < n) {
            const double o = fin_ta(k) + ro[k];
            dmax = ref_max(dmax, fabs(o - fin_ts(k)));
            gOut[s + k] = o;
          }
        }
      }
    }
  } else {
    double xn = Q;
    const int kl = R - 1;
    if (s + kl < n) {
      const double o = ld_ta(kl) + xn;
      tile_put(S.ex, e0 + kl, o);
      dmax = ref_max(dmax, fabs(o - ld_ts(kl)));
    }
    double x = up[R - 2] + Qprev * vp[R - 2] + wp * Q;
#pragma unroll
    for (int k = R - 2; k >= 0; --k) {
      if (k < R - 2) x = up[k] + Qprev * vp[k] - cp[k] * xn;
      if (s + k < n) {
        const double o = ld_ta(k) + x;
        tile_put(S.ex, e0 + k, o);
        dmax = ref_max(dmax, fabs(o - ld_ts(k)));
      }
      xn = x;
    }
  }
  __syncthreads();
  if (kDirect) {
    // stored directly above
  } else if ((A.ld & 1) == 0) {
    for (int e = 2 * tid; e < nseg; e += 2 * NT) {
      const double2 v = *reinterpret_cast<const double2*>(reinterpret_cast<const char*>(S.ex.v) + swz(e));
      if (e + 1 < nseg) {
        *reinterpret_cast<double2*>(gOut + seg0 + e) = v;
      } else {
        gOut[seg0 + e] = v.x;
      }
    }
  } else {
    for (int e = tid; e < nseg; e += NT) gOut[seg0 + e] = tile_get(S.ex, e);
  }
  dmax = warp_max(dmax);
  if ((tid & 31) == 0)
    atomicMax(&A.st->delta[A.it], static_cast<unsigned long long>(__double_as_longlong(dmax)));
}

// ---------------------------------------------------------------------------
// K3 (fast): expl_N = Lambda_z[T_cur] from the T-layout field, plus the
// N-layout copy of T_cur (the radial sweep's anchor). Lane = j (coalesced T
// reads), each face evaluated once and shared by shuffle; tiles of 32 lines
// are transposed through shared memory for the N-layout stores.
constexpr int kTl = 32;
__global__ void __launch_bounds__(256)
    k_expl_axial_fast(DevProblem P, const double* __restrict__ fT, double* __restrict__ explN,
                      double* __restrict__ TcN, DevStatus* st) {
  __shared__ double te[kTl][kTl + 1], tt[kTl][kTl + 1];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;  // 8 warps x 4 lines
  const int i0 = blockIdx.y * kTl, j0 = blockIdx.x * kTl;
  for (int ii = w * 4; ii < w * 4 + 4; ++ii) {
    const int i = i0 + ii;
    if (i >= P.nr) break;
    const int m = col_extent(P, i);
    const int L = P.layer[i];
    const int j = j0 + lane;
    const double* row = fT + static_cast<size_t>(i) * P.nz;
    const bool act = j < m;
    const double tj = act ? row[j] : 0.0;
    double fh = 0.0;
    if (act) {
      if (j < m - 1) {
        const double tn = row[j + 1];
        fh = face_lambda_fast(P, L, L, tj, tn, st, i) * P.inv_gap_z[j + 1] * (tn - tj);
      } else if (L == 0 && !P.all_neumann) {
        fh = mat_eval_fast(P, L, kLambda, P.T0, st, i) * (P.T0 - tj) * __drcp_rn(0.5 * P.width_z[j]);
      }
    }
    double flo = __shfl_up_sync(0xffffffffu, fh, 1);
    if (lane == 0) {
      flo = 0.0;
      if (act && j > 0) {
        const double tp = row[j - 1];
        flo = face_lambda_fast<false>(P, L, L, tp, tj, st, i) * P.inv_gap_z[j] * (tj - tp);
      }
    }
    te[ii][lane] = act ? (fh - flo) * P.inv_eta[j] : 0.0;
    tt[ii][lane] = tj;
  }
  __syncthreads();
  for (int jj = w * 4; jj < w * 4 + 4; ++jj) {
    const int j = j0 + jj, i = i0 + lane;
    if (j < P.nz && i < P.nr && j < col_extent(P, i)) {
      const size_t o = static_cast<size_t>(j) * P.nr + i;
      explN[o] = te[lane][jj];
      TcN[o] = tt[lane][jj];
    }
  }
}

// K4 (fast): from the N-layout half field, expl_T = Lambda_r[T_half] + X(T_half)
// and the T-layout copy of T_half (the axial sweep's anchor).
__global__ void __launch_bounds__(256)
    k_axial_rhs_fast(DevProblem P, double pulse, const double* __restrict__ hN,
                     const double* __restrict__ powN, double* __restrict__ explT,
                     double* __restrict__ hT, DevStatus* st) {
  __shared__ double te[kTl][kTl + 1], tt[kTl][kTl + 1];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int j0 = blockIdx.y * kTl, i0 = blockIdx.x * kTl;
  for (int jj = w * 4; jj < w * 4 + 4; ++jj) {
    const int j = j0 + jj;
    if (j >= P.nz) break;
    const int n = row_extent(P, j);
    const int i = i0 + lane;
    const double* row = hN + static_cast<size_t>(j) * P.nr;
    const bool act = i < n;
    const double ti = act ? row[i] : 0.0;
    double fh = 0.0;
    if (act && i < n - 1) {
      const double tn = row[i + 1];
      fh = P.face_r_lo[i + 1] * face_lambda_fast(P, P.layer[i], P.layer[i + 1], ti, tn, st, j) *
           P.inv_gap_r[i + 1] * (tn - ti);
    }
    double flo = __shfl_up_sync(0xffffffffu, fh, 1);
    if (lane == 0) {
      flo = 0.0;
      if (act && i > 0) {
        const double tp = row[i - 1];
        flo = P.face_r_lo[i] * face_lambda_fast<false>(P, P.layer[i - 1], P.layer[i], tp, ti, st, j) *
              P.inv_gap_r[i] * (ti - tp);
      }
    }
    double e = 0.0;
    if (act) {
      const int L = P.layer[i];
      const double fp = P.source_kind == PCGPU_SOURCE_FIELD
                            ? powN[static_cast<size_t>(j) * P.nr + i] : 0.0;
      e = (fh - flo) * P.inv_vol_r[i] + source_power_fast(P, pulse, L, ti, fp, st, j);
    }
    te[jj][lane] = e;
    tt[jj][lane] = ti;
  }
  __syncthreads();
  for (int ii = w * 4; ii < w * 4 + 4; ++ii) {
    const int i = i0 + ii, j = j0 + lane;
    if (i < P.nr && j < P.nz && j < col_extent(P, i)) {
      const size_t o = static_cast<size_t>(i) * P.nz + j;
      explT[o] = te[lane][ii];
      hT[o] = tt[lane][ii];
    }
  }
}

void report_launch_error(cudaError_t e) {
  // Surfaced to the host at the next synchronisation as a sticky error.
  fprintf(stderr, "pcgpu: k_line_fast launch failed: %s\n", cudaGetErrorString(e));
}

template <bool kAxial, bool kU2, int kLean, bool kDirect = false>
void launch_line_t(const DevProblem& P, const LineArgs& A, int nmax, cudaStream_t s) {
  const int CL = (nmax + SEG - 1) / SEG;
  // the direct variant never touches the staging tiles (the struct's tail)
  const size_t smem = kDirect ? offsetof(FastSmem, ts) : sizeof(FastSmem);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_line_fast<kAxial, kU2, kLean, kDirect>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(A.nlines * CL));
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr_cl[1];
  attr_cl[0].id = cudaLaunchAttributeClusterDimension;
  attr_cl[0].val.clusterDim.x = static_cast<unsigned>(CL);
  attr_cl[0].val.clusterDim.y = 1;
  attr_cl[0].val.clusterDim.z = 1;
  cfg.attrs = attr_cl;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, k_line_fast<kAxial, kU2, kLean, kDirect>, P, A);
  if (e != cudaSuccess) report_launch_error(e);
  ++g_launches;
}

template <bool kAxial>
void launch_line(const DevProblem& P, const LineArgs& A, int nmax, cudaStream_t s) {
  // Direct (register) row loads measured slower than the swizzled cp.async
  // tiles on B200 (4.3 vs 3.5 ms per cfg3 radial launch): opt-in only.
  static const bool direct = std::getenv("PCGPU_DIRECT") != nullptr;
  if (P.lean && direct && (A.ld & 1) == 0) {
    if (!kAxial && P.source_kind == PCGPU_SOURCE_JOULE)
      launch_line_t<kAxial, true, 2, true>(P, A, nmax, s);
    else
      launch_line_t<kAxial, true, 1, true>(P, A, nmax, s);
  } else if (P.lean) {
    if (!kAxial && P.source_kind == PCGPU_SOURCE_JOULE)
      launch_line_t<kAxial, true, 2>(P, A, nmax, s);
    else
      launch_line_t<kAxial, true, 1>(P, A, nmax, s);
  } else if (P.all_u2) {
    launch_line_t<kAxial, true, 0>(P, A, nmax, s);
  } else {
    launch_line_t<kAxial, false, 0>(P, A, nmax, s);
  }
}


// ---------------------------------------------------------------------------
// Slab variants for the partitioned (multi-GPU) stepper. A z-slab holds the
// radial lines j in [j0, j0+nj) in N layout (line stride nr); an r-slab holds
// the axial lines i in [i0, i0+ni) in T layout (line stride nz). The per-cell
// arithmetic is exactly the single-GPU fast kernels', so a partitioned run is
// bit-identical to a single-GPU fast run.

// Lambda_r[T] + X(T) on a z-slab, N layout in and out (k_axial_rhs_fast
// without the transpose).
__global__ void __launch_bounds__(256)
    k_rhs_zslab(DevProblem P, double pulse, int j0, int nj, const double* __restrict__ hN,
                double* __restrict__ eN, DevStatus* st) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int jl = blockIdx.y * 8 + w;
  if (jl >= nj) return;
  const int j = j0 + jl;
  const int n = row_extent(P, j);
  const int i = blockIdx.x * 32 + lane;
  const double* row = hN + static_cast<size_t>(jl) * P.nr;
  const bool act = i < n;
  const double ti = act ? row[i] : 0.0;
  double fh = 0.0;
  if (act && i < n - 1) {
    const double tn = row[i + 1];
    fh = P.face_r_lo[i + 1] * face_lambda_fast(P, P.layer[i], P.layer[i + 1], ti, tn, st, j) *
         P.inv_gap_r[i + 1] * (tn - ti);
  }
  double flo = __shfl_up_sync(0xffffffffu, fh, 1);
  if (lane == 0) {
    flo = 0.0;
    if (act && i > 0) {
      const double tp = row[i - 1];
      flo = P.face_r_lo[i] * face_lambda_fast<false>(P, P.layer[i - 1], P.layer[i], tp, ti, st, j) *
            P.inv_gap_r[i] * (ti - tp);
    }
  }
  if (act)
    eN[static_cast<size_t>(jl) * P.nr + i] =
        (fh - flo) * P.inv_vol_r[i] + source_power_fast(P, pulse, P.layer[i], ti, 0.0, st, j);
}

// Lambda_z[T] on an r-slab, T layout in and out (k_expl_axial_fast without the
// transpose).
__global__ void __launch_bounds__(256)
    k_expl_rslab(DevProblem P, int i0, int ni, const double* __restrict__ fT,
                 double* __restrict__ eT, DevStatus* st) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int il = blockIdx.y * 8 + w;
  if (il >= ni) return;
  const int i = i0 + il;
  const int m = col_extent(P, i);
  const int L = P.layer[i];
  const int j = blockIdx.x * 32 + lane;
  const double* row = fT + static_cast<size_t>(il) * P.nz;
  const bool act = j < m;
  const double tj = act ? row[j] : 0.0;
  double fh = 0.0;
  if (act) {
    if (j < m - 1) {
      const double tn = row[j + 1];
      fh = face_lambda_fast(P, L, L, tj, tn, st, i) * P.inv_gap_z[j + 1] * (tn - tj);
    } else if (L == 0 && !P.all_neumann) {
      fh = mat_eval_fast(P, L, kLambda, P.T0, st, i) * (P.T0 - tj) * __drcp_rn(0.5 * P.width_z[j]);
    }
  }
  double flo = __shfl_up_sync(0xffffffffu, fh, 1);
  if (lane == 0) {
    flo = 0.0;
    if (act && j > 0) {
      const double tp = row[j - 1];
      flo = face_lambda_fast<false>(P, L, L, tp, tj, st, i) * P.inv_gap_z[j] * (tj - tp);
    }
  }
  if (act) eT[static_cast<size_t>(il) * P.nz + j] = (fh - flo) * P.inv_eta[j];
}

}  // namespace

void launch_radial_fast_slab(const DevProblem& P, int it, double eps, double half_k, double pulse,
                             int j0, int nj, const double* TsN, const double* TcN,
                             const double* explN, double* outN, DevStatus* st, cudaStream_t s) {
  LineArgs A{TsN, TcN, explN, nullptr, outN, P.nr, nj, j0, it, eps, half_k, pulse, st};
  if (nj > 0) launch_line<false>(P, A, P.nr, s);
}

void launch_axial_fast_slab(const DevProblem& P, int it, double eps, double half_k, int i0,
                            int ni, const double* TsT, const double* ThT, const double* explT,
                            double* outT, DevStatus* st, cudaStream_t s) {
  LineArgs A{TsT, ThT, explT, nullptr, outT, P.nz, ni, i0, it, eps, half_k, 0.0, st};
  if (ni > 0) launch_line<true>(P, A, P.nz, s);
}

void launch_rhs_zslab(const DevProblem& P, double pulse, int j0, int nj, const double* hN,
                      double* eN, DevStatus* st, cudaStream_t s) {
  if (nj <= 0) return;
  dim3 grid((P.nr + 31) / 32, (nj + 7) / 8);
  k_rhs_zslab<<<grid, 256, 0, s>>>(P, pulse, j0, nj, hN, eN, st);
  ++g_launches;
}

void launch_expl_rslab(const DevProblem& P, int i0, int ni, const double* fT, double* eT,
                       DevStatus* st, cudaStream_t s) {
  if (ni <= 0) return;
  dim3 grid((P.nz + 31) / 32, (ni + 7) / 8);
  k_expl_rslab<<<grid, 256, 0, s>>>(P, i0, ni, fT, eT, st);
  ++g_launches;
}

namespace {
}  // namespace

bool fast_supported(const DevProblem& P) {
  return P.nr <= SEG * kMaxCluster && P.nz <= SEG * kMaxCluster;
}

void launch_radial_fast(const DevProblem& P, int it, double eps, double half_k, double pulse,
                        const double* TsN, const double* TcN, const double* explN,
                        const double* powN, double* outN, DevStatus* st, cudaStream_t s) {
  LineArgs A{TsN, TcN, explN, powN, outN, P.nr, P.nz, 0, it, eps, half_k, pulse, st};
  launch_line<false>(P, A, P.nr, s);
}

void launch_axial_fast(const DevProblem& P, int it, double eps, double half_k, const double* TsT,
                       const double* ThT, const double* explT, double* outT, DevStatus* st,
                       cudaStream_t s) {
  LineArgs A{TsT, ThT, explT, nullptr, outT, P.nz, P.nr, 0, it, eps, half_k, 0.0, st};
  launch_line<true>(P, A, P.nz, s);
}

void launch_explicit_axial_fast(const DevProblem& P, const double* fieldT, double* explN,
                                double* TcN, DevStatus* st, cudaStream_t s) {
  dim3 grid((P.nz + kTl - 1) / kTl, (P.nr + kTl - 1) / kTl);
  k_expl_axial_fast<<<grid, 256, 0, s>>>(P, fieldT, explN, TcN, st);
  ++g_launches;
}

void launch_axial_rhs_fast(const DevProblem& P, double pulse, const double* halfN,
                           const double* powN, double* explT, double* halfT, DevStatus* st,
                           cudaStream_t s) {
  dim3 grid((P.nr + kTl - 1) / kTl, (P.nz + kTl - 1) / kTl);
  k_axial_rhs_fast<<<grid, 256, 0, s>>>(P, pulse, halfN, powN, explT, halfT, st);
  ++g_launches;
}

}  // namespace pcgpu
