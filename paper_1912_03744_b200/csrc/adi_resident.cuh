// adi_resident.cuh -- the resident stepper: whole ADI steps (tau controller,
// Picard loops, accept-or-halve) in ONE cooperative launch per batch of steps.
// Included by adi_exact.cu inside its anonymous namespace (it reuses the
// exact line solver line_exact_ws and the K3/K4 tiles, --fmad=false).
//
// Reference control flow restated on the device (solver.cpp):
//   step            :356-373  tau = initial_tau (host schedule); attempts until
//                             both half-steps converge; tau *= 0.5 and the
//                             floor test on failure; accept = buffer rotation
//   radial_half_step:235-257  K3 (explicit_axial_pass) then Picard s = 1..max_iter,
//                             converged iff max-norm < epsilon (strict)
//   axial_half_step :334-354  K4 (axial_fixed_rhs_pass) then Picard
// Every decision reads the same device max-norm after a grid-wide barrier, so
// all CTAs take it identically; nothing returns to the host inside a batch.
//
// Layout: one CTA of 12 warps per SM (the axial "spread" roles of the line
// solver: warp 0 solves, 8 warps produce coefficients, 3 idle), line blocks of
// 32 lines strided over the grid; K3/K4 tiles (32 lines x 64 rows) by warps
// 0-7. Staging is cp.async (no tensor maps: the iterate buffers rotate on the
// device). Worth it where launches and host round trips dominate -- grids
// with at most ~2 line blocks per SM per sweep (resident_grid()).

__device__ __forceinline__ unsigned long long ld_volatile_u64(const unsigned long long* p) {
  return *reinterpret_cast<const volatile unsigned long long*>(p);
}

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void reset_status(DevStatus* st, int max_iter) {
  for (int q = 0; q <= max_iter; ++q) st->delta[q] = 0ull;
  st->err = kNoError;
}

__device__ __forceinline__ void bar_k34() {  // warps 0-7 (K3 / K4 tiles)
  asm volatile("bar.sync 2, %0;" ::"n"(kT3Threads) : "memory");
}

// kCluster: the whole grid is one thread-block cluster (at most 16 CTAs, one
// GPC): the phase barrier is the hardware cluster barrier instead of the
// cooperative grid barrier's global-memory atomics and polling (which cross
// the two dies).
template <int kX, bool kCluster>
__global__ void __launch_bounds__(kResThreads, 1)
    k_resident(const __grid_constant__ DevProblem P, const __grid_constant__ ResArgs A) {
  namespace cg = cooperative_groups;
  struct PhaseBarrier {
    __device__ void sync() const {
      if (kCluster)
        cg::this_cluster().sync();
      else
        cg::this_grid().sync();
    }
  } grid;
  extern __shared__ __align__(128) double sm[];
  const int tid = threadIdx.x;
  const bool lead = blockIdx.x == 0 && tid == 0;
  const int G = gridDim.x;
  const int nblk_r = (P.nz + 31) / 32, nblk_a = (P.nr + 31) / 32;
  const int k3x = (P.nr + 31) / 32, k3y = (P.nz + kT3Rows - 1) / kT3Rows;
  const int k4x = (P.nz + 31) / 32, k4y = (P.nr + kT3Rows - 1) / kT3Rows;
  const int max_iter = A.max_iter;
  const double eps = A.eps;
  int state = A.state0;
  int hs = 0;  // half-step counter: status buffers alternate
  double(*te)[kT3Rows + 1] = reinterpret_cast<double(*)[kT3Rows + 1]>(sm);
  // phase profile (lead thread only)
  unsigned long long t_last = 0, t_ph = 0;
  long long c_last = 0;
  auto mark = [&](int phase) {
    if (!A.profile) return;
    if (tid == 0) t_ph = global_ns();  // this CTA's phase start
    if (!lead) return;
    const long long c_now = clock64();
    A.ctl->prof_cyc += static_cast<unsigned long long>(c_now - c_last);
    c_last = c_now;
    const unsigned long long now = t_ph;
    A.ctl->prof_ns[phase] += now - t_last;
    A.ctl->prof_n[phase] += 1;
    A.ctl->prof_busy[phase] += atomicExch(&A.ctl->busy_max[phase], 0ull);
    t_last = now;
  };
  // before a barrier: this CTA's busy time in the phase that ends there
  auto busy = [&](int phase) {
    if (A.profile && tid == 0) atomicMax(&A.ctl->busy_max[phase], global_ns() - t_ph);
#ifdef PCGPU_TSPROF
    if (tid == 0 && blockIdx.x < 64 && (phase == 2 || phase == 4)) {
      g_rts[phase == 4][blockIdx.x][0] = t_ph;
      g_rts[phase == 4][blockIdx.x][6] = global_ns();
    }
#endif
  };
  // Status of half-step hs is st2[hs & 1]. Both start reset; the buffer of
  // the next half-step is reset by the lead thread after the first grid
  // barrier of the current one (its last readers are past that barrier).
  if (lead) {
    reset_status(A.st2, max_iter);
    reset_status(A.st2 + 1, max_iter);
    if (A.profile) {
      t_last = global_ns();
      c_last = clock64();
    }
  }
  grid.sync();
  mark(0);

  for (int k = 0; k < A.nsteps; ++k) {
    const ResSched& S = A.sched[k];
    double tau = S.tau0;
    int h = 0;
    double upd = 0.0;
    pcgpu_step_result res{};
    double* const cur = A.X[state];
    double* const xa = A.X[(state + 1) % 3];
    double* const xb = A.X[(state + 2) % 3];
    if (lead)  // clamp counters at the step start (restored if the host redoes it)
      for (int L = 0; L < P.n_layers; ++L) A.ctl->clamp_save[L] = P.clamp[L];
    int outcome = -1;  // accepted: the axial result buffer (1: xa, 2: xb)
    for (;;) {
      if (h > A.max_halv) {  // no precomputed pulse: the host redoes this step
        if (lead) {
          for (int L = 0; L < P.n_layers; ++L) P.clamp[L] = A.ctl->clamp_save[L];
          A.ctl->stop = kResNeedHost;
        }
        break;
      }
      const double pulse = S.pulse[h];
      const double hk = 2.0 / tau;
      // ---- radial half-step (solver.cpp:235-257) ----
      DevStatus* st = A.st2 + (hs & 1);
      DevStatus* st_next = A.st2 + (++hs & 1);
      if (tid < kT3Threads)  // K3: explicit_axial_pass (T_cur -> Lambda_z, T copy)
        for (int q = blockIdx.x; q < k3x * k3y; q += G) {
          explicit_axial_t3_tile<kX>(P, cur, A.ExplT, A.TcT, st, q % k3x, q / k3x, tid, te, te + 32,
                                     bar_k34);
          bar_k34();
        }
      busy(1);
      grid.sync();
      mark(1);
      if (lead) reset_status(st_next, max_iter);
      bool failed = ld_volatile_u64(&st->err) != kNoError;
      int conv = 0;
      for (int it = 1; it <= max_iter && !failed; ++it) {
        const double* src = it == 1 ? A.TcT : (it % 2 == 0 ? A.HalfT : xb);
        double* dst = it % 2 == 1 ? A.HalfT : xb;
        for (int vb = blockIdx.x; vb < nblk_r; vb += G) {
          if (A.short_r)
            line_exact_ws<false, kX, kNPAxial, true, true>(P, it, -1.0, hk, pulse, 0, P.nz, src,
                                                           A.TcT, A.ExplT, nullptr, dst, A.W,
                                                           A.Xs, st, nullptr, vb);
          else
            line_exact_ws<false, kX, kNPAxial, true>(P, it, -1.0, hk, pulse, 0, P.nz, src, A.TcT,
                                                     A.ExplT, nullptr, dst, A.W, A.Xs, st,
                                                     nullptr, vb);
        }
        busy(2);
        grid.sync();
        mark(2);
        failed = ld_volatile_u64(&st->err) != kNoError;
        const double dl = __longlong_as_double(static_cast<long long>(ld_volatile_u64(&st->delta[it])));
        upd += A.active;
        res.radial.iterations = it;
        res.radial.last_delta = dl;
        if (!failed && dl < eps) {
          conv = it;
          res.radial.converged = 1;
          break;
        }
      }
      if (failed) {
        if (lead) {
          A.ctl->stop = kResError;
          A.ctl->err = ld_volatile_u64(&st->err);
        }
        break;
      }
      if (conv) {
        // ---- axial half-step (solver.cpp:334-354) ----
        const double* halfT = conv % 2 == 1 ? A.HalfT : xb;
        DevStatus* sa = A.st2 + (hs & 1);
        DevStatus* sa_next = A.st2 + (++hs & 1);
        if (tid < kT3Threads) {  // K4: axial_fixed_rhs_pass (-> Lambda_r + X, T_half in N)
          for (int q = blockIdx.x; q < k4x * k4y; q += G) {
            if (A.kbarN)
              axial_rhs_t3_tile<kX, true>(P, hk, pulse, halfT, nullptr, A.kbarN, A.ExplT, A.TcT,
                                          sa, q % k4x, q / k4x, tid, sm, bar_k34);
            else
              axial_rhs_t3_tile<kX == 0 ? 1 : kX, false>(P, hk, pulse, halfT, nullptr, nullptr,
                                                         A.ExplT, A.TcT, sa, q % k4x, q / k4x,
                                                         tid, sm, bar_k34);
            bar_k34();
          }
        }
        busy(3);
        grid.sync();
        mark(3);
        if (lead) reset_status(sa_next, max_iter);
        failed = ld_volatile_u64(&sa->err) != kNoError;
        int aconv = 0;
        for (int it = 1; it <= max_iter && !failed; ++it) {
          const double* src = it == 1 ? A.TcT : (it % 2 == 0 ? xa : xb);
          double* dst = it % 2 == 1 ? xa : xb;
          for (int vb = blockIdx.x; vb < nblk_a; vb += G) {
            if (A.short_a)
              line_exact_ws<true, kX, kNPAxial, true, true>(P, it, -1.0, hk, 0.0, 0, P.nr, src,
                                                            A.TcT, A.ExplT, A.kbarN, dst, A.W,
                                                            A.Xs, sa, nullptr, vb);
            else
              line_exact_ws<true, kX, kNPAxial, true>(P, it, -1.0, hk, 0.0, 0, P.nr, src, A.TcT,
                                                      A.ExplT, A.kbarN, dst, A.W, A.Xs, sa,
                                                      nullptr, vb);
          }
          busy(4);
          grid.sync();
          mark(4);
          failed = ld_volatile_u64(&sa->err) != kNoError;
          const double dl = __longlong_as_double(static_cast<long long>(ld_volatile_u64(&sa->delta[it])));
          upd += A.active;
          res.axial.iterations = it;
          res.axial.last_delta = dl;
          if (!failed && dl < eps) {
            aconv = it;
            res.axial.converged = 1;
            break;
          }
        }
        if (failed) {
          if (lead) {
            A.ctl->stop = kResError;
            A.ctl->err = ld_volatile_u64(&sa->err);
          }
          break;
        }
        if (aconv) {
          outcome = aconv % 2 == 1 ? 1 : 2;
          res.tau_used = tau;
          break;
        }
      }
      // rejected attempt: halve (solver.cpp:369-371); only the accepted
      // attempt's iteration counts are reported
      tau *= 0.5;
      ++h;
      ++res.halvings;
      res.radial = pcgpu_outcome{};
      res.axial = pcgpu_outcome{};
      if (tau < A.tau_floor) {
        if (lead) {
          A.ctl->stop = kResFloor;
          A.ctl->tau = tau;
        }
        break;
      }
    }
    if (outcome < 0) {  // error / floor / need-host: the field stays X[state]
      if (lead) {
        A.ctl->steps = k;
        A.ctl->state = state;
        A.ctl->updates = upd;
      }
      return;
    }
    state = (state + outcome) % 3;
    mark(5);
    if (blockIdx.x == 0) {
      if (tid == 0) {
        A.log[k].r = res;
        A.log[k].updates = upd;
      }
      if (tid < A.n_probes) {  // the new field is complete (grid barrier above)
        const volatile double* f = A.X[state];
        A.log[k].probes[tid] = f[A.probe_off[tid]];
      }
    }
    if (res.halvings > 0 && k + 1 < A.nsteps) {  // the schedule assumed no halving
      if (lead) {
        A.ctl->steps = k + 1;
        A.ctl->state = state;
        A.ctl->stop = kResHalved;
      }
      return;
    }
  }
  if (lead) {
    A.ctl->steps = A.nsteps;
    A.ctl->state = state;
    A.ctl->stop = kResRan;
  }
}
