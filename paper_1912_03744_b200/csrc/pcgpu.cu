// pcgpu.cu -- host side of the C-ABI (include/pcgpu.h): the B200 AdiStepper.
//
// Mirrors pulsecell::AdiStepper (solver.hpp:66-106, solver.cpp:125-373):
//   ctor          -> pcgpu_create   (validation solver.cpp:33-42,133-138; buffers :140-159)
//   radial/axial  -> pcgpu_*_half_step (Picard loops solver.cpp:235-257, :334-354)
//   step          -> pcgpu_step     (tau halving controller solver.cpp:356-373)
// The Picard iterations run on the device; each iteration kernel early-exits
// once the previous iteration's device-side max-norm passed (< epsilon), so
// the host enqueues a predicted batch of iterations and synchronises once per
// half-step to read the outcome (no per-iteration round trip).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <string>
#include <type_traits>
#include <vector>

#include "../../include/pcgpu.h"
#include "extents.h"
#include "adi_kernels.h"

using namespace pcgpu;

namespace {

thread_local std::string g_create_error;

struct CudaError {
  cudaError_t e;
  const char* what;
};

#define CK(x)                                           \
  do {                                                  \
    cudaError_t e_ = (x);                               \
    if (e_ != cudaSuccess) throw CudaError{e_, #x};     \
  } while (0)

// Host restatement of pulse_value (source.cpp:18-45) -- same libm calls as
// the reference, so the same bits.
double host_pulse_value(const pcgpu_desc& d, double t) {
  const double phase = std::fmod(t, d.t_per);
  if (d.waveform == PCGPU_WAVE_RECTANGULAR) return phase < d.t_src ? 1.0 : 0.0;
  const double margin = d.t_trs / d.zeta * (1.0 + 6.5 / d.xi);
  const long elapsed = std::llround((t - phase) / d.t_per);
  const long back_hi =
      std::min(elapsed, 1 + static_cast<long>(std::ceil((d.t_src + margin) / d.t_per)));
  const double scale = d.xi * d.zeta / d.t_trs;
  double sum = 0.0;
  for (long m = -1; m <= back_hi; ++m) {
    const double u = phase + static_cast<double>(m) * d.t_per;
    sum += std::erf(scale * u - d.xi) - std::erf(scale * (u - d.t_src) - d.xi);
  }
  return 0.5 * sum;
}

// initial_tau (solver.cpp:44-51).
double host_initial_tau(const pcgpu_desc& d, double t) {
  const double phase = std::fmod(t, d.t_per);
  const bool in_transient =
      phase <= d.t_trs || (phase >= d.t_src && phase <= d.t_src + d.t_trs);
  return in_transient ? d.t_trs / d.tau_transient_divisor : d.t_src / d.tau_source_divisor;
}

std::string validate(const pcgpu_desc* d) {
  if (d->abi_version != PCGPU_ABI_VERSION) return "pcgpu: ABI version mismatch";
  // SolverConfig::validate (solver.cpp:33-42)
  if (!(d->epsilon > 0)) return "solver.epsilon: must be > 0";
  if (d->max_iter < 1) return "solver.max_iter: must be >= 1";
  if (d->max_iter > kMaxIter) return "solver.max_iter: exceeds the device limit";
  if (!(d->tau_transient_divisor > 0)) return "solver.tau_transient_divisor: must be > 0";
  if (!(d->tau_source_divisor > 0)) return "solver.tau_source_divisor: must be > 0";
  if (!(d->T0 > 0)) return "solver.T0: must be > 0";
  if (!(d->t_ceiling > d->T0)) return "solver.t_ceiling: must exceed T0";
  // SourceSpec::validate (source.cpp:9-17)
  if (!(d->t_per > 0)) return "source.t_per: must be > 0";
  if (!(d->t_src > 0 && d->t_src <= d->t_per))
    return "source.t_src: must satisfy 0 < t_src <= t_per";
  if (!(d->t_trs > 0 && d->t_trs < d->t_src)) return "source.t_trs: must satisfy 0 < t_trs < t_src";
  if (!(d->xi > 0)) return "source.xi: must be > 0";
  if (!(d->zeta > 0)) return "source.zeta: must be > 0";
  // Grid / wiring (solver.cpp:135-138)
  if (d->nr < 1 || d->nz < 1 || d->nr_core < 1 || d->nr_core > d->nr || d->nz_shared < 1 ||
      d->nz_shared > d->nz)
    return "stepper: invalid grid extents";
  if (!d->layer || !d->r_center || !d->gap_r || !d->width_z || !d->gap_z)
    return "stepper: null grid array";
  {
    const std::string e = check_extents(d);
    if (!e.empty()) return e;
  }
  if (d->n_layers < 1 || d->n_layers > kMaxLayers) return "stepper: one material required per layer";
  if (!d->materials) return "stepper: null material";
  for (int i = 0; i < d->nr; ++i)
    if (d->layer[i] < 0 || d->layer[i] >= d->n_layers)
      return "stepper: one material required per layer";
  // MaterialTable / PropertyTable invariants (materials.cpp:5-37)
  for (int m = 0; m < d->n_layers; ++m) {
    const pcgpu_material& mt = d->materials[m];
    if (!(mt.rho > 0)) return "material: rho must be > 0";
    if (mt.cv.n < 1) return "material: missing heat capacity table";
    if (mt.lambda.n < 1) return "material: missing conductivity table";
    const pcgpu_table* tabs[3] = {&mt.cv, &mt.lambda, &mt.chi};
    for (int p = 0; p < 3; ++p) {
      const pcgpu_table& t = *tabs[p];
      if (t.n < 0 || (t.n > 0 && (!t.t || !t.v))) return "property table: bad pointer";
      for (int k = 1; k < t.n; ++k)
        if (!(t.t[k] > t.t[k - 1]))
          return "property table: temperature knots must be strictly increasing";
      for (int k = 0; k < t.n; ++k) {
        if (p < 2 && !(t.v[k] > 0)) return "material: values must be > 0";
        if (p == 2 && t.v[k] < 0) return "material: resistivity values must be >= 0";
      }
    }
  }
  if (d->source_kind == PCGPU_SOURCE_JOULE) {
    if (d->source_layer < 0 || d->source_layer >= d->n_layers)
      return "domain.source_layer: out of range";
    if (!std::isfinite(d->amplitude)) return "source.S_C: must be > 0";
    if (d->amplitude != 0.0 && d->materials[d->source_layer].chi.n == 0)
      return "material: source layer needs a resistivity table";
  } else if (d->source_kind != PCGPU_SOURCE_NULL && d->source_kind != PCGPU_SOURCE_FIELD) {
    return "source: unknown kind";
  }
  if (d->mode != PCGPU_MODE_EXACT) return "pcgpu: unknown mode (only exact mode exists)";
  return "";
}

// dst[L] += sum of the first nslots counter rows (stride `stride`), L < n
__global__ void k_add_counters(unsigned long long* dst, const unsigned long long* slots, int n,
                               int stride, int nslots) {
  const int L = threadIdx.x;
  if (L >= n) return;
  unsigned long long sum = 0;
  for (int k = 0; k < nslots; ++k) sum += slots[static_cast<size_t>(k) * stride + L];
  dst[L] += sum;
}
void launch_add_counters(unsigned long long* dst, const unsigned long long* slots, int n,
                         int stride, int nslots, cudaStream_t s) {
  k_add_counters<<<1, 32, 0, s>>>(dst, slots, n, stride, nslots);
}

// Speculative batches (pcgpu_stepper::host_run). Reset: every status of the
// batch cleared, the clamp counters snapshot taken.
__global__ void k_spec_reset(DevStatus* st, int n, const unsigned long long* clamp,
                             unsigned long long* save, int n_layers) {
  for (int q = threadIdx.x; q < n; q += blockDim.x) {
    for (int it = 0; it <= kMaxIter; ++it) st[q].delta[it] = 0;
    st[q].err = kNoError;
  }
  if (threadIdx.x < n_layers) save[threadIdx.x] = clamp[threadIdx.x];
}
// Verify one half-step: it must have converged within its `launched`
// iterations without error; otherwise every later half-step of the batch is
// marked kSpecAbort (its kernels return at once, so the field it started from
// survives). `snapshot`: after a passing axial sweep, the clamp counters of the
// completed step become the restore point.
__global__ void k_spec_verify(const DevStatus* st, int launched, double eps, DevStatus* later,
                              int n_later, const unsigned long long* clamp,
                              unsigned long long* save, int n_layers, int snapshot) {
  __shared__ int ok;
  if (threadIdx.x == 0) {
    int conv = 0;
    if (st->err == kNoError)
      for (int it = 1; it <= launched && !conv; ++it)
        conv = __longlong_as_double(static_cast<long long>(st->delta[it])) < eps;
    ok = st->err == kSpecAbort ? 2 : conv;  // 2: aborted upstream, already marked
  }
  __syncthreads();
  if (ok == 0) {
    for (int q = threadIdx.x; q < n_later; q += blockDim.x) later[q].err = kSpecAbort;
  } else if (ok == 1 && snapshot && threadIdx.x < n_layers) {
    save[threadIdx.x] = clamp[threadIdx.x];
  }
}

template <typename T>
T* dev_upload(const std::vector<T>& v) {
  T* p = nullptr;
  CK(cudaMalloc(&p, sizeof(T) * std::max<size_t>(1, v.size())));
  if (!v.empty()) CK(cudaMemcpy(p, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice));
  return p;
}

}  // namespace

// Buffer roles. N = natural layout, T = transposed.
enum Buf {
  kTcT = 0,     // radial: transposed anchor T_cur   | axial: halfN
  kExpl,        // radial: Lambda_z[T_cur] (T)       | axial: expl (N)
  kHalfT,       // radial iterate / result (T)
  kIterT,       // radial ping-pong (T)              | axial: ping-pong (N)
  kW,           // Thomas work vector (exact mode)
  kX,           // Thomas x vector (exact mode)
  kKbar,        // axial: kbar (N)
  kNext,        // axial result (N)
  kField,       // pcgpu_run: resident field (N)
  kPowN,        // bound power field (N)
  kPowT,        // bound power field (T)
  kStage,       // host-API staging field (N), allocated on first use
  kNumBufs
};

// The last evolve's resampled probe-0 periods (pcgpu_detector_periods).
struct pcgpu_runner_state {
  std::vector<std::vector<double>> detector_rows;
  int samples = 0;
};

struct pcgpu_stepper {
  pcgpu_desc d{};
  pcgpu_runner_state* runner = nullptr;  // the last evolve's detector rows
  std::vector<int> col_ext_host;         // masked extent of every axial line
  DevProblem P{};
  std::vector<void*> dev_allocs;
  cudaStream_t stream = nullptr;
  DevStatus* st = nullptr;       // device
  DevStatus* st_host = nullptr;  // pinned mirror
  double* buf[kNumBufs] = {};
  double tau_floor = 0;
  int64_t active = 0;
  std::string err;
  int64_t err_line = -1;
  int pred_radial = 1, pred_axial = 1;
  bool pred_stable = false;  // the last two radial half-steps took the same iterations
  bool power_bound = false;
  // kernel timing
  bool timing = false;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  struct Timed { cudaEvent_t a, b; int sweep; int it; int tag; };  // tag: batch step + 1
  std::vector<Timed> pending;
  double radial_ms = 0, axial_ms = 0;
  int64_t radial_launches = 0, axial_launches = 0;
  unsigned long long launches0 = 0;
  // host-field steps with the copy-in pipelined into the radial sweep
  // (radial_pipelined): lazily allocated
  static constexpr int kPipeChunks = 8, kPipeMaxIter = 16;
  cudaStream_t copy_stream = nullptr;
  cudaStream_t chunk_stream[kPipeChunks] = {};
  cudaEvent_t pipe_ev[kPipeChunks + 1] = {};
  cudaEvent_t chunk_done[kPipeChunks] = {};
  // [(kPipeMaxIter + 1) * kPipeChunks]: per row block, K3 (k = 0) then one
  // status per iteration k -- index k * kPipeChunks + c
  DevStatus* st_pipe = nullptr;
  DevStatus* st_pipe_host = nullptr;  // pinned mirror
  unsigned long long* clamp_pipe = nullptr;  // [kPipeMaxIter + 1][kMaxLayers]
  double* pipe_spare = nullptr;       // third rotating radial iterate (T)
  const double* pipe_host = nullptr;  // set by pcgpu_step_host for its first attempt
  int64_t pipe_steps = 0, pipe_fallbacks = 0;
  // resident stepper (whole steps in one cooperative launch per batch):
  // grid size (0: not applicable), device control block, schedule and log
  static constexpr int kResBatch = 1024;
  int res_grid = 0;
  bool res_cluster = false;  // the resident grid is one thread-block cluster
  ResCtl* res_ctl = nullptr;       // device
  ResCtl* res_ctl_host = nullptr;  // pinned
  ResSched* res_sched = nullptr;   // device [kResBatch]
  ResSched* res_sched_host = nullptr;
  ResLog* res_log = nullptr;       // device [kResBatch]
  ResLog* res_log_host = nullptr;
  DevStatus* res_st2 = nullptr;    // device [2]
  int* res_probe_off = nullptr;    // device [kResProbes]
  int64_t res_batches = 0, res_steps = 0, res_host_steps = 0;
  // $PCGPU_RES_PROF=1: per-phase device time of the resident batches,
  // printed to stderr when the stepper is destroyed
  bool res_profile = std::getenv("PCGPU_RES_PROF") != nullptr;
  double res_prof_ns[8] = {}, res_prof_n[8] = {}, res_prof_busy[8] = {}, res_prof_cyc = 0;
  // the host functions behind the schedule (the reference's own through
  // pcgpu_set_host_clock, else the restatements below)
  pcgpu_clock_fn pulse_fn = nullptr, tau_fn = nullptr;
  void* clock_user = nullptr;

  ~pcgpu_stepper() {
    if (res_profile && res_batches) {
      static const char* names[6] = {"start", "K3", "radial_it", "K4", "axial_it", "epilogue"};
      double ns = 0;
      for (int q = 1; q < 8; ++q) ns += res_prof_ns[q];
      std::fprintf(stderr, "pcgpu resident profile (%lld batches, %lld steps, SM clock %.0f MHz):",
                   static_cast<long long>(res_batches), static_cast<long long>(res_steps),
                   ns > 0 ? res_prof_cyc / ns * 1e3 : 0.0);
      for (int q = 0; q < 6; ++q)
        std::fprintf(stderr, " %s %.2f us (busiest CTA %.2f) x %.0f;", names[q],
                     res_prof_n[q] ? res_prof_ns[q] / res_prof_n[q] / 1e3 : 0.0,
                     res_prof_n[q] ? res_prof_busy[q] / res_prof_n[q] / 1e3 : 0.0, res_prof_n[q]);
      if (P.prof) {  // solver warp of line block 0: cycles per row waiting / in the chain
        unsigned long long c[16] = {};
        cudaMemcpy(c, P.prof, sizeof c, cudaMemcpyDeviceToHost);
        std::fprintf(stderr, " solver cycles/row: radial wait %.1f chain %.1f, axial wait %.1f "
                     "chain %.1f;", c[4] ? 1.0 * c[0] / c[4] : 0.0, c[4] ? 1.0 * c[1] / c[4] : 0.0,
                     c[5] ? 1.0 * c[2] / c[5] : 0.0, c[5] ? 1.0 * c[3] / c[5] : 0.0);
        // per call (cycles): entry -> forward, forward end -> back start, back pass
        const double nr_ = res_prof_n[2] ? res_prof_n[2] : 1, na_ = res_prof_n[4] ? res_prof_n[4] : 1;
        std::fprintf(stderr, " per call cycles: radial pre %.0f bulk %.0f back %.0f, axial pre %.0f "
                     "bulk %.0f back %.0f;", c[6] / nr_, (1.0 * c[10] - c[8]) / nr_,
                     (1.0 * c[12] - c[10]) / nr_, c[7] / na_, (1.0 * c[11] - c[9]) / na_,
                     (1.0 * c[13] - c[11]) / na_);
        std::fprintf(stderr, " back loop alone: radial %.0f axial %.0f;", c[14] / nr_, c[15] / na_);
      }
      std::fprintf(stderr, "\n");
    }
    delete runner;
    if (stream) cudaStreamSynchronize(stream);
    if (copy_stream) {
      cudaStreamSynchronize(copy_stream);
      cudaStreamDestroy(copy_stream);
    }
    for (auto& cs : chunk_stream)
      if (cs) {
        cudaStreamSynchronize(cs);
        cudaStreamDestroy(cs);
      }
    for (auto& e : pipe_ev)
      if (e) cudaEventDestroy(e);
    for (auto& e : chunk_done)
      if (e) cudaEventDestroy(e);
    if (st_pipe_host) cudaFreeHost(st_pipe_host);
    if (res_ctl_host) cudaFreeHost(res_ctl_host);
    if (res_sched_host) cudaFreeHost(res_sched_host);
    if (res_log_host) cudaFreeHost(res_log_host);
    for (auto& e : ev_pool) cudaEventDestroy(e);
    for (void* p : dev_allocs) cudaFree(p);
    if (st_host) cudaFreeHost(st_host);
    if (stream) cudaStreamDestroy(stream);
  }

  int fail(int code, const std::string& msg, int64_t line = -1) {
    err = msg;
    err_line = line;
    return code;
  }

  size_t cells() const { return static_cast<size_t>(d.nr) * static_cast<size_t>(d.nz); }

  cudaEvent_t event() {
    if (ev_used == ev_pool.size()) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      ev_pool.push_back(e);
    }
    return ev_pool[ev_used++];
  }

  void reset_status() {
    // delta slots -> 0 (+0.0), err -> kNoError
    CK(cudaMemsetAsync(st->delta, 0, sizeof(st->delta), stream));
    CK(cudaMemsetAsync(&st->err, 0xff, sizeof(st->err), stream));
  }

  // Fetch delta[1..n] and err from the device (one sync).
  void fetch_status(int n) {
    CK(cudaMemcpyAsync(st_host->delta, st->delta, sizeof(unsigned long long) * (n + 1),
                       cudaMemcpyDeviceToHost, stream));
    CK(cudaMemcpyAsync(&st_host->err, &st->err, sizeof(st->err), cudaMemcpyDeviceToHost,
                       stream));
    CK(cudaStreamSynchronize(stream));
  }

  double delta_of(int it) const {
    double v;
    std::memcpy(&v, &st_host->delta[it], sizeof v);
    return v;
  }

  int check_line_error() {
    const unsigned long long e = st_host->err;
    if (e == kNoError) return PCGPU_OK;
    const int code = static_cast<int>(e & 7ull);
    const int64_t line = static_cast<int64_t>(e >> 3);
    const char* what = code == PCGPU_ERR_ZERO_PIVOT ? "thomas_solve: zero pivot"
                                                    : "property table range violation";
    return fail(code, "line " + std::to_string(line) + " failed: " + what, line);
  }

  double pulse_for(double t, double tau) const {
    // SourceModel::bind_time(t + tau/2) (solver.cpp:238, :337)
    if (d.source_kind != PCGPU_SOURCE_JOULE) return 0.0;
    const double tb = t + 0.5 * tau;
    return pulse_fn ? pulse_fn(clock_user, tb) : host_pulse_value(d, tb);
  }
  double initial_tau(double t) const {  // solver.cpp:44-51
    return tau_fn ? tau_fn(clock_user, t) : host_initial_tau(d, t);
  }

  void timed_begin(int sweep, int it, cudaEvent_t* a) {
    if (!timing) return;
    *a = event();
    CK(cudaEventRecord(*a, stream));
    (void)sweep;
    (void)it;
  }
  void timed_end(int sweep, int it, cudaEvent_t a, int tag = 0) {
    if (!timing) return;
    cudaEvent_t b = event();
    CK(cudaEventRecord(b, stream));
    pending.push_back({a, b, sweep, it, tag});
  }
  // After a sync: accumulate the durations of the iterations that ran (of
  // one sweep; tag < 0: every tag, else that batch step only).
  void collect_timing(int sweep, int ran, int tag = -1) {
    if (!timing) return;
    std::vector<Timed> keep;
    for (const Timed& t : pending) {
      if (t.sweep != sweep || (tag >= 0 && t.tag != tag)) { keep.push_back(t); continue; }
      if (t.it <= ran) {
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, t.a, t.b));
        if (sweep == 0) { radial_ms += ms; ++radial_launches; }
        else { axial_ms += ms; ++axial_launches; }
      }
    }
    pending.swap(keep);
    if (pending.empty()) ev_used = 0;
  }
  void drop_timing() {
    pending.clear();
    ev_used = 0;
  }

  // ---- Picard loop driver shared by both sweeps ----------------------------
  // `launch(it)` enqueues iteration it; returns the converged iteration or 0.
  template <typename Launch>
  int picard(int sweep, int& pred, Launch&& launch, pcgpu_outcome* o) {
    const int max_iter = d.max_iter;
    int launched = 0;
    int batch = std::min(max_iter, std::max(1, pred) + 1);
    o->converged = 0;
    o->iterations = 0;
    o->last_delta = 0;
    while (launched < max_iter) {
      const int upto = std::min(max_iter, launched + batch);
      for (int it = launched + 1; it <= upto; ++it) {
        cudaEvent_t a = nullptr;
        timed_begin(sweep, it, &a);
        launch(it);
        timed_end(sweep, it, a);
      }
      launched = upto;
      fetch_status(launched);
      int rc = check_line_error();
      if (rc) {
        collect_timing(sweep, launched);
        return -rc;
      }
      for (int it = 1; it <= launched; ++it) {
        const double dl = delta_of(it);
        if (dl < d.epsilon) {
          o->converged = 1;
          o->iterations = it;
          o->last_delta = dl;
          if (sweep == 0) pred_stable = it == pred;
          pred = it;
          collect_timing(sweep, it);
          return it;
        }
      }
      batch = 2;
    }
    o->iterations = max_iter;
    o->last_delta = delta_of(max_iter);
    collect_timing(sweep, max_iter);
    return 0;
  }

  // Radial half-step from the anchor `field` (N layout: the explicit pass
  // reads N and writes the T copies the sweep needs). On success *res points
  // at the result (T layout).
  int radial(const double* field, double t, double tau, const double** res, pcgpu_outcome* o) {
    const double pulse = pulse_for(t, tau);
    const double hk = 2.0 / tau;
    reset_status();
    auto dst_of = [&](int it) -> double* { return it % 2 == 1 ? buf[kHalfT] : buf[kIterT]; };
    auto src_of = [&](int it) -> const double* {
      return it == 1 ? buf[kTcT] : (it % 2 == 0 ? buf[kHalfT] : buf[kIterT]);
    };
    launch_explicit_axial_exact(P, field, buf[kExpl], buf[kTcT], st, stream);
    const int conv = picard(0, pred_radial, [&](int it) {
      launch_radial_exact(P, it, d.epsilon, hk, pulse, src_of(it), buf[kTcT], buf[kExpl],
                          buf[kPowT], dst_of(it), buf[kW], buf[kX], st, stream);
    }, o);
    if (conv < 0) return -conv;
    if (conv > 0) *res = dst_of(conv);
    return PCGPU_OK;
  }

  // ---- radial half-step with the host field arriving in row blocks ----------
  // The first attempt of a host-field step (pcgpu_step_host, exact mode): the
  // field is copied in as kPipeChunks row blocks on a copy stream, and K3 plus
  // Picard iterations 1..K (K = predicted + 1) of the radial lines in each
  // block run as soon as the block (and the next one, for K3's halo row) has
  // arrived -- a radial line needs only its own row. Lines are independent;
  // only the stopping rule couples them, so no iteration is skipped here:
  // iteration k of every block writes its delta / error into its own status
  // and its clamp events into its own counters. Afterwards the host applies
  // the reference's sequence -- K3's error, then per iteration its error and
  // the convergence test -- and keeps the counters of the iterations the
  // reference runs. Iterates rotate over three buffers, so the converged one
  // survives up to two speculative iterations; otherwise (and when iteration K
  // has not converged) the half-step is redone from the complete field on the
  // ordinary path. Same arithmetic, same bits.
  bool pipe_ready() {
    if (copy_stream) return true;
    CK(cudaStreamCreateWithFlags(&copy_stream, cudaStreamNonBlocking));
    for (auto& cs : chunk_stream) CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    for (auto& e : pipe_ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (auto& e : chunk_done) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    const size_t nst = static_cast<size_t>(kPipeMaxIter + 1) * kPipeChunks;
    CK(cudaMalloc(&st_pipe, sizeof(DevStatus) * nst));
    dev_allocs.push_back(st_pipe);
    CK(cudaMallocHost(&st_pipe_host, sizeof(DevStatus) * nst));
    CK(cudaMalloc(&clamp_pipe, sizeof(unsigned long long) * (kPipeMaxIter + 1) * kMaxLayers));
    dev_allocs.push_back(clamp_pipe);
    CK(cudaMalloc(&pipe_spare, sizeof(double) * cells()));
    dev_allocs.push_back(pipe_spare);
    return true;
  }

  // *fallback: redo the half-step on the ordinary path (the copy is complete).
  int radial_pipelined(const double* host, double* f, double t, double tau, const double** res,
                       pcgpu_outcome* o, bool* fallback) {
    pipe_ready();
    *fallback = false;
    const int nr = d.nr, nz = d.nz;
    // speculate one iteration beyond the prediction unless the last two radial
    // half-steps converged at the same count (then the tail is one iteration
    // shorter; a longer one falls back)
    const int K = std::min(std::min(d.max_iter, pred_radial + (pred_stable ? 0 : 1)),
                           kPipeMaxIter);
    const double pulse = pulse_for(t, tau);
    const double hk = 2.0 / tau;
    // row blocks: multiples of K3's 64-row tiles
    int jc[kPipeChunks + 1];
    const int rows = (nz + kPipeChunks * kK3RowTile - 1) / (kPipeChunks * kK3RowTile) * kK3RowTile;
    for (int c = 0; c <= kPipeChunks; ++c) jc[c] = std::min(c * rows, nz);
    // the copy stream starts after everything queued so far (f may still be read)
    CK(cudaEventRecord(pipe_ev[kPipeChunks], stream));
    CK(cudaStreamWaitEvent(copy_stream, pipe_ev[kPipeChunks], 0));
    for (int c = 0; c < kPipeChunks; ++c) {
      const size_t off = static_cast<size_t>(jc[c]) * nr;
      const size_t n = static_cast<size_t>(jc[c + 1] - jc[c]) * nr;
      if (n) CK(cudaMemcpyAsync(f + off, host + off, sizeof(double) * n, cudaMemcpyHostToDevice,
                                copy_stream));
      CK(cudaEventRecord(pipe_ev[c], copy_stream));
    }
    // statuses (per row block and iteration) and clamp counters (per iteration)
    const size_t nst = static_cast<size_t>(K + 1) * kPipeChunks;
    for (size_t q = 0; q < nst; ++q) {
      CK(cudaMemsetAsync(st_pipe[q].delta, 0, sizeof(st_pipe[q].delta), stream));
      CK(cudaMemsetAsync(&st_pipe[q].err, 0xff, sizeof(st_pipe[q].err), stream));
    }
    CK(cudaMemsetAsync(clamp_pipe, 0, sizeof(unsigned long long) * (K + 1) * kMaxLayers, stream));
    CK(cudaEventRecord(pipe_ev[kPipeChunks], stream));  // the resets are done
    double* rot[3] = {buf[kHalfT], buf[kIterT], pipe_spare};
    auto dst_of = [&](int k) { return rot[(k - 1) % 3]; };
    auto src_of = [&](int k) -> const double* { return k == 1 ? buf[kTcT] : dst_of(k - 1); };
    auto slot = [&](int k) {
      DevProblem Q = P;
      Q.clamp = clamp_pipe + static_cast<size_t>(k) * kMaxLayers;
      return Q;
    };
    const DevProblem Q0 = slot(0);
    const double* powT = buf[kPowT];
    // each row block on its own stream: blocks run concurrently once arrived
    // (one block's Picard iterations are bound by its lines' pivot chains)
    for (int c = 0; c < kPipeChunks; ++c) {
      cudaStream_t cs = chunk_stream[c];
      const int j0 = jc[c], nj = jc[c + 1] - jc[c];
      CK(cudaStreamWaitEvent(cs, pipe_ev[kPipeChunks], 0));
      if (nj > 0) {
        CK(cudaStreamWaitEvent(cs, pipe_ev[std::min(c + 1, kPipeChunks - 1)], 0));
        CK(cudaStreamWaitEvent(cs, pipe_ev[c], 0));
        launch_explicit_axial_exact_rows(Q0, f, buf[kExpl], buf[kTcT], &st_pipe[c], j0, j0 + nj,
                                         cs);
        for (int k = 1; k <= K; ++k) {
          const DevProblem Qk = slot(k);
          // eps < 0: no iteration is skipped (the stopping rule is applied below)
          launch_radial_exact_slab(Qk, k, -1.0, hk, pulse, j0, nj, src_of(k) + j0,
                                   buf[kTcT] + j0, buf[kExpl] + j0,
                                   powT ? powT + j0 : nullptr, dst_of(k) + j0, buf[kW] + j0,
                                   buf[kX] + j0, &st_pipe[k * kPipeChunks + c], cs, nz);
        }
      }
      CK(cudaEventRecord(chunk_done[c], cs));
      CK(cudaStreamWaitEvent(stream, chunk_done[c], 0));
    }
    CK(cudaMemcpyAsync(st_pipe_host, st_pipe, sizeof(DevStatus) * nst, cudaMemcpyDeviceToHost,
                       stream));
    CK(cudaStreamSynchronize(stream));
    ++pipe_steps;
    auto add_clamps = [&](int upto) {
      launch_add_counters(P.clamp, clamp_pipe, d.n_layers, kMaxLayers, upto + 1, stream);
    };
    // status k combined over the row blocks: lowest failing line, max delta
    auto err_of = [&](int k) {
      unsigned long long e = kNoError;
      for (int c = 0; c < kPipeChunks; ++c) e = std::min(e, st_pipe_host[k * kPipeChunks + c].err);
      return e;
    };
    auto delta_of_k = [&](int k) {
      unsigned long long m = 0;  // non-negative doubles: integer max == double max
      for (int c = 0; c < kPipeChunks; ++c) m = std::max(m, st_pipe_host[k * kPipeChunks + c].delta[k]);
      double v;
      std::memcpy(&v, &m, sizeof v);
      return v;
    };
    auto fail_with = [&](int k) {  // the reference stops at this kernel
      st_host->err = err_of(k);
      add_clamps(k);
      return check_line_error();
    };
    if (err_of(0) != kNoError) return -fail_with(0);
    for (int k = 1; k <= K; ++k) {
      if (err_of(k) != kNoError) return -fail_with(k);
      const double dl = delta_of_k(k);
      if (dl < d.epsilon) {
        if (K - k >= 3) break;  // the converged iterate was overwritten: redo
        add_clamps(k);
        o->converged = 1;
        o->iterations = k;
        o->last_delta = dl;
        pred_stable = k == pred_radial;
        pred_radial = k;
        *res = dst_of(k);
        return PCGPU_OK;
      }
    }
    ++pipe_fallbacks;
    *fallback = true;
    return PCGPU_OK;
  }

  // Axial half-step from the radial result `half` (T layout). `out` (N
  // layout) is the preferred destination; *res receives the buffer holding
  // the result (out or the ping-pong buffer).
  int axial(const double* half, double t, double tau, double* out, const double** res,
            pcgpu_outcome* o) {
    const double pulse = pulse_for(t, tau);
    const double hk = 2.0 / tau;
    reset_status();
    double* anchor = buf[kTcT];  // halfN
    auto src_of = [&](int it) -> const double* {
      return it == 1 ? anchor : (it % 2 == 0 ? out : buf[kIterT]);
    };
    auto dst_of = [&](int it) -> double* { return it % 2 == 1 ? out : buf[kIterT]; };
    // exact lookups: the axial sweep computes K-bar from T_half (no K-bar field)
    double* kbar = kbar_on_the_fly(P) ? nullptr : buf[kKbar];
    launch_axial_rhs_exact(P, hk, pulse, half, buf[kPowN], kbar, buf[kExpl], anchor, st, stream);
    const int conv = picard(1, pred_axial, [&](int it) {
      launch_axial_exact(P, it, d.epsilon, hk, src_of(it), anchor, kbar, buf[kExpl], dst_of(it),
                         buf[kW], buf[kX], st, stream);
    }, o);
    if (conv < 0) return -conv;
    if (conv > 0) *res = dst_of(conv);
    return PCGPU_OK;
  }

  // The user field and the resident state are both N layout.
  void to_state(const double* fieldN, double* state) {
    CK(cudaMemcpyAsync(state, fieldN, sizeof(double) * cells(), cudaMemcpyDeviceToDevice, stream));
  }
  void from_state(const double* state, double* fieldN) {
    if (state != fieldN)
      CK(cudaMemcpyAsync(fieldN, state, sizeof(double) * cells(), cudaMemcpyDeviceToDevice,
                         stream));
  }

  // step(): tau controller (solver.cpp:356-373). `field` is N layout; on
  // acceptance *accepted holds the N-layout buffer with the new field.
  int step(const double* field, double t, double* next, const double** accepted,
           pcgpu_step_result* r, double* attempt_updates, double tau0 = -1.0) {
    double tau = tau0 > 0 ? tau0 : initial_tau(t);
    std::memset(r, 0, sizeof *r);
    const double* host = pipe_host;  // first attempt only
    pipe_host = nullptr;
    for (;;) {
      const double* half = nullptr;
      int rc;
      bool redo = true;
      if (host) {
        rc = radial_pipelined(host, const_cast<double*>(field), t, tau, &half, &r->radial, &redo);
        host = nullptr;
        if (rc < 0) return -rc;
      }
      if (redo) {
        r->radial = pcgpu_outcome{};
        rc = radial(field, t, tau, &half, &r->radial);
      }
      if (rc) return rc;
      *attempt_updates += static_cast<double>(active) * r->radial.iterations;
      if (r->radial.converged) {
        rc = axial(half, t, tau, next, accepted, &r->axial);
        if (rc) return rc;
        *attempt_updates += static_cast<double>(active) * r->axial.iterations;
        if (r->axial.converged) {
          r->tau_used = tau;
          return PCGPU_OK;
        }
      }
      tau *= 0.5;
      ++r->halvings;
      if (tau < tau_floor) {
        char msg[160];
        std::snprintf(msg, sizeof msg, "time step %f fell below floor %f at t=%f", tau,
                      tau_floor, t);
        fail_tau = tau;
        fail_t = t;
        return fail(PCGPU_ERR_TAU_FLOOR, msg);
      }
      r->axial = pcgpu_outcome{};
    }
  }

  // ---- resident stepper ------------------------------------------------------
  bool res_ready() {
    if (!res_grid) return false;
    if (res_ctl) return true;
    CK(cudaMalloc(&res_ctl, sizeof(ResCtl)));
    dev_allocs.push_back(res_ctl);
    CK(cudaMallocHost(&res_ctl_host, sizeof(ResCtl)));
    CK(cudaMalloc(&res_sched, sizeof(ResSched) * kResBatch));
    dev_allocs.push_back(res_sched);
    CK(cudaMallocHost(&res_sched_host, sizeof(ResSched) * kResBatch));
    CK(cudaMalloc(&res_log, sizeof(ResLog) * kResBatch));
    dev_allocs.push_back(res_log);
    CK(cudaMallocHost(&res_log_host, sizeof(ResLog) * kResBatch));
    CK(cudaMalloc(&res_st2, sizeof(DevStatus) * 2));
    dev_allocs.push_back(res_st2);
    CK(cudaMalloc(&res_probe_off, sizeof(int) * kResProbes));
    dev_allocs.push_back(res_probe_off);
    return true;
  }

  // One schedule entry: the first attempt's tau and the pulse of every
  // attempt (tau halved h times, exactly as step() halves it).
  void res_entry(ResSched& e, double t, double tau0) const {
    e.tau0 = tau0;
    double tau = tau0;
    for (int q = 0; q <= kResHalv; ++q) {
      e.pulse[q] = pulse_for(t, tau);
      tau *= 0.5;
    }
  }

  // Runs res_sched_host[0..n) from field buffer X[state]; one host sync.
  // Returns the control block (copied to res_ctl_host); the accepted steps'
  // logs are in res_log_host[0..ctl.steps).
  const ResCtl& res_batch(double* const X[3], int state, int n, int n_probes) {
    ResArgs A{};
    for (int q = 0; q < 3; ++q) A.X[q] = X[q];
    A.TcT = buf[kTcT];
    A.ExplT = buf[kExpl];
    A.HalfT = buf[kHalfT];
    A.kbarN = kbar_on_the_fly(P) ? nullptr : buf[kKbar];
    A.W = buf[kW];
    A.Xs = buf[kX];
    A.st2 = res_st2;
    A.sched = res_sched;
    A.log = res_log;
    A.ctl = res_ctl;
    A.probe_off = res_probe_off;
    A.n_probes = n_probes;
    A.nsteps = n;
    A.state0 = state;
    A.max_iter = d.max_iter;
    const char* mh = std::getenv("PCGPU_RES_MAX_HALV");  // test knob
    A.max_halv = mh ? std::max(0, std::min(kResHalv, std::atoi(mh))) : kResHalv;
    A.eps = d.epsilon;
    A.profile = res_profile ? 1 : 0;
    A.tau_floor = tau_floor;
    A.active = static_cast<double>(active);
    CK(cudaMemcpyAsync(res_sched, res_sched_host, sizeof(ResSched) * n, cudaMemcpyHostToDevice,
                       stream));
    if (res_profile) {
      CK(cudaMemsetAsync(res_ctl->prof_ns, 0, sizeof(res_ctl->prof_ns), stream));
      CK(cudaMemsetAsync(res_ctl->prof_n, 0, sizeof(res_ctl->prof_n), stream));
      CK(cudaMemsetAsync(res_ctl->prof_busy, 0, sizeof(res_ctl->prof_busy), stream));
      CK(cudaMemsetAsync(res_ctl->busy_max, 0, sizeof(res_ctl->busy_max), stream));
      CK(cudaMemsetAsync(&res_ctl->prof_cyc, 0, sizeof(res_ctl->prof_cyc), stream));
    }
    launch_resident(P, A, res_grid, res_cluster, stream);
    CK(cudaMemcpyAsync(res_ctl_host, res_ctl, sizeof(ResCtl), cudaMemcpyDeviceToHost, stream));
    CK(cudaMemcpyAsync(res_log_host, res_log, sizeof(ResLog) * n, cudaMemcpyDeviceToHost,
                       stream));
    CK(cudaStreamSynchronize(stream));
    if (res_profile)
      for (int q = 0; q < 8; ++q) {
        res_prof_ns[q] += res_ctl_host->prof_ns[q];
        res_prof_n[q] += res_ctl_host->prof_n[q];
        res_prof_busy[q] += res_ctl_host->prof_busy[q];
      }
    if (res_profile) res_prof_cyc += static_cast<double>(res_ctl_host->prof_cyc);
    ++res_batches;
    res_steps += res_ctl_host->steps;
    return *res_ctl_host;
  }

  // A batch's stop other than "ran" / "halved" as a status (field intact at
  // X[ctl.state]): line error, tau floor. t = the failed step's time.
  int res_fail(const ResCtl& c, double t) {
    if (c.stop == kResError) {
      st_host->err = c.err;
      return check_line_error();
    }
    char msg[160];
    std::snprintf(msg, sizeof msg, "time step %f fell below floor %f at t=%f", c.tau, tau_floor, t);
    fail_tau = c.tau;
    fail_t = t;
    return fail(PCGPU_ERR_TAU_FLOOR, msg);
  }

  // The step the batch could not finish (more than kResHalv halvings) on the
  // host-driven path, from X[*state]; rotates *state. Same arithmetic, same bits.
  int res_host_step(double* const X[3], int* state, double t, double tau0,
                    pcgpu_step_result* r, double* upd) {
    const int s = *state;
    double* saved = buf[kIterT];
    buf[kIterT] = X[(s + 2) % 3];
    const double* acc = nullptr;
    const int rc = step(X[s], t, X[(s + 1) % 3], &acc, r, upd, tau0);
    buf[kIterT] = saved;
    ++res_host_steps;
    if (rc) return rc;
    *state = acc == X[(s + 1) % 3] ? (s + 1) % 3 : (s + 2) % 3;
    return PCGPU_OK;
  }

  // Controller above the resident batches. `next_tau(t, k)` gives the first
  // attempt's tau of step k (scheduled with no halvings before it);
  // `accept(r)` updates the controller with an accepted step's result and
  // returns false to stop. Stops after max_steps or when `more(t)` is false.
  template <typename Plan, typename Accept, typename More>
  int res_run(double* const X[3], int* state, double* t, int64_t max_steps, Plan&& plan,
              Accept&& accept, More&& more, pcgpu_step_result* results, pcgpu_run_stats* s,
              int n_probes = 0, const std::function<bool(int64_t, const ResLog&)>& on_log = {}) {
    res_ready();
    int64_t done = 0;
    while (done < max_steps && more(*t)) {
      // speculate: no halvings in the batch
      int n = 0;
      double tt = *t;
      typename std::decay<decltype(plan.state())>::type ps = plan.state();
      while (n < kResBatch && done + n < max_steps && (n == 0 || more(tt))) {
        const double tau0 = plan.next(ps, tt);
        res_entry(res_sched_host[n], tt, tau0);
        plan.advance(ps, tau0);
        tt += tau0;
        ++n;
      }
      const ResCtl& c = res_batch(X, *state, n, n_probes);
      for (int q = 0; q < c.steps; ++q) {
        const ResLog& lg = res_log_host[q];
        const pcgpu_step_result& r = lg.r;
        *t += r.tau_used;
        if (results) results[done] = r;
        s->steps += 1;
        s->halvings += r.halvings;
        s->radial_iterations += r.radial.iterations;
        s->axial_iterations += r.axial.iterations;
        s->cell_updates += lg.updates;
        s->cell_updates_accepted +=
            static_cast<double>(active) * (r.radial.iterations + r.axial.iterations);
        s->attempt_cells += 2.0 * static_cast<double>(active) * (r.halvings + 1);
        accept(r);
        ++done;
        if (on_log && !on_log(done, lg)) {
          *state = c.state;
          return PCGPU_OK;
        }
      }
      *state = c.state;
      if (c.stop == kResError || c.stop == kResFloor) return res_fail(c, *t);
      if (c.stop == kResNeedHost) {
        pcgpu_step_result r;
        double upd = 0;
        const double tau0 = plan.next(plan.state(), *t);
        const int rc = res_host_step(X, state, *t, tau0, &r, &upd);
        s->cell_updates += upd;
        if (rc) return rc;
        *t += r.tau_used;
        if (results) results[done] = r;
        s->steps += 1;
        s->halvings += r.halvings;
        s->radial_iterations += r.radial.iterations;
        s->axial_iterations += r.axial.iterations;
        s->cell_updates_accepted +=
            static_cast<double>(active) * (r.radial.iterations + r.axial.iterations);
        s->attempt_cells += 2.0 * static_cast<double>(active) * (r.halvings + 1);
        accept(r);
        ++done;
        if (on_log) {
          ResLog lg{};
          lg.r = r;
          lg.updates = upd;
          gather_probes_host(X[*state], n_probes, lg.probes);
          if (!on_log(done, lg)) return PCGPU_OK;
        }
      }
    }
    return PCGPU_OK;
  }

  void gather_probes_host(const double* field, int n, double* out) {
    if (n <= 0) return;
    std::vector<int> off(n);
    CK(cudaMemcpy(off.data(), res_probe_off, sizeof(int) * n, cudaMemcpyDeviceToHost));
    for (int k = 0; k < n; ++k)
      CK(cudaMemcpyAsync(out + k, field + off[k], sizeof(double), cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
  }
  double fail_tau = 0, fail_t = 0;

  // ---- speculative batches (grids too large for the resident stepper) -------
  // Host-driven runs read a status after every half-step. The Picard counts
  // of consecutive steps are nearly constant on the large grids, so instead a
  // batch of up to kSpecBatch steps is enqueued at once: each with its tau
  // from the schedule (no halving), each sweep launching its predicted count
  // + 1 iterations (those after convergence return at once, as in the
  // host-driven sweep). The iterate a sweep converged in depends on the count's
  // parity, so the next kernel (K4 after the radial sweep, the next step's K3
  // after the axial one) picks it on the device (SpecPick). A one-thread
  // verify kernel after each sweep checks convergence within the launched
  // count without error; on failure every later half-step is marked
  // kSpecAbort and does nothing. Steps alternate between two pairs of
  // iterate buffers, so the field a failed step started from is intact: the
  // steps before it are kept, the clamp counters go back to the snapshot
  // taken after the last good step, and that step is redone host-driven
  // (halving, error, longer sweep). One read per batch. Same kernels, same
  // arithmetic: bit-identical to the step-by-step path.
  static constexpr int kSpecBatch = 16;
  double* spec_n[4] = {};            // two pairs of N-layout iterate buffers
  bool spec_alloc_failed = false;
  DevStatus* spec_st = nullptr;      // [2 * kSpecBatch] status per half-step
  DevStatus* spec_st_host = nullptr;
  unsigned long long* spec_clamp_save = nullptr;  // [kMaxLayers]
  int64_t spec_batches = 0, spec_steps = 0, spec_rollbacks = 0;
  bool spec_ok() const {
    return P.exact_ws && d.source_kind != PCGPU_SOURCE_FIELD && !spec_alloc_failed &&
           std::getenv("PCGPU_NO_SPECULATE") == nullptr;
  }
  bool spec_ready() {
    if (spec_st) return true;
    if (spec_alloc_failed) return false;
    for (int q = 0; q < 4; ++q) {  // disjoint from buf[kField] / kNext / kIterT
      if (cudaMalloc(&spec_n[q], sizeof(double) * cells()) != cudaSuccess) {
        cudaGetLastError();  // not enough memory: run step by step
        for (int r = 0; r < q; ++r) cudaFree(spec_n[r]);
        for (auto& p : spec_n) p = nullptr;
        spec_alloc_failed = true;
        return false;
      }
    }
    for (double* p : spec_n) dev_allocs.push_back(p);
    CK(cudaMalloc(&spec_st, sizeof(DevStatus) * 2 * kSpecBatch));
    dev_allocs.push_back(spec_st);
    CK(cudaMallocHost(&spec_st_host, sizeof(DevStatus) * 2 * kSpecBatch));
    CK(cudaMalloc(&spec_clamp_save, sizeof(unsigned long long) * kMaxLayers));
    dev_allocs.push_back(spec_clamp_save);
    return true;
  }

  // Step k of a batch (statuses spec_st[2k], [2k+1]; n steps in all), from
  // `from` (the previous step's SpecPick; from.st == nullptr: the field C)
  // into the pair (Po, Qo): its result is Po after an odd axial count, Qo
  // after an even one. Lr / La: iterations launched per sweep.
  void spec_enqueue(int k, int n, const double* C, const SpecPick& from, double t, double tau,
                    int Lr, int La, double* Po, double* Qo) {
    const double pulse = pulse_for(t, tau);
    const double hk = 2.0 / tau;
    DevStatus* sr = spec_st + 2 * k;
    DevStatus* sa = sr + 1;
    const int nlater = 2 * (n - k);  // statuses after sr (sa included)
    launch_explicit_axial_exact(P, C, buf[kExpl], buf[kTcT], sr, stream, from);
    for (int it = 1; it <= Lr; ++it) {
      const double* src = it == 1 ? buf[kTcT] : (it % 2 == 0 ? buf[kHalfT] : buf[kIterT]);
      double* dst = it % 2 == 1 ? buf[kHalfT] : buf[kIterT];
      cudaEvent_t a = nullptr;
      timed_begin(0, it, &a);
      launch_radial_exact(P, it, d.epsilon, hk, pulse, src, buf[kTcT], buf[kExpl], buf[kPowT], dst,
                          buf[kW], buf[kX], sr, stream);
      timed_end(0, it, a, k + 1);
    }
    k_spec_verify<<<1, 32, 0, stream>>>(sr, Lr, d.epsilon, sa, nlater - 1, P.clamp,
                                        spec_clamp_save, d.n_layers, 0);
    SpecPick half;
    half.st = sr;
    half.odd = buf[kHalfT];
    half.even = buf[kIterT];
    half.eps = d.epsilon;
    double* kbar = kbar_on_the_fly(P) ? nullptr : buf[kKbar];
    double* anchor = buf[kTcT];  // halfN
    launch_axial_rhs_exact(P, hk, pulse, nullptr, buf[kPowN], kbar, buf[kExpl], anchor, sa, stream,
                           half);
    for (int it = 1; it <= La; ++it) {
      const double* src = it == 1 ? anchor : (it % 2 == 0 ? Po : Qo);
      double* dst = it % 2 == 1 ? Po : Qo;
      cudaEvent_t a = nullptr;
      timed_begin(1, it, &a);
      launch_axial_exact(P, it, d.epsilon, hk, src, anchor, kbar, buf[kExpl], dst, buf[kW],
                         buf[kX], sa, stream);
      timed_end(1, it, a, k + 1);
    }
    k_spec_verify<<<1, 32, 0, stream>>>(sa, La, d.epsilon, sa + 1, nlater - 2, P.clamp,
                                        spec_clamp_save, d.n_layers, 1);
    g_launches += 2;
  }

  // First converged iteration (<= launched) of a batch status, no error; 0 if none.
  int spec_conv(const DevStatus& x, int launched, double* last) const {
    if (x.err != kNoError) return 0;
    for (int it = 1; it <= launched; ++it) {
      double dl;
      std::memcpy(&dl, &x.delta[it], sizeof dl);
      if (dl < d.epsilon) {
        *last = dl;
        return it;
      }
    }
    return 0;
  }

  // Host-driven runs: speculative batches, each failed step redone step by
  // step. The field is buf[kField] in and out. Plan / accept / more as in
  // res_run.
  template <typename Plan, typename Accept, typename More>
  int host_run(double* t, int64_t max_steps, Plan&& plan, Accept&& accept, More&& more,
               pcgpu_step_result* results, pcgpu_run_stats* s) {
    int64_t done = 0;
    auto record = [&](const pcgpu_step_result& r, double upd) {
      *t += r.tau_used;
      if (results) results[done] = r;
      s->steps += 1;
      s->halvings += r.halvings;
      s->radial_iterations += r.radial.iterations;
      s->axial_iterations += r.axial.iterations;
      s->cell_updates += upd;
      s->cell_updates_accepted +=
          static_cast<double>(active) * (r.radial.iterations + r.axial.iterations);
      s->attempt_cells += 2.0 * static_cast<double>(active) * (r.halvings + 1);
      accept(r);
      ++done;
    };
    // one host-driven step of the field in buf[kField] (rotating kNext / kIterT)
    auto safe_step = [&]() -> int {
      pcgpu_step_result r;
      const double* acc = nullptr;
      double upd = 0;
      double* cur = buf[kField];
      const int rc = step(cur, *t, buf[kNext], &acc, &r, &upd, plan.next(plan.state(), *t));
      if (rc) return rc;
      double* accepted = const_cast<double*>(acc);
      if (accepted == buf[kNext]) std::swap(buf[kField], buf[kNext]);
      else std::swap(buf[kField], buf[kIterT]);
      record(r, upd);
      return PCGPU_OK;
    };
    bool learned = false;  // counts known from a host-driven step
    while (done < max_steps && more(*t)) {
      if (!learned || !spec_ok() || !spec_ready()) {
        const int rc = safe_step();
        if (rc) return rc;
        learned = true;
        continue;
      }
      const int Lr = std::min(d.max_iter, std::max(1, pred_radial) + 1);
      const int La = std::min(d.max_iter, std::max(1, pred_axial) + 1);
      int n = 0;
      double tt = *t;
      auto ps = plan.state();
      double taus[kSpecBatch];
      while (n < kSpecBatch && done + n < max_steps && (n == 0 || more(tt))) {
        taus[n] = plan.next(ps, tt);
        plan.advance(ps, taus[n]);
        tt += taus[n];
        ++n;
      }
      double* const C = buf[kField];  // the batch input: never written in the batch
      k_spec_reset<<<1, 32, 0, stream>>>(spec_st, 2 * n, P.clamp, spec_clamp_save, d.n_layers);
      ++g_launches;
      SpecPick from;  // step 0 reads C
      double ts = *t;
      for (int k = 0; k < n; ++k) {
        double* Po = spec_n[2 * (k & 1)];
        double* Qo = spec_n[2 * (k & 1) + 1];
        spec_enqueue(k, n, C, from, ts, taus[k], Lr, La, Po, Qo);
        from.st = spec_st + 2 * k + 1;
        from.odd = Po;
        from.even = Qo;
        from.eps = d.epsilon;
        ts += taus[k];
      }
      CK(cudaMemcpyAsync(spec_st_host, spec_st, sizeof(DevStatus) * 2 * n, cudaMemcpyDeviceToHost,
                         stream));
      CK(cudaStreamSynchronize(stream));
      ++spec_batches;
      // the steps that converged within their launches, in order
      int good = 0;
      int q = -1;  // index in spec_n of the last good step's result
      for (int k = 0; k < n; ++k) {
        double dr = 0, da = 0;
        const int cr = spec_conv(spec_st_host[2 * k], Lr, &dr);
        const int ca = cr ? spec_conv(spec_st_host[2 * k + 1], La, &da) : 0;
        if (!ca) break;
        if (timing) {
          collect_timing(0, cr, k + 1);
          collect_timing(1, ca, k + 1);
        }
        pcgpu_step_result r{};
        r.tau_used = taus[k];
        r.radial = pcgpu_outcome{1, cr, dr};
        r.axial = pcgpu_outcome{1, ca, da};
        record(r, static_cast<double>(active) * (cr + ca));
        pred_radial = cr;
        pred_axial = ca;
        q = 2 * (k & 1) + ((ca & 1) ? 0 : 1);
        ++good;
      }
      if (timing) drop_timing();  // the failed step's launches are redone
      spec_steps += good;
      if (q >= 0) {  // the result becomes the field; the old field takes its place
        buf[kField] = spec_n[q];
        spec_n[q] = C;
      }
      if (good < n) {
        // a sweep did not converge within its launches (or failed): redo that
        // step host-driven from the counters after the last good step
        ++spec_rollbacks;
        CK(cudaMemcpyAsync(P.clamp, spec_clamp_save, sizeof(unsigned long long) * d.n_layers,
                           cudaMemcpyDeviceToDevice, stream));
        if (done < max_steps && more(*t)) {
          const int rc = safe_step();
          if (rc) return rc;
        }
      }
    }
    return PCGPU_OK;
  }
};

// Schedules for the resident stepper's controller (pcgpu_stepper::res_run).
// A plan gives the first attempt's tau of the next step from its state and
// advances the state as if the step were accepted without halving.
struct FixedPlan {  // step(): tau = initial_tau(t) every step (solver.cpp:357)
  const pcgpu_stepper* h;
  struct State {};
  State state() const { return {}; }
  double next(const State&, double t) const { return h->initial_tau(t); }
  void advance(State&, double) const {}
};
struct GrowthPlan {  // the BASELINE growth policy (pcgpu_run_growth)
  double grow, tau_max;
  int easy_steps;
  struct State {
    double tau;
    int easy;
  } st;
  State state() const { return st; }
  double next(const State& s, double) const { return s.tau; }
  void advance(State& s, double tau_used) const { update(s, tau_used, 0); }
  void update(State& s, double tau_used, int halvings) const {
    s.tau = tau_used;
    s.easy = halvings == 0 ? s.easy + 1 : 0;
    if (s.easy >= easy_steps) {
      s.tau = std::min(s.tau * grow, tau_max);
      s.easy = 0;
    }
  }
};

// DevProblem from the descriptor: metric reciprocals and flattened tables,
// uploaded to the current device. Shared by the
// single-GPU stepper and the partitioned (multi-GPU) stepper.
void build_dev_problem(const pcgpu_desc* d, DevProblem& P, std::vector<void*>& allocs) {
  const int nr = d->nr, nz = d->nz;
    // Metric reciprocals exactly as the reference stepper computes them
    // (solver.cpp:146-159; geometry.hpp:87-94). Host code is compiled with
    // -ffp-contract=off, so these are the reference's bits.
    std::vector<double> face_r_lo(nr), inv_gap_r(nr + 1), inv_vol_r(nr);
    std::vector<double> inv_gap_z(nz + 1), inv_eta(nz), control_z(nz), gap_z(nz + 1), width_z(nz);
    for (int i = 0; i < nr; ++i) {
      face_r_lo[i] = i == 0 ? 0.0 : 0.5 * (d->r_center[i - 1] + d->r_center[i]);
      const double control_r = 0.5 * (d->gap_r[i] + d->gap_r[i + 1]);
      inv_vol_r[i] = 1.0 / (d->r_center[i] * control_r);
      inv_gap_r[i] = 1.0 / d->gap_r[i];
    }
    inv_gap_r[nr] = 1.0 / d->gap_r[nr];
    for (int j = 0; j < nz; ++j) {
      control_z[j] = 0.5 * (d->gap_z[j] + d->gap_z[j + 1]);
      inv_eta[j] = 1.0 / control_z[j];
      inv_gap_z[j] = 1.0 / d->gap_z[j];
      width_z[j] = d->width_z[j];
    }
    inv_gap_z[nz] = 1.0 / d->gap_z[nz];
    for (int j = 0; j <= nz; ++j) gap_z[j] = d->gap_z[j];
    std::vector<int> layer(d->layer, d->layer + nr);

    // Tables, flattened.
    std::vector<double> knots, vals, xpair;
    
    P.n_layers = d->n_layers;
    for (int m = 0; m < d->n_layers; ++m) {
      const pcgpu_material& mt = d->materials[m];
      P.mats[m].rho = mt.rho;
      const pcgpu_table* tabs[3] = {&mt.cv, &mt.lambda, &mt.chi};
      for (int p = 0; p < 3; ++p) {
        const pcgpu_table& t = *tabs[p];
        P.mats[m].off[p] = static_cast<int>(knots.size());
        P.mats[m].n[p] = t.n;
        P.mats[m].uniform[p] = 0;
        P.mats[m].inv_h[p] = 0.0;
        for (int k = 0; k < t.n; ++k) {
          knots.push_back(t.t[k]);
          vals.push_back(t.v[k]);
          xpair.push_back(t.v[k]);
          xpair.push_back(k + 1 < t.n ? t.v[k + 1] - t.v[k] : 0.0);
        }
        if (t.n > 0) {
          P.mats[m].t_first[p] = t.t[0];
          P.mats[m].t_last[p] = t.t[t.n - 1];
          P.mats[m].v_first[p] = t.v[0];
          P.mats[m].v_last[p] = t.v[t.n - 1];
        }
        P.mats[m].xmode[p] = 0;
        if (t.n == 2) {
          // a single interval: the bracket is always k = 1
          P.mats[m].uniform[p] = 2;
          P.mats[m].inv_h[p] = 0.0;
          P.mats[m].xmode[p] = 2;
          P.mats[m].rdt[p] = 1.0 / (t.t[1] - t.t[0]);  // RN(1/(t1 - t0)) for div_rn
        } else if (t.n >= 3) {
          // Uniform-knot bracket guess (exactness is kept by the device fix-up).
          const double inv_h = (t.n - 1) / (t.t[t.n - 1] - t.t[0]);
          double worst = 0;
          for (int k = 0; k < t.n; ++k)
            worst = std::max(worst, std::fabs((t.t[k] - t.t[0]) * inv_h - k));
          if (worst < 0.5) {
            P.mats[m].uniform[p] = 1;
            P.mats[m].inv_h[p] = inv_h;
            // Exactly uniform with a power-of-two step: the bracket is exact.
            const double h = t.t[1] - t.t[0];
            int ex;
            const bool pow2 = h > 0 && std::frexp(h, &ex) == 0.5;
            bool exact = pow2 && std::isfinite(t.t[0]);
            for (int k = 0; exact && k < t.n; ++k)
              exact = t.t[k] == t.t[0] + k * h && (t.t[k] - t.t[0]) * (1.0 / h) == k;
            if (exact) {
              P.mats[m].uniform[p] = 2;
              P.mats[m].inv_h[p] = 1.0 / h;
              P.mats[m].xmode[p] = 1;
              P.mats[m].h[p] = h;
            }
          }
        }
      }
    }
    // exact kernels' branch-free lookups: lambda/cv tables xmode 1 whose t0 >= 0
    // is a multiple of h and whose top knot's ulp is below h (T - t0 exact), chi
    // a single interval or absent; MeanTemperature faces.
    P.exact_x = d->halfpoint_rule == PCGPU_HALFPOINT_MEAN_TEMPERATURE;
    for (int m = 0; m < d->n_layers && P.exact_x; ++m) {
      for (int p = 0; p < 2; ++p) {
        const DevMaterial& dm = P.mats[m];
        if (dm.xmode[p] != 1) { P.exact_x = 0; break; }
        const double h = dm.h[p];
        const double q = dm.t_first[p] / h;
        if (dm.t_first[p] < 0 || q != std::floor(q) || std::nextafter(dm.t_last[p], 1e300) - dm.t_last[p] > h)
          P.exact_x = 0;
      }
      if (P.mats[m].n[2] > 0 && P.mats[m].xmode[2] != 2) P.exact_x = 0;
    }
    if (std::getenv("PCGPU_NO_EXACTX")) P.exact_x = 0;
    // exact lean: exact_x and one knot grid per property (cv, lambda) across
    // layers -- per-property lookup constants, guard pairs for the clamps
    P.exact_lean = P.exact_x && d->n_layers <= kMaxLayers;
    for (int p = 0; p < 2 && P.exact_lean; ++p) {
      const DevMaterial& a = P.mats[0];
      for (int m = 1; m < d->n_layers; ++m) {
        const DevMaterial& b = P.mats[m];
        if (a.n[p] != b.n[p] || a.t_first[p] != b.t_first[p] || a.t_last[p] != b.t_last[p] ||
            a.inv_h[p] != b.inv_h[p])
          P.exact_lean = 0;
      }
    }
    if (std::getenv("PCGPU_NO_EXACTLEAN")) P.exact_lean = 0;
    // div_rn precondition: every per-row / per-table denominator it divides by
    // has |b| in [2^-100, 2^100]
    {
      auto in = [](double b) { b = std::fabs(b); return b >= 0x1p-100 && b <= 0x1p100; };
      P.div_ok = 1;
      for (int j = 0; j < nz; ++j)
        if (!in(d->gap_z[j]) || !in(0.5 * (d->gap_z[j] + d->gap_z[j + 1]))) P.div_ok = 0;
      if (!in(d->gap_z[nz])) P.div_ok = 0;
      for (int m = 0; m < d->n_layers; ++m)
        if (P.mats[m].xmode[2] == 2 && !in(P.mats[m].t_last[2] - P.mats[m].t_first[2]))
          P.div_ok = 0;
    }
    std::vector<double> xe;
    if (P.exact_lean) {
      for (int p = 0; p < 2; ++p) {
        const int n = P.mats[0].n[p];
        P.xe_t0[p] = P.mats[0].t_first[p];
        P.xe_tK[p] = P.mats[0].t_last[p];
        P.xe_inv_h[p] = P.mats[0].inv_h[p];
        P.xe_n[p] = n;
        P.xe_base[p] = static_cast<int>(xe.size() / 2);
        for (int m = 0; m < d->n_layers; ++m) {
          const pcgpu_table& t = p == 0 ? d->materials[m].cv : d->materials[m].lambda;
          xe.push_back(t.v[0]);
          xe.push_back(0.0);
          for (int k = 1; k < n; ++k) {
            xe.push_back(t.v[k - 1]);
            xe.push_back(t.v[k] - t.v[k - 1]);
          }
          xe.push_back(t.v[n - 1]);
          xe.push_back(0.0);
        }
      }
      for (int m = 0; m < d->n_layers; ++m) P.xe_rho[m] = P.mats[m].rho;
    }
    P.exact_ws = std::getenv("PCGPU_NO_EXACTWS") ? 0 : 1;
    // test knob: every full tile of the line solvers takes the reciprocal redo path
    P.rcp_redo = std::getenv("PCGPU_RCP_REDO") ? 1 : 0;
    P.prof = nullptr;
    if (std::getenv("PCGPU_RES_PROF")) {  // solver-warp cycle counters (resident profile)
      unsigned long long* pc = nullptr;
      CK(cudaMalloc(&pc, sizeof(unsigned long long) * 16));
      CK(cudaMemset(pc, 0, sizeof(unsigned long long) * 16));
      allocs.push_back(pc);
      P.prof = pc;
    }
    P.nr = nr;
    P.nz = nz;
    P.nr_core = d->nr_core;
    P.nz_shared = d->nz_shared;
    {
      const std::vector<int> re = desc_row_extent(d), ce = desc_col_extent(d);
      int* dre = nullptr;
      int* dce = nullptr;
      CK(cudaMalloc(&dre, sizeof(int) * re.size()));
      CK(cudaMalloc(&dce, sizeof(int) * ce.size()));
      allocs.push_back(dre);
      allocs.push_back(dce);
      CK(cudaMemcpy(dre, re.data(), sizeof(int) * re.size(), cudaMemcpyHostToDevice));
      CK(cudaMemcpy(dce, ce.data(), sizeof(int) * ce.size(), cudaMemcpyHostToDevice));
      P.row_ext = dre;
      P.col_ext = dce;
    }
    auto up = [&](const std::vector<double>& v) {
      double* p = dev_upload(v);
      allocs.push_back(p);
      return p;
    };
    int* dlayer = dev_upload(layer);
    allocs.push_back(dlayer);
    P.layer = dlayer;
    P.face_r_lo = up(face_r_lo);
    std::vector<double> gfac(nr + 1, 0.0);
    for (int i = 0; i < nr; ++i) gfac[i] = face_r_lo[i] * inv_gap_r[i];
    P.gfac_r = up(gfac);
    P.inv_gap_r = up(inv_gap_r);
    P.inv_vol_r = up(inv_vol_r);
    P.gap_z = up(gap_z);
    P.inv_gap_z = up(inv_gap_z);
    P.inv_eta = up(inv_eta);
    P.control_z = up(control_z);
    P.width_z = up(width_z);
    P.knots = up(knots);
    P.vals = up(vals);
    P.xpair = up(xpair);
    if (P.exact_lean) P.xe_tab = up(xe);
    P.source_kind = d->source_kind;
    P.source_layer = d->source_layer;
    if (d->source_kind == PCGPU_SOURCE_JOULE) {  // chi_x2's constants
      const DevMaterial& m = P.mats[P.source_layer];
      P.chi_t0 = m.t_first[kChi];
      P.chi_tK = m.t_last[kChi];
      P.chi_vl = m.v_first[kChi];
      P.chi_vh = m.v_last[kChi];
      P.chi_dt = P.chi_tK - P.chi_t0;
      P.chi_dv = P.chi_vh - P.chi_vl;
      P.chi_rdt = m.rdt[kChi];
    }
    P.amplitude = d->amplitude;
    P.halfpoint_rule = d->halfpoint_rule;
    P.range_policy = d->range_policy;
    P.all_neumann = d->all_neumann;
    P.T0 = d->T0;
    unsigned long long* clamp = nullptr;
    CK(cudaMalloc(&clamp, sizeof(unsigned long long) * d->n_layers));
    CK(cudaMemset(clamp, 0, sizeof(unsigned long long) * d->n_layers));
    allocs.push_back(clamp);
    P.clamp = clamp;
}

// Exported for pcgpu_dist.cu.
std::string pcgpu_validate_desc(const pcgpu_desc* d) { return validate(d); }
double pcgpu_host_initial_tau(const pcgpu_desc& d, double t) { return host_initial_tau(d, t); }
double pcgpu_host_pulse_value(const pcgpu_desc& d, double t) { return host_pulse_value(d, t); }

#define GUARD_BEGIN DeviceGuard dg_(h->d.device); try {
#define GUARD_END(h)                                                                  \
  }                                                                                   \
  catch (const CudaError& ce) {                                                       \
    return (h)->fail(PCGPU_ERR_CUDA, std::string(ce.what) + ": " + cudaGetErrorString(ce.e)); \
  }

// Steps bound a FIELD source's power per half-step (the caller binds it
// before every half-step); the whole-step entry points cannot.
static int reject_field_source(pcgpu_stepper* h) {
  if (h->d.source_kind != PCGPU_SOURCE_FIELD) return PCGPU_OK;
  return h->fail(PCGPU_ERR_CONFIG,
                 "a FIELD source is bound per half-step (pcgpu_bind_power_field): drive "
                 "radial_half_step / axial_half_step instead of step / run / evolve");
}

// The resident stepper on the rotation X = {field buffer, next, spare}; the
// field enters X[0] and leaves X[state]; the stepper's buffer roles follow.
template <typename Run>
static int resident_run(pcgpu_stepper* h, double* field, Run&& run) {
  double* X[3] = {h->buf[kField], h->buf[kNext], h->buf[kIterT]};
  h->to_state(field, X[0]);
  int state = 0;
  const int rc = run(X, &state);
  h->from_state(X[state], field);
  h->buf[kField] = X[state];
  h->buf[kNext] = X[(state + 1) % 3];
  h->buf[kIterT] = X[(state + 2) % 3];
  CK(cudaStreamSynchronize(h->stream));
  return rc;
}

extern "C" {

int32_t pcgpu_abi_version(void) { return PCGPU_ABI_VERSION; }

int pcgpu_device_count(int32_t* count) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) n = 0;
  *count = n;
  return PCGPU_OK;
}

int pcgpu_create(const pcgpu_desc* d, pcgpu_stepper** out) {
  if (!d || !out) return PCGPU_ERR_ARG;
  *out = nullptr;
  const std::string v = validate(d);
  if (!v.empty()) {
    g_create_error = v;
    return PCGPU_ERR_CONFIG;
  }
  DeviceGuard dg(d->device);
  if (!dg.ok) {
    g_create_error = "pcgpu_create: cannot select device " + std::to_string(d->device);
    return PCGPU_ERR_CUDA;
  }
  auto h = std::make_unique<pcgpu_stepper>();
  try {
    h->d = *d;
    CK(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
    const int nr = d->nr, nz = d->nz;
    h->tau_floor = d->tau_min > 0 ? d->tau_min : 1e-12 * d->t_per;  // solver.hpp:28-30
    h->col_ext_host = desc_col_extent(d);
    for (int i = 0; i < nr; ++i) h->active += h->col_ext_host[i];
    (void)nz;

    build_dev_problem(d, h->P, h->dev_allocs);
    // the caller's arrays are copied; the stepper keeps no pointer to them
    h->d.row_extent = h->d.col_extent = nullptr;

    CK(cudaMalloc(&h->st, sizeof(DevStatus)));
    h->dev_allocs.push_back(h->st);
    CK(cudaMallocHost(&h->st_host, sizeof(DevStatus)));

    // Field buffers (the reference's half_, next_, iter_buf_, expl_, kbar_,
    // solver.cpp:140-144, plus the layout copies and Thomas work vectors).
    // Filled with T0 like the reference's half_/next_/iter_buf_.
    const size_t bytes = sizeof(double) * h->cells();
    std::vector<double> t0fill(h->cells(), d->T0);
    for (int b = 0; b < kNumBufs; ++b) {
      if ((b == kPowN || b == kPowT) && d->source_kind != PCGPU_SOURCE_FIELD) continue;
      if (b == kKbar && kbar_on_the_fly(h->P)) continue;  // computed inside the axial sweep
      if (b == kStage) continue;  // lazily, by the *_host entry points
      double* p = nullptr;
      CK(cudaMalloc(&p, bytes));
      h->dev_allocs.push_back(p);
      if (b == kPowN || b == kPowT)  // no power until pcgpu_bind_power_field
        CK(cudaMemset(p, 0, bytes));
      else
        CK(cudaMemcpy(p, t0fill.data(), bytes, cudaMemcpyHostToDevice));
      h->buf[b] = p;
    }
    CK(cudaDeviceSynchronize());
    // the resident stepper where it applies ($PCGPU_RESIDENT=0: host-driven steps)
    const char* rv = std::getenv("PCGPU_RESIDENT");
    h->res_grid = (rv && std::atoi(rv) == 0) ? 0 : resident_grid(h->P);
    h->res_cluster = h->res_grid > 0 && resident_cluster(h->P, h->res_grid);
    // the speculative batches' buffers up front (not inside a timed run)
    if (!h->res_grid && h->spec_ok()) h->spec_ready();  // outside any timed region
    h->launches0 = g_launches;
  } catch (const CudaError& ce) {
    g_create_error = std::string(ce.what) + ": " + cudaGetErrorString(ce.e);
    return PCGPU_ERR_CUDA;
  }
  *out = h.release();
  return PCGPU_OK;
}

void pcgpu_destroy(pcgpu_stepper* h) {
  if (!h) return;
  DeviceGuard dg(h->d.device);
  delete h;
}

const char* pcgpu_last_error(const pcgpu_stepper* h) {
  return h ? h->err.c_str() : g_create_error.c_str();
}

int64_t pcgpu_error_line(const pcgpu_stepper* h) { return h ? h->err_line : -1; }

double pcgpu_initial_tau(const pcgpu_stepper* h, double t) { return h->initial_tau(t); }
double pcgpu_pulse_value(const pcgpu_stepper* h, double t) {
  return h->pulse_fn ? h->pulse_fn(h->clock_user, t) : host_pulse_value(h->d, t);
}
int64_t pcgpu_active_cells(const pcgpu_stepper* h) { return h->active; }

int pcgpu_set_host_clock(pcgpu_stepper* h, pcgpu_clock_fn pulse_value, pcgpu_clock_fn initial_tau,
                         void* user) {
  if (!h) return PCGPU_ERR_ARG;
  h->pulse_fn = pulse_value;
  h->tau_fn = initial_tau;
  h->clock_user = user;
  return PCGPU_OK;
}

int pcgpu_last_tau_floor(const pcgpu_stepper* h, double* tau, double* floor, double* t) {
  if (!h || !tau || !floor || !t) return PCGPU_ERR_ARG;
  *tau = h->fail_tau;
  *floor = h->tau_floor;
  *t = h->fail_t;
  return PCGPU_OK;
}

int pcgpu_speculation_stats(const pcgpu_stepper* h, int64_t* batches, int64_t* steps,
                            int64_t* rollbacks) {
  if (!h || !batches || !steps || !rollbacks) return PCGPU_ERR_ARG;
  *batches = h->spec_batches;
  *steps = h->spec_steps;
  *rollbacks = h->spec_rollbacks;
  return PCGPU_OK;
}

int pcgpu_resident_stats(const pcgpu_stepper* h, int32_t* grid, int64_t* batches, int64_t* steps,
                         int64_t* host_steps) {
  if (!h || !grid || !batches || !steps || !host_steps) return PCGPU_ERR_ARG;
  *grid = h->res_grid;
  *batches = h->res_batches;
  *steps = h->res_steps;
  *host_steps = h->res_host_steps;
  return PCGPU_OK;
}
void* pcgpu_stream(const pcgpu_stepper* h) { return h->stream; }
int64_t pcgpu_launch_count(const pcgpu_stepper* h) {
  return static_cast<int64_t>(g_launches - h->launches0);
}

int32_t pcgpu_describe(const pcgpu_stepper* h, char* buf, int32_t len) {
  std::string s;
  s = "mode=exact lines=";
  s += h->P.exact_ws ? "ws" : "thread";
  s += " lookups=";
  s += h->P.exact_lean ? "exact-lean" : (h->P.exact_x ? "exact-x" : "generic");
  s += " steps=";
  s += h->res_grid ? (std::string("resident:") + std::to_string(h->res_grid) +
                      (h->res_cluster ? "-cta-cluster" : "-cta-cooperative"))
                   : std::string("host-driven");
  if (buf && len > 0) {
    const size_t n = std::min(s.size(), static_cast<size_t>(len - 1));
    std::memcpy(buf, s.data(), n);
    buf[n] = 0;
  }
  return static_cast<int32_t>(s.size());
}

int pcgpu_bind_power_field(pcgpu_stepper* h, const double* power_dev) {
  if (h->d.source_kind != PCGPU_SOURCE_FIELD || !power_dev)
    return h->fail(PCGPU_ERR_ARG, "bind_power_field: source kind is not FIELD");
  GUARD_BEGIN
  CK(cudaMemcpyAsync(h->buf[kPowN], power_dev, sizeof(double) * h->cells(),
                     cudaMemcpyDeviceToDevice, h->stream));
  launch_transpose_N2T(h->P, h->buf[kPowN], h->buf[kPowT], h->stream);
  h->power_bound = true;
  GUARD_END(h)
  return PCGPU_OK;
}

// A FIELD source's power array is bound for one half-step at a time (the
// reference binds the source's time inside every half-step, solver.cpp:238,
// :337): each half-step consumes the binding.
static int consume_power_binding(pcgpu_stepper* h) {
  if (h->d.source_kind != PCGPU_SOURCE_FIELD) return PCGPU_OK;
  if (!h->power_bound)
    return h->fail(PCGPU_ERR_CONFIG,
                   "FIELD source: pcgpu_bind_power_field must precede every half-step");
  h->power_bound = false;
  return PCGPU_OK;
}

int pcgpu_radial_half_step(pcgpu_stepper* h, const double* T_cur, double t, double tau,
                           double* out, pcgpu_outcome* o) {
  if (!h || !T_cur || !out || !o || out == T_cur) return PCGPU_ERR_ARG;
  if (const int e = consume_power_binding(h)) return e;
  GUARD_BEGIN
  const double* res = nullptr;
  const int rc = h->radial(T_cur, t, tau, &res, o);
  if (rc) return rc;
  if (o->converged) launch_transpose_T2N(h->P, res, out, h->stream);
  CK(cudaStreamSynchronize(h->stream));
  GUARD_END(h)
  return PCGPU_OK;
}

int pcgpu_axial_half_step(pcgpu_stepper* h, const double* T_half, double t, double tau,
                          double* out, pcgpu_outcome* o) {
  if (!h || !T_half || !out || !o || out == T_half) return PCGPU_ERR_ARG;
  if (const int e = consume_power_binding(h)) return e;
  GUARD_BEGIN
  launch_transpose_N2T(h->P, T_half, h->buf[kHalfT], h->stream);
  const double* res = nullptr;
  const int rc = h->axial(h->buf[kHalfT], t, tau, out, &res, o);
  if (rc) return rc;
  if (o->converged) h->from_state(res, out);
  CK(cudaStreamSynchronize(h->stream));
  GUARD_END(h)
  return PCGPU_OK;
}

int pcgpu_step(pcgpu_stepper* h, double* field, double t, pcgpu_step_result* r) {
  if (!h || !field || !r) return PCGPU_ERR_ARG;
  if (const int e = reject_field_source(h)) return e;
  if (h->res_grid) {
    // one resident step on X = {field, next, spare}; the result is copied into
    // the caller's array (field.swap(next_), solver.cpp:364)
    GUARD_BEGIN
    double* X[3] = {field, h->buf[kNext], h->buf[kIterT]};
    int state = 0;
    double tt = t;
    pcgpu_run_stats s{};
    *r = pcgpu_step_result{};
    const int rc = h->res_run(X, &state, &tt, 1, FixedPlan{h}, [](const pcgpu_step_result&) {},
                              [](double) { return true; }, r, &s);
    if (rc) return rc;
    if (state != 0) {
      CK(cudaMemcpyAsync(field, X[state], sizeof(double) * h->cells(), cudaMemcpyDeviceToDevice,
                         h->stream));
      // keep the three roles distinct: the other buffer stays the spare
      h->buf[kNext] = X[state];
      h->buf[kIterT] = X[state == 1 ? 2 : 1];
    }
    CK(cudaStreamSynchronize(h->stream));
    GUARD_END(h)
    return PCGPU_OK;
  }
  GUARD_BEGIN
  const double* acc = nullptr;
  double upd = 0;
  const int rc = h->step(field, t, h->buf[kNext], &acc, r, &upd);
  if (rc) return rc;
  // field.swap(next_) (solver.cpp:364): the caller's array receives the result.
  h->from_state(acc, field);
  CK(cudaStreamSynchronize(h->stream));
  GUARD_END(h)
  return PCGPU_OK;
}

int pcgpu_run(pcgpu_stepper* h, double* field, double t0, int32_t nsteps,
              pcgpu_step_result* results, pcgpu_run_stats* stats) {
  if (!h || !field || nsteps < 0) return PCGPU_ERR_ARG;
  if (const int e = reject_field_source(h)) return e;
  pcgpu_run_stats s{};
  double t = t0;
  int rc = PCGPU_OK;
  if (h->res_grid) {
    GUARD_BEGIN
    rc = resident_run(h, field, [&](double* const X[3], int* state) {
      return h->res_run(X, state, &t, nsteps, FixedPlan{h}, [](const pcgpu_step_result&) {},
                        [](double) { return true; }, results, &s);
    });
    GUARD_END(h)
    s.t_end = t;
    if (stats) *stats = s;
    return rc;
  }
  GUARD_BEGIN
  // the field stays resident in buf[kField] (buffer roles rotate, no copies)
  h->to_state(field, h->buf[kField]);
  rc = h->host_run(&t, nsteps, FixedPlan{h}, [](const pcgpu_step_result&) {},
                   [](double) { return true; }, results, &s);
  h->from_state(h->buf[kField], field);
  CK(cudaStreamSynchronize(h->stream));
  GUARD_END(h)
  s.t_end = t;
  if (stats) *stats = s;
  return rc;
}

int pcgpu_run_growth(pcgpu_stepper* h, double* field, double t0, double t_end, int32_t max_steps,
                     double tau_start, double grow, int32_t easy_steps, double tau_max,
                     pcgpu_step_result* results, pcgpu_run_stats* stats) {
  if (!h || !field || max_steps < 0 || !(tau_start > 0) || !(grow >= 1.0)) return PCGPU_ERR_ARG;
  if (const int e = reject_field_source(h)) return e;
  pcgpu_run_stats s{};
  double t = t0, tau = std::min(tau_start, tau_max);
  int easy = 0, rc = PCGPU_OK;
  if (h->res_grid) {
    GUARD_BEGIN
    GrowthPlan plan{grow, tau_max, easy_steps, {tau, 0}};
    rc = resident_run(h, field, [&](double* const X[3], int* state) {
      return h->res_run(
          X, state, &t, max_steps, plan,
          [&](const pcgpu_step_result& r) { plan.update(plan.st, r.tau_used, r.halvings); },
          [&](double tt) { return tt < t_end; }, results, &s);
    });
    GUARD_END(h)
    s.t_end = t;
    if (stats) *stats = s;
    return rc;
  }
  GUARD_BEGIN
  GrowthPlan plan{grow, tau_max, easy_steps, {tau, easy}};
  h->to_state(field, h->buf[kField]);
  rc = h->host_run(
      &t, max_steps, plan,
      [&](const pcgpu_step_result& r) { plan.update(plan.st, r.tau_used, r.halvings); },
      [&](double tt) { return tt < t_end; }, results, &s);
  h->from_state(h->buf[kField], field);
  CK(cudaStreamSynchronize(h->stream));
  GUARD_END(h)
  s.t_end = t;
  if (stats) *stats = s;
  return rc;
}

static void ensure_stage(pcgpu_stepper* h) {
  if (h->buf[kStage]) return;
  double* p = nullptr;
  CK(cudaMalloc(&p, sizeof(double) * h->cells()));
  h->dev_allocs.push_back(p);
  CK(cudaMemsetAsync(p, 0, sizeof(double) * h->cells(), h->stream));
  h->buf[kStage] = p;
}

int pcgpu_pipeline_stats(const pcgpu_stepper* h, int64_t* steps, int64_t* fallbacks) {
  if (!h || !steps || !fallbacks) return PCGPU_ERR_ARG;
  *steps = h->pipe_steps;
  *fallbacks = h->pipe_fallbacks;
  return PCGPU_OK;
}

int pcgpu_step_host(pcgpu_stepper* h, double* field_host, double t, pcgpu_step_result* r) {
  if (!h || !field_host) return PCGPU_ERR_ARG;
  GUARD_BEGIN
  ensure_stage(h);
  double* f = h->buf[kStage];
  const bool no_pipe = std::getenv("PCGPU_NO_PIPELINE") != nullptr;
  const char* mv = std::getenv("PCGPU_PIPELINE_MIN_NZ");  // tests: pipeline small grids
  const int min_nz = mv ? std::atoi(mv) : 2048;
  if (h->P.exact_ws && !no_pipe && h->d.nz >= min_nz && !h->res_grid) {
    // the copy-in overlaps K3 and the first radial iterations (radial_pipelined);
    // the accepted buffer goes straight back to the host
    const double* acc = nullptr;
    double upd = 0;
    h->pipe_host = field_host;
    const int rc = h->step(f, t, h->buf[kNext], &acc, r, &upd);
    h->pipe_host = nullptr;
    if (rc) return rc;
    CK(cudaMemcpyAsync(field_host, acc, sizeof(double) * h->cells(), cudaMemcpyDeviceToHost,
                       h->stream));
    CK(cudaStreamSynchronize(h->stream));
    return PCGPU_OK;
  }
  CK(cudaMemcpyAsync(f, field_host, sizeof(double) * h->cells(), cudaMemcpyHostToDevice,
                     h->stream));
  const int rc = pcgpu_step(h, f, t, r);
  if (rc) return rc;
  CK(cudaMemcpyAsync(field_host, f, sizeof(double) * h->cells(), cudaMemcpyDeviceToHost,
                     h->stream));
  CK(cudaStreamSynchronize(h->stream));
  GUARD_END(h)
  return PCGPU_OK;
}

static int half_host(pcgpu_stepper* h, bool radial, const double* in_host, double t, double tau,
                     double* out_host, pcgpu_outcome* o) {
  GUARD_BEGIN
  ensure_stage(h);
  double* in = h->buf[kField];
  double* out = h->buf[kStage];
  CK(cudaMemcpyAsync(in, in_host, sizeof(double) * h->cells(), cudaMemcpyHostToDevice,
                     h->stream));
  CK(cudaMemcpyAsync(out, out_host, sizeof(double) * h->cells(), cudaMemcpyHostToDevice,
                     h->stream));
  const int rc = radial ? pcgpu_radial_half_step(h, in, t, tau, out, o)
                        : pcgpu_axial_half_step(h, in, t, tau, out, o);
  if (rc) return rc;
  CK(cudaMemcpyAsync(out_host, out, sizeof(double) * h->cells(), cudaMemcpyDeviceToHost,
                     h->stream));
  CK(cudaStreamSynchronize(h->stream));
  GUARD_END(h)
  return PCGPU_OK;
}

int pcgpu_radial_half_step_host(pcgpu_stepper* h, const double* T_cur_host, double t,
                                double tau, double* out_host, pcgpu_outcome* o) {
  if (!h || !T_cur_host || !out_host || !o) return PCGPU_ERR_ARG;
  return half_host(h, true, T_cur_host, t, tau, out_host, o);
}

int pcgpu_axial_half_step_host(pcgpu_stepper* h, const double* T_half_host, double t,
                               double tau, double* out_host, pcgpu_outcome* o) {
  if (!h || !T_half_host || !out_host || !o) return PCGPU_ERR_ARG;
  return half_host(h, false, T_half_host, t, tau, out_host, o);
}

int pcgpu_clamp_events(const pcgpu_stepper* h, uint64_t* counts) {
  if (!h || !counts) return PCGPU_ERR_ARG;
  DeviceGuard dg(h->d.device);
  if (cudaStreamSynchronize(h->stream) != cudaSuccess) return PCGPU_ERR_CUDA;
  if (cudaMemcpy(counts, h->P.clamp, sizeof(uint64_t) * h->d.n_layers, cudaMemcpyDeviceToHost) !=
      cudaSuccess)
    return PCGPU_ERR_CUDA;
  return PCGPU_OK;
}

int pcgpu_enable_kernel_timing(pcgpu_stepper* h, int32_t on) {
  h->timing = on != 0;
  h->radial_ms = h->axial_ms = 0;
  h->radial_launches = h->axial_launches = 0;
  return PCGPU_OK;
}

int pcgpu_kernel_timing(const pcgpu_stepper* h, double* radial_ms, int64_t* radial_launches,
                        double* axial_ms, int64_t* axial_launches) {
  *radial_ms = h->radial_ms;
  *radial_launches = h->radial_launches;
  *axial_ms = h->axial_ms;
  *axial_launches = h->axial_launches;
  return PCGPU_OK;
}

}  // extern "C"

// ---- Device-resident runner --------------------------------
namespace {

// PhaseResampler (runner.cpp:35-62): resamples an adaptively stepped trace
// onto samples_per_period fixed phases of each period by linear interpolation.
struct PhaseResamplerGpu {
  double t_per = 1, dt = 1;
  int samples = 1;
  long next_sample = 0;
  bool seeded = false;
  double t_prev = 0, v_prev = 0;
  std::vector<double> current;
  std::vector<std::vector<double>> rows;
  PhaseResamplerGpu(double tp, int s) : t_per(tp), dt(tp / s), samples(s), current(s, 0.0) {}
  void seed(double t, double v) {
    t_prev = t;
    v_prev = v;
    seeded = true;
    next_sample = static_cast<long>(std::ceil(t / dt));
  }
  void feed(double t, double v) {
    if (!seeded) {
      seed(t, v);
      return;
    }
    while (static_cast<double>(next_sample) * dt <= t) {
      const double pt = static_cast<double>(next_sample) * dt;
      double val = v_prev;
      if (t > t_prev) val = v_prev + (v - v_prev) * ((pt - t_prev) / (t - t_prev));
      current[next_sample % samples] = val;
      if (next_sample % samples == samples - 1) rows.push_back(current);
      ++next_sample;
    }
    t_prev = t;
    v_prev = v;
  }
};

// RegimeDetector::update (runner.cpp:76-95): fires once `min_periods`
// consecutive period pairs agree phase-wise within `tol` (max |difference|,
// NaN-ignoring maximum like the reference's reduction).
struct RegimeDetectorGpu {
  PhaseResamplerGpu rs;
  double tol;
  int min_periods;
  size_t checked = 1;
  int consecutive = 0;
  bool fired = false;
  RegimeDetectorGpu(double tp, int samples, double tol_, int minp)
      : rs(tp, samples), tol(tol_), min_periods(minp) {}
  bool update(double t, double v) {
    rs.feed(t, v);
    while (checked < rs.rows.size()) {
      const std::vector<double>& a = rs.rows[checked];
      const std::vector<double>& b = rs.rows[checked - 1];
      double diff = std::abs(a[0] - b[0]);
      for (size_t q = 1; q < a.size(); ++q) {
        const double d = std::abs(a[q] - b[q]);
        if (diff < d) diff = d;
      }
      consecutive = diff < tol ? consecutive + 1 : 0;
      ++checked;
      if (!fired && consecutive >= min_periods) {
        fired = true;
        return true;
      }
    }
    return false;
  }
};

__global__ void k_gather_probes(const double* __restrict__ f, const int* __restrict__ off, int n,
                                double* __restrict__ out) {
  const int k = threadIdx.x;
  if (k < n) out[k] = f[off[k]];
}

}  // namespace

extern "C" {

int pcgpu_evolve(pcgpu_stepper* h, double* field, const pcgpu_runner_cfg* cfg,
                 pcgpu_step_cb on_step, pcgpu_snapshot_cb on_snapshot, void* user,
                 pcgpu_evolve_result* res) {
  if (!h || !field || !cfg || !res) return PCGPU_ERR_ARG;
  if (const int e = reject_field_source(h)) return e;
  // RunnerConfig::validate (runner.hpp:96-102)
  if (!(cfg->t_end > 0)) return h->fail(PCGPU_ERR_CONFIG, "runner.t_end: must be > 0");
  if (cfg->detector_samples_per_period < 1)
    return h->fail(PCGPU_ERR_CONFIG, "detector.samples_per_period: must be >= 1");
  if (!(cfg->detector_tolerance > 0))
    return h->fail(PCGPU_ERR_CONFIG, "detector.tolerance: must be > 0");
  if (cfg->detector_min_periods < 1)
    return h->fail(PCGPU_ERR_CONFIG, "detector.min_periods: must be >= 1");
  std::vector<double> pending(cfg->snapshot_times, cfg->snapshot_times + cfg->n_snapshot_times);
  for (double ts : pending)
    if (ts < 0) return h->fail(PCGPU_ERR_CONFIG, "runner.snapshot_times: must be >= 0");
  std::sort(pending.begin(), pending.end());
  const int np = cfg->n_probes;
  if (np < 0 || np > 1024) return PCGPU_ERR_ARG;
  const pcgpu_desc& d = h->d;
  std::vector<int> off(np);
  for (int k = 0; k < np; ++k) {
    const int i = cfg->probe_i[k], j = cfg->probe_j[k];
    const bool in_mask = i >= 0 && i < d.nr && j >= 0 && j < h->col_ext_host[i];
    if (!in_mask) return h->fail(PCGPU_ERR_CONFIG, "probe cell falls outside the domain");
    off[k] = j * d.nr + i;
  }
  *res = pcgpu_evolve_result{};
  res->fire_t = -1;
  GUARD_BEGIN
  int* d_off = nullptr;
  double* d_vals = nullptr;
  double* h_vals = nullptr;
  CK(cudaMalloc(&d_off, sizeof(int) * std::max(np, 1)));
  CK(cudaMalloc(&d_vals, sizeof(double) * std::max(np, 1)));
  CK(cudaMallocHost(&h_vals, sizeof(double) * std::max(np, 1)));
  struct Free {
    int* a;
    double* b;
    double* c;
    ~Free() {
      cudaFree(a);
      cudaFree(b);
      cudaFreeHost(c);
    }
  } free_guard{d_off, d_vals, h_vals};
  if (np) CK(cudaMemcpy(d_off, off.data(), sizeof(int) * np, cudaMemcpyHostToDevice));
  const bool resident = h->res_grid && np <= kResProbes && h->res_ready();
  if (resident && np)
    CK(cudaMemcpy(h->res_probe_off, off.data(), sizeof(int) * np, cudaMemcpyHostToDevice));
  // field rotation X[state] (resident) / cur, nxt, spare (host-driven steps)
  double* X[3] = {h->buf[kField], h->buf[kNext], h->buf[kIterT]};
  int state = 0;
  h->to_state(field, X[0]);
  auto gather = [&](const double* f) {  // probe values of field f into h_vals
    if (!np) return;
    k_gather_probes<<<1, 1024, 0, h->stream>>>(f, d_off, np, d_vals);
    ++g_launches;
    CK(cudaMemcpyAsync(h_vals, d_vals, sizeof(double) * np, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
  };
  auto snapshot = [&](int kind, double ts, const double* f) {  // N layout, device
    if (!on_snapshot) return;
    if (!f) throw CudaError{cudaErrorUnknown, "evolve: snapshot inside a multi-step batch"};
    CK(cudaStreamSynchronize(h->stream));
    on_snapshot(user, kind, ts, f);
  };
  // Regime detection over probe 0: the caller's detector (e.g. the
  // reference's own RegimeDetector through the C++ drop-in) or the
  // restatement of runner.cpp:35-95 below.
  const bool detect = cfg->source_on && np > 0;
  RegimeDetectorGpu det(d.t_per, cfg->detector_samples_per_period, cfg->detector_tolerance,
                        cfg->detector_min_periods);
  auto det_seed = [&](double t, double v) {
    if (cfg->detect) cfg->detect(cfg->detect_user, 1, t, v);
    else det.rs.seed(t, v);
  };
  auto det_update = [&](double t, double v) {
    return cfg->detect ? cfg->detect(cfg->detect_user, 0, t, v) != 0 : det.update(t, v);
  };
  if (detect) {
    gather(X[0]);
    det_seed(0.0, h_vals[0]);
  }
  long period_idx = 1, off_idx = 0;
  const double off_offset = d.t_src + d.t_trs;
  size_t next_time = 0;
  double t = 0, comp = 0;
  int stop = PCGPU_STOP_REACHED_TIME;
  // The reference's per-step bookkeeping (runner.cpp:140-180) for an accepted
  // step from field `prev` to field `cur` with probe values `vals`. Returns
  // true when the regime detector fired.
  auto after_step = [&](const pcgpu_step_result& r, const double* prev, const double* cur,
                        const double* vals) {
    const double t_before = t;
    {  // Kahan accumulation of the accepted steps (runner.cpp:141-146)
      const double y = r.tau_used - comp;
      const double tt = t + y;
      comp = (tt - t) - y;
      t = tt;
    }
    res->steps += 1;
    if (on_step) on_step(user, res->steps, t, r.tau_used, vals);
    const double edge = static_cast<double>(period_idx) * d.t_per;
    if (cfg->snapshot_pre_on && t >= edge && t_before < edge)
      snapshot(PCGPU_SNAP_PRE_ON, t_before, prev);
    while (t >= static_cast<double>(period_idx) * d.t_per) ++period_idx;
    if (cfg->snapshot_post_off && t >= static_cast<double>(off_idx) * d.t_per + off_offset) {
      snapshot(PCGPU_SNAP_POST_OFF, t, cur);
      while (t >= static_cast<double>(off_idx) * d.t_per + off_offset) ++off_idx;
    }
    while (next_time < pending.size() && t >= pending[next_time]) {
      snapshot(PCGPU_SNAP_AT_TIME, t, cur);
      ++next_time;
    }
    if (detect && det_update(t, vals[0])) {
      res->fire_t = t;
      stop = PCGPU_STOP_PERIODIC;
      return true;
    }
    return false;
  };
  // Could an accepted step from tb to ta trigger a snapshot or complete a
  // resampled period (the only time the detector can fire)? Such steps run
  // as single-step batches, so that their input field is still intact.
  const double dt_s = d.t_per / cfg->detector_samples_per_period;
  const long S = cfg->detector_samples_per_period;
  auto eventful = [&](double tb, double ta) {
    const long pi = std::max(period_idx, static_cast<long>(std::floor(tb / d.t_per)));
    for (long q = pi - 1; q <= pi + 1; ++q) {
      const double e = static_cast<double>(q) * d.t_per;
      if (cfg->snapshot_pre_on && ta >= e && tb < e) return true;
    }
    if (cfg->snapshot_post_off && ta >= static_cast<double>(off_idx) * d.t_per + off_offset)
      return true;
    for (size_t q = next_time; q < pending.size(); ++q)
      if (ta >= pending[q]) return true;
    if (detect) {  // a sample index k = S-1 (mod S) with tb <= k*dt <= ta
      // (>= tb: conservative at the seed's sample 0)
      long k = static_cast<long>(std::floor(tb / dt_s));
      k = k - ((k % S) + S) % S + (S - 1);
      while (static_cast<double>(k) * dt_s < tb) k += S;
      while (k >= S && static_cast<double>(k - S) * dt_s >= tb) k -= S;
      if (static_cast<double>(k) * dt_s <= ta) return true;
    }
    return false;
  };
  bool fired = false;
  while (!fired) {
    if (t >= cfg->t_end) {
      stop = PCGPU_STOP_REACHED_TIME;
      break;
    }
    if (resident) {
      // schedule: steps from (t, comp) assuming no halving, ending before an
      // eventful step (or with it alone), or once t_end is reached
      int n = 0;
      double tt = t, cc = comp;
      while (n < pcgpu_stepper::kResBatch && tt < cfg->t_end) {
        const double tau0 = h->initial_tau(tt);
        const double y = tau0 - cc;
        const double ta = tt + y;
        const bool ev = eventful(tt, ta);
        if (ev && n > 0) break;
        h->res_entry(h->res_sched_host[n], tt, tau0);
        ++n;
        cc = (ta - tt) - y;
        tt = ta;
        if (ev) break;
      }
      const int s0 = state;
      const ResCtl c = h->res_batch(X, state, n, np);
      for (int q = 0; q < c.steps && !fired; ++q) {
        const ResLog& lg = h->res_log_host[q];
        // single-step batches keep the step's input field intact
        const int sq = c.steps == 1 ? c.state : -1;
        fired = after_step(lg.r, c.steps == 1 ? X[s0] : nullptr, sq >= 0 ? X[sq] : nullptr,
                           lg.probes);
      }
      state = c.state;
      if (fired) break;
      if (c.stop == kResFloor) {  // the field stays the last accepted one
        h->res_fail(c, t);
        stop = PCGPU_STOP_TAU_FLOOR;
        break;
      }
      if (c.stop == kResError) {
        const int rc = h->res_fail(c, t);
        h->buf[kField] = X[state];
        h->buf[kNext] = X[(state + 1) % 3];
        h->buf[kIterT] = X[(state + 2) % 3];
        return rc;
      }
      if (c.stop == kResNeedHost) {
        const int s1 = state;
        pcgpu_step_result r;
        double upd = 0;
        const int rc = h->res_host_step(X, &state, t, -1.0, &r, &upd);
        if (rc == PCGPU_ERR_TAU_FLOOR) {
          stop = PCGPU_STOP_TAU_FLOOR;
          break;
        }
        if (rc) return rc;
        gather(X[state]);
        fired = after_step(r, X[s1], X[state], h_vals);
      }
      continue;
    }
    // host-driven step on the rotation
    const int s1 = state;
    pcgpu_step_result r;
    double upd = 0;
    const int rc = h->res_host_step(X, &state, t, -1.0, &r, &upd);
    if (rc == PCGPU_ERR_TAU_FLOOR) {  // the field stays the last accepted one
      stop = PCGPU_STOP_TAU_FLOOR;
      break;
    }
    if (rc) {
      h->buf[kField] = X[state];
      h->buf[kNext] = X[(state + 1) % 3];
      h->buf[kIterT] = X[(state + 2) % 3];
      return rc;
    }
    gather(X[state]);
    fired = after_step(r, X[s1], X[state], h_vals);
  }
  h->buf[kField] = X[state];
  h->buf[kNext] = X[(state + 1) % 3];
  h->buf[kIterT] = X[(state + 2) % 3];
  h->from_state(X[state], field);
  CK(cudaStreamSynchronize(h->stream));
  res->t = t;
  res->reason = stop;
  if (!h->runner) h->runner = new pcgpu_runner_state();
  h->runner->detector_rows =
      detect && !cfg->detect ? det.rs.rows : std::vector<std::vector<double>>{};
  h->runner->samples = cfg->detector_samples_per_period;
  res->detector_periods = static_cast<int32_t>(h->runner->detector_rows.size());
  GUARD_END(h)
  return PCGPU_OK;
}

int pcgpu_evolve_host(pcgpu_stepper* h, double* field_host, const pcgpu_runner_cfg* cfg,
                      pcgpu_step_cb on_step, pcgpu_snapshot_cb on_snapshot, void* user,
                      pcgpu_evolve_result* res) {
  if (!h || !field_host) return PCGPU_ERR_ARG;
  DeviceGuard dg(h->d.device);
  // Trampolines: the step callback passes through, snapshots are copied to a
  // host buffer first.
  struct Ctx {
    pcgpu_step_cb step;
    pcgpu_snapshot_cb snap;
    void* user;
    std::vector<double> host;
    size_t cells;
    bool copy_failed = false;
  } ctx{on_step, on_snapshot, user, {}, h->cells()};
  auto step_tr = [](void* u, int64_t k, double t, double tau, const double* v) {
    Ctx* c = static_cast<Ctx*>(u);
    if (c->step) c->step(c->user, k, t, tau, v);
  };
  auto snap_tr = [](void* u, int32_t kind, double t, const double* fdev) {
    Ctx* c = static_cast<Ctx*>(u);
    if (!c->snap) return;
    c->host.resize(c->cells);
    if (cudaMemcpy(c->host.data(), fdev, sizeof(double) * c->cells, cudaMemcpyDeviceToHost) !=
        cudaSuccess) {
      c->copy_failed = true;
      return;
    }
    c->snap(c->user, kind, t, c->host.data());
  };
  double* dev = nullptr;
  GUARD_BEGIN
  CK(cudaMalloc(&dev, sizeof(double) * h->cells()));
  GUARD_END(h)
  int rc = PCGPU_OK;
  if (cudaMemcpy(dev, field_host, sizeof(double) * h->cells(), cudaMemcpyHostToDevice) !=
      cudaSuccess)
    rc = h->fail(PCGPU_ERR_CUDA, "evolve: field copy failed");
  if (rc == PCGPU_OK) rc = pcgpu_evolve(h, dev, cfg, step_tr, snap_tr, &ctx, res);
  if (rc == PCGPU_OK && ctx.copy_failed)
    rc = h->fail(PCGPU_ERR_CUDA, "evolve: snapshot copy failed");
  if (rc == PCGPU_OK &&
      cudaMemcpy(field_host, dev, sizeof(double) * h->cells(), cudaMemcpyDeviceToHost) !=
          cudaSuccess)
    rc = h->fail(PCGPU_ERR_CUDA, "evolve: field copy failed");
  cudaFree(dev);
  return rc;
}

int pcgpu_detector_periods(const pcgpu_stepper* h, double* rows, int32_t max_rows) {
  if (!h || !rows) return PCGPU_ERR_ARG;
  if (!h->runner) return PCGPU_OK;
  const auto& R = h->runner->detector_rows;
  for (size_t k = 0; k < R.size() && static_cast<int32_t>(k) < max_rows; ++k)
    std::copy(R[k].begin(), R[k].end(), rows + k * h->runner->samples);
  return PCGPU_OK;
}

}  // extern "C"
