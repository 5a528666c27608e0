// pulsecell_gpu/adi_stepper.hpp -- drop-in GPU AdiStepper for the reference's
// C++ interface (header-only; links against libpcgpu.so through pcgpu.h).
//
// Mirrors class pulsecell::AdiStepper (proj/include/pulsecell/solver.hpp:66-106)
// method for method: same constructor arguments (the LinePool is replaced by
// a DeviceOptions), same radial_half_step / axial_half_step / step signatures on
// pulsecell::Array2, same exceptions (ConfigError, TauFloorError, LineError).
// The Grid, the MaterialTables and the SourceModel are borrowed exactly like
// the reference borrows them; their data are marshalled once into a
// pcgpu_desc. Device-native sources: NullSource and JouleSource (recognised by
// dynamic_cast, source.hpp:57-83); anything else is rejected with ConfigError.
// The time stepping runs on the reference's own host functions (pulse_value,
// initial_tau), registered with pcgpu_set_host_clock.
//
// Usage inside the reference tree:
//   #include "pulsecell_gpu/adi_stepper.hpp"
//   pulsecell::gpu::AdiStepper stepper(grid, layers, source, timing, cfg, {});
//   auto r = stepper.step(field, t);   // field is a pulsecell::Array2
#pragma once

#include <cstring>
#include <string>
#include <vector>

#include "pcgpu.h"
#include "pulsecell/errors.hpp"
#include "pulsecell/geometry.hpp"
#include "pulsecell/materials.hpp"
#include "pulsecell/runner.hpp"
#include "pulsecell/solver.hpp"
#include "pulsecell/source.hpp"

namespace pulsecell {
namespace gpu {

struct DeviceOptions {
  int device = 0;  // CUDA device ordinal (the kernels are bit-identical to the CPU AdiStepper)
};

class AdiStepper {
 public:
  AdiStepper(const Grid& grid, LayerMaterials mats, SourceModel& source, const SourceSpec& timing,
             SolverConfig cfg, DeviceOptions opt = {})
      : grid_(grid), mats_(std::move(mats)), source_(source), timing_(timing), cfg_(cfg) {
    cfg_.validate();     // solver.cpp:133
    timing_.validate();  // solver.cpp:134
    if (static_cast<int>(mats_.size()) != grid_.domain().layer_count())
      throw ConfigError("stepper: one material required per layer");
    for (const auto* m : mats_)
      if (m == nullptr) throw ConfigError("stepper: null material");
    // Grid metrics exactly as the reference Grid holds them (geometry.hpp:60-100).
    const Index nr = grid_.nr(), nz = grid_.nz();
    layer_.resize(nr);
    r_center_.resize(nr);
    gap_r_.resize(nr + 1);
    width_z_.resize(nz);
    gap_z_.resize(nz + 1);
    for (Index i = 0; i < nr; ++i) {
      layer_[i] = grid_.layer(i);
      r_center_[i] = grid_.r_center(i);
    }
    for (Index i = 0; i <= nr; ++i) gap_r_[i] = grid_.gap_r(i);
    for (Index j = 0; j < nz; ++j) width_z_[j] = grid_.width_z(j);
    for (Index j = 0; j <= nz; ++j) gap_z_[j] = grid_.gap_z(j);
    mat_.resize(mats_.size());
    for (size_t m = 0; m < mats_.size(); ++m) {
      const MaterialTable& t = *mats_[m];
      mat_[m].rho = t.rho();
      mat_[m].cv = table(t.table(Property::HeatCapacity));
      mat_[m].lambda = table(t.table(Property::Conductivity));
      mat_[m].chi = table(t.table(Property::Resistivity));
    }
    pcgpu_desc d{};
    d.abi_version = PCGPU_ABI_VERSION;
    d.nr = static_cast<int32_t>(nr);
    d.nz = static_cast<int32_t>(nz);
    d.nr_core = static_cast<int32_t>(grid_.nr_core());
    d.nz_shared = static_cast<int32_t>(grid_.nz_shared());
    d.layer = layer_.data();
    d.r_center = r_center_.data();
    d.gap_r = gap_r_.data();
    d.width_z = width_z_.data();
    d.gap_z = gap_z_.data();
    d.n_layers = static_cast<int32_t>(mat_.size());
    d.materials = mat_.data();
    if (auto* js = dynamic_cast<JouleSource*>(&source_)) {
      d.source_kind = PCGPU_SOURCE_JOULE;
      d.source_layer = grid_.domain().source_layer;
      d.amplitude = js->spec().current_factor();
    } else if (dynamic_cast<NullSource*>(&source_)) {
      d.source_kind = PCGPU_SOURCE_NULL;
    } else {
      throw ConfigError("gpu stepper: only NullSource and JouleSource are device-native");
    }
    d.t_per = timing_.t_per;
    d.t_src = timing_.t_src;
    d.t_trs = timing_.t_trs;
    d.xi = timing_.xi;
    d.zeta = timing_.zeta;
    d.waveform = timing_.waveform == Waveform::Rectangular ? PCGPU_WAVE_RECTANGULAR
                                                           : PCGPU_WAVE_TRANSIENT;
    d.epsilon = cfg_.epsilon;
    d.max_iter = cfg_.max_iter;
    d.tau_min = cfg_.tau_min;
    d.tau_transient_divisor = cfg_.tau_transient_divisor;
    d.tau_source_divisor = cfg_.tau_source_divisor;
    d.halfpoint_rule = static_cast<int32_t>(cfg_.halfpoint_rule);
    d.range_policy = static_cast<int32_t>(cfg_.range_policy);
    d.all_neumann = cfg_.all_neumann ? 1 : 0;
    d.T0 = cfg_.T0;
    d.t_ceiling = cfg_.t_ceiling;
    d.mode = PCGPU_MODE_EXACT;
    d.device = opt.device;
    const int rc = pcgpu_create(&d, &h_);
    if (rc != PCGPU_OK) raise(rc, pcgpu_last_error(nullptr));
    // the reference's own host functions drive the time stepping:
    // pulse_value (source.cpp:42-45) and initial_tau (solver.cpp:44-51)
    pcgpu_set_host_clock(h_, &AdiStepper::pulse_cb, &AdiStepper::tau_cb, this);
  }
  ~AdiStepper() { pcgpu_destroy(h_); }
  AdiStepper(const AdiStepper&) = delete;
  AdiStepper& operator=(const AdiStepper&) = delete;

  HalfStepOutcome radial_half_step(const Array2& T_cur, Real t, Real tau, Array2& out) {
    pcgpu_outcome o{};
    check(pcgpu_radial_half_step_host(h_, T_cur.data(), t, tau, out.data(), &o));
    return outcome(o);
  }
  HalfStepOutcome axial_half_step(const Array2& T_half, Real t, Real tau, Array2& out) {
    pcgpu_outcome o{};
    check(pcgpu_axial_half_step_host(h_, T_half.data(), t, tau, out.data(), &o));
    return outcome(o);
  }
  StepResult step(Array2& field, Real t) {
    pcgpu_step_result r{};
    check(pcgpu_step_host(h_, field.data(), t, &r));
    StepResult s;
    s.tau_used = r.tau_used;
    s.halvings = r.halvings;
    s.radial = outcome(r.radial);
    s.axial = outcome(r.axial);
    return s;
  }
  const SolverConfig& config() const { return cfg_; }
  const Grid& grid() const { return grid_; }
  pcgpu_stepper* handle() { return h_; }

 private:
  static double pulse_cb(void* u, double t) {
    return pulse_value(t, static_cast<const AdiStepper*>(u)->timing_);
  }
  static double tau_cb(void* u, double t) {
    const AdiStepper* s = static_cast<const AdiStepper*>(u);
    return initial_tau(t, s->timing_, s->cfg_);
  }
  static pcgpu_table table(const PropertyTable& t) {
    return pcgpu_table{static_cast<int32_t>(t.size()), t.empty() ? nullptr : t.knots().data(),
                       t.empty() ? nullptr : t.values().data()};
  }
  static HalfStepOutcome outcome(const pcgpu_outcome& o) {
    HalfStepOutcome r;
    r.converged = o.converged != 0;
    r.iterations = o.iterations;
    r.last_delta = o.last_delta;
    return r;
  }
  [[noreturn]] void raise(int rc, const char* msg) const {
    const std::string m = msg ? msg : "";
    switch (rc) {
      case PCGPU_ERR_CONFIG: throw ConfigError(m);
      case PCGPU_ERR_TAU_FLOOR: {  // TauFloorError(tau, floor, t) as solver.cpp:371 throws it
        double tau = 0, floor = 0, t = 0;
        if (h_) pcgpu_last_tau_floor(h_, &tau, &floor, &t);
        throw TauFloorError(tau, floor, t);
      }
      case PCGPU_ERR_TABLE_RANGE:
        throw LineError(h_ ? pcgpu_error_line(h_) : -1, "TableRangeError: " + m);
      case PCGPU_ERR_ZERO_PIVOT:
        throw LineError(h_ ? pcgpu_error_line(h_) : -1, m);
      default: throw Error("pcgpu: " + m);
    }
  }
  void check(int rc) const {
    if (rc != PCGPU_OK) raise(rc, pcgpu_last_error(h_));
  }

  const Grid& grid_;
  LayerMaterials mats_;
  SourceModel& source_;
  SourceSpec timing_;
  SolverConfig cfg_;
  std::vector<int32_t> layer_;
  std::vector<double> r_center_, gap_r_, width_z_, gap_z_;
  std::vector<pcgpu_material> mat_;
  pcgpu_stepper* h_ = nullptr;
};

/// pulsecell::evolve (runner.cpp:97-190) for the GPU stepper, with the same
/// arguments and EvolutionResult: the field stays on the device for the whole
/// run (pcgpu_evolve_host); only probe values cross each step and snapshots
/// when they occur. The probe cells are the reference's own probe_cell, and
/// the regime detection is the reference's own RegimeDetector.
inline EvolutionResult evolve(AdiStepper& stepper, const SourceSpec& timing, Array2 initial,
                              Real t_end, const RunnerConfig& cfg) {
  cfg.validate();
  const Grid& grid = stepper.grid();
  std::vector<int32_t> pi, pj;
  for (const auto& p : cfg.probes) {
    const auto c = probe_cell(grid, p.r, p.z);
    pi.push_back(static_cast<int32_t>(c.first));
    pj.push_back(static_cast<int32_t>(c.second));
  }
  pcgpu_runner_cfg c{};
  c.t_end = t_end;
  c.n_probes = static_cast<int32_t>(pi.size());
  c.probe_i = pi.data();
  c.probe_j = pj.data();
  c.n_snapshot_times = static_cast<int32_t>(cfg.snapshot_times.size());
  c.snapshot_times = cfg.snapshot_times.data();
  c.snapshot_pre_on = cfg.snapshot_pre_on;
  c.snapshot_post_off = cfg.snapshot_post_off;
  c.detector_samples_per_period = cfg.detector.samples_per_period;
  c.detector_min_periods = cfg.detector.min_periods;
  c.detector_tolerance = cfg.detector.tolerance;
  c.source_on = timing.I0 > 0;
  // the reference's own RegimeDetector (runner.cpp:35-95) over probe 0
  RegimeDetector detector(timing.t_per, cfg.detector);
  c.detect = [](void* u, int32_t seed, double t, double v) -> int32_t {
    RegimeDetector* d = static_cast<RegimeDetector*>(u);
    if (seed) {
      d->seed(t, v);
      return 0;
    }
    return d->update(t, v) ? 1 : 0;
  };
  c.detect_user = &detector;
  EvolutionResult res;
  res.field = std::move(initial);
  struct Sink {
    EvolutionResult* r;
    const Grid* g;
    size_t np;
  } sink{&res, &grid, pi.size()};
  auto on_step = [](void* u, int64_t, double t, double tau, const double* v) {
    Sink* s = static_cast<Sink*>(u);
    TraceEntry e;
    e.t = t;
    e.tau = tau;
    e.values.assign(v, v + s->np);
    s->r->trace.push_back(std::move(e));
  };
  auto on_snap = [](void* u, int32_t kind, double t, const double* f) {
    Sink* s = static_cast<Sink*>(u);
    Array2 a(s->g->nr(), s->g->nz());
    std::memcpy(a.data(), f, sizeof(double) * a.size());
    Snapshot snap{t, std::move(a)};
    if (kind == PCGPU_SNAP_PRE_ON) s->r->pre_on = std::move(snap);
    else if (kind == PCGPU_SNAP_POST_OFF) s->r->post_off = std::move(snap);
    else s->r->at_times.push_back(std::move(snap));
  };
  pcgpu_evolve_result out{};
  const int rc = pcgpu_evolve_host(stepper.handle(), res.field.data(), &c, on_step, on_snap,
                                   &sink, &out);
  if (rc != PCGPU_OK) throw Error(std::string("pcgpu_evolve: ") + pcgpu_last_error(stepper.handle()));
  res.t = out.t;
  res.steps = out.steps;
  res.reason = static_cast<StopReason>(out.reason);
  res.fire_t = out.fire_t;
  if (res.reason == StopReason::TauFloor) res.error = pcgpu_last_error(stepper.handle());
  if (c.source_on && !pi.empty()) res.detector_periods = detector.resampler().periods();
  return res;
}

}  // namespace gpu
}  // namespace pulsecell
