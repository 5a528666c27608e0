// ref_bridge.cpp -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
//
// Thin C wrapper over the reference's own pulsecell library, compiled
// unchanged from /root/reference/proj/src (see oracle/Makefile). Nothing here
// re-implements reference arithmetic: every number comes from the reference's
// Grid, MaterialTable, JouleSource, AdiStepper, thomas_solve_inplace and
// LinePool. Exceptions are mapped onto pcgpu_status codes.
#include "ref_bridge.h"

#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "pulsecell/errors.hpp"
#include "pulsecell/geometry.hpp"
#include "pulsecell/materials.hpp"
#include "pulsecell/parallel.hpp"
#include "pulsecell/runner.hpp"
#include "pulsecell/snapshot_io.hpp"
#include "pulsecell/solver.hpp"
#include "pulsecell/source.hpp"
#include "pulsecell/tridiagonal.hpp"

using namespace pulsecell;

namespace {

// T-independent per-cell power bound by the host (the acceptance suite's
// ManufacturedSource pattern, acceptance_main.cpp:262-274).
class ArraySource final : public SourceModel {
 public:
  ArraySource(Index nr, Index nz) : p_(static_cast<size_t>(nr * nz), 0.0), nr_(nr) {}
  void bind_time(Real) override {}
  Real power(Index i, Index j, int, Real) const override { return p_[j * nr_ + i]; }
  void set(const double* p) { std::memcpy(p_.data(), p, p_.size() * sizeof(double)); }

 private:
  std::vector<double> p_;
  Index nr_;
};

PropertyTable make_table(const pcgpu_table& t) {
  if (t.n <= 0) return PropertyTable();
  return PropertyTable(std::vector<Real>(t.t, t.t + t.n), std::vector<Real>(t.v, t.v + t.n));
}

int classify(const std::exception& e) {
  if (dynamic_cast<const TauFloorError*>(&e)) return PCGPU_ERR_TAU_FLOOR;
  if (dynamic_cast<const TableRangeError*>(&e)) return PCGPU_ERR_TABLE_RANGE;
  if (dynamic_cast<const ConfigError*>(&e)) return PCGPU_ERR_CONFIG;
  const std::string w = e.what();
  if (w.find("zero pivot") != std::string::npos) return PCGPU_ERR_ZERO_PIVOT;
  if (w.find("outside table range") != std::string::npos ||
      w.find("property table missing") != std::string::npos)
    return PCGPU_ERR_TABLE_RANGE;
  return PCGPU_ERR_CONFIG;
}

thread_local std::string g_create_error;

}  // namespace

struct pcref {
  DomainSpec domain;
  GridSpec gridspec;
  MaterialSet materials;
  std::unique_ptr<Grid> grid;
  LayerMaterials layers;
  SourceSpec timing;
  std::unique_ptr<SourceModel> source;
  ArraySource* array_source = nullptr;
  SolverConfig cfg;
  std::unique_ptr<LinePool> pool;
  std::unique_ptr<AdiStepper> stepper;
  std::string error;
  int64_t error_line = -1;

  int fail(const std::exception& e) {
    error = e.what();
    error_line = -1;
    if (auto* le = dynamic_cast<const LineError*>(&e)) error_line = le->line();
    return classify(e);
  }
};

extern "C" {

int pcref_create(const pcref_spec* s, pcref** out) {
  *out = nullptr;
  auto h = std::make_unique<pcref>();
  try {
    for (int m = 0; m < s->n_layers; ++m) {
      h->domain.layer_radii.push_back(s->layer_radii[m]);
      h->domain.layer_materials.push_back("layer" + std::to_string(m));
      h->gridspec.radial_divisions.push_back(s->radial_divisions[m]);
    }
    h->domain.core_length = s->core_length;
    h->domain.outer_length = s->outer_length;
    h->domain.source_layer = s->source_layer;
    h->gridspec.axial_divisions_core = s->axial_divisions_core;
    h->gridspec.axial_divisions_outer = s->axial_divisions_outer;
    h->grid = std::make_unique<Grid>(h->domain, h->gridspec);
    for (int m = 0; m < s->n_layers; ++m) {
      const pcgpu_material& pm = s->materials[m];
      h->materials.add(MaterialTable(h->domain.layer_materials[m], pm.rho, make_table(pm.cv),
                                     make_table(pm.lambda), make_table(pm.chi)));
    }
    h->layers = resolve_layers(h->materials, h->domain.layer_materials);

    h->timing.t_per = s->t_per;
    h->timing.t_src = s->t_src;
    h->timing.t_trs = s->t_trs;
    h->timing.xi = s->xi;
    h->timing.zeta = s->zeta;
    h->timing.I0 = s->I0;
    h->timing.S_C = s->S_C;
    h->timing.waveform = s->waveform == PCGPU_WAVE_RECTANGULAR ? Waveform::Rectangular
                                                               : Waveform::Transient;
    h->timing.joule_dimensional = s->joule_dimensional != 0;
    if (h->timing.S_C <= 0) h->timing.S_C = h->domain.source_cross_section();  // config.cpp:207

    h->cfg.epsilon = s->epsilon;
    h->cfg.max_iter = s->max_iter;
    h->cfg.tau_min = s->tau_min;
    h->cfg.tau_transient_divisor = s->tau_transient_divisor;
    h->cfg.tau_source_divisor = s->tau_source_divisor;
    h->cfg.halfpoint_rule = static_cast<HalfPointRule>(s->halfpoint_rule);
    h->cfg.range_policy = static_cast<RangePolicy>(s->range_policy);
    h->cfg.all_neumann = s->all_neumann != 0;
    h->cfg.T0 = s->T0;
    h->cfg.t_ceiling = s->t_ceiling;

    if (s->source_kind == PCGPU_SOURCE_JOULE) {
      h->source = std::make_unique<JouleSource>(h->timing, s->source_layer,
                                                *h->layers[s->source_layer], h->cfg.range_policy);
    } else if (s->source_kind == PCGPU_SOURCE_FIELD) {
      auto a = std::make_unique<ArraySource>(h->grid->nr(), h->grid->nz());
      h->array_source = a.get();
      h->source = std::move(a);
    } else {
      h->source = std::make_unique<NullSource>();
    }
    ExecPlan plan;
    plan.workers = s->workers < 1 ? 1 : s->workers;
    plan.chunking = s->chunking == 1 ? Chunking::StaticInterleave : Chunking::StaticBlock;
    h->pool = std::make_unique<LinePool>(plan);
    h->stepper = std::make_unique<AdiStepper>(*h->grid, h->layers, *h->source, h->timing,
                                              h->cfg, *h->pool);
  } catch (const std::exception& e) {
    g_create_error = e.what();
    return classify(e);
  }
  *out = h.release();
  return PCGPU_OK;
}

void pcref_destroy(pcref* h) { delete h; }

const char* pcref_last_error(const pcref* h) {
  return h ? h->error.c_str() : g_create_error.c_str();
}

int64_t pcref_error_line(const pcref* h) { return h->error_line; }

void pcref_grid_dims(const pcref* h, int64_t* nr, int64_t* nz, int64_t* nr_core,
                     int64_t* nz_shared, int64_t* active) {
  const Grid& g = *h->grid;
  *nr = g.nr();
  *nz = g.nz();
  *nr_core = g.nr_core();
  *nz_shared = g.nz_shared();
  *active = g.active_cells();
}

void pcref_grid_arrays(const pcref* h, double* r_center, double* width_r, double* gap_r,
                       double* z_center, double* width_z, double* gap_z, int32_t* layer) {
  const Grid& g = *h->grid;
  for (Index i = 0; i < g.nr(); ++i) {
    r_center[i] = g.r_center(i);
    width_r[i] = g.width_r(i);
    layer[i] = g.layer(i);
  }
  for (Index i = 0; i <= g.nr(); ++i) gap_r[i] = g.gap_r(i);
  for (Index j = 0; j < g.nz(); ++j) {
    z_center[j] = g.z_center(j);
    width_z[j] = g.width_z(j);
  }
  for (Index j = 0; j <= g.nz(); ++j) gap_z[j] = g.gap_z(j);
}

double pcref_source_amplitude(const pcref* h) { return h->timing.current_factor(); }
double pcref_tau_floor(const pcref* h) { return h->cfg.effective_tau_min(h->timing.t_per); }
double pcref_initial_tau(const pcref* h, double t) { return initial_tau(t, h->timing, h->cfg); }
double pcref_pulse_value(const pcref* h, double t) { return pulse_value(t, h->timing); }

int pcref_bind_power_field(pcref* h, const double* power) {
  if (!h->array_source) return PCGPU_ERR_ARG;
  h->array_source->set(power);
  return PCGPU_OK;
}

static Array2 to_array(const pcref* h, const double* p) {
  Array2 a(h->grid->nr(), h->grid->nz());
  std::memcpy(a.data(), p, sizeof(double) * a.size());
  return a;
}

int pcref_radial_half_step(pcref* h, const double* T_cur, double t, double tau, double* out,
                           pcgpu_outcome* o) {
  try {
    const Array2 tc = to_array(h, T_cur);
    Array2 dst = to_array(h, out);
    const HalfStepOutcome r = h->stepper->radial_half_step(tc, t, tau, dst);
    std::memcpy(out, dst.data(), sizeof(double) * dst.size());
    o->converged = r.converged;
    o->iterations = r.iterations;
    o->last_delta = r.last_delta;
  } catch (const std::exception& e) {
    return h->fail(e);
  }
  return PCGPU_OK;
}

int pcref_axial_half_step(pcref* h, const double* T_half, double t, double tau, double* out,
                          pcgpu_outcome* o) {
  try {
    const Array2 th = to_array(h, T_half);
    Array2 dst = to_array(h, out);
    const HalfStepOutcome r = h->stepper->axial_half_step(th, t, tau, dst);
    std::memcpy(out, dst.data(), sizeof(double) * dst.size());
    o->converged = r.converged;
    o->iterations = r.iterations;
    o->last_delta = r.last_delta;
  } catch (const std::exception& e) {
    return h->fail(e);
  }
  return PCGPU_OK;
}

static void copy_result(const StepResult& r, pcgpu_step_result* o) {
  o->tau_used = r.tau_used;
  o->halvings = r.halvings;
  o->radial.converged = r.radial.converged;
  o->radial.iterations = r.radial.iterations;
  o->radial.last_delta = r.radial.last_delta;
  o->axial.converged = r.axial.converged;
  o->axial.iterations = r.axial.iterations;
  o->axial.last_delta = r.axial.last_delta;
}

int pcref_step(pcref* h, double* field, double t, pcgpu_step_result* result) {
  try {
    Array2 f = to_array(h, field);
    const StepResult r = h->stepper->step(f, t);
    std::memcpy(field, f.data(), sizeof(double) * f.size());
    copy_result(r, result);
  } catch (const std::exception& e) {
    return h->fail(e);
  }
  return PCGPU_OK;
}

// nsteps x step() with t += tau_used, exactly the bench harness loop
// (bench.cpp:20-22). Stats count the accepted attempt's iterations (step()
// reports only those, solver.hpp:56-60).
int pcref_evolve(pcref* h, double* field, pcref_evolve_io* io) {
  try {
    RunnerConfig rc;
    rc.t_end = io->t_end;
    rc.detector.samples_per_period = io->detector_samples_per_period;
    rc.detector.min_periods = io->detector_min_periods;
    rc.detector.tolerance = io->detector_tolerance;
    for (int32_t k = 0; k < io->n_probes; ++k) {
      rc.probes.push_back(ProbeSpec{io->probe_r[k], io->probe_z[k]});
      const auto c = probe_cell(*h->grid, io->probe_r[k], io->probe_z[k]);
      if (k < 16) {
        io->probe_i[k] = static_cast<int32_t>(c.first);
        io->probe_j[k] = static_cast<int32_t>(c.second);
      }
    }
    rc.snapshot_times.assign(io->snapshot_times, io->snapshot_times + io->n_snapshot_times);
    rc.snapshot_pre_on = io->snapshot_pre_on != 0;
    rc.snapshot_post_off = io->snapshot_post_off != 0;
    SourceSpec timing = h->timing;
    timing.I0 = io->I0;
    EvolutionResult r = evolve(*h->stepper, timing, to_array(h, field), io->t_end, rc);
    std::memcpy(field, r.field.data(), sizeof(double) * r.field.size());
    io->t = r.t;
    io->steps = r.steps;
    io->reason = static_cast<int32_t>(r.reason);
    io->fire_t = r.fire_t;
    const size_t cells = static_cast<size_t>(r.field.size());
    for (size_t k = 0; k < r.trace.size() && static_cast<int64_t>(k) < io->trace_cap; ++k) {
      io->trace_t[k] = r.trace[k].t;
      io->trace_tau[k] = r.trace[k].tau;
      for (int32_t p = 0; p < io->n_probes; ++p)
        io->trace_values[k * io->n_probes + p] = r.trace[k].values[p];
    }
    io->has_pre_on = r.pre_on.has_value();
    if (r.pre_on) {
      io->pre_on_t = r.pre_on->t;
      if (io->pre_on_field) std::memcpy(io->pre_on_field, r.pre_on->field.data(), sizeof(double) * cells);
    }
    io->has_post_off = r.post_off.has_value();
    if (r.post_off) {
      io->post_off_t = r.post_off->t;
      if (io->post_off_field)
        std::memcpy(io->post_off_field, r.post_off->field.data(), sizeof(double) * cells);
    }
    io->at_count = static_cast<int32_t>(r.at_times.size());
    for (int32_t k = 0; k < io->at_count && k < io->at_cap; ++k) {
      io->at_t[k] = r.at_times[k].t;
      std::memcpy(io->at_fields + k * cells, r.at_times[k].field.data(), sizeof(double) * cells);
    }
    io->det_rows = static_cast<int32_t>(r.detector_periods.size());
    for (int32_t k = 0; k < io->det_rows && k < io->det_cap; ++k)
      for (int32_t q = 0; q < io->detector_samples_per_period; ++q)
        io->det_values[k * io->detector_samples_per_period + q] = r.detector_periods[k][q];
    if (r.reason == StopReason::TauFloor) h->error = r.error;
  } catch (const std::exception& e) {
    return h->fail(e);
  }
  return PCGPU_OK;
}

int pcref_write_snapshot(pcref* h, const double* field, const char* path, int32_t format,
                         const char* header) {
  try {
    write_snapshot(*h->grid, to_array(h, field), path,
                   format == 0 ? SnapshotFormat::Csv : SnapshotFormat::VtkStructured, header);
  } catch (const std::exception& e) {
    return h->fail(e);
  }
  return PCGPU_OK;
}

int pcref_write_trace(pcref* h, const double* t, const double* values, int64_t n,
                      int32_t n_probes, const char* path, const char* header) {
  try {
    std::vector<TraceEntry> tr(static_cast<size_t>(n));
    for (int64_t k = 0; k < n; ++k) {
      tr[k].t = t[k];
      tr[k].values.assign(values + k * n_probes, values + (k + 1) * n_probes);
    }
    write_trace(tr, static_cast<size_t>(n_probes), path, header);
  } catch (const std::exception& e) {
    return h->fail(e);
  }
  return PCGPU_OK;
}

int pcref_write_phase_trace(pcref* h, const double* rows, int32_t n_rows, int32_t samples,
                            double t_per, const char* path, const char* header) {
  try {
    std::vector<Vector> p;
    for (int32_t r = 0; r < n_rows; ++r) {
      Vector v(samples);
      for (int32_t q = 0; q < samples; ++q) v[q] = rows[r * samples + q];
      p.push_back(v);
    }
    write_phase_trace(p, t_per, path, header);
  } catch (const std::exception& e) {
    return h->fail(e);
  }
  return PCGPU_OK;
}

int pcref_run(pcref* h, double* field, double t0, int32_t nsteps, pcgpu_step_result* results,
              pcgpu_run_stats* stats) {
  pcgpu_run_stats st{};
  const Grid& g = *h->grid;
  double t = t0;
  try {
    Array2 f = to_array(h, field);
    for (int32_t k = 0; k < nsteps; ++k) {
      const StepResult r = h->stepper->step(f, t);
      t += r.tau_used;
      if (results) copy_result(r, &results[k]);
      st.steps += 1;
      st.halvings += r.halvings;
      st.radial_iterations += r.radial.iterations;
      st.axial_iterations += r.axial.iterations;
      const double cells = static_cast<double>(g.active_cells());
      st.cell_updates_accepted += cells * (r.radial.iterations + r.axial.iterations);
      st.attempt_cells += 2.0 * cells;
    }
    std::memcpy(field, f.data(), sizeof(double) * f.size());
  } catch (const std::exception& e) {
    st.t_end = t;
    st.cell_updates = st.cell_updates_accepted;
    if (stats) *stats = st;
    return h->fail(e);
  }
  st.t_end = t;
  st.cell_updates = st.cell_updates_accepted;
  if (stats) *stats = st;
  return PCGPU_OK;
}

int pcref_clamp_events(const pcref* h, uint64_t* counts) {
  for (size_t m = 0; m < h->layers.size(); ++m) counts[m] = h->layers[m]->clamp_events();
  return PCGPU_OK;
}

double pcref_apply_lambda_r(const pcref* h, const double* field, int64_t i, int64_t j) {
  return apply_lambda_r(*h->grid, h->layers, to_array(h, field), i, j, h->cfg);
}
double pcref_apply_lambda_z(const pcref* h, const double* field, int64_t i, int64_t j) {
  return apply_lambda_z(*h->grid, h->layers, to_array(h, field), i, j, h->cfg);
}
double pcref_weighted_heat_sum(const pcref* h, const double* field) {
  return weighted_heat_sum(*h->grid, h->layers, to_array(h, field));
}

int pcref_eval(const pcref* h, int32_t layer, int32_t prop, double T, double* value) {
  try {
    *value = h->layers[layer]->eval(static_cast<Property>(prop), T, h->cfg.range_policy);
  } catch (const std::exception& e) {
    return classify(e);
  }
  return PCGPU_OK;
}

int pcref_thomas_batch(const double* lower, const double* diag, const double* upper,
                       const double* rhs, double* x, int64_t n, int64_t batch, int32_t layout,
                       int32_t workers, int64_t* failed_system) {
  *failed_system = -1;
  try {
    ExecPlan plan;
    plan.workers = workers < 1 ? 1 : workers;
    LinePool pool(plan);
    pool.for_lines(batch, [&](Index s) {
      thread_local std::vector<double> a, b, c, d, xx, w;
      if (layout == PCGPU_LAYOUT_CONTIGUOUS) {
        w.resize(static_cast<size_t>(n));
        const size_t off = static_cast<size_t>(s) * static_cast<size_t>(n);
        thomas_solve_inplace(lower + off, diag + off, upper + off, rhs + off, x + off,
                             w.data(), n);
      } else {
        // Strided layout: gather the line, solve, scatter (the reference's
        // axial_line pattern, solver.cpp:293-299,325-330).
        a.resize(n); b.resize(n); c.resize(n); d.resize(n); xx.resize(n); w.resize(n);
        for (Index k = 0; k < n; ++k) {
          const size_t idx = static_cast<size_t>(k) * static_cast<size_t>(batch) + s;
          a[k] = lower[idx]; b[k] = diag[idx]; c[k] = upper[idx]; d[k] = rhs[idx];
        }
        thomas_solve_inplace(a.data(), b.data(), c.data(), d.data(), xx.data(), w.data(), n);
        for (Index k = 0; k < n; ++k)
          x[static_cast<size_t>(k) * static_cast<size_t>(batch) + s] = xx[k];
      }
    });
  } catch (const LineError& e) {
    *failed_system = e.line();
    return PCGPU_ERR_ZERO_PIVOT;
  } catch (const std::exception& e) {
    return classify(e);
  }
  return PCGPU_OK;
}

// The BASELINE growth policy (pcgpu_run_growth) driven through the
// reference's own public half-step API (solver.hpp:70-78), the way the
// reference's acceptance suite drives half-steps (acceptance_main.cpp:311-332,
// MmsRun::march): each step tries radial then axial at the controller's tau,
// halves on non-convergence and throws TauFloorError below the floor like
// AdiStepper::step (solver.cpp:356-373); accepted steps swap the field. The
// controller itself (grow x`grow` after `easy_steps` steps without halving,
// cap tau_max) is the policy shared with the GPU and the C restatement.
int pcref_run_growth(pcref* h, double* field, double t0, double t_end, int32_t max_steps,
                     double tau_start, double grow, int32_t easy_steps, double tau_max,
                     pcgpu_step_result* results, pcgpu_run_stats* stats) {
  pcgpu_run_stats st{};
  const Grid& g = *h->grid;
  const double cells = static_cast<double>(g.active_cells());
  const double floor = h->cfg.effective_tau_min(h->timing.t_per);
  double t = t0, tau_next = tau_start < tau_max ? tau_start : tau_max;
  int easy = 0;
  int rc = PCGPU_OK;
  try {
    Array2 f = to_array(h, field);
    Array2 half = make_field(g, h->cfg.T0), next = make_field(g, h->cfg.T0);
    for (int32_t k = 0; k < max_steps && t < t_end; ++k) {
      pcgpu_step_result r{};
      double tau = tau_next;
      for (;;) {
        const HalfStepOutcome rad = h->stepper->radial_half_step(f, t, tau, half);
        st.cell_updates += cells * rad.iterations;
        r.radial = pcgpu_outcome{rad.converged ? 1 : 0, rad.iterations, rad.last_delta};
        r.axial = pcgpu_outcome{};
        if (rad.converged) {
          const HalfStepOutcome ax = h->stepper->axial_half_step(half, t, tau, next);
          st.cell_updates += cells * ax.iterations;
          r.axial = pcgpu_outcome{ax.converged ? 1 : 0, ax.iterations, ax.last_delta};
          if (ax.converged) break;
        }
        tau *= 0.5;
        ++r.halvings;
        if (tau < floor) throw TauFloorError(tau, floor, t);
      }
      f.swap(next);
      r.tau_used = tau;
      t += tau;
      if (results) results[k] = r;
      st.steps += 1;
      st.halvings += r.halvings;
      st.radial_iterations += r.radial.iterations;
      st.axial_iterations += r.axial.iterations;
      st.cell_updates_accepted += cells * (r.radial.iterations + r.axial.iterations);
      st.attempt_cells += 2.0 * cells * (r.halvings + 1);
      easy = r.halvings == 0 ? easy + 1 : 0;
      tau_next = tau;
      if (easy >= easy_steps) {
        tau_next = tau * grow < tau_max ? tau * grow : tau_max;
        easy = 0;
      }
    }
    std::memcpy(field, f.data(), sizeof(double) * f.size());
  } catch (const std::exception& e) {
    rc = h->fail(e);
  }
  st.t_end = t;
  if (stats) *stats = st;
  return rc;
}

}  // extern "C"
