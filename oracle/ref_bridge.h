/* ref_bridge.h -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * C entry points over the reference's own, unmodified pulsecell library
 * (compiled from /root/reference/proj/src by oracle/Makefile into
 * oracle/_ref/libpcref.so). Used by tests/ and bench.py's cpu_baseline /
 * --impl reference leg only. Spec-level inputs: the bridge builds the
 * reference's DomainSpec / GridSpec / MaterialSet / Grid / SourceModel /
 * SolverConfig / LinePool / AdiStepper itself, so the reference's own code
 * computes every metric.
 */
#ifndef PCREF_BRIDGE_H
#define PCREF_BRIDGE_H

#include "../include/pcgpu.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pcref_spec {
  /* DomainSpec (geometry.hpp:14-27) + GridSpec (:29-35) */
  int32_t n_layers;
  const double* layer_radii;         /* [n_layers] */
  const int32_t* radial_divisions;   /* [n_layers] */
  double core_length, outer_length;
  int32_t axial_divisions_core, axial_divisions_outer;
  int32_t source_layer;
  const pcgpu_material* materials;   /* [n_layers], layer order */
  /* SourceModel choice + SourceSpec (source.hpp:14-29) */
  int32_t source_kind;               /* pcgpu_source_kind */
  double t_per, t_src, t_trs, xi, zeta, I0, S_C; /* S_C <= 0: derived (config.cpp:207) */
  int32_t waveform, joule_dimensional;
  /* SolverConfig (solver.hpp:12-31) */
  double epsilon;
  int32_t max_iter;
  double tau_min, tau_transient_divisor, tau_source_divisor;
  int32_t halfpoint_rule, range_policy, all_neumann;
  double T0, t_ceiling;
  /* ExecPlan (parallel.hpp:18-27) */
  int32_t workers, chunking; /* chunking: 0 static-block, 1 static-interleave */
} pcref_spec;

typedef struct pcref pcref;

int pcref_create(const pcref_spec* spec, pcref** out);
void pcref_destroy(pcref* h);
const char* pcref_last_error(const pcref* h);
int64_t pcref_error_line(const pcref* h);

/* Grid accessors (geometry.hpp:55-100). Arrays sized nr, nr+1, nz, nz+1. */
void pcref_grid_dims(const pcref* h, int64_t* nr, int64_t* nz, int64_t* nr_core,
                     int64_t* nz_shared, int64_t* active_cells);
void pcref_grid_arrays(const pcref* h, double* r_center, double* width_r, double* gap_r,
                       double* z_center, double* width_z, double* gap_z, int32_t* layer);
double pcref_source_amplitude(const pcref* h);
double pcref_tau_floor(const pcref* h);

double pcref_initial_tau(const pcref* h, double t);
double pcref_pulse_value(const pcref* h, double t);

int pcref_bind_power_field(pcref* h, const double* power); /* PCGPU_SOURCE_FIELD, host nr*nz */
int pcref_radial_half_step(pcref* h, const double* T_cur, double t, double tau, double* out,
                           pcgpu_outcome* outcome);
int pcref_axial_half_step(pcref* h, const double* T_half, double t, double tau, double* out,
                          pcgpu_outcome* outcome);
int pcref_step(pcref* h, double* field, double t, pcgpu_step_result* result);
int pcref_run(pcref* h, double* field, double t0, int32_t nsteps, pcgpu_step_result* results,
              pcgpu_run_stats* stats);
int pcref_clamp_events(const pcref* h, uint64_t* counts);
/* The BASELINE growth policy over the reference's own radial_half_step /
 * axial_half_step (same controller as pcgpu_run_growth / oracle_run_growth). */
int pcref_run_growth(pcref* h, double* field, double t0, double t_end, int32_t max_steps,
                     double tau_start, double grow, int32_t easy_steps, double tau_max,
                     pcgpu_step_result* results, pcgpu_run_stats* stats);

/* pulsecell::evolve (runner.cpp:97-190) on the reference stepper, with
 * probes at (r, z). field: initial in, final out. Trace arrays hold
 * trace_cap entries (values: trace_cap x n_probes); snapshot fields nr*nz. */
typedef struct pcref_evolve_io {
  double t_end;
  int32_t n_probes;
  const double* probe_r;
  const double* probe_z;
  int32_t n_snapshot_times;
  const double* snapshot_times;
  int32_t snapshot_pre_on, snapshot_post_off;
  int32_t detector_samples_per_period, detector_min_periods;
  double detector_tolerance;
  double I0; /* SourceSpec::I0 (the detector engages only when > 0) */
  /* outputs */
  double t, fire_t;
  int64_t steps;
  int32_t reason;
  int64_t trace_cap;
  double *trace_t, *trace_tau, *trace_values;
  int32_t has_pre_on, has_post_off;
  double pre_on_t, post_off_t;
  double *pre_on_field, *post_off_field;
  int32_t at_cap, at_count;
  double *at_t, *at_fields;
  int32_t det_cap, det_rows;
  double* det_values; /* det_cap x samples */
  int32_t probe_i[16], probe_j[16]; /* probe_cell of each probe (<= 16) */
} pcref_evolve_io;
int pcref_evolve(pcref* h, double* field, pcref_evolve_io* io);

/* snapshot_io.cpp (the reference's writers): format 0 CSV, 1 VTK structured.
 * Trace: n steps of (t, values[n_probes]); phase trace: rows x samples. */
int pcref_write_snapshot(pcref* h, const double* field, const char* path, int32_t format,
                         const char* header);
int pcref_write_trace(pcref* h, const double* t, const double* values, int64_t n,
                      int32_t n_probes, const char* path, const char* header);
int pcref_write_phase_trace(pcref* h, const double* rows, int32_t n_rows, int32_t samples,
                            double t_per, const char* path, const char* header);

/* Operators and diagnostics (solver.cpp:53-119). */
double pcref_apply_lambda_r(const pcref* h, const double* field, int64_t i, int64_t j);
double pcref_apply_lambda_z(const pcref* h, const double* field, int64_t i, int64_t j);
double pcref_weighted_heat_sum(const pcref* h, const double* field);

/* Property evaluation MaterialTable::eval (materials.hpp:78-82); prop 0 cv, 1 lambda, 2 chi.
 * Returns PCGPU_ERR_TABLE_RANGE in strict mode out of range. */
int pcref_eval(const pcref* h, int32_t layer, int32_t prop, double T, double* value);

/* thomas_solve_inplace (tridiagonal.hpp:25-42) over a batch, run through a
 * LinePool of `workers` threads (parallel.cpp:95-116). layout: pcgpu_layout. */
int pcref_thomas_batch(const double* lower, const double* diag, const double* upper,
                       const double* rhs, double* x, int64_t n, int64_t batch, int32_t layout,
                       int32_t workers, int64_t* failed_system);

#ifdef __cplusplus
}
#endif
#endif
