/* pcgpu.h -- C-ABI of the B200-native ADI hot path of pulsecell
 * (arXiv 1912.03744 reference, /root/reference/proj).
 *
 * This is the drop-in boundary for `class pulsecell::AdiStepper`
 * (proj/include/pulsecell/solver.hpp:66-106, proj/src/solver.cpp:125-373).
 * Plain pointers and sizes only; no C++ exceptions cross it. Every entry point
 * returns a pcgpu_status; the C++ wrapper (include/pulsecell_gpu/adi_stepper.hpp)
 * and the Python mirror (paper_1912_03744_b200/solver.py) map the codes back to
 * the reference exception types (errors.hpp:10-54).
 *
 * Fields are FP64, column-major nr x nz -- element (i, j) at j*nr + i -- the
 * reference's Array2 layout (types.hpp:10-14). Field pointers passed to the
 * half-step / step entry points are DEVICE pointers (cudaMalloc / torch);
 * the *_host variants take host pointers and copy.
 */
#ifndef PCGPU_H
#define PCGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PCGPU_ABI_VERSION 3

/* Status codes. Reference equivalents in brackets. */
enum pcgpu_status {
  PCGPU_OK = 0,
  PCGPU_ERR_CONFIG = 1,      /* ConfigError: SolverConfig::validate (solver.cpp:33-42),
                                stepper wiring (solver.cpp:133-138), SourceSpec (source.cpp:9-17) */
  PCGPU_ERR_TAU_FLOOR = 2,   /* TauFloorError (solver.cpp:369-371) */
  PCGPU_ERR_TABLE_RANGE = 3, /* TableRangeError in a line body (materials.cpp:60-69), re-thrown
                                as LineError(lowest line) (parallel.cpp:68-93,115) */
  PCGPU_ERR_ZERO_PIVOT = 4,  /* Error("thomas_solve: zero pivot") (tridiagonal.hpp:27,33) */
  PCGPU_ERR_CUDA = 5,        /* CUDA runtime failure (no reference equivalent) */
  PCGPU_ERR_ARG = 6          /* bad pointer / size at the boundary */
};

/* Enumerations mirror the reference's enum classes value-for-value. */
enum pcgpu_halfpoint_rule { /* materials.hpp:16-20 */
  PCGPU_HALFPOINT_MEAN_TEMPERATURE = 0,
  PCGPU_HALFPOINT_MEAN_LAMBDA = 1,
  PCGPU_HALFPOINT_TWO_SIDED_HARMONIC = 2
};
enum pcgpu_range_policy { PCGPU_RANGE_CLAMP = 0, PCGPU_RANGE_STRICT = 1 }; /* materials.hpp:14 */
enum pcgpu_waveform { PCGPU_WAVE_RECTANGULAR = 0, PCGPU_WAVE_TRANSIENT = 1 }; /* source.hpp:9 */
enum pcgpu_source_kind {
  PCGPU_SOURCE_NULL = 0,   /* NullSource (source.hpp:57-61) */
  PCGPU_SOURCE_JOULE = 1,  /* JouleSource (source.hpp:63-83) */
  PCGPU_SOURCE_FIELD = 2   /* T-independent per-cell power (e.g. the acceptance suite's
                              ManufacturedSource, acceptance_main.cpp:262-274): the host binds
                              an nr x nz power array per half-step (pcgpu_bind_power_field). */
};
enum pcgpu_mode {
  /* Bit-identical to the reference CPU path: the reference's operation order
   * (SURVEY Appendix A), no FMA contraction, sequential Thomas per line. The
   * only mode (the round-1 partitioned "fast" line solver is retired: off the
   * bit-exact path it cannot meet the 1e-9 fixed-dt bar on the stiff grids,
   * DESIGN.md section 4.2). */
  PCGPU_MODE_EXACT = 0
};

/* Piecewise-linear property table: n strictly increasing knots t[] and values v[]
 * (PropertyTable, materials.hpp:24-53). n == 0 means "absent" (an empty chi). */
typedef struct pcgpu_table {
  int32_t n;
  const double* t;
  const double* v;
} pcgpu_table;

/* MaterialTable (materials.hpp:57-95): constant rho and three tables. */
typedef struct pcgpu_material {
  double rho;
  pcgpu_table cv;     /* Property::HeatCapacity */
  pcgpu_table lambda; /* Property::Conductivity */
  pcgpu_table chi;    /* Property::Resistivity (may be empty) */
} pcgpu_material;

/* Everything the stepper needs, marshalled from the reference objects
 * (Grid, LayerMaterials, SourceModel, SourceSpec, SolverConfig). Arrays are
 * copied by pcgpu_create; the caller may free them afterwards. */
typedef struct pcgpu_desc {
  int32_t abi_version; /* must be PCGPU_ABI_VERSION */

  /* Grid (geometry.hpp:48-115), metrics exactly as Grid computes them. */
  int32_t nr, nz;          /* Grid::nr(), Grid::nz() */
  int32_t nr_core;         /* Grid::nr_core()   -- row_extent(j) = j < nz_shared ? nr : nr_core */
  int32_t nz_shared;       /* Grid::nz_shared() -- col_extent(i) = i < nr_core ? nz : nz_shared */
  const int32_t* layer;    /* [nr]   Grid::layer(i) */
  const double* r_center;  /* [nr]   Grid::r_center(i) */
  const double* gap_r;     /* [nr+1] Grid::gap_r(i) (mirror-ghost ends) */
  const double* width_z;   /* [nz]   Grid::width_z(j) */
  const double* gap_z;     /* [nz+1] Grid::gap_z(j) (mirror-ghost ends) */

  /* LayerMaterials: one material per layer (solver.cpp:135-138). */
  int32_t n_layers;
  const pcgpu_material* materials; /* [n_layers] */

  /* SourceModel. amplitude = SourceSpec::current_factor() (source.hpp:26-28). */
  int32_t source_kind;  /* pcgpu_source_kind */
  int32_t source_layer;
  double amplitude;

  /* SourceSpec timing (source.hpp:14-29), for initial_tau / pulse_value on the host. */
  double t_per, t_src, t_trs, xi, zeta;
  int32_t waveform; /* pcgpu_waveform */

  /* SolverConfig (solver.hpp:12-31). */
  double epsilon;
  int32_t max_iter;
  double tau_min; /* <= 0 means 1e-12 * t_per (effective_tau_min) */
  double tau_transient_divisor;
  double tau_source_divisor;
  int32_t halfpoint_rule; /* pcgpu_halfpoint_rule */
  int32_t range_policy;   /* pcgpu_range_policy */
  int32_t all_neumann;
  double T0;
  double t_ceiling;

  /* Device options (not part of the reference schema). */
  int32_t mode;   /* pcgpu_mode */
  int32_t device; /* CUDA device ordinal */

  /* Generalised stepped domain (beyond the reference's
   * two-level Grid): when both are non-NULL they give the masked extent of
   * every line -- non-increasing, consistent prefix masks (i < row_extent[j]
   * iff j < col_extent[i]). NULL: the reference's rule from nr_core /
   * nz_shared above. */
  const int32_t* row_extent; /* [nz] cells of radial line j */
  const int32_t* col_extent; /* [nr] cells of axial line i */
} pcgpu_desc;

/* HalfStepOutcome (solver.hpp:50-54). */
typedef struct pcgpu_outcome {
  int32_t converged;
  int32_t iterations;
  double last_delta;
} pcgpu_outcome;

/* StepResult (solver.hpp:56-60). */
typedef struct pcgpu_step_result {
  double tau_used;
  int32_t halvings;
  pcgpu_outcome radial, axial;
} pcgpu_step_result;

/* Counters accumulated over a pcgpu_run: every half-step attempt's active
 * cells x Picard iterations (SURVEY 8(d) "cell-update"), rejected attempts
 * included; and the same for accepted attempts only. */
typedef struct pcgpu_run_stats {
  double t_end;
  int64_t steps;
  int64_t halvings;
  int64_t radial_iterations;
  int64_t axial_iterations;
  double cell_updates;
  double cell_updates_accepted;
  double attempt_cells; /* sum over attempts of active cells (x2 half-steps) */
} pcgpu_run_stats;

typedef struct pcgpu_stepper pcgpu_stepper;

/* Library / device introspection. */
int32_t pcgpu_abi_version(void);
int pcgpu_device_count(int32_t* count);

/* AdiStepper(grid, mats, source, timing, cfg, pool) -- solver.cpp:125-160.
 * Validates like the reference and allocates the device buffers (the
 * reference's half_, next_, iter_buf_, expl_, kbar_). */
int pcgpu_create(const pcgpu_desc* desc, pcgpu_stepper** out);
void pcgpu_destroy(pcgpu_stepper* h);

/* Last error message for h (or for the last failed pcgpu_create when h is NULL). */
const char* pcgpu_last_error(const pcgpu_stepper* h);
/* Lowest failing line of the last PCGPU_ERR_TABLE_RANGE / PCGPU_ERR_ZERO_PIVOT
 * (LineError::line(), errors.hpp:46-54); -1 if none. */
int64_t pcgpu_error_line(const pcgpu_stepper* h);

/* Reference free function initial_tau(t, timing, cfg) (solver.cpp:44-51). */
double pcgpu_initial_tau(const pcgpu_stepper* h, double t);
/* Reference free function pulse_value(t, spec) (source.cpp:42-45). */
double pcgpu_pulse_value(const pcgpu_stepper* h, double t);
/* Active cells of the grid (Grid::active_cells, geometry.cpp:95). */
int64_t pcgpu_active_cells(const pcgpu_stepper* h);

/* The host functions behind the time stepping: pulse_value(t, spec)
 * (source.cpp:42-45) and initial_tau(t, timing, cfg) (solver.cpp:44-51). By
 * default the library uses its own restatements; a caller holding the
 * reference objects (the C++ drop-in) passes the reference's functions here so
 * that the stepper runs on exactly the reference's host arithmetic. Either
 * pointer may be NULL (keep the default). */
typedef double (*pcgpu_clock_fn)(void* user, double t);
int pcgpu_set_host_clock(pcgpu_stepper* h, pcgpu_clock_fn pulse_value, pcgpu_clock_fn initial_tau,
                         void* user);
/* After PCGPU_ERR_TAU_FLOOR: TauFloorError's tau(), floor() and time()
 * (errors.hpp, solver.cpp:371). */
int pcgpu_last_tau_floor(const pcgpu_stepper* h, double* tau, double* floor, double* t);

/* Resident stepper (whole steps -- tau controller, Picard loops with their
 * device max-norm tests, accept-or-halve -- in one cooperative launch per
 * batch of steps; used by pcgpu_step / pcgpu_run / pcgpu_run_growth /
 * pcgpu_evolve on grids of at most one 32-line block per SM and sweep;
 * $PCGPU_RESIDENT=0 disables it): grid size (0 = not used), batches launched,
 * steps they accepted, steps redone host-driven (> 8 halvings in one step). */
int pcgpu_resident_stats(const pcgpu_stepper* h, int32_t* grid, int64_t* batches, int64_t* steps,
                         int64_t* host_steps);
/* Host-driven runs (grids the resident stepper does not take, e.g. configs[3];
 * pcgpu_run / pcgpu_run_growth): batches of steps enqueued with the predicted
 * Picard counts and no host read inside a batch, verified by one read at its
 * end; a misprediction, halving or error undoes the batch (its input field is
 * never written; clamp counters restored) and replays it step by step
 * ($PCGPU_NO_SPECULATE=1: always step by step). Batches, steps they accepted,
 * batches undone. */
int pcgpu_speculation_stats(const pcgpu_stepper* h, int64_t* batches, int64_t* steps,
                            int64_t* rollbacks);

/* Per-cell power for PCGPU_SOURCE_FIELD: device pointer, nr x nz column-major,
 * read by the next half-step (the SourceModel::power(i, j, ...) values for the
 * half-step's bind_time). */
int pcgpu_bind_power_field(pcgpu_stepper* h, const double* power_dev);

/* AdiStepper::radial_half_step (solver.cpp:235-257). Device pointers; out != T_cur.
 * `out` holds the half-layer field when outcome->converged. */
int pcgpu_radial_half_step(pcgpu_stepper* h, const double* T_cur, double t, double tau,
                           double* out, pcgpu_outcome* outcome);
/* AdiStepper::axial_half_step (solver.cpp:334-354). Device pointers; out != T_half. */
int pcgpu_axial_half_step(pcgpu_stepper* h, const double* T_half, double t, double tau,
                          double* out, pcgpu_outcome* outcome);
/* AdiStepper::step (solver.cpp:356-373) on a device field, in place.
 * Returns PCGPU_ERR_TAU_FLOOR when halving passes the floor. */
int pcgpu_step(pcgpu_stepper* h, double* field, double t, pcgpu_step_result* result);
/* Host-memory variants (H2D copy, step, D2H copy). */
int pcgpu_step_host(pcgpu_stepper* h, double* field_host, double t, pcgpu_step_result* result);
/* pcgpu_step_host copies the field in as row blocks overlapped with K3 and the
 * first radial Picard iterations (exact mode, nz >= 2048 or
 * $PCGPU_PIPELINE_MIN_NZ; off with $PCGPU_NO_PIPELINE). Counts of the steps
 * that took that path and of those whose radial half-step had to be redone
 * on the ordinary path (iteration count not as predicted). */
int pcgpu_pipeline_stats(const pcgpu_stepper* h, int64_t* steps, int64_t* fallbacks);
int pcgpu_radial_half_step_host(pcgpu_stepper* h, const double* T_cur_host, double t,
                                double tau, double* out_host, pcgpu_outcome* outcome);
int pcgpu_axial_half_step_host(pcgpu_stepper* h, const double* T_half_host, double t,
                               double tau, double* out_host, pcgpu_outcome* outcome);

/* nsteps calls of step() with t += tau_used (the bench harness loop,
 * bench.cpp:20-22), keeping the field resident on the device between steps.
 * `field` is a device pointer (in/out). Per-step results are written to
 * `results` when non-NULL ([nsteps]). */
int pcgpu_run(pcgpu_stepper* h, double* field, double t0, int32_t nsteps,
              pcgpu_step_result* results, pcgpu_run_stats* stats);

/* The BASELINE adaptive policy (configs[2]/[4]) above step(): start at
 * tau_start, halve on non-convergence exactly like step() (solver.cpp:369-371),
 * grow by `grow` after `easy_steps` consecutive steps accepted without
 * halving, never above tau_max; stop at t_end or after max_steps. Not in the
 * reference (halving only); the CPU oracle implements the same
 * policy (oracle_run_growth) so both paths take identical decisions. */
int pcgpu_run_growth(pcgpu_stepper* h, double* field, double t0, double t_end, int32_t max_steps,
                     double tau_start, double grow, int32_t easy_steps, double tau_max,
                     pcgpu_step_result* results, pcgpu_run_stats* stats);

/* MaterialTable::clamp_events() per layer (materials.hpp:85, materials.cpp:68).
 * counts has n_layers entries. Counted per out-of-range evaluation on the device. */
int pcgpu_clamp_events(const pcgpu_stepper* h, uint64_t* counts);

/* Stream the stepper launches on (a cudaStream_t as void*), for CUDA-event timing. */
void* pcgpu_stream(const pcgpu_stepper* h);

/* Time spent in the dominant kernel: the last run's accumulated device time
 * (CUDA events around each launch of the Picard line kernels) and launch count. */
int pcgpu_kernel_timing(const pcgpu_stepper* h, double* radial_ms, int64_t* radial_launches,
                        double* axial_ms, int64_t* axial_launches);
int pcgpu_enable_kernel_timing(pcgpu_stepper* h, int32_t on);
/* Number of this library's kernels launched since creation. */
int64_t pcgpu_launch_count(const pcgpu_stepper* h);
/* The kernel variants this stepper selected, as text (e.g.
 * "mode=exact lines=ws lookups=exact-x"), into buf (NUL-terminated, at most
 * len bytes). Returns the full length. */
int32_t pcgpu_describe(const pcgpu_stepper* h, char* buf, int32_t len);

/* ---- Device-resident runner -------------------------------
 * pulsecell::evolve (runner.cpp:97-190) with the field resident on the
 * device: steps from t = 0 (Kahan-accumulated time) until t_end, the
 * periodic-regime detector fires, or the step hits its floor. Per step only
 * the probe values come back (a device gather); snapshots are handed to the
 * caller as device pointers valid during the callback; the pre-turn-on
 * capture copies the field on the device only for steps that can cross a
 * period boundary. The regime detector (PhaseResampler / RegimeDetector,
 * runner.cpp:35-95) runs on the host over probe 0. Probe cells are the
 * caller's pulsecell::probe_cell(grid, r, z) (runner.cpp:20-28). */
typedef struct pcgpu_runner_cfg {
  double t_end;
  int32_t n_probes;
  const int32_t* probe_i; /* radial cell of each probe */
  const int32_t* probe_j; /* axial cell of each probe */
  int32_t n_snapshot_times;
  const double* snapshot_times; /* any order (sorted by the runner) */
  int32_t snapshot_pre_on;
  int32_t snapshot_post_off;
  int32_t detector_samples_per_period;
  int32_t detector_min_periods;
  double detector_tolerance;
  int32_t source_on; /* SourceSpec::I0 > 0: regime detection engages with >= 1 probe */
  /* The regime detector: NULL = the library's restatement of
   * PhaseResampler / RegimeDetector (runner.cpp:35-95); otherwise the
   * caller's (the C++ drop-in passes the reference's own RegimeDetector),
   * called with seed = 1 once at t = 0 (RegimeDetector::seed), then with
   * seed = 0 after every accepted step (RegimeDetector::update), returning
   * nonzero when the periodic criterion fires. pcgpu_detector_periods then
   * reports nothing (the caller's detector holds the periods). */
  int32_t (*detect)(void* user, int32_t seed, double t, double v);
  void* detect_user;
} pcgpu_runner_cfg;

typedef enum { PCGPU_STOP_REACHED_TIME = 0, PCGPU_STOP_PERIODIC = 1, PCGPU_STOP_TAU_FLOOR = 2 } pcgpu_stop;
typedef enum { PCGPU_SNAP_PRE_ON = 0, PCGPU_SNAP_POST_OFF = 1, PCGPU_SNAP_AT_TIME = 2 } pcgpu_snap;

/* Called after every accepted step with the step count, t, tau_used and the
 * n_probes probe values (TraceEntry, runner.hpp:29-33). */
typedef void (*pcgpu_step_cb)(void* user, int64_t step, double t, double tau,
                              const double* probe_values);
/* Snapshot (runner.hpp:106-109): field_dev is an nr x nz column-major device
 * field valid until the callback returns. */
typedef void (*pcgpu_snapshot_cb)(void* user, int32_t kind, double t, const double* field_dev);

typedef struct pcgpu_evolve_result {
  double t;
  int64_t steps;
  int32_t reason; /* pcgpu_stop */
  double fire_t;  /* -1 unless the detector fired */
  int32_t detector_periods; /* completed resampled periods of probe 0 */
} pcgpu_evolve_result;

/* field_dev is the initial field in, the final field out (the last accepted
 * one on a TauFloor stop; pcgpu_last_error() holds the reason). Returns
 * PCGPU_OK for all three stop reasons. */
int pcgpu_evolve(pcgpu_stepper* h, double* field_dev, const pcgpu_runner_cfg* cfg,
                 pcgpu_step_cb on_step, pcgpu_snapshot_cb on_snapshot, void* user,
                 pcgpu_evolve_result* result);
/* Host-field variant (for callers without CUDA, e.g. the C++ drop-in's
 * evolve): the field is copied in and out, and snapshots are handed over as
 * host nr x nz column-major fields valid during the callback. */
int pcgpu_evolve_host(pcgpu_stepper* h, double* field_host, const pcgpu_runner_cfg* cfg,
                      pcgpu_step_cb on_step, pcgpu_snapshot_cb on_snapshot, void* user,
                      pcgpu_evolve_result* result);
/* The last evolve's resampled periods of probe 0 (detector_periods rows of
 * detector_samples_per_period values), into rows (capacity max_rows). */
int pcgpu_detector_periods(const pcgpu_stepper* h, double* rows, int32_t max_rows);

/* ---- Asynchronous snapshot writer --------------------------
 * write_snapshot (snapshot_io.cpp:26-60) off the critical path: submitting a
 * device field enqueues a device-to-device copy into one of `slots` slots on
 * `stream` (stream-ordered after the kernels that produced it), a copy to
 * pinned host memory on the writer's copy stream, and the formatting and
 * file write on a writer thread. Formats: 0 CSV (masked cells, z-major,
 * "%.17g"), 1 VTK legacy structured grid -- the reference's bytes. Submit
 * blocks only while every slot is in flight. z_center: the grid's nz axial
 * cell centres (Grid::z_center). */
typedef struct pcgpu_writer pcgpu_writer;
int pcgpu_writer_create(const pcgpu_desc* desc, const double* z_center, int32_t slots,
                        pcgpu_writer** out);
void pcgpu_writer_destroy(pcgpu_writer* w); /* finishes pending writes */
int pcgpu_writer_submit(pcgpu_writer* w, const double* field_dev, void* stream,
                        const char* path, int32_t format, const char* header);
/* Waits for every submitted snapshot; written = files completed so far. */
int pcgpu_writer_flush(pcgpu_writer* w, int64_t* written);
const char* pcgpu_writer_last_error(const pcgpu_writer* w);

/* ---- Partitioned stepper: one node of B200s ------------------
 * z-slabs (radial lines j) for the radial sweep, r-slabs (axial lines i) for
 * the axial sweep, all-to-all transposes between them, allreduce(max) of the
 * Picard norm every iteration, bit-identical to the single-GPU stepper. With
 * nccl_id == NULL the library emulates
 * `nranks` ranks in this process on desc->device (test/validation mode);
 * otherwise this process is rank `rank` of an NCCL communicator created from
 * the 128-byte id produced by pcgpu_nccl_unique_id on one rank and shared by
 * the caller (e.g. torch.distributed broadcast). No reference equivalent: the
 * reference is shared-memory only. */
typedef struct pcgpu_dist pcgpu_dist;
int pcgpu_nccl_unique_id(void* id128);
int pcgpu_dist_create(const pcgpu_desc* desc, int32_t rank, int32_t nranks, const void* nccl_id,
                      pcgpu_dist** out);
void pcgpu_dist_destroy(pcgpu_dist* h);
const char* pcgpu_dist_last_error(const pcgpu_dist* h);
/* Slab boundaries for nranks ranks (host only): zb/rb have nranks+1 entries;
 * rank p owns radial lines j in [zb[p], zb[p+1]) and axial lines i in
 * [rb[p], rb[p+1]). Balanced by active cells. */
int pcgpu_dist_plan(const pcgpu_desc* desc, int32_t nranks, int32_t* zb, int32_t* rb);
int pcgpu_dist_slabs(const pcgpu_dist* h, int32_t* z0, int32_t* z1, int32_t* r0, int32_t* r1);
/* Every rank passes the full initial field (device, nr x nz column-major). */
int pcgpu_dist_set_field(pcgpu_dist* h, const double* field_dev);
/* Writes this process's lines -- the r-slab columns (axial lines) -- into the
 * full-size device field. */
int pcgpu_dist_get_field(pcgpu_dist* h, double* field_dev);
/* Exact mode, host fields (nr x nz column-major, ideally pinned): copy only
 * this process's state lines -- the r-slab columns (axial lines) -- in from /
 * out to the full-size host field, so that each rank moves 1/nranks of the
 * field over its own PCIe link. set_field_host also refreshes the z-slab copy
 * (NCCL transpose) when the peer transport is off. */
int pcgpu_dist_set_field_host(pcgpu_dist* h, const double* field_host);
int pcgpu_dist_get_field_host(pcgpu_dist* h, double* field_host);
/* Exact mode transport: 1 = peer stores from the fused slab passes (the
 * default for emulated ranks; after pcgpu_dist_ipc_import for processes),
 * 0 = NCCL all-to-all transposes. */
int32_t pcgpu_dist_transport(const pcgpu_dist* h);
/* Peer transport across processes (exact mode, one process per GPU): each
 * rank exports PCGPU_DIST_IPC_BYTES of CUDA IPC handles for its slabs, the
 * caller all-gathers them (rank order) and every rank imports the
 * nranks * PCGPU_DIST_IPC_BYTES block; the fused K3/K4 passes then store into
 * the peers' slabs over NVLink, ordered by an NCCL barrier. */
#define PCGPU_DIST_IPC_BYTES 256
int pcgpu_dist_ipc_export(pcgpu_dist* h, void* handles);
int pcgpu_dist_ipc_import(pcgpu_dist* h, const void* all_handles);
/* Close the imported peer mappings and return to the NCCL transport. The
 * transport must be the same on every rank: when any rank's import failed,
 * every rank calls this (the Python mirror agrees on it with an all-gather). */
int pcgpu_dist_peer_off(pcgpu_dist* h);
/* nsteps x step() with t += tau_used on the partitioned state. */
int pcgpu_dist_run(pcgpu_dist* h, double t0, int32_t nsteps, pcgpu_step_result* results,
                   pcgpu_run_stats* stats);
void* pcgpu_dist_stream(const pcgpu_dist* h);
/* Kernels launched by this library in this process so far. */
int64_t pcgpu_dist_launch_count(const pcgpu_dist* h);
int pcgpu_dist_enable_timing(pcgpu_dist* h, int32_t on);
/* Accumulated all-to-all transpose time (pack + exchange + unpack), counts,
 * and Picard line-kernel time, since timing was enabled. */
int pcgpu_dist_timing(const pcgpu_dist* h, double* transpose_ms, int64_t* transposes,
                      int64_t* allreduces, double* radial_ms, double* axial_ms);

/* ---- Batched tridiagonal systems (BASELINE configs[1]) ----------
 * thomas_solve_inplace (tridiagonal.hpp:25-42) applied to `batch` independent
 * systems of size n, all device pointers. Layouts:
 *   PCGPU_LAYOUT_CONTIGUOUS: system s, row k at s*n + k   (line-contiguous)
 *   PCGPU_LAYOUT_STRIDED:    system s, row k at k*batch + s (interleaved / transposed)
 * lower[k=0] and upper[k=n-1] are ignored like the reference. x may alias rhs.
 * `exact` = 1: the reference's operation order, bit-identical per system;
 * 0: the fastest variant (currently the same kernels). Contiguous layout only,
 * for comparison: 2 = the legacy warp-tiled kernel, 3 = the transpose path
 * (32x32 transposes around the strided kernel); otherwise the fused TMA kernel
 * when n is even and the bands are 16-B aligned. Returns PCGPU_ERR_ZERO_PIVOT
 * (error_line = lowest failing system) on a zero pivot. */
enum pcgpu_layout { PCGPU_LAYOUT_CONTIGUOUS = 0, PCGPU_LAYOUT_STRIDED = 1 };
int pcgpu_tridiag_batch(const double* lower, const double* diag, const double* upper,
                        const double* rhs, double* x, int64_t n, int64_t batch,
                        int32_t layout, int32_t exact, void* stream, int64_t* failed_system);

#ifdef __cplusplus
}
#endif

#endif /* PCGPU_H */
