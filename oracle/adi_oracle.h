/* adi_oracle.h -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * Plain-C restatement of the reference ADI hot path
 * (pulsecell::AdiStepper, /root/reference/proj/src/solver.cpp:125-373, and
 * what it inlines). Takes the same pcgpu_desc as the CUDA library, so the
 * tests can run both on identical inputs. Pinned against the reference itself
 * (oracle/_ref/libpcref.so, built from the reference sources) bit-for-bit by
 * tests/test_oracle_pin.py, and against committed fixtures in tests/golden/.
 */
#ifndef ADI_ORACLE_H
#define ADI_ORACLE_H

#include "../include/pcgpu.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct oracle oracle;

int oracle_create(const pcgpu_desc* d, oracle** out);
void oracle_destroy(oracle* o);
const char* oracle_last_error(const oracle* o);
int64_t oracle_error_line(const oracle* o);
double oracle_initial_tau(const oracle* o, double t);
double oracle_pulse_value(const oracle* o, double t);
int oracle_bind_power_field(oracle* o, const double* power);
int oracle_radial_half_step(oracle* o, const double* T_cur, double t, double tau, double* out,
                            pcgpu_outcome* res);
int oracle_axial_half_step(oracle* o, const double* T_half, double t, double tau, double* out,
                           pcgpu_outcome* res);
int oracle_step(oracle* o, double* field, double t, pcgpu_step_result* res);
int oracle_run(oracle* o, double* field, double t0, int32_t nsteps, pcgpu_step_result* results,
               pcgpu_run_stats* stats);
int oracle_run_growth(oracle* o, double* field, double t0, double t_end, int32_t max_steps,
                      double tau_start, double grow, int32_t easy_steps, double tau_max,
                      pcgpu_step_result* results, pcgpu_run_stats* stats);
int oracle_clamp_events(const oracle* o, uint64_t* counts);
/* thomas_solve_inplace (tridiagonal.hpp:25-42); returns PCGPU_ERR_ZERO_PIVOT. */
int oracle_thomas(const double* lower, const double* diag, const double* upper,
                  const double* rhs, double* x, double* work, int64_t n);
int oracle_thomas_batch(const double* lower, const double* diag, const double* upper,
                        const double* rhs, double* x, int64_t n, int64_t batch, int32_t layout,
                        int64_t* failed_system);

#ifdef __cplusplus
}
#endif
#endif
