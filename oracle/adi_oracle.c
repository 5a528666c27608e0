/* adi_oracle.c -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * Plain-C restatement of the reference's ADI step (pulsecell::AdiStepper).
 * Each function cites the reference file:line it restates. Arithmetic follows
 * the reference expression trees operation for operation,
 * compiled with -ffp-contract=off, so results are bit-identical to the
 * reference built with its own Release flags -- which tests/test_oracle_pin.py
 * checks against oracle/_ref/libpcref.so (the reference compiled from its
 * sources). Single-threaded: the reference output is bitwise independent of
 * its worker count (solver.hpp:62-65).
 */
#include "adi_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  int n;
  double* t;
  double* v;
} otable;

typedef struct {
  double rho;
  otable prop[3]; /* 0 cv, 1 lambda, 2 chi -- Property order, materials.hpp:12 */
} omaterial;

enum { P_CV = 0, P_LAMBDA = 1, P_CHI = 2 };

struct oracle {
  pcgpu_desc d; /* scalars; array pointers below are owned copies */
  int nr, nz, nr_core, nz_shared;
  int *row_ext, *col_ext; /* masked extents (generalised stepped domain) */
  int* layer;
  double *r_center, *gap_r, *width_z, *gap_z;
  omaterial* mats;
  double tau_floor;
  /* stepper state, solver.hpp:98-101 */
  double *half, *next, *iter_buf, *expl, *kbar, *line_delta;
  double *inv_vol_r, *inv_eta, *inv_gap_r, *inv_gap_z;
  double* power_field; /* PCGPU_SOURCE_FIELD */
  double pulse;        /* JouleSource::pulse_ after bind_time */
  uint64_t* clamp;     /* per layer */
  /* line scratch (solver.cpp:11-27) */
  double *a, *b, *c, *dd, *x, *w, *fcoef, *tt, *k0, *r0;
  char err[256];
  int64_t err_line;
  int line_status; /* first error inside the current line sweep */
};

static double* dup_d(const double* p, size_t n) {
  double* q = (double*)malloc(sizeof(double) * (n ? n : 1));
  if (n) memcpy(q, p, sizeof(double) * n);
  return q;
}

/* ---- materials.hpp:39-46 PropertyTable::operator() ---------------------- */
static double table_value(const otable* tb, double T) {
  if (T <= tb->t[0]) return tb->v[0];
  if (T >= tb->t[tb->n - 1]) return tb->v[tb->n - 1];
  int k = 1;
  while (tb->t[k] < T) ++k;
  const double w = (T - tb->t[k - 1]) / (tb->t[k] - tb->t[k - 1]);
  return tb->v[k - 1] + w * (tb->v[k] - tb->v[k - 1]);
}

/* ---- materials.hpp:78-82 MaterialTable::eval + materials.cpp:60-69 ------- */
static double mat_eval(oracle* o, int layer, int prop, double T, int64_t line) {
  const otable* tb = &o->mats[layer].prop[prop];
  const int in_range = tb->n > 0 && T >= tb->t[0] && T <= tb->t[tb->n - 1];
  if (!in_range) {
    if (tb->n == 0 || o->d.range_policy == PCGPU_RANGE_STRICT) {
      if (!o->line_status || line < o->err_line) {
        o->line_status = PCGPU_ERR_TABLE_RANGE;
        o->err_line = line;
        snprintf(o->err, sizeof o->err, "line %lld failed: T=%g outside table range",
                 (long long)line, T);
      }
      return 0.0; /* line result discarded: the sweep reports the error */
    }
    o->clamp[layer] += 1;
  }
  return table_value(tb, T);
}

/* ---- materials.hpp:101-124 face_lambda (own = lower-index side) --------- */
static double face_lambda(oracle* o, int own, int other, double Ta, double Tb, int64_t line) {
  switch (o->d.halfpoint_rule) {
    case PCGPU_HALFPOINT_MEAN_LAMBDA:
      return 0.5 * (mat_eval(o, own, P_LAMBDA, Ta, line) + mat_eval(o, own, P_LAMBDA, Tb, line));
    case PCGPU_HALFPOINT_TWO_SIDED_HARMONIC: {
      const double la = mat_eval(o, own, P_LAMBDA, Ta, line);
      const double lb = mat_eval(o, other, P_LAMBDA, Tb, line);
      return 2.0 * la * lb / (la + lb);
    }
    default:
      return mat_eval(o, own, P_LAMBDA, 0.5 * (Ta + Tb), line);
  }
}

/* ---- source.hpp:68-72 JouleSource::power / NullSource / field source ----- */
static double source_power(oracle* o, int i, int j, int layer, double T, int64_t line) {
  switch (o->d.source_kind) {
    case PCGPU_SOURCE_JOULE:
      if (layer != o->d.source_layer || o->pulse == 0.0) return 0.0;
      return mat_eval(o, o->d.source_layer, P_CHI, T, line) * o->d.amplitude * o->pulse;
    case PCGPU_SOURCE_FIELD:
      return o->power_field[(size_t)j * o->nr + i];
    default:
      return 0.0;
  }
}

/* ---- source.cpp:18-45 pulse_rect / pulse_transient / pulse_value --------- */
static double pulse_value(const pcgpu_desc* d, double t) {
  const double phase = fmod(t, d->t_per);
  if (d->waveform == PCGPU_WAVE_RECTANGULAR) return phase < d->t_src ? 1.0 : 0.0;
  const double margin = d->t_trs / d->zeta * (1.0 + 6.5 / d->xi);
  const long elapsed = (long)llround((t - phase) / d->t_per);
  long back_hi = 1 + (long)ceil((d->t_src + margin) / d->t_per);
  if (elapsed < back_hi) back_hi = elapsed;
  const double scale = d->xi * d->zeta / d->t_trs;
  double sum = 0.0;
  for (long m = -1; m <= back_hi; ++m) {
    const double u = phase + (double)m * d->t_per;
    sum += erf(scale * u - d->xi) - erf(scale * (u - d->t_src) - d->xi);
  }
  return 0.5 * sum;
}

static void bind_time(oracle* o, double t) { o->pulse = pulse_value(&o->d, t); }

/* ---- solver.cpp:44-51 initial_tau --------------------------------------- */
double oracle_initial_tau(const oracle* o, double t) {
  const pcgpu_desc* d = &o->d;
  const double phase = fmod(t, d->t_per);
  const int in_transient =
      phase <= d->t_trs || (phase >= d->t_src && phase <= d->t_src + d->t_trs);
  return in_transient ? d->t_trs / d->tau_transient_divisor : d->t_src / d->tau_source_divisor;
}

double oracle_pulse_value(const oracle* o, double t) { return pulse_value(&o->d, t); }

/* ---- tridiagonal.hpp:25-42 thomas_solve_inplace ------------------------- */
int oracle_thomas(const double* lower, const double* diag, const double* upper,
                  const double* rhs, double* x, double* work, int64_t n) {
  double piv = diag[0];
  if (piv == 0.0) return PCGPU_ERR_ZERO_PIVOT;
  double inv = 1.0 / piv;
  work[0] = upper[0] * inv;
  x[0] = rhs[0] * inv;
  for (int64_t k = 1; k < n; ++k) {
    piv = diag[k] - lower[k] * work[k - 1];
    if (piv == 0.0) return PCGPU_ERR_ZERO_PIVOT;
    inv = 1.0 / piv;
    work[k] = upper[k] * inv;
    x[k] = (rhs[k] - lower[k] * x[k - 1]) * inv;
  }
  for (int64_t k = n - 2; k >= 0; --k) x[k] -= work[k] * x[k + 1];
  return PCGPU_OK;
}

int oracle_thomas_batch(const double* lower, const double* diag, const double* upper,
                        const double* rhs, double* x, int64_t n, int64_t batch, int32_t layout,
                        int64_t* failed_system) {
  double* buf = (double*)malloc(sizeof(double) * 6 * (size_t)n);
  double *a = buf, *b = buf + n, *c = buf + 2 * n, *d = buf + 3 * n, *xx = buf + 4 * n,
         *w = buf + 5 * n;
  int status = PCGPU_OK;
  *failed_system = -1;
  for (int64_t s = 0; s < batch; ++s) {
    int rc;
    if (layout == PCGPU_LAYOUT_CONTIGUOUS) {
      const size_t off = (size_t)s * (size_t)n;
      rc = oracle_thomas(lower + off, diag + off, upper + off, rhs + off, x + off, w, n);
    } else {
      for (int64_t k = 0; k < n; ++k) {
        const size_t idx = (size_t)k * (size_t)batch + (size_t)s;
        a[k] = lower[idx];
        b[k] = diag[idx];
        c[k] = upper[idx];
        d[k] = rhs[idx];
      }
      rc = oracle_thomas(a, b, c, d, xx, w, n);
      if (rc == PCGPU_OK)
        for (int64_t k = 0; k < n; ++k) x[(size_t)k * (size_t)batch + (size_t)s] = xx[k];
    }
    if (rc != PCGPU_OK && status == PCGPU_OK) {
      status = rc;
      *failed_system = s;
    }
  }
  free(buf);
  return status;
}

/* ---- solver.cpp:33-42 SolverConfig::validate, source.cpp:9-17, ctor ----- */
int oracle_create(const pcgpu_desc* d, oracle** out) {
  *out = NULL;
  if (d->abi_version != PCGPU_ABI_VERSION) return PCGPU_ERR_ARG;
  if (!(d->epsilon > 0) || d->max_iter < 1 || !(d->tau_transient_divisor > 0) ||
      !(d->tau_source_divisor > 0) || !(d->T0 > 0) || !(d->t_ceiling > d->T0))
    return PCGPU_ERR_CONFIG;
  if (!(d->t_per > 0) || !(d->t_src > 0 && d->t_src <= d->t_per) ||
      !(d->t_trs > 0 && d->t_trs < d->t_src) || !(d->xi > 0) || !(d->zeta > 0))
    return PCGPU_ERR_CONFIG;
  if (d->n_layers < 1 || !d->materials || d->nr < 1 || d->nz < 1) return PCGPU_ERR_CONFIG;

  oracle* o = (oracle*)calloc(1, sizeof(oracle));
  o->d = *d;
  o->nr = d->nr;
  o->nz = d->nz;
  o->nr_core = d->nr_core;
  o->nz_shared = d->nz_shared;
  const int nr = o->nr, nz = o->nz;
  /* The reference's two-level Grid (geometry.hpp:72-74), or the explicit
   * extents of a generalised stepped domain (beyond the reference). */
  o->row_ext = (int*)malloc(sizeof(int) * nz);
  o->col_ext = (int*)malloc(sizeof(int) * nr);
  for (int j = 0; j < nz; ++j)
    o->row_ext[j] = d->row_extent ? d->row_extent[j] : (j < d->nz_shared ? nr : d->nr_core);
  for (int i = 0; i < nr; ++i)
    o->col_ext[i] = d->col_extent ? d->col_extent[i] : (i < d->nr_core ? nz : d->nz_shared);
  o->d.row_extent = o->d.col_extent = NULL;
  o->layer = (int*)malloc(sizeof(int) * nr);
  for (int i = 0; i < nr; ++i) o->layer[i] = d->layer[i];
  o->r_center = dup_d(d->r_center, nr);
  o->gap_r = dup_d(d->gap_r, nr + 1);
  o->width_z = dup_d(d->width_z, nz);
  o->gap_z = dup_d(d->gap_z, nz + 1);
  o->mats = (omaterial*)calloc(d->n_layers, sizeof(omaterial));
  for (int m = 0; m < d->n_layers; ++m) {
    const pcgpu_table* src[3] = {&d->materials[m].cv, &d->materials[m].lambda,
                                 &d->materials[m].chi};
    o->mats[m].rho = d->materials[m].rho;
    for (int p = 0; p < 3; ++p) {
      o->mats[m].prop[p].n = src[p]->n;
      o->mats[m].prop[p].t = dup_d(src[p]->t, src[p]->n);
      o->mats[m].prop[p].v = dup_d(src[p]->v, src[p]->n);
    }
  }
  o->clamp = (uint64_t*)calloc(d->n_layers, sizeof(uint64_t));
  o->tau_floor = d->tau_min > 0 ? d->tau_min : 1e-12 * d->t_per; /* solver.hpp:28-30 */
  const size_t cells = (size_t)nr * nz;
  o->half = (double*)malloc(sizeof(double) * cells);
  o->next = (double*)malloc(sizeof(double) * cells);
  o->iter_buf = (double*)malloc(sizeof(double) * cells);
  for (size_t k = 0; k < cells; ++k) o->half[k] = o->next[k] = o->iter_buf[k] = d->T0;
  o->expl = (double*)calloc(cells, sizeof(double));
  o->kbar = (double*)calloc(cells, sizeof(double));
  o->power_field = (double*)calloc(cells, sizeof(double));
  const int nmax = nr > nz ? nr : nz;
  o->line_delta = (double*)calloc(nmax, sizeof(double));
  /* solver.cpp:146-159 metric reciprocals */
  o->inv_vol_r = (double*)malloc(sizeof(double) * nr);
  o->inv_gap_r = (double*)malloc(sizeof(double) * (nr + 1));
  for (int i = 0; i < nr; ++i) {
    const double control_r = 0.5 * (o->gap_r[i] + o->gap_r[i + 1]); /* geometry.hpp:87 */
    o->inv_vol_r[i] = 1.0 / (o->r_center[i] * control_r);
    o->inv_gap_r[i] = 1.0 / o->gap_r[i];
  }
  o->inv_gap_r[nr] = 1.0 / o->gap_r[nr];
  o->inv_eta = (double*)malloc(sizeof(double) * nz);
  o->inv_gap_z = (double*)malloc(sizeof(double) * (nz + 1));
  for (int j = 0; j < nz; ++j) {
    o->inv_eta[j] = 1.0 / (0.5 * (o->gap_z[j] + o->gap_z[j + 1]));
    o->inv_gap_z[j] = 1.0 / o->gap_z[j];
  }
  o->inv_gap_z[nz] = 1.0 / o->gap_z[nz];
  double** scr[] = {&o->a, &o->b, &o->c, &o->dd, &o->x, &o->w, &o->tt, &o->k0, &o->r0};
  for (size_t s = 0; s < sizeof scr / sizeof scr[0]; ++s)
    *scr[s] = (double*)calloc(nmax + 1, sizeof(double));
  o->fcoef = (double*)calloc(nmax + 2, sizeof(double));
  o->err_line = -1;
  *out = o;
  return PCGPU_OK;
}

void oracle_destroy(oracle* o) {
  if (!o) return;
  free(o->row_ext); free(o->col_ext);
  free(o->layer); free(o->r_center); free(o->gap_r); free(o->width_z); free(o->gap_z);
  for (int m = 0; m < o->d.n_layers; ++m)
    for (int p = 0; p < 3; ++p) { free(o->mats[m].prop[p].t); free(o->mats[m].prop[p].v); }
  free(o->mats); free(o->clamp);
  free(o->half); free(o->next); free(o->iter_buf); free(o->expl); free(o->kbar);
  free(o->power_field); free(o->line_delta);
  free(o->inv_vol_r); free(o->inv_gap_r); free(o->inv_eta); free(o->inv_gap_z);
  free(o->a); free(o->b); free(o->c); free(o->dd); free(o->x); free(o->w); free(o->tt);
  free(o->k0); free(o->r0); free(o->fcoef);
  free(o);
}

const char* oracle_last_error(const oracle* o) { return o->err; }
int64_t oracle_error_line(const oracle* o) { return o->err_line; }

int oracle_bind_power_field(oracle* o, const double* p) {
  memcpy(o->power_field, p, sizeof(double) * (size_t)o->nr * o->nz);
  return PCGPU_OK;
}

int oracle_clamp_events(const oracle* o, uint64_t* counts) {
  for (int m = 0; m < o->d.n_layers; ++m) counts[m] = o->clamp[m];
  return PCGPU_OK;
}

static int row_extent(const oracle* o, int j) { return o->row_ext[j]; }
static int col_extent(const oracle* o, int i) { return o->col_ext[i]; }
/* geometry.hpp:92-94 */
static double face_r_lo(const oracle* o, int i) {
  return i == 0 ? 0.0 : 0.5 * (o->r_center[i - 1] + o->r_center[i]);
}

static void thomas_line(oracle* o, int n, int64_t line) {
  if (oracle_thomas(o->a, o->b, o->c, o->dd, o->x, o->w, n) != PCGPU_OK) {
    if (!o->line_status || line < o->err_line) {
      o->line_status = PCGPU_ERR_ZERO_PIVOT;
      o->err_line = line;
      snprintf(o->err, sizeof o->err, "line %lld failed: thomas_solve: zero pivot",
               (long long)line);
    }
  }
}

/* ---- solver.cpp:162-189 explicit_axial_pass: out = Lambda_z[src] -------- */
static void explicit_axial_pass(oracle* o, const double* src, double* out) {
  const int nr = o->nr;
  for (int i = 0; i < nr; ++i) {
    const int m = col_extent(o, i);
    const int L = o->layer[i];
    const int dirichlet_top = L == 0 && !o->d.all_neumann;
    double* t = o->tt;
    for (int j = 0; j < m; ++j) t[j] = src[(size_t)j * nr + i];
    double flux_lo = 0;
    for (int j = 0; j < m; ++j) {
      double flux_hi;
      if (j < m - 1) {
        const double coef = face_lambda(o, L, L, t[j], t[j + 1], i) / o->gap_z[j + 1];
        flux_hi = coef * (t[j + 1] - t[j]);
      } else if (dirichlet_top) {
        const double lam = mat_eval(o, L, P_LAMBDA, o->d.T0, i);
        flux_hi = lam * (o->d.T0 - t[j]) / (0.5 * o->width_z[j]);
      } else {
        flux_hi = 0;
      }
      const double control_z = 0.5 * (o->gap_z[j] + o->gap_z[j + 1]);
      out[(size_t)j * nr + i] = (flux_hi - flux_lo) / control_z;
      flux_lo = flux_hi;
    }
  }
}

/* ---- solver.cpp:191-233 radial_line (increment form around T_cur) ------- */
static void radial_line(oracle* o, int j, const double* T_iter, const double* T_cur,
                        double half_k, double* out) {
  const int nr = o->nr;
  const int n = row_extent(o, j);
  const double* Ts = T_iter + (size_t)j * nr;
  const double* Tc = T_cur + (size_t)j * nr;
  for (int f = 1; f < n; ++f) {
    o->fcoef[f] = face_r_lo(o, f) *
                  face_lambda(o, o->layer[f - 1], o->layer[f], Ts[f - 1], Ts[f], j) *
                  o->inv_gap_r[f];
    o->r0[f] = o->fcoef[f] * (Tc[f] - Tc[f - 1]);
  }
  for (int i = 0; i < n; ++i) {
    const int L = o->layer[i];
    const double inv_vol = o->inv_vol_r[i];
    const double A = i > 0 ? o->fcoef[i] * inv_vol : 0.0;
    const double C = i < n - 1 ? o->fcoef[i + 1] * inv_vol : 0.0;
    const double K = o->mats[L].rho * mat_eval(o, L, P_CV, Ts[i], j) * half_k;
    const double flux_lo = i > 0 ? o->r0[i] : 0.0;
    const double flux_hi = i < n - 1 ? o->r0[i + 1] : 0.0;
    o->a[i] = -A;
    o->b[i] = K + A + C;
    o->c[i] = -C;
    o->dd[i] = (flux_hi - flux_lo) * inv_vol + o->expl[(size_t)j * nr + i] +
               source_power(o, i, j, L, Ts[i], j);
  }
  thomas_line(o, n, j);
  double* op = out + (size_t)j * nr;
  double dmax = 0;
  for (int i = 0; i < n; ++i) {
    op[i] = Tc[i] + o->x[i];
    const double dv = fabs(op[i] - Ts[i]);
    dmax = dmax < dv ? dv : dmax; /* std::max(dmax, dv): NaN-ignoring */
  }
  o->line_delta[j] = dmax;
}

static double max_of(const double* v, int n) {
  double m = v[0];
  for (int k = 1; k < n; ++k)
    if (m < v[k]) m = v[k];
  return m;
}

/* ---- solver.cpp:235-257 radial_half_step -------------------------------- */
int oracle_radial_half_step(oracle* o, const double* T_cur, double t, double tau, double* out,
                            pcgpu_outcome* res) {
  const size_t bytes = sizeof(double) * (size_t)o->nr * o->nz;
  bind_time(o, t + 0.5 * tau);
  o->line_status = 0;
  o->err_line = -1;
  explicit_axial_pass(o, T_cur, o->expl);
  if (o->line_status) return o->line_status;
  const double half_k = 2.0 / tau;
  const double* src = T_cur;
  res->converged = 0;
  res->iterations = 0;
  res->last_delta = 0;
  for (int s = 1; s <= o->d.max_iter; ++s) {
    double* dst = (src == out) ? o->iter_buf : out;
    for (int j = 0; j < o->nz; ++j) radial_line(o, j, src, T_cur, half_k, dst);
    if (o->line_status) return o->line_status;
    res->iterations = s;
    res->last_delta = max_of(o->line_delta, o->nz);
    if (res->last_delta < o->d.epsilon) {
      if (dst != out) memcpy(out, dst, bytes);
      res->converged = 1;
      return PCGPU_OK;
    }
    src = dst;
  }
  return PCGPU_OK;
}

/* ---- solver.cpp:259-284 axial_fixed_rhs_pass ---------------------------- */
static void axial_fixed_rhs_pass(oracle* o, const double* T_half, double half_k) {
  const int nr = o->nr;
  for (int j = 0; j < o->nz; ++j) {
    const int n = row_extent(o, j);
    const double* Th = T_half + (size_t)j * nr;
    for (int f = 1; f < n; ++f)
      o->fcoef[f] = face_r_lo(o, f) *
                    face_lambda(o, o->layer[f - 1], o->layer[f], Th[f - 1], Th[f], j) *
                    o->inv_gap_r[f];
    double flux_lo = 0;
    for (int i = 0; i < n; ++i) {
      const int L = o->layer[i];
      const double flux_hi = i < n - 1 ? o->fcoef[i + 1] * (Th[i + 1] - Th[i]) : 0.0;
      const double lam_r = (flux_hi - flux_lo) * o->inv_vol_r[i];
      o->kbar[(size_t)j * nr + i] = o->mats[L].rho * mat_eval(o, L, P_CV, Th[i], j) * half_k;
      o->expl[(size_t)j * nr + i] = lam_r + source_power(o, i, j, L, Th[i], j);
      flux_lo = flux_hi;
    }
  }
}

/* ---- solver.cpp:286-332 axial_line -------------------------------------- */
static void axial_line(oracle* o, int i, const double* T_iter, const double* T_half,
                       double* out) {
  const int nr = o->nr;
  const int m = col_extent(o, i);
  const int L = o->layer[i];
  const int dirichlet_top = L == 0 && !o->d.all_neumann;
  for (int j = 0; j < m; ++j) {
    const size_t idx = (size_t)j * nr + i;
    o->tt[j] = T_iter[idx];
    o->r0[j] = T_half[idx];
    o->k0[j] = o->kbar[idx];
    o->dd[j] = o->expl[idx];
  }
  for (int f = 1; f < m; ++f)
    o->fcoef[f] = face_lambda(o, L, L, o->tt[f - 1], o->tt[f], i) * o->inv_gap_z[f];
  for (int j = 0; j < m; ++j) {
    const double inv_eta = o->inv_eta[j];
    const double A = j > 0 ? o->fcoef[j] * inv_eta : 0.0;
    const double C = j < m - 1 ? o->fcoef[j + 1] * inv_eta : 0.0;
    const double flux_lo = j > 0 ? o->fcoef[j] * (o->r0[j] - o->r0[j - 1]) : 0.0;
    double flux_hi = j < m - 1 ? o->fcoef[j + 1] * (o->r0[j + 1] - o->r0[j]) : 0.0;
    o->a[j] = -A;
    o->b[j] = o->k0[j] + A + C;
    o->c[j] = -C;
    if (j == m - 1 && dirichlet_top) {
      const double face = mat_eval(o, L, P_LAMBDA, o->d.T0, i) / (0.5 * o->width_z[j]);
      o->b[j] += face * inv_eta;
      flux_hi += face * (o->d.T0 - o->r0[j]);
    }
    o->dd[j] += (flux_hi - flux_lo) * inv_eta;
  }
  thomas_line(o, m, i);
  double dmax = 0;
  for (int j = 0; j < m; ++j) {
    const double v = o->r0[j] + o->x[j];
    const double dv = fabs(v - o->tt[j]);
    dmax = dmax < dv ? dv : dmax;
    out[(size_t)j * nr + i] = v;
  }
  o->line_delta[i] = dmax;
}

/* ---- solver.cpp:334-354 axial_half_step --------------------------------- */
int oracle_axial_half_step(oracle* o, const double* T_half, double t, double tau, double* out,
                           pcgpu_outcome* res) {
  const size_t bytes = sizeof(double) * (size_t)o->nr * o->nz;
  bind_time(o, t + 0.5 * tau);
  o->line_status = 0;
  o->err_line = -1;
  axial_fixed_rhs_pass(o, T_half, 2.0 / tau);
  if (o->line_status) return o->line_status;
  const double* src = T_half;
  res->converged = 0;
  res->iterations = 0;
  res->last_delta = 0;
  for (int s = 1; s <= o->d.max_iter; ++s) {
    double* dst = (src == out) ? o->iter_buf : out;
    for (int i = 0; i < o->nr; ++i) axial_line(o, i, src, T_half, dst);
    if (o->line_status) return o->line_status;
    res->iterations = s;
    res->last_delta = max_of(o->line_delta, o->nr);
    if (res->last_delta < o->d.epsilon) {
      if (dst != out) memcpy(out, dst, bytes);
      res->converged = 1;
      return PCGPU_OK;
    }
    src = dst;
  }
  return PCGPU_OK;
}

/* ---- solver.cpp:356-373 step: tau controller ---------------------------- */
static int step_tau(oracle* o, double* field, double t, double tau, pcgpu_step_result* res);

int oracle_step(oracle* o, double* field, double t, pcgpu_step_result* res) {
  return step_tau(o, field, t, oracle_initial_tau(o, t), res);
}

/* solver.cpp:356-373 with the first tau supplied by the caller. */
static int step_tau(oracle* o, double* field, double t, double tau, pcgpu_step_result* res) {
  const size_t bytes = sizeof(double) * (size_t)o->nr * o->nz;
  memset(res, 0, sizeof *res);
  for (;;) {
    int rc = oracle_radial_half_step(o, field, t, tau, o->half, &res->radial);
    if (rc) return rc;
    if (res->radial.converged) {
      rc = oracle_axial_half_step(o, o->half, t, tau, o->next, &res->axial);
      if (rc) return rc;
      if (res->axial.converged) {
        /* field.swap(next_): the caller's array receives next_'s contents and
         * next_ keeps the caller's previous buffer (solver.cpp:364). */
        double* tmp = (double*)malloc(bytes);
        memcpy(tmp, field, bytes);
        memcpy(field, o->next, bytes);
        memcpy(o->next, tmp, bytes);
        free(tmp);
        res->tau_used = tau;
        return PCGPU_OK;
      }
    }
    tau *= 0.5;
    ++res->halvings;
    if (tau < o->tau_floor) {
      snprintf(o->err, sizeof o->err, "time step %g fell below floor %g at t=%g", tau,
               o->tau_floor, t);
      return PCGPU_ERR_TAU_FLOOR;
    }
  }
}

int oracle_run(oracle* o, double* field, double t0, int32_t nsteps, pcgpu_step_result* results,
               pcgpu_run_stats* stats) {
  pcgpu_run_stats st;
  memset(&st, 0, sizeof st);
  double cells = 0;
  for (int i = 0; i < o->nr; ++i) cells += col_extent(o, i);
  double t = t0;
  int rc = PCGPU_OK;
  for (int32_t k = 0; k < nsteps; ++k) {
    pcgpu_step_result r;
    rc = oracle_step(o, field, t, &r);
    if (rc) break;
    t += r.tau_used;
    if (results) results[k] = r;
    st.steps += 1;
    st.halvings += r.halvings;
    st.radial_iterations += r.radial.iterations;
    st.axial_iterations += r.axial.iterations;
    st.cell_updates_accepted += cells * (r.radial.iterations + r.axial.iterations);
    st.attempt_cells += 2.0 * cells;
  }
  st.t_end = t;
  st.cell_updates = st.cell_updates_accepted;
  if (stats) *stats = st;
  return rc;
}

/* The BASELINE growth policy (see pcgpu_run_growth in include/pcgpu.h): the
 * same controller over the same step semantics, so the GPU and the oracle
 * take identical decisions on identical results. */
int oracle_run_growth(oracle* o, double* field, double t0, double t_end, int32_t max_steps,
                      double tau_start, double grow, int32_t easy_steps, double tau_max,
                      pcgpu_step_result* results, pcgpu_run_stats* stats) {
  pcgpu_run_stats st;
  memset(&st, 0, sizeof st);
  double cells = 0;
  for (int i = 0; i < o->nr; ++i) cells += col_extent(o, i);
  double t = t0, tau = tau_start < tau_max ? tau_start : tau_max;
  int easy = 0, rc = PCGPU_OK;
  for (int32_t k = 0; k < max_steps && t < t_end; ++k) {
    pcgpu_step_result r;
    rc = step_tau(o, field, t, tau, &r);
    if (rc) break;
    t += r.tau_used;
    if (results) results[k] = r;
    st.steps += 1;
    st.halvings += r.halvings;
    st.radial_iterations += r.radial.iterations;
    st.axial_iterations += r.axial.iterations;
    st.cell_updates_accepted += cells * (r.radial.iterations + r.axial.iterations);
    tau = r.tau_used;
    easy = r.halvings == 0 ? easy + 1 : 0;
    if (easy >= easy_steps) {
      tau = tau * grow < tau_max ? tau * grow : tau_max;
      easy = 0;
    }
  }
  st.t_end = t;
  st.cell_updates = st.cell_updates_accepted;
  if (stats) *stats = st;
  return rc;
}
