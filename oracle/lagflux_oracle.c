/*
 * lagflux_oracle.c -- CPU restatement of the reference Lagrange-flux step.
 * TEST INFRASTRUCTURE ONLY (see lagflux_oracle.h).  Compiled with
 * -O2 -ffp-contract=off so every expression rounds exactly as the shipped
 * reference build does (no FMA, SSE2 scalar).
 *
 * Every function names the reference file:line it restates.  Parenthesised
 * expressions keep the C++ left-to-right evaluation order of the reference.
 */
#include "lagflux_oracle.h"

#include <float.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

struct lfo_solver {
  lfo_grid g;
  lfo_scheme s;
  int64_t cells;           /* nxt*nyt */
  double* prim[2][4];      /* solver.hpp:125 prim_ */
  double* fx[2][4];        /* FluxSet::x   (nx+1)*ny  (flux1_, flux2_) */
  double* fy[2][4];        /* FluxSet::y   nx*(ny+1) */
  double* ustar_x[2];
  double* ustar_y[2];
  double* pred[4];         /* predictor_ */
  /* multimaterial (solver.hpp:126-130): NULL / 0 without a material set */
  int n_mat;
  double mat_gamma[LFO_MAX_MATERIALS];
  double* gamma_cells[2];                 /* gamma_[slot] */
  double* frac[2][LFO_MAX_MATERIALS];     /* frac_[slot][k] */
  double* pred_mat[LFO_MAX_MATERIALS];    /* predictor_mat_ */
};

static int nxt_of(const lfo_grid* g) { return g->nx + 2 * g->gx; }
static int nyt_of(const lfo_grid* g) { return g->ny + 2 * g->gy; }
static int64_t idx_of(const lfo_grid* g, int i, int j) { return (int64_t)j * nxt_of(g) + i; }

/* std::to_string(double) is "%f" (libstdc++). */
static void fmt_f(char* buf, size_t n, double v) { snprintf(buf, n, "%f", v); }

static void set_err(lfo_error* e, int kind) {
  if (!e) return;
  memset(e, 0, sizeof *e);
  e->kind = kind;
  e->i = e->j = e->step = -1;
}

/* grid.cpp:23-56 */
int lfo_make_grid_1d(int nx, double x_min, double x_max, lfo_grid* g) {
  if (nx < 1 || !(x_max > x_min)) return LFO_ERR_CONFIG;
  memset(g, 0, sizeof *g);
  g->dim = 1; g->nx = nx; g->ny = 1;
  g->dx = (x_max - x_min) / nx; g->dy = 1.0;
  g->x0 = x_min; g->y0 = 0.0; g->gx = 2; g->gy = 0;
  return 0;
}

int lfo_make_grid_2d(int nx, int ny, double x_min, double x_max, double y_min, double y_max,
                     lfo_grid* g) {
  if (nx < 1 || ny < 1 || !(x_max > x_min) || !(y_max > y_min)) return LFO_ERR_CONFIG;
  memset(g, 0, sizeof *g);
  g->dim = 2; g->nx = nx; g->ny = ny;
  g->dx = (x_max - x_min) / nx; g->dy = (y_max - y_min) / ny;
  g->x0 = x_min; g->y0 = y_min; g->gx = 2; g->gy = 2;
  return 0;
}

/* grid.cpp:72-114: x sides over interior rows first, then y sides over every
 * column so the corners pick up the fresh x ghosts.  parity 0 even, 1 flip_x,
 * 2 flip_y (GhostParity, grid.hpp:60). */
void lfo_fill_ghosts(const lfo_grid* g, const int bc[4], int parity, double* f) {
  const int nxt = nxt_of(g);
  const double sx = parity == 1 ? -1.0 : 1.0;
  const double sy = parity == 2 ? -1.0 : 1.0;
#define AT(i, j) f[(int64_t)(j) * nxt + (i)]
  for (int j = g->gy; j < g->gy + g->ny; ++j) {
    for (int l = 1; l <= g->gx; ++l) {
      const int lo = g->gx - l;
      const int hi = g->gx + g->nx - 1 + l;
      switch (bc[0]) {
        case LFO_TRANSMISSIVE: AT(lo, j) = AT(g->gx, j); break;
        case LFO_REFLECTIVE: AT(lo, j) = sx * AT(g->gx + l - 1, j); break;
        default: AT(lo, j) = AT(g->gx + ((g->nx - l) % g->nx + g->nx) % g->nx, j); break;
      }
      switch (bc[1]) {
        case LFO_TRANSMISSIVE: AT(hi, j) = AT(g->gx + g->nx - 1, j); break;
        case LFO_REFLECTIVE: AT(hi, j) = sx * AT(g->gx + g->nx - l, j); break;
        default: AT(hi, j) = AT(g->gx + (l - 1) % g->nx, j); break;
      }
    }
  }
  if (g->gy == 0) return;
  for (int i = 0; i < nxt; ++i) {
    for (int l = 1; l <= g->gy; ++l) {
      const int lo = g->gy - l;
      const int hi = g->gy + g->ny - 1 + l;
      switch (bc[2]) {
        case LFO_TRANSMISSIVE: AT(i, lo) = AT(i, g->gy); break;
        case LFO_REFLECTIVE: AT(i, lo) = sy * AT(i, g->gy + l - 1); break;
        default: AT(i, lo) = AT(i, g->gy + ((g->ny - l) % g->ny + g->ny) % g->ny); break;
      }
      switch (bc[3]) {
        case LFO_TRANSMISSIVE: AT(i, hi) = AT(i, g->gy + g->ny - 1); break;
        case LFO_REFLECTIVE: AT(i, hi) = sy * AT(i, g->gy + g->ny - l); break;
        default: AT(i, hi) = AT(i, g->gy + (l - 1) % g->ny); break;
      }
    }
  }
#undef AT
}

/* grid.cpp:116-121 */
void lfo_apply_boundary(const lfo_grid* g, const int bc[4], double* const field[4]) {
  lfo_fill_ghosts(g, bc, 0, field[0]);
  lfo_fill_ghosts(g, bc, 1, field[1]);
  lfo_fill_ghosts(g, bc, 2, field[2]);
  lfo_fill_ghosts(g, bc, 0, field[3]);
}

/* grid.cpp:123-134 */
void lfo_interior_totals(const lfo_grid* g, double* const field[4], double tot[4]) {
  const double vol = g->dim == 2 ? g->dx * g->dy : g->dx;
  for (int c = 0; c < 4; ++c) {
    double sum = 0.0;
    for (int j = g->gy; j < g->gy + g->ny; ++j)
      for (int i = g->gx; i < g->gx + g->nx; ++i) sum += field[c][idx_of(g, i, j)];
    tot[c] = sum * vol;
  }
}

/* libstdc++ std::min/std::max tie semantics. */
static inline double smin(double a, double b) { return (b < a) ? b : a; }
static inline double smax(double a, double b) { return (a < b) ? b : a; }

/* reconstruct.hpp:24-30 */
double lfo_sweby(double a, double b, double beta) {
  if (!(a * b > 0.0)) return 0.0;
  const double aa = fabs(a);
  const double ab = fabs(b);
  const double m = smax(smin(aa, beta * ab), smin(beta * aa, ab));
  return a > 0.0 ? m : -m;
}

/* reconstruct.hpp:33-35, 44-49 */
static inline void face_trace(double q0, double q1, double q2, double q3, double beta,
                              double* minus, double* plus) {
  const double s1 = lfo_sweby(q2 - q1, q1 - q0, beta);
  const double s2 = lfo_sweby(q3 - q2, q2 - q1, beta);
  *minus = q1 + 0.5 * s1;
  *plus = q2 - 0.5 * s2;
}

/* riemann_hll.hpp:27-40 with sound_speed euler.hpp:99-104 */
void lfo_lagrangian_hll(const double wl[4], const double wr[4], double nx, double ny,
                        double gamma_l, double gamma_r, double* p_star, double* u_star) {
  const double ul = wl[1] * nx + wl[2] * ny;
  const double ur = wr[1] * nx + wr[2] * ny;
  const double cl = sqrt(gamma_l * wl[3] / wl[0]);
  const double cr = sqrt(gamma_r * wr[3] / wr[0]);
  const double cmax = smax(cl, cr);
  const double rho_sum = wl[0] + wr[0];
  *p_star = (wr[0] * wl[3] + wl[0] * wr[3]) / rho_sum -
            (wl[0] * wr[0] / rho_sum) * cmax * (ur - ul);
  *u_star = (wl[0] * ul + wr[0] * ur) / rho_sum - (wr[3] - wl[3]) / (cmax * rho_sum);
}

/* euler.hpp:87-97 (the positivity guard is the caller's, solver.cpp:222) */
static inline void cons_from_prim(const double w[4], double gamma, double u[4]) {
  u[0] = w[0];
  u[1] = w[0] * w[1];
  u[2] = w[0] * w[2];
  u[3] = w[3] / (gamma - 1.0) + 0.5 * w[0] * (w[1] * w[1] + w[2] * w[2]);
}

/* solver.cpp:26-43 */
static inline void contact_flux(const double um[4], const double up[4], double nx, double ny,
                                double p_star, double u_star, double f[4]) {
  double ua[4];
  if (u_star > 0.0) {
    memcpy(ua, um, sizeof ua);
  } else if (u_star < 0.0) {
    memcpy(ua, up, sizeof ua);
  } else {
    for (int c = 0; c < 4; ++c) ua[c] = 0.5 * (um[c] + up[c]);
  }
  f[0] = ua[0] * u_star;
  f[1] = ua[1] * u_star + p_star * nx;
  f[2] = ua[2] * u_star + p_star * ny;
  f[3] = ua[3] * u_star + p_star * u_star;
}

/* solver.cpp:47-53 */
void lfo_edge_flux(const double wm[4], const double wp[4], double nx, double ny, double gamma,
                   double f[4]) {
  double ps, us, um[4], up[4];
  lfo_lagrangian_hll(wm, wp, nx, ny, gamma, gamma, &ps, &us);
  cons_from_prim(wm, gamma, um);
  cons_from_prim(wp, gamma, up);
  contact_flux(um, up, nx, ny, ps, us, f);
}

/* solver.cpp:61-88 */
lfo_solver* lfo_create(const lfo_grid* g, const lfo_scheme* s, lfo_error* err) {
  set_err(err, 0);
  if (g->nx < 1 || g->ny < 1) {
    set_err(err, LFO_ERR_CONFIG);
    if (err) snprintf(err->message, sizeof err->message, "grid has no interior cells");
    return NULL;
  }
  if (g->gx < 2 || (g->dim == 2 && g->gy < 2)) {
    set_err(err, LFO_ERR_CONFIG);
    if (err) snprintf(err->message, sizeof err->message, "MUSCL stencils need at least two ghost layers");
    return NULL;
  }
  /* validate_boundary, grid.cpp:65-70 */
  if ((s->bc[0] == LFO_PERIODIC) != (s->bc[1] == LFO_PERIODIC)) {
    set_err(err, LFO_ERR_CONFIG);
    if (err) snprintf(err->message, sizeof err->message, "periodic boundary in x must be set on both sides");
    return NULL;
  }
  if (g->dim == 2 && (s->bc[2] == LFO_PERIODIC) != (s->bc[3] == LFO_PERIODIC)) {
    set_err(err, LFO_ERR_CONFIG);
    if (err) snprintf(err->message, sizeof err->message, "periodic boundary in y must be set on both sides");
    return NULL;
  }
  lfo_solver* so = (lfo_solver*)calloc(1, sizeof *so);
  so->g = *g;
  so->s = *s;
  so->cells = (int64_t)nxt_of(g) * nyt_of(g);
  const size_t nex = (size_t)(g->nx + 1) * g->ny;
  const size_t ney = g->dim == 2 ? (size_t)g->nx * (g->ny + 1) : 0;
  for (int k = 0; k < 2; ++k) {
    for (int c = 0; c < 4; ++c) {
      so->prim[k][c] = (double*)calloc((size_t)so->cells, sizeof(double));
      so->fx[k][c] = (double*)calloc(nex ? nex : 1, sizeof(double));
      so->fy[k][c] = (double*)calloc(ney ? ney : 1, sizeof(double));
    }
    so->ustar_x[k] = (double*)calloc(nex ? nex : 1, sizeof(double));
    so->ustar_y[k] = (double*)calloc(ney ? ney : 1, sizeof(double));
  }
  for (int c = 0; c < 4; ++c) so->pred[c] = (double*)calloc((size_t)so->cells, sizeof(double));
  return so;
}

void lfo_destroy(lfo_solver* so) {
  if (!so) return;
  for (int k = 0; k < 2; ++k) {
    for (int c = 0; c < 4; ++c) {
      free(so->prim[k][c]);
      free(so->fx[k][c]);
      free(so->fy[k][c]);
    }
    free(so->ustar_x[k]);
    free(so->ustar_y[k]);
  }
  for (int c = 0; c < 4; ++c) free(so->pred[c]);
  for (int s2 = 0; s2 < 2; ++s2) {
    free(so->gamma_cells[s2]);
    for (int k = 0; k < so->n_mat; ++k) free(so->frac[s2][k]);
  }
  for (int k = 0; k < so->n_mat; ++k) free(so->pred_mat[k]);
  free(so);
}

/* solver.cpp:434-480 */
int lfo_compute_dt(lfo_solver* so, double* const field[4], double cfl, double time,
                   double limit_time, double* dt_out, lfo_error* err) {
  const lfo_grid* g = &so->g;
  const double gamma0 = so->s.gamma;
  const double* gamma_cells = so->n_mat ? so->gamma_cells[0] : NULL;
  const int nx = g->nx, ny = g->ny;
  const int dim2 = g->dim == 2;
  const int64_t n_cells = (int64_t)nx * ny;
  int64_t fail = INT64_MAX;
  double rate = 0.0;
  set_err(err, 0);
  for (int64_t cc = 0; cc < n_cells; ++cc) {
    const int64_t cell = idx_of(g, g->gx + (int)(cc % nx), g->gy + (int)(cc / nx));
    const double r = field[0][cell];
    if (!(r > 0.0)) {
      if (cc < fail) fail = cc;
      continue;
    }
    const double inv = 1.0 / r;
    const double u = field[1][cell] * inv;
    const double v = field[2][cell] * inv;
    const double gamma = gamma_cells ? gamma_cells[cell] : gamma0;
    const double p = (gamma - 1.0) *
                     (field[3][cell] -
                      0.5 * (field[1][cell] * field[1][cell] + field[2][cell] * field[2][cell]) *
                          inv);
    if (!(p > 0.0)) {
      if (cc < fail) fail = cc;
      continue;
    }
    const double c = sqrt(gamma * p * inv);
    double rr = (fabs(u) + c) / g->dx;
    if (dim2) rr += (fabs(v) + c) / g->dy;
    rate = smax(rate, rr);
  }
  if (fail != INT64_MAX) {
    set_err(err, LFO_ERR_DT_STATE);
    err->i = fail % nx;
    err->j = fail / nx;
    snprintf(err->message, sizeof err->message,
             "non-physical state while computing the time step at cell (%lld,%lld)",
             (long long)err->i, (long long)err->j);
    return LFO_ERR_DT_STATE;
  }
  double dt = cfl / rate;
  if (time + dt > limit_time) dt = limit_time - time;
  if (!(dt > 0.0)) {
    set_err(err, LFO_ERR_DT_NONPOS);
    err->dt = dt;
    snprintf(err->message, sizeof err->message,
             "non-positive time step (time limit already reached?)");
    return LFO_ERR_DT_NONPOS;
  }
  *dt_out = dt;
  return 0;
}

/* solver.cpp:131-171 */
static int build_primitives(lfo_solver* so, double* const field[4], int slot, int64_t step,
                            lfo_error* err) {
  const lfo_grid* g = &so->g;
  const double gamma0 = so->s.gamma;
  const double* gamma_cells = so->n_mat ? so->gamma_cells[slot] : NULL;
  double* rho = so->prim[slot][0];
  double* u = so->prim[slot][1];
  double* v = so->prim[slot][2];
  double* p = so->prim[slot][3];
  const double* rin = field[0];
  const double* mx = field[1];
  const double* my = field[2];
  const double* re = field[3];
  int64_t fail = INT64_MAX;
  for (int64_t c = 0; c < so->cells; ++c) {
    const double r = rin[c];
    if (!(r > 0.0)) {
      if (c < fail) fail = c;
      rho[c] = u[c] = v[c] = p[c] = 0.0;
      continue;
    }
    const double inv = 1.0 / r;
    const double uu = mx[c] * inv;
    const double vv = my[c] * inv;
    const double g0 = gamma_cells ? gamma_cells[c] : gamma0;
    const double pp = (g0 - 1.0) * (re[c] - 0.5 * (mx[c] * mx[c] + my[c] * my[c]) * inv);
    rho[c] = r;
    u[c] = uu;
    v[c] = vv;
    p[c] = pp;
    if (!(pp > 0.0)) {
      if (c < fail) fail = c;
    }
  }
  if (fail == INT64_MAX) return 0;
  /* primitive_from_conserved with CellContext (euler.hpp:73-85, 56-66) */
  const int64_t c = fail;
  const double g0 = gamma_cells ? gamma_cells[c] : gamma0;
  set_err(err, LFO_ERR_PRIMITIVE);
  err->i = c % nxt_of(g) - g->gx;
  err->j = c / nxt_of(g) - g->gy;
  err->step = step;
  char num[64], suffix[96];
  const char* what;
  if (!(rin[c] > 0.0)) {
    what = "non-positive density";
    err->value = rin[c];
  } else {
    const double inv = 1.0 / rin[c];
    err->value = (g0 - 1.0) * (re[c] - 0.5 * (mx[c] * mx[c] + my[c] * my[c]) * inv);
    what = "non-positive pressure";
  }
  fmt_f(num, sizeof num, err->value);
  if (step >= 0)
    snprintf(suffix, sizeof suffix, " at cell (%lld,%lld) step %lld", (long long)err->i,
             (long long)err->j, (long long)step);
  else
    snprintf(suffix, sizeof suffix, " at cell (%lld,%lld)", (long long)err->i, (long long)err->j);
  snprintf(err->message, sizeof err->message, "%s = %s%s", what, num, suffix);
  return LFO_ERR_PRIMITIVE;
}

/* solver.cpp:173-256 */
static int compute_fluxes(lfo_solver* so, int fs, int slot, int64_t step, lfo_error* err) {
  const lfo_grid* g = &so->g;
  const double* rho = so->prim[slot][0];
  const double* u = so->prim[slot][1];
  const double* v = so->prim[slot][2];
  const double* p = so->prim[slot][3];
  const double gamma0 = so->s.gamma;
  const double* gamma_cells = so->n_mat ? so->gamma_cells[slot] : NULL;
  const double beta = so->s.beta;
  const int muscl = so->s.spatial_order >= 2;
  const int nx = g->nx, ny = g->ny, nxt = nxt_of(g);
  const int64_t nex = (int64_t)(nx + 1) * ny;
  int64_t fail = INT64_MAX;

  for (int axis = 0; axis < (g->dim == 2 ? 2 : 1); ++axis) {
    const int is_x = axis == 0;
    const int64_t n_edges = is_x ? nex : (int64_t)nx * (ny + 1);
    const int64_t stride = is_x ? 1 : nxt;
    const int along = is_x ? nx + 1 : nx;
    const double nrm_x = is_x ? 1.0 : 0.0;
    const double nrm_y = is_x ? 0.0 : 1.0;
    double* const* out = is_x ? so->fx[fs] : so->fy[fs];
    double* ustar = is_x ? so->ustar_x[fs] : so->ustar_y[fs];
    for (int64_t e = 0; e < n_edges; ++e) {
      const int a = (int)(e % along);
      const int b = (int)(e / along);
      const int64_t chigh = idx_of(g, g->gx + a, g->gy + b);
      const int64_t clow = chigh - stride;
      double wm[4], wp[4];
      if (muscl) {
        face_trace(rho[clow - stride], rho[clow], rho[chigh], rho[chigh + stride], beta, &wm[0], &wp[0]);
        face_trace(u[clow - stride], u[clow], u[chigh], u[chigh + stride], beta, &wm[1], &wp[1]);
        face_trace(v[clow - stride], v[clow], v[chigh], v[chigh + stride], beta, &wm[2], &wp[2]);
        face_trace(p[clow - stride], p[clow], p[chigh], p[chigh + stride], beta, &wm[3], &wp[3]);
      } else {
        wm[0] = rho[clow]; wm[1] = u[clow]; wm[2] = v[clow]; wm[3] = p[clow];
        wp[0] = rho[chigh]; wp[1] = u[chigh]; wp[2] = v[chigh]; wp[3] = p[chigh];
      }
      if (!(wm[0] > 0.0) || !(wm[3] > 0.0) || !(wp[0] > 0.0) || !(wp[3] > 0.0)) {
        const int64_t code = (is_x ? 0 : nex) + e;
        if (code < fail) fail = code;
        ustar[e] = 0.0;
        for (int c = 0; c < 4; ++c) out[c][e] = 0.0;
        continue;
      }
      double ps, us, um[4], up[4], f[4];
      const double el = gamma_cells ? gamma_cells[clow] : gamma0;
      const double er = gamma_cells ? gamma_cells[chigh] : gamma0;
      lfo_lagrangian_hll(wm, wp, nrm_x, nrm_y, el, er, &ps, &us);
      ustar[e] = us;
      cons_from_prim(wm, el, um);
      cons_from_prim(wp, er, up);
      contact_flux(um, up, nrm_x, nrm_y, ps, us, f);
      for (int c = 0; c < 4; ++c) out[c][e] = f[c];
    }
  }
  if (fail == INT64_MAX) return 0;
  const int is_x = fail < nex;
  const int64_t e = is_x ? fail : fail - nex;
  const int along = is_x ? nx + 1 : nx;
  set_err(err, LFO_ERR_TRACE);
  err->axis = is_x ? 0 : 1;
  err->i = e % along;
  err->j = e / along;
  err->step = step;
  snprintf(err->message, sizeof err->message,
           "non-physical reconstructed trace at %s-face (%lld,%lld) step %lld", is_x ? "x" : "y",
           (long long)err->i, (long long)err->j, (long long)step);
  return LFO_ERR_TRACE;
}

/* solver.cpp:258-329.  fa/fb are flux-set indices (fb < 0: single stage). */
static int apply_update(lfo_solver* so, double* const base[4], int fa, int fb, double dt,
                        double* const out[4], int64_t step, double* min_rho, double* min_p,
                        lfo_error* err) {
  const lfo_grid* g = &so->g;
  const int nx = g->nx, ny = g->ny;
  const double lam_x = dt / g->dx;
  const double lam_y = dt / g->dy;
  const int two = fb >= 0;
  const int dim2 = g->dim == 2;
  const int64_t n_cells = (int64_t)nx * ny;
  int64_t fail = INT64_MAX;
  double mr = INFINITY, me = INFINITY;
  for (int64_t cc = 0; cc < n_cells; ++cc) {
    const int i = (int)(cc % nx);
    const int j = (int)(cc / nx);
    const int64_t cell = idx_of(g, g->gx + i, g->gy + j);
    const size_t exl = (size_t)j * (nx + 1) + i;
    const size_t exr = exl + 1;
    const size_t eyb = (size_t)j * nx + i;
    const size_t eyt = eyb + (size_t)nx;
    double vals[4];
    for (int c = 0; c < 4; ++c) {
      const double* ax = so->fx[fa][c];
      const double fxl = two ? 0.5 * (ax[exl] + so->fx[fb][c][exl]) : ax[exl];
      const double fxr = two ? 0.5 * (ax[exr] + so->fx[fb][c][exr]) : ax[exr];
      double val = base[c][cell] - lam_x * (fxr - fxl);
      if (dim2) {
        const double* ay = so->fy[fa][c];
        const double fyb = two ? 0.5 * (ay[eyb] + so->fy[fb][c][eyb]) : ay[eyb];
        const double fyt = two ? 0.5 * (ay[eyt] + so->fy[fb][c][eyt]) : ay[eyt];
        val -= lam_y * (fyt - fyb);
      }
      vals[c] = val;
    }
    out[0][cell] = vals[0];
    out[1][cell] = vals[1];
    out[2][cell] = vals[2];
    out[3][cell] = vals[3];
    const double eint = vals[3] - 0.5 * (vals[1] * vals[1] + vals[2] * vals[2]) / vals[0];
    if (!(vals[0] > 0.0) || !(eint > 0.0)) {
      if (cc < fail) fail = cc;
    } else {
      mr = smin(mr, vals[0]);
      me = smin(me, eint);
    }
  }
  if (fail != INT64_MAX) {
    const int64_t i = fail % nx, j = fail / nx;
    const int64_t cell = idx_of(g, (int)(g->gx + i), (int)(g->gy + j));
    const double r = out[0][cell];
    const double eint =
        out[3][cell] - 0.5 * (out[1][cell] * out[1][cell] + out[2][cell] * out[2][cell]) / r;
    char rs[64], es[64], ds[64];
    fmt_f(rs, sizeof rs, r);
    fmt_f(es, sizeof es, eint);
    fmt_f(ds, sizeof ds, dt);
    set_err(err, LFO_ERR_POSITIVITY);
    err->i = i;
    err->j = j;
    err->step = step;
    err->dt = dt;
    err->value = r;
    err->value2 = eint;
    snprintf(err->message, sizeof err->message,
             "update lost positivity at cell (%lld,%lld): rho = %s, internal energy density = %s, "
             "step %lld, dt %s",
             (long long)i, (long long)j, rs, es, (long long)step, ds);
    return LFO_ERR_POSITIVITY;
  }
  if (min_rho) *min_rho = mr;
  if (min_p) *min_p = me;
  return 0;
}

/* solver.cpp:406-432 */
static void accumulate_boundary_outflow(lfo_solver* so, int fa, int fb, double dt, double acc[4]) {
  const lfo_grid* g = &so->g;
  const int nx = g->nx, ny = g->ny;
  const double ax = dt * (g->dim == 1 ? 1.0 : g->dy);
  for (int c = 0; c < 4; ++c) {
    const double* a = so->fx[fa][c];
    const double* b = fb >= 0 ? so->fx[fb][c] : a;
    double s = 0.0;
    for (int j = 0; j < ny; ++j) {
      const size_t row = (size_t)j * (nx + 1);
      const double r = fb >= 0 ? 0.5 * (a[row + nx] + b[row + nx]) : a[row + nx];
      const double l = fb >= 0 ? 0.5 * (a[row] + b[row]) : a[row];
      s += r - l;
    }
    acc[c] += ax * s;
  }
  if (g->dim == 2) {
    const double ay = dt * g->dx;
    for (int c = 0; c < 4; ++c) {
      const double* a = so->fy[fa][c];
      const double* b = fb >= 0 ? so->fy[fb][c] : a;
      double s = 0.0;
      for (int i = 0; i < nx; ++i) {
        const size_t t = (size_t)ny * nx + i;
        const double tv = fb >= 0 ? 0.5 * (a[t] + b[t]) : a[t];
        const double bv = fb >= 0 ? 0.5 * (a[i] + b[i]) : a[i];
        s += tv - bv;
      }
      acc[c] += ay * s;
    }
  }
}

/* solver.cpp:482-487 */
int lfo_euler_stage(lfo_solver* so, double* const in[4], double dt, double* const out[4],
                    int64_t step, lfo_error* err) {
  set_err(err, 0);
  lfo_apply_boundary(&so->g, so->s.bc, in);
  int rc = build_primitives(so, in, 0, step, err);
  if (rc) return rc;
  rc = compute_fluxes(so, 0, 0, step, err);
  if (rc) return rc;
  return apply_update(so, in, 0, -1, dt, out, step, NULL, NULL, err);
}

/* ---- multimaterial (multimat.cpp:7-44; solver.cpp:90-129, 331-404) ---- */

/* make_material_set, multimat.cpp:7-15 */
int lfo_set_materials(lfo_solver* so, int n, const double* gammas, lfo_error* err) {
  set_err(err, 0);
  char msg[160];
  msg[0] = 0;
  if (n < 1) snprintf(msg, sizeof msg, "material set needs at least one material");
  else if (n > LFO_MAX_MATERIALS) snprintf(msg, sizeof msg, "at most 16 materials are supported");
  else
    for (int k = 0; k < n; ++k)
      if (!(gammas[k] > 1.0) || !(gammas[k] <= 3.0)) {
        char num[64];
        fmt_f(num, sizeof num, gammas[k]);
        snprintf(msg, sizeof msg, "material adiabatic index must lie in (1, 3], got %s", num);
        break;
      }
  if (msg[0]) {
    set_err(err, LFO_ERR_CONFIG);
    if (err) snprintf(err->message, sizeof err->message, "%s", msg);
    return LFO_ERR_CONFIG;
  }
  if (so->n_mat) return LFO_ERR_CONFIG; /* once, like the constructor argument */
  so->n_mat = n;
  for (int k = 0; k < n; ++k) so->mat_gamma[k] = gammas[k];
  for (int s2 = 0; s2 < 2; ++s2) {
    /* solver.cpp:80-83: gamma_[s].assign(cells, eos.gamma), frac_ zeros */
    so->gamma_cells[s2] = (double*)malloc((size_t)so->cells * sizeof(double));
    for (int64_t c = 0; c < so->cells; ++c) so->gamma_cells[s2][c] = so->s.gamma;
    for (int k = 0; k < n; ++k) so->frac[s2][k] = (double*)calloc((size_t)so->cells, sizeof(double));
  }
  for (int k = 0; k < n; ++k) so->pred_mat[k] = (double*)calloc((size_t)so->cells, sizeof(double));
  return 0;
}

/* clamped_fraction, multimat.cpp:17-23 (without the CellContext variant) */
int lfo_clamped_fraction(double partial, double rho, double* y_out) {
  const double y = partial / rho;
  if (y >= 0.0 && y <= 1.0) {
    *y_out = y;
    return 0;
  }
  if (y < -1e-11 || y > 1.0 + 1e-11) return LFO_ERR_FRACTION;
  *y_out = y < 0.0 ? 0.0 : 1.0;
  return 0;
}

/* mixed_cell_gamma, multimat.cpp:25-32 */
double lfo_mixed_cell_gamma(int n, const double* gammas, const double* fractions) {
  double s = 0.0;
  for (int k = 0; k < n; ++k) {
    if (fractions[k] == 1.0) return gammas[k];
    s += fractions[k] / (gammas[k] - 1.0);
  }
  return 1.0 + 1.0 / s;
}

/* mass_fraction_fluxes, multimat.cpp:34-44 */
void lfo_mass_fraction_fluxes(double mass_flux, int n, const double* y_upwind, double* out) {
  double rest = mass_flux;
  for (int k = 0; k + 1 < n; ++k) {
    out[k] = mass_flux * y_upwind[k];
    rest -= out[k];
  }
  out[n - 1] = rest;
}

/* fill_all_ghosts, solver.cpp:90-129: ghost cells of the field and of every
 * partial density (even parity), then the clamped fractions and the mixed-cell
 * gamma of every (ghosted) cell into slot `slot`. */
static int fill_all_ghosts(lfo_solver* so, double* const field[4], double* const* partials,
                           int slot, lfo_error* err) {
  const lfo_grid* g = &so->g;
  lfo_apply_boundary(g, so->s.bc, field);
  if (partials == NULL || so->n_mat == 0) return 0;
  const int n_mat = so->n_mat;
  for (int k = 0; k < n_mat; ++k) lfo_fill_ghosts(g, so->s.bc, 0, partials[k]);
  const double* rho = field[0];
  int64_t fail = INT64_MAX;
  for (int64_t c = 0; c < so->cells; ++c) {
    double ysum_gamma = 0.0;
    int pure = -1;
    for (int k = 0; k < n_mat; ++k) {
      const double raw = partials[k][c] / rho[c];
      double y = raw;
      if (y < 0.0 || y > 1.0) {
        if (raw < -1e-11 || raw > 1.0 + 1e-11) {
          if (c < fail) fail = c;
          y = 0.0;
        } else {
          y = raw < 0.0 ? 0.0 : 1.0;
        }
      }
      so->frac[slot][k][c] = y;
      if (y == 1.0) pure = k;
      ysum_gamma += y / (so->mat_gamma[k] - 1.0);
    }
    so->gamma_cells[slot][c] = pure >= 0 ? so->mat_gamma[pure] : 1.0 + 1.0 / ysum_gamma;
  }
  if (fail == INT64_MAX) return 0;
  set_err(err, LFO_ERR_FRACTION);
  err->i = fail % nxt_of(g) - g->gx;
  err->j = fail / nxt_of(g) - g->gy;
  snprintf(err->message, sizeof err->message,
           "mass fraction out of [0,1] beyond round-off at cell (%lld,%lld)", (long long)err->i,
           (long long)err->j);
  return LFO_ERR_FRACTION;
}

/* update_partials, solver.cpp:331-404.  Stage fluxes: mass component of flux
 * set fa (and fb), u* of the same sets, fractions of slot sa (and sb). */
static void edge_material_flux(const lfo_solver* so, int fs, int slot, int is_x, size_t e,
                               int64_t clow, int64_t chigh, double* out_k) {
  const double mass = is_x ? so->fx[fs][0][e] : so->fy[fs][0][e];
  const double us = is_x ? so->ustar_x[fs][e] : so->ustar_y[fs][e];
  const int64_t up = us > 0.0 ? clow : chigh;
  double rest = mass;
  for (int k = 0; k < so->n_mat - 1; ++k) {
    const double fk = us == 0.0 ? 0.0 : mass * so->frac[slot][k][up];
    out_k[k] = fk;
    rest -= fk;
  }
  out_k[so->n_mat - 1] = us == 0.0 ? 0.0 : rest;
}

static void update_partials(lfo_solver* so, double* const* base, int fa, int fb, double dt,
                            int sa, int sb, double* const* out) {
  const lfo_grid* g = &so->g;
  const int n_mat = so->n_mat;
  const int nx = g->nx, ny = g->ny;
  const double lam_x = dt / g->dx;
  const double lam_y = dt / g->dy;
  const int dim2 = g->dim == 2;
  const int nxt = nxt_of(g);
  for (int64_t cc = 0; cc < (int64_t)nx * ny; ++cc) {
    const int i = (int)(cc % nx), j = (int)(cc / nx);
    const int64_t cell = idx_of(g, g->gx + i, g->gy + j);
    const size_t exl = (size_t)j * (nx + 1) + i, exr = exl + 1;
    const size_t eyb = (size_t)j * nx + i, eyt = eyb + (size_t)nx;
    double fl[LFO_MAX_MATERIALS], fr[LFO_MAX_MATERIALS], fb2[LFO_MAX_MATERIALS],
        ft[LFO_MAX_MATERIALS];
    for (int k = 0; k < n_mat; ++k) fl[k] = fr[k] = fb2[k] = ft[k] = 0.0;
    for (int stage = 0; stage < (fb >= 0 ? 2 : 1); ++stage) {
      const int fs = stage == 0 ? fa : fb, slot = stage == 0 ? sa : sb;
      const double w = fb >= 0 ? 0.5 : 1.0;
      double tl[LFO_MAX_MATERIALS], tr[LFO_MAX_MATERIALS], tb[LFO_MAX_MATERIALS],
          tt[LFO_MAX_MATERIALS];
      edge_material_flux(so, fs, slot, 1, exl, cell - 1, cell, tl);
      edge_material_flux(so, fs, slot, 1, exr, cell, cell + 1, tr);
      if (dim2) {
        edge_material_flux(so, fs, slot, 0, eyb, cell - nxt, cell, tb);
        edge_material_flux(so, fs, slot, 0, eyt, cell, cell + nxt, tt);
      }
      for (int k = 0; k < n_mat; ++k) {
        fl[k] += w * tl[k];
        fr[k] += w * tr[k];
        if (dim2) {
          fb2[k] += w * tb[k];
          ft[k] += w * tt[k];
        }
      }
    }
    for (int k = 0; k < n_mat; ++k) {
      double val = base[k][cell] - lam_x * (fr[k] - fl[k]);
      if (dim2) val -= lam_y * (ft[k] - fb2[k]);
      out[k][cell] = val;
    }
  }
}

/* solver.cpp:519-540: with materials, min p from the fresh partial masses */
static double mat_min_p(const lfo_solver* so, double* const field[4], double* const* partials) {
  const lfo_grid* g = &so->g;
  const int nx = g->nx, ny = g->ny;
  double min_p = INFINITY;
  for (int64_t cc = 0; cc < (int64_t)nx * ny; ++cc) {
    const int64_t cell = idx_of(g, g->gx + (int)(cc % nx), g->gy + (int)(cc / nx));
    const double r = field[0][cell];
    double s = 0.0;
    for (int k = 0; k < so->n_mat; ++k) s += (partials[k][cell] / r) / (so->mat_gamma[k] - 1.0);
    const double eint =
        field[3][cell] - 0.5 * (field[1][cell] * field[1][cell] + field[2][cell] * field[2][cell]) / r;
    min_p = smin(min_p, eint / s);
  }
  return min_p;
}

/* solver.cpp:489-546.  partials: the MaterialCells (n_mat arrays in grid
 * layout, updated in place) or NULL without a material set. */
int lfo_heun_step_mat(lfo_solver* so, double* const field[4], double* const* partials,
                      double cfl, double limit_time, double* time, int64_t* step,
                      double* boundary_outflow, lfo_step_out* out, lfo_error* err) {
  set_err(err, 0);
  if (so->n_mat == 0) partials = NULL;
  if (so->n_mat && partials == NULL) {
    /* the reference dereferences the missing MaterialCells (solver.cpp:529) */
    set_err(err, LFO_ERR_CONFIG);
    snprintf(err->message, sizeof err->message, "multimaterial step needs material storage");
    return LFO_ERR_CONFIG;
  }
  int rc = fill_all_ghosts(so, field, partials, 0, err);
  if (rc) return rc;
  double dt = 0.0;
  rc = lfo_compute_dt(so, field, cfl, *time, limit_time, &dt, err);
  if (rc) return rc;
  const int hits_limit = *time + dt >= limit_time;

  rc = build_primitives(so, field, 0, *step, err);
  if (rc) return rc;
  rc = compute_fluxes(so, 0, 0, *step, err);
  if (rc) return rc;
  double min_rho = 0.0, min_eint = 0.0;
  rc = apply_update(so, field, 0, -1, dt, so->pred, *step, &min_rho, &min_eint, err);
  if (rc) return rc;
  if (partials) update_partials(so, partials, 0, -1, dt, 0, -1, so->pred_mat);

  if (so->s.time_order >= 2) {
    rc = fill_all_ghosts(so, so->pred, partials ? so->pred_mat : NULL, 1, err);
    if (rc) return rc;
    rc = build_primitives(so, so->pred, 1, *step, err);
    if (rc) return rc;
    rc = compute_fluxes(so, 1, 1, *step, err);
    if (rc) return rc;
    rc = apply_update(so, field, 0, 1, dt, field, *step, &min_rho, &min_eint, err);
    if (rc) return rc;
    if (partials) update_partials(so, partials, 0, 1, dt, 0, 1, partials);
    accumulate_boundary_outflow(so, 0, 1, dt, boundary_outflow);
  } else {
    /* std::swap(state.field.comp, predictor_.comp) (and the partials): copy out */
    for (int c = 0; c < 4; ++c) memcpy(field[c], so->pred[c], (size_t)so->cells * sizeof(double));
    if (partials)
      for (int k = 0; k < so->n_mat; ++k)
        memcpy(partials[k], so->pred_mat[k], (size_t)so->cells * sizeof(double));
    accumulate_boundary_outflow(so, 0, -1, dt, boundary_outflow);
  }
  const double min_p = partials ? mat_min_p(so, field, partials) : (so->s.gamma - 1.0) * min_eint;
  *time = hits_limit ? limit_time : *time + dt;
  *step += 1;
  if (out) {
    out->dt = dt;
    out->hits_limit = hits_limit;
    out->time = *time;
    out->step = *step;
    out->min_rho = min_rho;
    out->min_p = min_p;
    for (int c = 0; c < 4; ++c) out->boundary_outflow[c] = boundary_outflow[c];
  }
  return 0;
}

/* solver.cpp:489-546 without materials */
int lfo_heun_step(lfo_solver* so, double* const field[4], double cfl, double limit_time,
                  double* time, int64_t* step, double* boundary_outflow, lfo_step_out* out,
                  lfo_error* err) {
  return lfo_heun_step_mat(so, field, NULL, cfl, limit_time, time, step, boundary_outflow, out,
                           err);
}

/* ---- Seeded smooth-perturbation generator ----
 * std::mt19937_64 restated (seed_seq-free integer seeding).  Each field k and
 * mode m draws, in order, kx, ky (1 + raw % 8), amplitude a = (raw>>11)*2^-53
 * and phase phi = 2*pi*((raw>>11)*2^-53).  The mode is
 *   a * sin(2 pi (kx x + ky y) + phi)
 *     = a * (sin(2 pi kx x + phi) cos(2 pi ky y) + cos(2 pi kx x + phi) sin(2 pi ky y)),
 * and the generator is DEFINED by the separable right-hand side evaluated from
 * 1D tables, so host and device produce identical bits. */
typedef struct { uint64_t mt[312]; int mti; } mt64;

static void mt64_seed(mt64* s, uint64_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
  s->mti = 312;
}

static uint64_t mt64_next(mt64* s) {
  static const uint64_t mag01[2] = {0ULL, 0xB5026F5AA96619E9ULL};
  const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
  if (s->mti >= 312) {
    int i;
    for (i = 0; i < 312 - 156; ++i) {
      uint64_t x = (s->mt[i] & UM) | (s->mt[i + 1] & LM);
      s->mt[i] = s->mt[i + 156] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
    }
    for (; i < 311; ++i) {
      uint64_t x = (s->mt[i] & UM) | (s->mt[i + 1] & LM);
      s->mt[i] = s->mt[i + (156 - 312)] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
    }
    uint64_t x = (s->mt[311] & UM) | (s->mt[0] & LM);
    s->mt[311] = s->mt[155] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
    s->mti = 0;
  }
  uint64_t x = s->mt[s->mti++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}

void lfo_fourier_tables(uint64_t seed, int nx, int ny, double x0, double y0, double dx,
                        double dy, double* tx, double* ty, double* amp) {
  const double two_pi = 6.283185307179586476925286766559;
  mt64 rng;
  mt64_seed(&rng, seed);
  for (int k = 0; k < 4; ++k) {
    for (int m = 0; m < 8; ++m) {
      const int kx = 1 + (int)(mt64_next(&rng) % 8ULL);
      const int ky = 1 + (int)(mt64_next(&rng) % 8ULL);
      const double a = (double)(mt64_next(&rng) >> 11) * 0x1.0p-53;
      const double phi = two_pi * ((double)(mt64_next(&rng) >> 11) * 0x1.0p-53);
      amp[k * 8 + m] = a;
      double* sx = tx + ((size_t)(k * 8 + m) * 2) * nx;
      double* cx = sx + nx;
      for (int i = 0; i < nx; ++i) {
        const double x = x0 + (i + 0.5) * dx;
        const double arg = two_pi * (kx * x) + phi;
        sx[i] = sin(arg);
        cx[i] = cos(arg);
      }
      double* sy = ty + ((size_t)(k * 8 + m) * 2) * ny;
      double* cy = sy + ny;
      for (int j = 0; j < ny; ++j) {
        const double y = y0 + (j + 0.5) * dy;
        const double arg = two_pi * (ky * y);
        sy[j] = sin(arg);
        cy[j] = cos(arg);
      }
    }
  }
}

/* The whole seeded smooth-flow initial state (cases.py initial_field, "fourier"):
 * f_k = sum_m a (sx cy + cx sy) in mode order, normalised by max |f_k| over the
 * interior, rho = 1 + 0.2 f1, u = 0.5 f2, v = 0.5 f3, p = 1 + 0.2 f4, then
 * conserved_from_primitive (euler.hpp:87-97).  Bit-identical to the Python
 * generator (every cell is independent; the maxima are order-free), so rows
 * may be split over `threads` OpenMP threads.  Used to give the reference arm
 * of bench.py the 16384^2 state without the Python generator's minutes. */
void lfo_init_fourier(uint64_t seed, const lfo_grid* g, double gamma, double* const field[4],
                      int threads) {
  const int nx = g->nx, ny = g->ny, gx = g->gx, gy = g->gy;
  const int64_t nxt = nx + 2 * gx;
  double* tx = (double*)malloc(sizeof(double) * 64 * (size_t)nx);
  double* ty = (double*)malloc(sizeof(double) * 64 * (size_t)ny);
  double amp[32];
  lfo_fourier_tables(seed, nx, ny, g->x0, g->y0, g->dx, g->dy, tx, ty, amp);
  if (threads < 1) threads = 1;
  double mx[4] = {0.0, 0.0, 0.0, 0.0};
  for (int k = 0; k < 4; ++k) {
    double m = 0.0;
#pragma omp parallel for num_threads(threads) reduction(max : m) schedule(static)
    for (int j = 0; j < ny; ++j) {
      double* row = field[k] + (int64_t)(j + gy) * nxt + gx;
      for (int i = 0; i < nx; ++i) row[i] = 0.0;
      for (int md = 0; md < 8; ++md) {
        const double* sx = tx + ((size_t)(k * 8 + md) * 2) * nx;
        const double* cx = sx + nx;
        const double* sy = ty + ((size_t)(k * 8 + md) * 2) * ny;
        const double* cy = sy + ny;
        const double a = amp[k * 8 + md], syj = sy[j], cyj = cy[j];
        for (int i = 0; i < nx; ++i) row[i] = row[i] + a * (sx[i] * cyj + cx[i] * syj);
      }
      for (int i = 0; i < nx; ++i) {
        const double v = fabs(row[i]);
        if (v > m) m = v;
      }
    }
    mx[k] = m;
  }
  const double gm1 = gamma - 1.0;
#pragma omp parallel for num_threads(threads) schedule(static)
  for (int j = 0; j < ny; ++j) {
    const int64_t o = (int64_t)(j + gy) * nxt + gx;
    for (int i = 0; i < nx; ++i) {
      const double rho = 1.0 + 0.2 * (field[0][o + i] / mx[0]);
      const double u = 0.5 * (field[1][o + i] / mx[1]);
      const double v = 0.5 * (field[2][o + i] / mx[2]);
      const double p = 1.0 + 0.2 * (field[3][o + i] / mx[3]);
      field[0][o + i] = rho;
      field[1][o + i] = rho * u;
      field[2][o + i] = rho * v;
      field[3][o + i] = p / gm1 + (0.5 * rho) * (u * u + v * v);
    }
  }
  free(tx);
  free(ty);
}
