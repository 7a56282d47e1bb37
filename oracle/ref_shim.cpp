// ref_shim.cpp -- C entry points over the UNMODIFIED reference solver.
//
// TEST INFRASTRUCTURE ONLY.  oracle/Makefile compiles this file together with
// the reference's own sources (/root/reference/proj/src/solver.cpp, grid.cpp)
// into oracle/_ref/libref_lagflux.so.  It is the "reference" CPU arm of
// bench.py and the pin for the C restatement (oracle/lagflux_oracle.c).
// Nothing in this file restates the algorithm: it only marshals arrays into a
// lagflux::SolverState and calls lagflux::LagfluxSolver (solver.hpp:78-131).
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <exception>
#include <string>

#ifdef _OPENMP
#include <omp.h>
#endif

#include "lagflux/csv.hpp"
#include "lagflux/error.hpp"
#include "lagflux/multimat.hpp"
#include "lagflux/solver.hpp"
#include "lagflux_oracle.h"

using namespace lagflux;

struct lfr_solver {
  CartesianGrid g;
  BoundaryCondition bc;
  PerfectGasEos eos;
  SchemeParams params;
  LagfluxSolver* solver = nullptr;
  SolverState state;
  CellField scratch;  // euler_stage output
  MaterialSet materials;   // outlives `solver` (constructor argument by pointer)
  MaterialCells mat;
};

namespace {

BcKind bc_kind(int k) {
  return k == LFO_REFLECTIVE ? BcKind::reflective
                             : (k == LFO_PERIODIC ? BcKind::periodic : BcKind::transmissive);
}

void clear(lfo_error* e) {
  if (!e) return;
  std::memset(e, 0, sizeof *e);
  e->i = e->j = e->step = -1;
}

int map_exception(lfo_error* e, int default_kind) {
  clear(e);
  int kind = default_kind;
  try {
    throw;
  } catch (const PositivityError& x) {
    kind = LFO_ERR_POSITIVITY;
    if (e) {
      e->i = x.cell_i;
      e->j = x.cell_j;
      e->step = x.step;
      e->dt = x.dt;
      std::snprintf(e->message, sizeof e->message, "%s", x.what());
    }
  } catch (const ConfigError& x) {
    kind = LFO_ERR_CONFIG;
    if (e) std::snprintf(e->message, sizeof e->message, "%s", x.what());
  } catch (const InvalidStateError& x) {
    const std::string w = x.what();
    if (w.rfind("non-physical state while computing the time step", 0) == 0)
      kind = LFO_ERR_DT_STATE;
    else if (w.rfind("mass fraction out of [0,1]", 0) == 0)
      kind = LFO_ERR_FRACTION;
    else if (w.rfind("non-physical reconstructed trace", 0) == 0)
      kind = LFO_ERR_TRACE;
    else
      kind = LFO_ERR_PRIMITIVE;
    if (e) std::snprintf(e->message, sizeof e->message, "%s", x.what());
  } catch (const Error& x) {
    kind = LFO_ERR_DT_NONPOS;
    if (e) std::snprintf(e->message, sizeof e->message, "%s", x.what());
  } catch (const std::exception& x) {
    if (e) std::snprintf(e->message, sizeof e->message, "%s", x.what());
  }
  if (e) e->kind = kind;
  return kind;
}

CartesianGrid to_grid(const lfo_grid* g) {
  CartesianGrid c;
  c.dim = g->dim;
  c.nx = g->nx;
  c.ny = g->ny;
  c.dx = g->dx;
  c.dy = g->dy;
  c.x0 = g->x0;
  c.y0 = g->y0;
  c.gx = g->gx;
  c.gy = g->gy;
  return c;
}

void copy_in(CellField& f, double* const src[4]) {
  for (int c = 0; c < 4; ++c)
    std::memcpy(f.comp[c].data(), src[c], f.comp[c].size() * sizeof(double));
}

void copy_out(const CellField& f, double* const dst[4]) {
  for (int c = 0; c < 4; ++c)
    std::memcpy(dst[c], f.comp[c].data(), f.comp[c].size() * sizeof(double));
}

}  // namespace

extern "C" {

// n_mat > 0: the solver gets make_material_set(gammas) (multimat.cpp:7-15).
lfr_solver* lfr_create_mat(const lfo_grid* g, const lfo_scheme* s, int threads, int n_mat,
                           const double* gammas, lfo_error* err) {
  clear(err);
  auto* r = new lfr_solver;
  try {
    r->g = to_grid(g);
    r->bc = {bc_kind(s->bc[0]), bc_kind(s->bc[1]), bc_kind(s->bc[2]), bc_kind(s->bc[3])};
    r->eos = PerfectGasEos{s->gamma};
    r->params.limiter = LimiterParams{s->beta};
    r->params.spatial_order = s->spatial_order;
    r->params.time_order = s->time_order;
    if (n_mat > 0) {
      r->materials = make_material_set(std::vector<double>(gammas, gammas + n_mat));
      r->mat = MaterialCells(r->g, r->materials.count());
    }
    r->solver = new LagfluxSolver(r->g, r->bc, r->eos, r->params, threads,
                                  n_mat > 0 ? &r->materials : nullptr);
    r->state.field = CellField(r->g);
    r->scratch = CellField(r->g);
  } catch (...) {
    map_exception(err, LFO_ERR_CONFIG);
    delete r->solver;
    delete r;
    return nullptr;
  }
  return r;
}

lfr_solver* lfr_create(const lfo_grid* g, const lfo_scheme* s, int threads, lfo_error* err) {
  return lfr_create_mat(g, s, threads, 0, nullptr, err);
}

// make_material_set's validation alone (0 or LFO_ERR_CONFIG with the message).
int lfr_make_material_set(int n, const double* gammas, lfo_error* err) {
  clear(err);
  try {
    (void)make_material_set(std::vector<double>(gammas, gammas + n));
  } catch (...) {
    return map_exception(err, LFO_ERR_CONFIG);
  }
  return 0;
}

void lfr_set_partials(lfr_solver* r, double* const* partials) {
  for (int k = 0; k < r->mat.count(); ++k)
    std::memcpy(r->mat.partial[size_t(k)].data(), partials[k],
                r->mat.partial[size_t(k)].size() * sizeof(double));
}

void lfr_get_partials(lfr_solver* r, double* const* partials) {
  for (int k = 0; k < r->mat.count(); ++k)
    std::memcpy(partials[k], r->mat.partial[size_t(k)].data(),
                r->mat.partial[size_t(k)].size() * sizeof(double));
}

double lfr_clamped_fraction(double partial, double rho, int* failed) {
  *failed = 0;
  try {
    return clamped_fraction(partial, rho);
  } catch (...) {
    *failed = 1;
    return 0.0;
  }
}

double lfr_mixed_cell_gamma(int n, const double* gammas, const double* fractions) {
  const MaterialSet set{std::vector<double>(gammas, gammas + n)};
  return mixed_cell_gamma(set, std::span<const double>(fractions, size_t(n)));
}

void lfr_mass_fraction_fluxes(double mass_flux, int n, const double* y_upwind, double* out) {
  mass_fraction_fluxes(mass_flux, std::span<const double>(y_upwind, size_t(n)),
                       std::span<double>(out, size_t(n)));
}

// field_csv (csv.cpp:26-83) of the internal state (and material cells): returns
// the length; copies min(len, cap) bytes into buf when buf != NULL.  -1 and the
// error record when field_csv throws.
int64_t lfr_field_csv(lfr_solver* r, uint64_t digest, double time, char* buf, int64_t cap,
                      lfo_error* err) {
  clear(err);
  try {
    const bool mm = r->mat.count() > 0;
    const std::string s = field_csv(r->g, r->state.field, r->eos, mm ? &r->materials : nullptr,
                                    mm ? &r->mat : nullptr, digest, time);
    if (buf) std::memcpy(buf, s.data(), size_t(std::min<int64_t>(cap, int64_t(s.size()))));
    return int64_t(s.size());
  } catch (...) {
    map_exception(err, LFO_ERR_PRIMITIVE);
    return -1;
  }
}

// diagnostics_csv (csv.cpp:104-114) of n records {step, time, dt, min_rho, min_p}
// (5 doubles each, step as a double): length, min(len, cap) bytes into buf.
int64_t lfr_diagnostics_csv(int n, const double* rec, char* buf, int64_t cap) {
  std::vector<StepDiagnostics> diag(static_cast<size_t>(n));
  for (int k = 0; k < n; ++k) {
    diag[size_t(k)].step = std::int64_t(rec[5 * k]);
    diag[size_t(k)].time = rec[5 * k + 1];
    diag[size_t(k)].dt = rec[5 * k + 2];
    diag[size_t(k)].min_rho = rec[5 * k + 3];
    diag[size_t(k)].min_p = rec[5 * k + 4];
  }
  const std::string s = diagnostics_csv(diag);
  if (buf) std::memcpy(buf, s.data(), size_t(std::min<int64_t>(cap, int64_t(s.size()))));
  return int64_t(s.size());
}

void lfr_destroy(lfr_solver* r) {
  if (!r) return;
  delete r->solver;
  delete r;
}

// Replace the solver state (field, time, step, outflow; diagnostics cleared).
void lfr_set_state(lfr_solver* r, double* const field[4], double time, int64_t step) {
  copy_in(r->state.field, field);
  r->state.time = time;
  r->state.step = step;
  r->state.diagnostics.clear();
  for (double& b : r->state.boundary_outflow) b = 0.0;
}

void lfr_get_state(lfr_solver* r, double* const field[4], double* time, int64_t* step,
                   double* outflow) {
  copy_out(r->state.field, field);
  if (time) *time = r->state.time;
  if (step) *step = r->state.step;
  if (outflow)
    for (int c = 0; c < 4; ++c) outflow[c] = r->state.boundary_outflow[size_t(c)];
}

// n calls of LagfluxSolver::heun_step on the internal state (bench.cpp:70-75).
// dts/diag (optional, n entries / n*5 doubles) receive the per-step record
// {dt, time, min_rho, min_p, step}.  Returns 0 or the error kind; *done = steps taken.
int lfr_heun_steps(lfr_solver* r, int n, double cfl, double limit_time, double* dts,
                   double* diag, int* done, lfo_error* err) {
  clear(err);
  TimeControls controls{cfl, limit_time, INT64_MAX};
  int k = 0;
  try {
    for (; k < n; ++k) {
      const double dt = r->solver->heun_step(r->state, controls, limit_time,
                                             r->mat.count() > 0 ? &r->mat : nullptr);
      if (dts) dts[k] = dt;
      if (diag) {
        const StepDiagnostics& d = r->state.diagnostics.back();
        diag[5 * k + 0] = d.dt;
        diag[5 * k + 1] = d.time;
        diag[5 * k + 2] = d.min_rho;
        diag[5 * k + 3] = d.min_p;
        diag[5 * k + 4] = double(d.step);
      }
    }
  } catch (...) {
    if (done) *done = k;
    return map_exception(err, LFO_ERR_PRIMITIVE);
  }
  if (done) *done = k;
  return 0;
}

// LagfluxSolver::compute_dt on the internal state field.
int lfr_compute_dt(lfr_solver* r, double cfl, double time, double limit_time, double* dt,
                   lfo_error* err) {
  clear(err);
  try {
    apply_boundary(r->g, r->bc, r->state.field);
    TimeControls controls{cfl, limit_time, INT64_MAX};
    *dt = r->solver->compute_dt(r->state.field, controls, time, limit_time);
  } catch (...) {
    return map_exception(err, LFO_ERR_DT_STATE);
  }
  return 0;
}

// LagfluxSolver::euler_stage(state.field, dt, out): out is returned in `out`
// (ghosts as the reference leaves them: zero-initialised scratch).
int lfr_euler_stage(lfr_solver* r, double dt, int64_t step, double* const out[4],
                    lfo_error* err) {
  clear(err);
  try {
    for (auto& c : r->scratch.comp) std::fill(c.begin(), c.end(), 0.0);
    r->solver->euler_stage(r->state.field, dt, r->scratch, step);
  } catch (...) {
    return map_exception(err, LFO_ERR_PRIMITIVE);
  }
  copy_out(r->scratch, out);
  return 0;
}

// Element functions for known-answer tests.
// lagflux::interior_totals (grid.cpp:122-133) of the solver's current state.
void lfr_interior_totals(lfr_solver* r, double tot[4]) {
  const std::array<double, 4> t = interior_totals(r->g, r->state.field);
  for (int c = 0; c < 4; ++c) tot[c] = t[size_t(c)];
}

void lfr_fill_ghosts(const lfo_grid* g, const int bc[4], int parity, double* f) {
  const CartesianGrid cg = to_grid(g);
  const BoundaryCondition b{bc_kind(bc[0]), bc_kind(bc[1]), bc_kind(bc[2]), bc_kind(bc[3])};
  fill_ghosts(cg, b, parity == 1 ? GhostParity::flip_x
                                 : (parity == 2 ? GhostParity::flip_y : GhostParity::even),
              f);
}

double lfr_sweby(double a, double b, double beta) { return sweby_limiter(a, b, LimiterParams{beta}); }

void lfr_lagrangian_hll(const double wl[4], const double wr[4], double nx, double ny,
                        double gamma, double* p_star, double* u_star) {
  const ContactSolution s = lagrangian_hll({wl[0], wl[1], wl[2], wl[3]},
                                           {wr[0], wr[1], wr[2], wr[3]}, Vec2{nx, ny},
                                           PerfectGasEos{gamma});
  *p_star = s.p_star;
  *u_star = s.u_star;
}

void lfr_edge_flux(const double wm[4], const double wp[4], double nx, double ny, double gamma,
                   double f[4]) {
  const EdgeFlux e = edge_flux({wm[0], wm[1], wm[2], wm[3]}, {wp[0], wp[1], wp[2], wp[3]},
                               Vec2{nx, ny}, PerfectGasEos{gamma});
  f[0] = e.mass;
  f[1] = e.mom_x;
  f[2] = e.mom_y;
  f[3] = e.energy;
}

// edge_flux / lagrangian_hll with one EOS per side (solver.cpp:45-53,
// riemann_hll.hpp:27-45); 0, or 1 with the exception's what() in msg.
int lfr_edge_flux2(const double wm[4], const double wp[4], double nx, double ny, double gm,
                   double gp, double f[4], double cs[2], char* msg, int cap) {
  try {
    const PrimitiveState a{wm[0], wm[1], wm[2], wm[3]}, b{wp[0], wp[1], wp[2], wp[3]};
    const ContactSolution s = lagrangian_hll(a, b, Vec2{nx, ny}, PerfectGasEos{gm}, PerfectGasEos{gp});
    const EdgeFlux e = edge_flux(a, b, Vec2{nx, ny}, PerfectGasEos{gm}, PerfectGasEos{gp});
    f[0] = e.mass;
    f[1] = e.mom_x;
    f[2] = e.mom_y;
    f[3] = e.energy;
    cs[0] = s.p_star;
    cs[1] = s.u_star;
    return 0;
  } catch (const std::exception& x) {
    std::snprintf(msg, (size_t)cap, "%s", x.what());
    return 1;
  }
}

int lfr_omp_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

}  // extern "C"
