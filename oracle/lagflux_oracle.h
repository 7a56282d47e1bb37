/*
 * lagflux_oracle.h -- CPU restatement of the reference Lagrange-flux time step.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the parity checker for the CUDA path in
 * paper_1607_08710_b200/.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.  The product never links it.
 *
 * It restates, in plain C with the reference's exact operation order, the
 * hot path of /root/reference/proj, single- and multimaterial:
 *   LagfluxSolver::heun_step        src/solver.cpp:489-546
 *   LagfluxSolver::euler_stage      src/solver.cpp:482-487
 *   LagfluxSolver::compute_dt       src/solver.cpp:434-480
 *   build_primitives                src/solver.cpp:131-171
 *   compute_fluxes                  src/solver.cpp:173-256
 *   apply_update                    src/solver.cpp:258-329
 *   accumulate_boundary_outflow     src/solver.cpp:406-432
 *   fill_ghosts / apply_boundary    src/grid.cpp:72-121
 *   lagrangian_hll                  include/lagflux/riemann_hll.hpp:27-40
 *   sweby_limiter / muscl_face_trace include/lagflux/reconstruct.hpp:24-49
 *   conserved_from_primitive        include/lagflux/euler.hpp:87-97
 *   fill_all_ghosts (materials)     src/solver.cpp:90-129
 *   update_partials                 src/solver.cpp:331-404
 *   multimaterial min p             src/solver.cpp:519-540
 *   make_material_set, clamped_fraction, mixed_cell_gamma,
 *   mass_fraction_fluxes            src/multimat.cpp:7-44
 *
 * Parity is pinned two ways (see tests/test_oracle_cpu.py):
 *   - bit-for-bit against the reference itself, compiled from its own sources
 *     by oracle/Makefile into oracle/_ref/ (ref_shim.cpp drives it);
 *   - against golden vectors in tests/golden/ generated from oracle/_ref by
 *     tests/golden/make_golden.py, and the reference's own known-answer tests.
 *
 * Build with -ffp-contract=off: the shipped reference has no FMA.
 */
#ifndef LAGFLUX_ORACLE_H
#define LAGFLUX_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Boundary kinds, same order as lagflux::BcKind (grid.hpp:51). */
enum { LFO_TRANSMISSIVE = 0, LFO_REFLECTIVE = 1, LFO_PERIODIC = 2 };

/* Error kinds (shared numbering with include/lagflux_b200.h). */
enum {
  LFO_OK = 0,
  LFO_ERR_CONFIG = 1,        /* ConfigError */
  LFO_ERR_DT_STATE = 2,      /* InvalidStateError from compute_dt (solver.cpp:471-475) */
  LFO_ERR_DT_NONPOS = 3,     /* Error "non-positive time step" (solver.cpp:478) */
  LFO_ERR_PRIMITIVE = 4,     /* InvalidStateError from build_primitives (solver.cpp:164-170) */
  LFO_ERR_TRACE = 5,         /* InvalidStateError from compute_fluxes (solver.cpp:245-255) */
  LFO_ERR_POSITIVITY = 6,    /* PositivityError from apply_update (solver.cpp:310-326) */
  LFO_ERR_FRACTION = 9       /* InvalidStateError from fill_all_ghosts (solver.cpp:122-127) */
};

#define LFO_MAX_MATERIALS 16   /* make_material_set, multimat.cpp:10 */

typedef struct {
  int dim;          /* 1 or 2 */
  int nx, ny;       /* interior cells */
  int gx, gy;       /* ghost layers (2, and 0 in y for 1D) */
  double dx, dy;
  double x0, y0;
} lfo_grid;

typedef struct {
  double gamma;
  double beta;         /* Sweby coefficient */
  int spatial_order;   /* 1 or 2 */
  int time_order;      /* 1 or 2 */
  int bc[4];           /* x_low, x_high, y_low, y_high */
} lfo_scheme;

typedef struct {
  int kind;
  int axis;            /* 0 = x-face, 1 = y-face (LFO_ERR_TRACE) */
  int64_t i, j;        /* cell or face index as the reference reports it */
  int64_t step;
  double dt;
  double value;        /* offending value (density, pressure, ...) */
  double value2;       /* second value (PositivityError: internal energy) */
  char message[320];   /* the reference's what() text */
} lfo_error;

typedef struct {
  double dt;
  int hits_limit;
  double time;           /* state.time after the step */
  int64_t step;          /* state.step after the step */
  double min_rho;        /* StepDiagnostics::min_rho */
  double min_p;          /* StepDiagnostics::min_p = (gamma-1) * min e_int */
  double boundary_outflow[4]; /* running SolverState::boundary_outflow */
} lfo_step_out;

typedef struct lfo_solver lfo_solver;

/* Grid helpers (grid.cpp:23-56). Return 0 or LFO_ERR_CONFIG. */
int lfo_make_grid_1d(int nx, double x_min, double x_max, lfo_grid* g);
int lfo_make_grid_2d(int nx, int ny, double x_min, double x_max, double y_min, double y_max,
                     lfo_grid* g);

/* Solver lifetime (solver.cpp:61-88). */
lfo_solver* lfo_create(const lfo_grid* g, const lfo_scheme* s, lfo_error* err);
void lfo_destroy(lfo_solver* s);

/* Field arrays are four ghosted row-major arrays of nxt*nyt doubles
 * (rho, rho u, rho v, rho E), exactly lagflux::CellField. */
int lfo_compute_dt(lfo_solver* s, double* const field[4], double cfl, double time,
                   double limit_time, double* dt, lfo_error* err);
int lfo_euler_stage(lfo_solver* s, double* const in[4], double dt, double* const out[4],
                    int64_t step, lfo_error* err);
/* state: field (in place), time/step in-out, boundary_outflow in-out (4). */
/* Multimaterial (solver.cpp:90-129, 331-404, 519-540; multimat.cpp:7-44):
 * lfo_set_materials is the constructor's MaterialSet (make_material_set's
 * validation); lfo_heun_step_mat is heun_step(state, controls, limit, &mat)
 * with the partial densities as n_mat arrays in the ghosted grid layout. */
int lfo_set_materials(lfo_solver* s, int n, const double* gammas, lfo_error* err);
int lfo_heun_step_mat(lfo_solver* s, double* const field[4], double* const* partials,
                      double cfl, double limit_time, double* time, int64_t* step,
                      double* boundary_outflow, lfo_step_out* out, lfo_error* err);
int lfo_clamped_fraction(double partial, double rho, double* y_out);
double lfo_mixed_cell_gamma(int n, const double* gammas, const double* fractions);
void lfo_mass_fraction_fluxes(double mass_flux, int n, const double* y_upwind, double* out);
int lfo_heun_step(lfo_solver* s, double* const field[4], double cfl, double limit_time,
                  double* time, int64_t* step, double* boundary_outflow, lfo_step_out* out,
                  lfo_error* err);

/* Element functions for the known-answer tests. */
void lfo_fill_ghosts(const lfo_grid* g, const int bc[4], int parity, double* f);
void lfo_apply_boundary(const lfo_grid* g, const int bc[4], double* const field[4]);
double lfo_sweby(double a, double b, double beta);
void lfo_lagrangian_hll(const double wl[4], const double wr[4], double nx, double ny,
                        double gamma_l, double gamma_r, double* p_star, double* u_star);
/* edge_flux (solver.cpp:47-53); traces must be physical. */
void lfo_edge_flux(const double wm[4], const double wp[4], double nx, double ny, double gamma,
                   double f[4]);
void lfo_interior_totals(const lfo_grid* g, double* const field[4], double tot[4]);

/* Seeded smooth-perturbation generator (BASELINE configs 4-5):
 * fills the interior of a ghosted field.  Tables come from lfo_fourier_tables. */
void lfo_fourier_tables(uint64_t seed, int nx, int ny, double x0, double y0, double dx,
                        double dy, double* tx /* 4*8*2*nx */, double* ty /* 4*8*2*ny */,
                        double* amp /* 4*8 */);
/* The whole initial state into the interior of a ghosted field (rows split over
 * `threads` OpenMP threads; bit-identical to cases.py initial_field). */
void lfo_init_fourier(uint64_t seed, const lfo_grid* g, double gamma, double* const field[4],
                      int threads);

#ifdef __cplusplus
}
#endif

#endif
