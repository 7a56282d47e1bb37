// kernels.h -- host-side launchers for the device kernels (internal to the .so).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "lagflux_device.cuh"
#include "layout.cuh"

namespace lfb {

// Per-step device scalars.  Mins/maxes are kept as order-preserving 64-bit keys
// so the reductions are exact atomics (max/min are order independent, exactly
// like the reference's OpenMP reduction(max/min), solver.cpp:272,449).
struct Scalars {
  unsigned long long rate_bits;      // max CFL rate over interior cells (double bits, >= 0)
  long long fail_dt;                 // smallest failing interior index in compute_dt
  long long fail_prim;               // smallest failing ghosted index in build_primitives
  long long fail_trace;              // smallest failing face code in compute_fluxes
  long long fail_update;             // smallest failing interior index in apply_update
  unsigned long long min_rho_bits;   // min rho over updated cells
  unsigned long long min_eint_bits;  // min internal energy density over updated cells
  double dt;                         // step dt (device-resident runs)
  double time;                       // state time after the step (device-resident runs)
  int hits;                          // time + dt >= limit
  int status;                        // 0 ok, else an LF_ERR_* kind detected in this step
  long long fail_frac;               // smallest failing ghosted index in the fraction closure
  unsigned long long min_p_key;      // multimaterial min p (order-preserving key of a double)
};

// Slab geometry: local rows [0, ny) are global rows [y0, y0+ny) of ny_global.
struct Slab {
  int y0 = 0;
  int ny_global = 0;
  int fill_lo = 1;   // apply the y_low BC locally (else the halo came from a neighbour)
  int fill_hi = 1;
};

// Face flux storage (reference FluxSet, solver.hpp:100-105): x faces (nx+1) x ny,
// y faces nx x (ny+1), 4 components each, pitched rows.
struct FluxArr {
  double* p;
  int64_t pitch;
  int64_t fstride;
};

// Process-wide count of kernels launched by this library (lf_launch_count).
void count_launch(int n = 1);
long long launch_count();

void reset_scalars(Scalars* s, cudaStream_t st);

// ghost fill (grid.cpp:72-114), 4 layers: x sides over interior rows, then
// (after any halo exchange) y sides over every column at the domain edges.
// ncomp components; component odd_x flips sign in a reflective x image,
// odd_y in a y image (a conserved field: 1 and 2; partial densities: none, -1).
void launch_fill_x(const Field& f, const Layout& L, const int bc[4], cudaStream_t st,
                   int ncomp = 4, int odd_x = 1);
// x and y sides in one launch; needs nx >= NG and (2D) ny >= NG
// f2 (may be NULL): ncomp2 more components of even parity in the same launch
void launch_fill_xy(const Field& f, const Layout& L, const int bc[4], const Slab& sl, bool dim2,
                    cudaStream_t st, int ncomp, int odd_x, int odd_y, const Field* f2 = nullptr,
                    int ncomp2 = 0);
void launch_fill_y_only(const Field& f, const Layout& L, const int bc[4], const Slab& sl,
                        cudaStream_t st, int ncomp = 4, int odd_y = 2);

// Boundary-face fluxes for accumulate_boundary_outflow (solver.cpp:406-432):
// out = [left 4 x ny | right 4 x ny | bottom 4 x nx | top 4 x nx], Heun-averaged when two.
void launch_gather_boundary(const FluxArr& fxa, const FluxArr& fya, const FluxArr& fxb,
                            const FluxArr& fyb, const Layout& L, bool two, double* out,
                            cudaStream_t st);

void launch_rate(const Field& u, const Layout& L, const Slab& sl, const Consts& k, int dim2,
                 Scalars* s, cudaStream_t st);

void launch_prims(const Field& u, const Field& w, const Layout& L, const Slab& sl, double gm1,
                  int dim2, Scalars* s, cudaStream_t st);

void launch_fluxes(const Field& w, const FluxArr& fx, const FluxArr& fy, const Layout& L,
                   const Slab& sl, const Consts& k, int muscl, int dim2, Scalars* s,
                   cudaStream_t st);

// out = base - lam*(dF); fb == nullptr: single stage; else F = 0.5*(Fa+Fb)
void launch_update(const Field& base, const FluxArr& fxa, const FluxArr& fya,
                   const FluxArr* fxb, const FluxArr* fyb, const Field& out, const Layout& L,
                   const Slab& sl, double dt, double dx, double dy, int dim2, Scalars* s,
                   cudaStream_t st);

// Fourier initial condition (cases.py fourier_*): raw sums then normalisation.
void launch_fourier_raw(const Field& f, const Layout& L, const double* tx, const double* ty,
                        const double* amp, cudaStream_t st);
void launch_absmax(const Field& f, const Layout& L, unsigned long long* out4, cudaStream_t st);
void launch_fourier_finish(const Field& f, const Layout& L, const unsigned long long* max4,
                           double gamma, cudaStream_t st);

// ---------------------------------------------------------------- multimaterial
// (solver.cpp:90-129, 331-404, 519-540; csrc/material_kernels.cu)
constexpr int MAX_MATERIALS = 16;
struct MatConsts {
  int n;
  double gamma[MAX_MATERIALS];
};

// fill_all_ghosts' closure over the reference's ghosted cells: clamped
// fractions y_k = partial_k / rho into y (n comps) and the mixed-cell gamma
// into gcell (1 comp); failures -> s->fail_frac.
void launch_mat_fractions(const Field& u, const Field& part, const Field& y, const Field& gcell,
                          const Layout& L, const Slab& sl, const MatConsts& mc, int dim2,
                          Scalars* s, cudaStream_t st);
// compute_dt / build_primitives / compute_fluxes with the per-cell gamma;
// the fluxes also store u* per face (us.p: component 0 of a FluxArr).
void launch_rate_g(const Field& u, const Field& gcell, const Layout& L, const Slab& sl,
                   const Consts& k, int dim2, Scalars* s, cudaStream_t st);
void launch_prims_g(const Field& u, const Field& w, const Field& gcell, const Layout& L,
                    const Slab& sl, int dim2, Scalars* s, cudaStream_t st);
void launch_fluxes_g(const Field& w, const Field& gcell, const FluxArr& fx, const FluxArr& fy,
                     const FluxArr& usx, const FluxArr& usy, const Layout& L, const Slab& sl,
                     const Consts& k, int muscl, int dim2, Scalars* s, cudaStream_t st);
// update_partials: out_k = base_k - lam (per-material face fluxes of set a
// [and b]); fractions of the upwind cells from ya [yb].
void launch_update_partials(const Field& base, const FluxArr& fxa, const FluxArr& fya,
                            const FluxArr& usxa, const FluxArr& usya, const Field& ya,
                            const FluxArr* fxb, const FluxArr* fyb, const FluxArr* usxb,
                            const FluxArr* usyb, const Field* yb, const Field& out,
                            const Layout& L, int n_mat, double dt, double dx, double dy,
                            int dim2, cudaStream_t st);
// solver.cpp:522-538: min over interior cells of e_int / sum_k (y_k / (gamma_k - 1))
void launch_mat_min_p(const Field& u, const Field& part, const Layout& L, const MatConsts& mc,
                      Scalars* s, cudaStream_t st);
void fill_value(double* p, int64_t n, double v, cudaStream_t st);
// initialize_hydro for InitKind::regions (run.cpp:29-78): reg = nreg x {x_min,
// x_max, y_min, y_max, rho, u, v, p, material}; failures -> atomicMin(fail, index)
void launch_init_regions(const Field& u, const Field& part, const Layout& L, const Slab& sl,
                         double x0, double y0, double dx, double dy, int dim2, const double* reg,
                         int nreg, const MatConsts& mc, double gamma0, unsigned long long* fail,
                         cudaStream_t st);
// field_csv's per-cell columns (csv.cpp:40-57): rho, u, v, p, e_internal, y_1..y_n as
// planes of nx*ny; clamp failures -> atomicMin(fail, row-major global interior index)
// edge_flux (solver.cpp:45-53) of n faces: w = n x {rho, u, v, p}, nrm = n x {nx, ny},
// one gamma per side and face; flux n x 4, contact n x {p*, u*} (may be NULL);
// fail: min over failing faces of 4 i + check (init ~0)
void launch_edge_flux(int64_t n, const double* wm, const double* wp, const double* nrm,
                      const double* gm, const double* gp, double* flux, double* contact,
                      unsigned long long* fail, cudaStream_t st);
// interior_totals' ordered per-component sums (grid.cpp:122-133) over one slab,
// starting from s_in[4] (NULL: 0.0); u at the interior origin
void launch_interior_sums(const double* u, int64_t fstride, int pitch, int nx, int ny,
                          const double* s_in, double* s_out, cudaStream_t st);
void launch_csv_derive(const Field& u, const Field& part, const Layout& L, const Slab& sl,
                       double gamma0, const MatConsts& mc, double* out, unsigned long long* fail,
                       cudaStream_t st);
// the n partial densities of the cell launch_csv_derive flagged (nothing if none)
void launch_csv_failcell(const Field& part, int n, const Layout& L, const Slab& sl,
                         const unsigned long long* fail, double* out, cudaStream_t st);

}  // namespace lfb
