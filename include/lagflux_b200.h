/*
 * lagflux_b200.h -- C ABI of the B200-native Lagrange-flux time step.
 *
 * Drop-in boundary for lagflux::LagfluxSolver (reference
 * /root/reference/proj/include/lagflux/solver.hpp:78-131).  A handle owns the
 * device copy of one SolverState::field plus all scratch; the field stays
 * resident on the GPU between steps (upload once, download for dumps).  Plain
 * pointers and sizes only; errors are returned as an int status plus a record
 * (the reference's exceptions, error.hpp:9-64).  One host thread per handle,
 * like the reference object (not thread-safe, mutable scratch).
 *
 * Entry point                      replaces (reference file:line)
 *   lf_create / lf_destroy         LagfluxSolver::LagfluxSolver  solver.cpp:61-88
 *   lf_create_dist                 (new) one y-slab per rank, NCCL halos + dt max
 *   lf_upload / lf_download        SolverState::field host <-> device (CellField,
 *                                  grid.hpp:73-92; ghosted row-major, ld = nxt)
 *   lf_compute_dt                  LagfluxSolver::compute_dt     solver.cpp:434-480
 *   lf_euler_stage                 LagfluxSolver::euler_stage    solver.cpp:482-487
 *   lf_heun_step                   LagfluxSolver::heun_step      solver.cpp:489-546
 *   lf_advance                     the run.cpp:180-210 step loop with the dt /
 *                                  time / diagnostics kept on the device
 *   lf_init_fourier                (new) on-device seeded smooth-flow IC (BASELINE 4-5)
 *   lf_init_regions                initialize_hydro, InitKind::regions  run.cpp:29-78
 *   lf_interior_totals             interior_totals(grid, state.field)  grid.cpp:122-133
 *   lf_edge_flux                   edge_flux (free function)      solver.cpp:45-53,
 *                                  solver.hpp:31-37 (batched, on the device)
 *   lf_last_error                  the exception object (what(), PositivityError fields)
 *   lf_write_field_csv             field_csv + write_text_file   csv.cpp:26-83, run.cpp:162-168
 *   lf_write_field_csv_async /     (new) the same dump, snapshotted in stream order and
 *   lf_wait_dumps                  copied / formatted / written on a host thread
 *   lf_set_materials               the constructor's `const MaterialSet*` (solver.cpp:61-88)
 *                                  with make_material_set's checks (multimat.cpp:7-15)
 *   lf_upload_partials /           MaterialCells::partial host <-> device
 *   lf_download_partials           (multimat.hpp:21-30); heun_step(state, controls,
 *                                  limit, &mat) is lf_heun_step once they are resident
 */
#ifndef LAGFLUX_B200_H
#define LAGFLUX_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LF_ABI_VERSION 1

/* BcKind (grid.hpp:51) */
enum { LF_TRANSMISSIVE = 0, LF_REFLECTIVE = 1, LF_PERIODIC = 2 };

/* status / error kinds */
enum {
  LF_OK = 0,
  LF_ERR_CONFIG = 1,       /* ConfigError */
  LF_ERR_DT_STATE = 2,     /* InvalidStateError in compute_dt (solver.cpp:471-475) */
  LF_ERR_DT_NONPOS = 3,    /* Error "non-positive time step" (solver.cpp:478) */
  LF_ERR_PRIMITIVE = 4,    /* InvalidStateError in build_primitives (solver.cpp:164-170) */
  LF_ERR_TRACE = 5,        /* InvalidStateError in compute_fluxes (solver.cpp:245-255) */
  LF_ERR_POSITIVITY = 6,   /* PositivityError in apply_update (solver.cpp:310-326) */
  LF_ERR_DEVICE = 7,       /* CUDA / NCCL failure (no reference counterpart) */
  LF_ERR_ARGUMENT = 8,     /* invalid argument to this ABI */
  LF_ERR_FRACTION = 9      /* InvalidStateError in fill_all_ghosts (solver.cpp:122-127) */
};

/* Heun-step implementation for lf_heun_step / lf_advance (all give identical results):
 *   AUTO     SMALL for grids of up to 2^17 cells in 2D (2^15 with materials) and every 1D
 *            grid (up to 2^22 cells) on one device (BASELINE config 1); FUSED for every
 *            larger 2D slab (Heun, no materials: BASELINE configs 2-5) -- always from 2^23
 *            cells (2^22 in LF_MATH_CONTRACT), and below that from 5 * 2^14 cells when nx
 *            fills its 120-column strips to 80 % or more; TWOPASS for narrow mid-size
 *            grids, for time_order 1 and for materials; FUSED also when the two-pass
 *            scratch does not fit in device memory.  lf_resolved_path reports the choice.
 *   FUSED    one kernel per step (U^n read once, U^{n+1} written once)
 *   STAGED   the reference's phase structure, one kernel per loop (also the
 *            exact diagnosis path for every failure, euler_stage and more than 8
 *            materials)
 *   TWOPASS  predictor and corrector as two warp-independent streaming kernels
 *            (1-8 materials included)
 *   SMALL    a whole lf_advance batch (up to 4096 steps) in one launch of one thread-block
 *            cluster (up to 16 blocks), or of one cooperative grid beyond 16 x 224 cells
 *            (batches of 256 steps): up to 8 materials, one slab, nx >= 2 (and ny >= 2
 *            in 2D), up to 2^22 cells; the reference's bits */
enum { LF_PATH_AUTO = 0, LF_PATH_FUSED = 1, LF_PATH_STAGED = 2, LF_PATH_TWOPASS = 3,
       LF_PATH_SMALL = 4 };
/* Arithmetic of the fast kernels (two-pass and fused).  LF_MATH_EXACT (default): the
 * reference's operation order without contraction, bit-identical to it.
 * LF_MATH_CONTRACT: FMA contraction and quotients as products by a refined
 * reciprocal -- fewer fp64 instructions, results within the north star's
 * tolerance of the reference (relative L1 <= 1e-10 per conserved field, dt to
 * 1e-12), not bit-identical.  The stage-wise kernels, the material kernels and the
 * re-run of every step the fast kernels flag always compute in LF_MATH_EXACT. */
enum { LF_MATH_EXACT = 0, LF_MATH_CONTRACT = 1 };

typedef struct lf_desc {
  int dim;              /* 1 or 2 (CartesianGrid::dim) */
  int nx, ny;           /* global interior cells (ny = 1 in 1D) */
  double dx, dy;        /* CartesianGrid::dx, dy (pass them; do not recompute) */
  double x0, y0;
  double gamma;         /* PerfectGasEos::gamma */
  double beta;          /* LimiterParams::beta */
  int spatial_order;    /* SchemeParams::spatial_order (1 or 2) */
  int time_order;       /* SchemeParams::time_order (1 or 2) */
  int bc[4];            /* x_low, x_high, y_low, y_high */
} lf_desc;

typedef struct lf_error {
  int kind;
  int axis;             /* LF_ERR_TRACE: 0 x-face, 1 y-face */
  int64_t i, j;         /* cell / face indices exactly as the reference reports them */
  int64_t step;
  double dt;
  double value;         /* offending density / pressure (LF_ERR_PRIMITIVE), rho (POSITIVITY) */
  double value2;        /* internal energy density (POSITIVITY) */
  char message[320];    /* the reference's what() text */
} lf_error;

typedef struct lf_step_out {
  double dt;
  int hits_limit;
  double time;          /* SolverState::time after the step */
  int64_t step;         /* SolverState::step after the step */
  double min_rho;       /* StepDiagnostics::min_rho */
  double min_p;         /* StepDiagnostics::min_p */
} lf_step_out;

typedef struct lf_handle lf_handle;

int lf_abi_version(void);

/* Single process.  ndev == 1: one GPU.  ndev > 1: the grid is split into ndev
 * y-slabs driven from this process (devices may repeat: several slabs on one
 * GPU run the identical slab code path, which is how the decomposition is
 * checked on a 1-GPU machine). */
int lf_create(const lf_desc* desc, const int* devices, int ndev, lf_handle** out);

/* One rank of an nranks-way y-slab decomposition (one process per GPU).
 * nccl_id: 128 bytes from lf_nccl_unique_id() on rank 0, broadcast by the caller. */
int lf_nccl_unique_id(void* id128);
int lf_create_dist(const lf_desc* desc, int device, int rank, int nranks, const void* nccl_id,
                   lf_handle** out);

void lf_destroy(lf_handle* h);

/* Rows [row0, row0 + nrows) of this handle's slab, as global rows. */
int lf_local_rows(lf_handle* h, int* row0, int* nrows);
/* The y-slab partition used by lf_create / lf_create_dist (host only, no GPU):
 * rank's first global row and row count for ny rows over nranks slabs. */
int lf_slab_partition(int ny, int nranks, int rank, int* row0, int* nrows);

/* Host <-> device field transfer in the reference's ghosted layout:
 * component c of cell (i, j) (total indices, ghosts included) at field[c][j*ld + i],
 * ld >= nx + 4.  Distributed handles transfer their own slab rows only, at the
 * same global positions; a rank that allocates only its own rows (total rows
 * y0 .. y0 + rows + 3 in 2D) passes component pointers biased by -y0 * ld, and
 * fill_ghosts = 0 (lf_local_rows gives y0, rows).  Download writes interior cells; fill_ghosts != 0
 * additionally applies the boundary conditions to the host ghosts
 * (apply_boundary, grid.cpp:116-121). */
int lf_upload(lf_handle* h, double* const field[4], int64_t ld);
int lf_download(lf_handle* h, double* const field[4], int64_t ld, int fill_ghosts);

/* Multimaterial partial-density transport (solver.cpp:90-129, 331-404, 519-540).
 * lf_set_materials: once, before stepping; n in [1, 16], gammas in (1, 3]
 * (LF_ERR_CONFIG with make_material_set's message otherwise).  With a material
 * set every Heun step also advects the n partial densities rho*y_k, uses the
 * mixed-cell gamma of each cell (each face side its own EOS), reports a fraction
 * outside [0,1] beyond round-off as LF_ERR_FRACTION, and returns the min
 * pressure from the fresh partials.  The two-pass material kernels run these
 * steps for 1-8 materials in 2D, the small-grid path for 1D and small 2D grids, the
 * stage-wise kernels for more than 8.
 * Partials: n arrays in the ghosted field layout (partials[k][j*ld + i],
 * ld >= nx + 4); interior cells are transferred. */
int lf_set_materials(lf_handle* h, int n, const double* gammas);
int lf_upload_partials(lf_handle* h, double* const* partials, int64_t ld);
int lf_download_partials(lf_handle* h, double* const* partials, int64_t ld);

/* field_csv (csv.cpp:26-83) of the current state written to `path` (run.cpp's
 * dump, write_text_file): "# config <digest hex> time <t>", the column line, then
 * x[,y],rho,u[,v],p,e_internal[,y1..yn] per interior cell, %.17g, row-major.
 * The per-cell quantities are derived on the device with the reference's
 * expressions; `threads` host threads format rows in parallel (0: all cores).
 * A mass fraction beyond round-off fails with LF_ERR_FRACTION (clamped_fraction's
 * text) and writes nothing.  A distributed handle writes its own rows only. */
int lf_write_field_csv(lf_handle* h, const char* path, uint64_t digest, double time,
                       int threads);

/* lf_write_field_csv without the wait: the columns of the current state are derived
 * into a device snapshot in stream order (later steps do not change the dump), and a
 * host thread copies them back (on a stream of its own), checks the fractions and
 * formats / writes the file while the caller keeps stepping.  Same bytes as
 * lf_write_field_csv at the same state.  Errors found at this call (null path,
 * missing material storage) return here; the dump's own (LF_ERR_FRACTION, I/O) are
 * returned by lf_wait_dumps, which joins every pending dump of the handle (first
 * error wins).  lf_destroy waits for pending dumps.  The snapshot holds
 * (5 + materials) x interior doubles of device memory until its copy ends. */
int lf_write_field_csv_async(lf_handle* h, const char* path, uint64_t digest, double time,
                             int threads);
int lf_wait_dumps(lf_handle* h);

/* Region initial state generated on the device (initialize_hydro, run.cpp:29-78,
 * InitKind::regions): regions = nreg x {x_min, x_max, y_min, y_max, rho, u, v, p,
 * material (1-based)}; every interior cell centre must lie in exactly one region
 * (LF_ERR_CONFIG with run.cpp's message otherwise).  Energy from the material's
 * gamma (the eos gamma without a material set); with materials the partial
 * densities are set too (rho in the cell's material, 0 elsewhere). */
int lf_init_regions(lf_handle* h, const double* regions, int nreg);

/* Seeded smooth-perturbation initial state (BASELINE configs 4-5), generated on the device. */
int lf_init_fourier(lf_handle* h, uint64_t seed);

int lf_compute_dt(lf_handle* h, double cfl, double time, double limit_time, double* dt);
/* state <- euler_stage(state, dt) (the reference writes `out`; the C++ adapter
 * uploads `in` and downloads into `out`) */
int lf_euler_stage(lf_handle* h, double dt, int64_t step);
/* boundary_outflow: SolverState::boundary_outflow, updated in place (may be NULL). */
int lf_heun_step(lf_handle* h, double cfl, double time, double limit_time, int64_t step,
                 double* boundary_outflow, lf_step_out* out);
/* Up to nsteps Heun steps while time < t_final (run.cpp:180), dt/time on the
 * device and no host synchronisation until the end.  per_step: nsteps records
 * (may be NULL).  *taken receives the steps executed. */
int lf_advance(lf_handle* h, int nsteps, double cfl, double t_final, double* time,
               int64_t* step, double* boundary_outflow, lf_step_out* per_step, int* taken);

/* interior_totals (grid.cpp:122-133) of the device-resident state: per
 * component, the row-major ordered sum over the interior times the cell volume,
 * bit-equal to the reference.  A distributed handle chains the sums over the
 * ranks in row order and returns the global totals on every rank (collective). */
int lf_interior_totals(lf_handle* h, double tot[4]);

/* The reference's free edge_flux(w_minus, w_plus, n, eos_minus, eos_plus)
 * (solver.cpp:45-53) for n faces on `device`: w_* = n x {rho, u, v, p},
 * normals = n x {nx, ny}, gamma_* = n per-side gammas; flux = n x {mass, mom_x,
 * mom_y, energy}; contact (may be NULL) = n x {p*, u*} of lagrangian_hll.
 * Bit-equal to the reference (general normals, no axis specialisation).  A
 * non-physical trace returns LF_ERR_PRIMITIVE with sound_speed's message for the
 * smallest such face (err->i = face index; err may be NULL). */
int lf_edge_flux(int64_t n, const double* w_minus, const double* w_plus, const double* normals,
                 const double* gamma_minus, const double* gamma_plus, double* flux,
                 double* contact, int device, lf_error* err);

int lf_last_error(lf_handle* h, lf_error* err);

/* ---- measurement / tuning hooks (used by bench.py; no reference counterpart) ---- */
int lf_set_stream(lf_handle* h, void* cuda_stream);   /* NULL: the handle's own stream */
int lf_set_path(lf_handle* h, int path);               /* LF_PATH_* */
int lf_set_math(lf_handle* h, int math);               /* LF_MATH_* (default EXACT) */
/* The path the next step takes: LF_PATH_TWOPASS, LF_PATH_FUSED, LF_PATH_STAGED or
 * LF_PATH_SMALL.
 * LF_PATH_AUTO runs the two-pass kernels when their scratch (four more states'
 * worth) fits in device memory, else the one-kernel step (e.g. 32768^2 on one GPU). */
int lf_resolved_path(lf_handle* h, int* path);
/* Time n device-resident steps with CUDA events around each launch of the
 * dominant kernel.  kernel_ms: summed kernel time; step_ms: whole-loop time. */
int lf_time_steps(lf_handle* h, int nsteps, double cfl, double* kernel_ms, double* step_ms,
                  int* kernel_launches);
int lf_device_bytes(lf_handle* h, int64_t* bytes);
/* The device's own ghost fill of the current state (the kernels' fill, not the
 * host apply_boundary of lf_download), downloaded with the reference's two
 * ghost layers (corners included) into the ghosted row-major layout. */
int lf_download_ghosted(lf_handle* h, double* const field[4], int64_t ld);
/* Kernels launched by this library in this process so far (all handles). */
int lf_launch_count(lf_handle* h, int64_t* launches);
/* One scalar per interior cell: the CFL rate field is not kept; this returns the
 * max rate of the current state (diagnostic for tests). */
int lf_max_rate(lf_handle* h, double* rate);
/* Device self-check of the exact fast-path division / sqrt / limiter on n random
 * operands (csrc/selftest.cu).  counts[10] = {tested, div valid, div mismatches,
 * shared-reciprocal mismatches, sqrt valid, sqrt mismatches, limiter mismatches,
 * tiny-dividend divisions tested, their mismatches vs '/', their out-of-range}. */
int lf_selftest_fastmath(int64_t n, uint64_t seed, int64_t* counts);
/* Device self-check of the cell box (csrc/face_fast.cuh): n random faces whose
 * four stencil cells lie in the box, extremes and one-ulp neighbours
 * over-represented; every division / square root of the face solves and of the
 * primitives must pass its fast-path range check.  counts[2] = {faces solved,
 * faces with a failed range check}. */
int lf_selftest_box(int64_t n, uint64_t seed, int64_t* counts);
/* Device self-check of the corrector epilogue's box (csrc/face_fast.cuh,
 * cell_epilogue_box): n random updated cells at the box edges; counts[3] =
 * {cells the box accepts, of those failing a per-operation check, of those
 * whose rate or e_int differs}. */
int lf_selftest_epilogue(int64_t n, uint64_t seed, int64_t* counts);
/* Measured fp64 throughput of `device` (csrc/fp64_peak.cu), the fp64 roof of the
 * step: out[6] = {DFMA burst, DFMA sustained, DMUL burst, DMUL sustained, DADD
 * burst, DADD sustained} in fp64 thread instructions per second (a DFMA counts
 * once).  Burst: one launch of ~burst_ms; sustained: back-to-back launches for
 * ~sustain_ms (0: burst only). */
int lf_fp64_peak(int device, double burst_ms, double sustain_ms, double* out);

#ifdef __cplusplus
}
#endif

#endif /* LAGFLUX_B200_H */
