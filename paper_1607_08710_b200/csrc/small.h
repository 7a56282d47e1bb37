// small.h -- LF_PATH_SMALL (small_step.cu): the step loop of a small grid in one
// persistent thread-block cluster.
#pragma once

#include <cstdint>

#include "handle.h"

namespace lfb {

// LF_PATH_SMALL accepts grids up to this size; LF_PATH_AUTO takes it up to the measured
// crossovers (tools/small_sweep.py, profiles/r02_small_sweep.json): in 2D against the
// two-pass kernels (2^17 cells: 51 vs 64 us per step; 512^2: 95 vs 74), in 1D always
// (the stage-wise kernels: 2.4 ms per step at 2^18 cells against 52 us).  Up to one
// cluster's worth of cells (16 x 224) the path runs as one thread-block cluster, beyond
// it as a cooperative grid of one block per SM (small_step.cu).
constexpr int64_t SMALL_MAX_CELLS = (int64_t)1 << 22;
constexpr int64_t SMALL_AUTO_CELLS_1D = SMALL_MAX_CELLS;
constexpr int64_t SMALL_AUTO_CELLS_2D = (int64_t)1 << 17;
// with materials (the IEEE closures of every stencil cell): 2D to 2^15 cells
// (tools/small_mat_sweep.py: the triple point at 70x30 / 256x110 84 us per step against
// 107 / 110 on the two-pass material kernels, 512x220 296 vs 111); 1D always (a 400-cell
// contact: 27 vs 160 us stage-wise)
constexpr int64_t SMALL_AUTO_CELLS_2D_MAT = (int64_t)1 << 15;
constexpr int SMALL_BATCH = 4096;   // steps per launch of lf_advance
constexpr int SMALL_GRID_BATCH = 256;   // grid mode (its boundary-face history per step)
constexpr int SMALL_MAX_PERIMETER = 1280;   // cluster mode, 2D: nx + ny (boundary faces
                                            // of two steps in shared memory, 160 KB)

bool small_supported(lf_handle* h);
bool prefer_small(lf_handle* h);
void small_invalidate(lf_handle* h);
void small_release(lf_handle* h);
int small_heun(lf_handle* h, double cfl, double time, double limit, int64_t step,
               double* outflow, lf_step_out* out);
int small_advance(lf_handle* h, int nsteps, double cfl, double t_final, double* time,
                  int64_t* step, double* outflow, lf_step_out* per_step, int* taken);
int small_time_steps(lf_handle* h, int nsteps, double cfl, double* kernel_ms, double* step_ms,
                     int* launches);

}  // namespace lfb
