// small.h -- LF_PATH_SMALL (small_step.cu): the step loop of a small grid in one
// persistent thread-block cluster.
#pragma once

#include <cstdint>

#include "handle.h"

namespace lfb {

// LF_PATH_SMALL accepts grids up to this size (one cluster of at most 16 blocks;
// beyond it the other paths are faster by far); LF_PATH_AUTO takes it up to the
// measured crossovers (tools/small_sweep.py, profiles/r02_small_sweep.json: 2D 128^2
// 56 vs 62 us per step on the two-pass kernels, 256^2 196 vs 63; 1D 65536 cells 97 us).
constexpr int64_t SMALL_MAX_CELLS = (int64_t)1 << 22;
constexpr int64_t SMALL_AUTO_CELLS_1D = (int64_t)1 << 17;
constexpr int64_t SMALL_AUTO_CELLS_2D = (int64_t)1 << 14;
constexpr int SMALL_BATCH = 4096;   // steps per launch of lf_advance
constexpr int SMALL_MAX_PERIMETER = 1280;   // 2D: nx + ny (boundary faces in shared memory)

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
