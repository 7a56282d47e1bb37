// fused.h -- the fused Heun step (fused_step.cu): one kernel per time step.
#pragma once

#include "handle.h"

namespace lfb {

bool fused_supported(lf_handle* h);
// LF_PATH_AUTO resolves to the one-kernel step (fused_step.cu); below this many cells
// per slab the small-grid path (small.h) or the two-pass kernels are faster
// (tools/chunk_sweep.py: 256^2 38 us per step against 28 on the small-grid path,
// 320^2 42 against 48)
constexpr int64_t FUSED_AUTO_MIN_CELLS = (int64_t)5 << 14;
bool prefer_fused(lf_handle* h);
int fused_heun(lf_handle* h, double cfl, double time, double limit, int64_t step,
               double* outflow, lf_step_out* out);
int fused_advance(lf_handle* h, int nsteps, double cfl, double t_final, double* time,
                  int64_t* step, double* outflow, lf_step_out* per_step, int* taken);
int fused_time_steps(lf_handle* h, int nsteps, double cfl, double* kernel_ms, double* step_ms,
                     int* launches);
void fused_release(lf_handle* h);
// a fast-path step of this handle runs the two-pass kernels (else the one-kernel step)
bool twopass_selected(lf_handle* h);
int64_t fused_bytes(lf_handle* h);

}  // namespace lfb
