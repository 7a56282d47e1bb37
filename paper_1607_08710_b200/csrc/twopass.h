// twopass.h -- the two-pass (predictor / corrector) Heun step kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "fused_common.cuh"

namespace lfb {

#ifndef LF_TP_THREADS
#define LF_TP_THREADS 128
#endif
constexpr int TP_THREADS = LF_TP_THREADS;   // independent warps per block x 32
constexpr int TP_MAX_MATERIALS = 8;   // the two-pass material kernels (more: stage-wise)

struct PassArgs {
  const double* x;      // stage input, ghost-filled: U^n (predictor) or U* (corrector)
  const double* base;   // U^n (both passes update from U^n, solver.cpp:500,507)
  double* out;          // U* (predictor) or U^{n+1} (corrector)
  const double* fx;     // corrector: F^n x-faces  [4][ny][pitch]  face c = left face of column c
  const double* fy;     // corrector: F^n y-faces  [4][ny+1][pitch] face j = bottom face of row j
  double* fxo;          // predictor: F^n x-faces written
  double* fyo;          // predictor: F^n y-faces written
  int64_t pitch, fstride, fx_stride, fy_stride;
  int nx, ny;           // local interior
  int y0g, nyg;         // global row of local row 0, global rows
  int strips, rows_per_chunk;
  double gamma, gm1, beta, dx, dy;
  double cfl, limit;
  const StepCtl* ctl;
  StepAcc* acc;
  double* bnd;          // corrector: boundary faces [left 4*nyg | right 4*nyg | bottom 4*nx | top 4*nx]
  int heun;             // corrector: 1 the Heun average with the stage-a faces; 0 the single
                        // forward-Euler stage of time_order 1 (x = base = U^n, F alone,
                        // solver.cpp:510-514)
};

// Multimaterial operands of the two passes (csrc/twopass_mat_kernel.cu):
// partial densities with the field's Layout strides, and the predictor's
// per-material face fluxes (the corrector's stage-a term) with the F^n strides.
struct MatPassArgs {
  const double* px;      // partials of the pass input: P^n (predictor) or P* (corrector)
  const double* pbase;   // P^n
  double* pout;          // P* or P^{n+1}
  const double* mfx;     // corrector: stage-a material fluxes, x faces [K][ny][pitch]
  const double* mfy;     // corrector: y faces [K][ny+1][pitch]
  double* mfxo;          // predictor: written
  double* mfyo;
  int64_t mfx_stride, mfy_stride;
};

int tp_strips(int nx);
bool tp_fits(int64_t pitch, int ny);  // 32-bit offsets suffice for the slab
// resident warps per SM of the corrector kernel: k_pass (nmat 0) or k_pass_mat<nmat>
int tp_resident_warps(int nmat);
int tp_resident_warps_mat(int nmat);
// rows per chunk for a slab of ny rows: whole waves of independent warps
int tp_choose_rows(int nx, int ny, int sms, int warps_per_sm);
// exact: the kernels that complete shock-precursor quotients exactly (see
// twopass_kernel.cu); the plain ones flag such steps (StepAcc::fail = 2)
void launch_pass(const PassArgs& a, bool corr, bool muscl, bool exact, cudaStream_t st);
// LF_MATH_CONTRACT: the same kernels built with FMA contraction and reciprocal
// multiplication (twopass_contract.cu); held to the north-star tolerance
void launch_pass_contract(const PassArgs& a, bool corr, bool muscl, cudaStream_t st);
struct MatConsts;
void launch_pass_mat(const PassArgs& a, const MatPassArgs& m, const MatConsts& mc, bool corr,
                     bool muscl, cudaStream_t st);

}  // namespace lfb
