// fused_common.cuh -- types shared by the fused-step kernels and their host driver.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace lfb {

#ifndef LF_FUSED_NC
#define LF_FUSED_NC 128
#endif
constexpr int FUSED_NC = LF_FUSED_NC;         // columns per strip (threads per warp group)
constexpr int FUSED_TXO = FUSED_NC - 8;       // output columns per strip
constexpr int FUSED_THREADS = 2 * FUSED_NC;   // predictor group + corrector group
constexpr unsigned long long NINF_KEY = ~0x7ff0000000000000ull;  // ~bits(+inf)

// Per-step control record, written by the host (first step) or k_finalize.
struct StepCtl {
  double time;                    // SolverState::time at the start of the step
  unsigned long long rate_bits;   // CFL rate of the state at the start of the step
  int done;                       // 1: skip (limit reached or an earlier step failed)
  int dtfail;                     // the rate check of this step's input failed
};

// Per-step accumulators: every field reduces with max (min via ~bits), so one
// atomicMax per warp and one NCCL max across ranks combine them exactly.
struct StepAcc {
  unsigned long long rate_next;   // CFL rate of U^{n+1}
  unsigned long long fail;        // any failure flag in this step
  unsigned long long nmin_rho;    // ~bits(min rho of U^{n+1})
  unsigned long long nmin_eint;   // ~bits(min e_int of U^{n+1})
  unsigned long long dtfail_next; // rate check of U^{n+1} failed
  unsigned long long nmin_p;      // ~bits(min p of U^{n+1}) from the partials (multimaterial)
  unsigned long long pad[2];
};
constexpr int STEP_ACC_WORDS = 6;

// Per-step record handed back to the host.
struct StepRec {
  double dt;
  double time;       // time after the step
  double min_rho;
  double min_eint;
  double min_p_mat;  // multimaterial min p (solver.cpp:522-538); +inf without
  int hits;
  int status;        // 0 ok, 1 failure flag (host diagnoses), 2 skipped (done),
                     // 3 precursor velocities: re-run with the exact two-pass kernels
};

// The step's constant divisors' shared reciprocals (face_fast.cuh FK), computed once
// per handle on the device (fused_make_fk: bit-identical to the kernel computing them)
// and passed as launch parameters: they live in the constant bank instead of registers.
struct FKBits {
  double gamma, gm1, beta;
  double rgm1_b, rgm1_y, rdx_b, rdx_y, rdy_b, rdy_y;
};

struct FusedArgs {
  const double* __restrict__ u;   // U^n, component 0 at (0, 0)
  double* __restrict__ un;        // U^{n+1}
  int64_t pitch, fstride;
  int nx, ny;                     // local interior
  int y0g;                        // global row of local row 0
  int nyg;                        // global rows
  int rows_per_chunk;
  int chunk0, chunk_step;         // row chunk of block y: chunk0 + blockIdx.y * chunk_step
  double gamma, gm1, beta, dx, dy;
  double cfl, limit;
  int bc_xlo, bc_xhi, bc_ylo, bc_yhi;
  int bottom_edge, top_edge;      // non-periodic domain edge at this slab's bottom / top
  const StepCtl* ctl;
  StepAcc* acc;
  double* bnd;                    // [left 4*nyg | right 4*nyg | bottom 4*nx | top 4*nx]
  FKBits fk;                      // make_fk(gamma, gm1, beta, dx, dy) of this build's arithmetic
};

size_t fused_smem_bytes();
// make_fk on the device in each build's arithmetic (the contract build refines less)
FKBits fused_make_fk(double gamma, double gm1, double beta, double dx, double dy);
FKBits fused_make_fk_contract(double gamma, double gm1, double beta, double dx, double dy);
void fused_configure();
int fused_blocks_per_sm();   // resident blocks of k_fused_step (after fused_configure)
void launch_fused_step(const FusedArgs& a, bool muscl, dim3 grid, cudaStream_t st);
// LF_MATH_CONTRACT (fused_contract.cu)
void fused_configure_contract();
void launch_fused_step_contract(const FusedArgs& a, bool muscl, dim3 grid, cudaStream_t st);
// dt, time, diagnostics and the next control record of a step; outflow_zero:
// every axis periodic, the outflow update is the += of +0.0 sums done here
void launch_finalize(const StepCtl* ctl, StepAcc* acc, StepCtl* nxt, StepRec* rec,
                     double* outflow, bool outflow_zero, double dx, double dy, double cfl,
                     double limit, double t_final, cudaStream_t st);
// the boundary-outflow sums of the step recorded in `rec` (no-op unless it completed)
void launch_outflow(const StepRec* rec, const double* bnd, double* outflow, int nx, int nyg,
                    bool sum_x, bool sum_y, double dx, double dy, cudaStream_t st);
void launch_acc_init(StepAcc* acc, cudaStream_t st);

}  // namespace lfb
