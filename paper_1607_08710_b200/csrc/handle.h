// handle.h -- the object behind lf_handle (internal to the .so).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/lagflux_b200.h"
#include "kernels.h"

namespace lfb {

// One y-slab of the grid, resident on one GPU.
struct SlabState {
  int device = 0;
  Layout L;
  Slab sl;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;     // own_stream or a caller stream (lf_set_stream)
  double* U = nullptr;               // current state U^n (4 components, Layout)
  double* U2 = nullptr;              // next state (fused output / corrector output)
  // staged-path scratch (allocated on first use)
  double* Us = nullptr;              // predictor U*
  double* W = nullptr;               // primitives
  double* FX[2] = {nullptr, nullptr};
  double* FY[2] = {nullptr, nullptr};
  int64_t fx_stride = 0, fy_stride = 0;
  // boundary-face gather for the outflow diagnostic
  double* bnd = nullptr;             // device, 2 sets x 4 comps x (2 ny + 2 nx)
  double* bnd_host = nullptr;        // pinned mirror
  Scalars* scal = nullptr;           // device: [0] step scalars, [1] stage-2 scalars, [2..] spare
  Scalars* scal_host = nullptr;      // pinned mirror
  unsigned long long* aux = nullptr; // device scratch (Fourier maxima)
  cudaEvent_t ev_a = nullptr, ev_b = nullptr;
  // multimaterial (lf_set_materials; same Layout strides, n_mat components)
  double* P = nullptr;               // partial densities of U
  double* Ps = nullptr;              // partial densities of U* (predictor_mat_)
  double* Y[2] = {nullptr, nullptr}; // clamped fractions per slot (frac_)
  double* GC[2] = {nullptr, nullptr};  // mixed-cell gamma per slot (gamma_), 1 component
  double* USX[2] = {nullptr, nullptr}; // u* of the x faces of flux set k (ustar_x)
  double* USY[2] = {nullptr, nullptr}; // u* of the y faces (ustar_y)
  double* P2 = nullptr;              // two-pass path: partial densities of U^{n+1}
  double* MFX = nullptr;             // two-pass path: predictor's material x-face fluxes
  double* MFY = nullptr;             //                and y-face fluxes (F^n strides)

  Field field(double* p) const { return Field{p + L.origin(), L.pitch, L.fstride}; }
  FluxArr fluxx(int k) const { return FluxArr{FX[k], L.pitch, fx_stride}; }
  FluxArr fluxy(int k) const { return FluxArr{FY[k], L.pitch, fy_stride}; }
  FluxArr ustx(int k) const { return FluxArr{USX[k], L.pitch, fx_stride}; }
  FluxArr usty(int k) const { return FluxArr{USY[k], L.pitch, fy_stride}; }
};

struct Nccl;  // nccl.cpp

}  // namespace lfb

struct lf_handle {
  lf_desc d{};
  lfb::Consts k{};
  int dim2 = 1;
  int path = LF_PATH_AUTO;
  int math = LF_MATH_EXACT;   // arithmetic of the two-pass kernels (lf_set_math)
  std::vector<lfb::SlabState> slabs;
  // distributed (one slab per process)
  int rank = 0, nranks = 1;
  lfb::Nccl* nccl = nullptr;
  bool rate_valid = false;           // scal[0].rate_bits holds the rate of the current U
  void* fused = nullptr;             // lfb::FusedState (fused_step.cu)
  void* small = nullptr;             // lfb::SmallState (small_step.cu)
  lf_error err{};
  // multimaterial: material table and whether partial densities were uploaded
  lfb::MatConsts mc{};
  int partials_ready = 0;
  // the two-pass path has met shock-precursor velocities: use its exact kernels
  // until a new state is uploaded (set by a step with status 3)
  int tp_exact = 0;
  // LF_PATH_SMALL met a cell outside the fast arithmetic's box: its IEEE kernels until
  // a new state is uploaded
  int small_ieee = 0;
  // LF_PATH_AUTO: -1 undecided, 1 the two-pass scratch fits in device memory, 0 it
  // does not (then the one-kernel step, which needs two states, runs instead)
  int tp_mem_ok = -1;
};

namespace lfb {
// api.cu services used by the fused path
void fill_all_public(lf_handle* h, double* SlabState::*buf);
bool fill_local_public(lf_handle* h, double* SlabState::*buf);
void fill_partials_public(lf_handle* h, double* SlabState::*buf);
// conserved field and partial densities together (one fill launch per slab)
void fill_state_public(lf_handle* h, double* SlabState::*ubuf, double* SlabState::*pbuf);
void alloc_staged_public(lf_handle* h);
Scalars rate_of_current(lf_handle* h);
int staged_heun_public(lf_handle* h, double cfl, double time, double limit, int64_t step,
                       double* outflow, lf_step_out* out);
void fused_invalidate(lf_handle* h);
}  // namespace lfb
