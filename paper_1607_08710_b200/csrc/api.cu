// api.cu -- the C ABI (include/lagflux_b200.h) over the device kernels.
//
// Host orchestration of LagfluxSolver::heun_step (solver.cpp:489-546):
//   fill ghosts -> (halo exchange between y-slabs) -> CFL rate -> predictor ->
//   fill ghosts of U* -> corrector -> diagnostics and boundary outflow,
// reporting failures with the reference's exception kinds, indices and text.
#include <cuda_runtime.h>

#include <algorithm>
#include <charconv>
#include <cinttypes>
#include <climits>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <limits>
#include <new>
#include <stdexcept>
#include <string>
#include <thread>
#include <mutex>
#include <memory>
#include <map>
#include <vector>

#include "fused.h"
#include "small.h"
#include "handle.h"
#include "host_util.h"
#include "nccl_comm.h"
#include "trace.h"
#include "twopass.h"

using namespace lfb;

namespace {

struct DeviceFail {
  std::string what;
};

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess)                                                           \
      throw DeviceFail{std::string(#x) + ": " + cudaGetErrorString(e_)};             \
  } while (0)

void clear_err(lf_error* e) {
  std::memset(e, 0, sizeof *e);
  e->i = e->j = e->step = -1;
}

int set_err(lf_handle* h, int kind, const char* fmt, ...) __attribute__((format(printf, 3, 4)));
int set_err(lf_handle* h, int kind, const char* fmt, ...) {
  clear_err(&h->err);
  h->err.kind = kind;
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(h->err.message, sizeof h->err.message, fmt, ap);
  va_end(ap);
  return kind;
}

std::string fmt_f(double v) {  // std::to_string(double) == "%f"
  char b[64];
  snprintf(b, sizeof b, "%f", v);
  return b;
}

double bits_to_double(unsigned long long b) {
  double d;
  std::memcpy(&d, &b, sizeof d);
  return d;
}

// ---------------------------------------------------------------- allocation
void alloc_state(SlabState& s) {
  CK(cudaSetDevice(s.device));
  const size_t bytes = (size_t)s.L.alloc * sizeof(double);
  CK(cudaMalloc(&s.U, bytes));
  CK(cudaMalloc(&s.U2, bytes));
  CK(cudaMemsetAsync(s.U, 0, bytes, s.stream));
  CK(cudaMemsetAsync(s.U2, 0, bytes, s.stream));
  CK(cudaMalloc(&s.scal, 4 * sizeof(Scalars)));
  CK(cudaHostAlloc(&s.scal_host, 4 * sizeof(Scalars), cudaHostAllocDefault));
  CK(cudaMalloc(&s.aux, 8 * sizeof(unsigned long long)));
  CK(cudaEventCreate(&s.ev_a));
  CK(cudaEventCreate(&s.ev_b));
}

void alloc_staged(SlabState& s) {
  if (s.Us) return;
  CK(cudaSetDevice(s.device));
  const size_t bytes = (size_t)s.L.alloc * sizeof(double);
  CK(cudaMalloc(&s.Us, bytes));
  CK(cudaMalloc(&s.W, bytes));
  CK(cudaMemsetAsync(s.Us, 0, bytes, s.stream));
  CK(cudaMemsetAsync(s.W, 0, bytes, s.stream));
  s.fx_stride = s.L.pitch * (int64_t)s.L.ny;
  s.fy_stride = s.L.pitch * (int64_t)(s.L.ny + 1);
  for (int k = 0; k < 2; ++k) {
    CK(cudaMalloc(&s.FX[k], 4 * s.fx_stride * sizeof(double)));
    CK(cudaMalloc(&s.FY[k], 4 * s.fy_stride * sizeof(double)));
  }
  const size_t nb = 2 * 4 * (size_t)(2 * s.L.ny + 2 * s.L.nx);
  CK(cudaMalloc(&s.bnd, nb * sizeof(double)));
  CK(cudaHostAlloc(&s.bnd_host, nb * sizeof(double), cudaHostAllocDefault));
}

void free_slab(SlabState& s) {
  cudaSetDevice(s.device);
  cudaFree(s.U);
  cudaFree(s.U2);
  cudaFree(s.Us);
  cudaFree(s.W);
  for (int k = 0; k < 2; ++k) {
    cudaFree(s.FX[k]);
    cudaFree(s.FY[k]);
  }
  cudaFree(s.bnd);
  cudaFreeHost(s.bnd_host);
  cudaFree(s.scal);
  cudaFreeHost(s.scal_host);
  cudaFree(s.aux);
  cudaFree(s.P);
  cudaFree(s.Ps);
  cudaFree(s.P2);
  cudaFree(s.MFX);
  cudaFree(s.MFY);
  for (int k = 0; k < 2; ++k) {
    cudaFree(s.Y[k]);
    cudaFree(s.GC[k]);
    cudaFree(s.USX[k]);
    cudaFree(s.USY[k]);
  }
  if (s.ev_a) cudaEventDestroy(s.ev_a);
  if (s.ev_b) cudaEventDestroy(s.ev_b);
  if (s.own_stream) cudaStreamDestroy(s.own_stream);
}

// ---------------------------------------------------------------- validation
int validate_desc(lf_handle* h, const lf_desc* d) {
  if (d->dim != 1 && d->dim != 2) return set_err(h, LF_ERR_CONFIG, "dimension must be 1 or 2");
  if (d->nx < 1 || d->ny < 1) return set_err(h, LF_ERR_CONFIG, "grid has no interior cells");
  if (d->dim == 1 && d->ny != 1) return set_err(h, LF_ERR_CONFIG, "a 1D grid has ny = 1");
  for (int b = 0; b < 4; ++b)
    if (d->bc[b] < 0 || d->bc[b] > 2) return set_err(h, LF_ERR_CONFIG, "unknown boundary kind");
  // validate_boundary, grid.cpp:65-70
  if ((d->bc[0] == LF_PERIODIC) != (d->bc[1] == LF_PERIODIC))
    return set_err(h, LF_ERR_CONFIG, "periodic boundary in x must be set on both sides");
  if (d->dim == 2 && (d->bc[2] == LF_PERIODIC) != (d->bc[3] == LF_PERIODIC))
    return set_err(h, LF_ERR_CONFIG, "periodic boundary in y must be set on both sides");
  if (d->spatial_order != 1 && d->spatial_order != 2)
    return set_err(h, LF_ERR_CONFIG, "spatial_order must be 1 or 2");
  if (d->time_order != 1 && d->time_order != 2)
    return set_err(h, LF_ERR_CONFIG, "time_order must be 1 or 2");
  return 0;
}

void init_common(lf_handle* h, const lf_desc* d) {
  h->d = *d;
  h->dim2 = d->dim == 2;
  h->k.gamma = d->gamma;
  h->k.gm1 = d->gamma - 1.0;
  h->k.beta = d->beta;
  h->k.dx = d->dx;
  h->k.dy = d->dy;
}

// Split ny rows into n slabs (first slabs take the remainder).
void slab_rows(int ny, int n, int s, int* y0, int* rows) {
  const int base = ny / n, rem = ny % n;
  *rows = base + (s < rem ? 1 : 0);
  *y0 = s * base + std::min(s, rem);
}

// ---------------------------------------------------------------- halos
// Copy the NG boundary rows (full padded width, x ghosts included, so corners
// wrap as in grid.cpp:98-113) between neighbouring in-process slabs.
void exchange_local(lf_handle* h, double* SlabState::*buf, int ncomp = 4) {
  const int n = (int)h->slabs.size();
  if (n == 1) return;
  const bool periodic = h->d.bc[2] == LF_PERIODIC;
  for (auto& s : h->slabs) {
    CK(cudaSetDevice(s.device));
    CK(cudaEventRecord(s.ev_a, s.stream));
  }
  for (int t = 0; t < n; ++t) {
    SlabState& dst = h->slabs[t];
    CK(cudaSetDevice(dst.device));
    for (int side = 0; side < 2; ++side) {
      int src_i = side == 0 ? t - 1 : t + 1;
      if (src_i < 0 || src_i >= n) {
        if (!periodic) continue;
        src_i = (src_i + n) % n;
      }
      SlabState& src = h->slabs[src_i];
      CK(cudaStreamWaitEvent(dst.stream, src.ev_a, 0));
      const int src_row = side == 0 ? src.L.ny - NG : 0;
      const int dst_row = side == 0 ? -NG : dst.L.ny;
      for (int c = 0; c < ncomp; ++c) {
        const double* sp = (src.*buf) + src.L.origin() + c * src.L.fstride +
                           (int64_t)src_row * src.L.pitch - NG;
        double* dp = (dst.*buf) + dst.L.origin() + c * dst.L.fstride +
                     (int64_t)dst_row * dst.L.pitch - NG;
        CK(cudaMemcpy2DAsync(dp, dst.L.pitch * sizeof(double), sp, src.L.pitch * sizeof(double),
                             (size_t)(dst.L.nx + 2 * NG) * sizeof(double), NG,
                             cudaMemcpyDefault, dst.stream));
      }
    }
  }
  // the copies read the neighbours' rows: nobody may overwrite them before done
  for (auto& s : h->slabs) {
    CK(cudaSetDevice(s.device));
    CK(cudaEventRecord(s.ev_b, s.stream));
  }
  for (auto& s : h->slabs)
    for (auto& o : h->slabs) {
      if (&o == &s) continue;
      CK(cudaSetDevice(s.device));
      CK(cudaStreamWaitEvent(s.stream, o.ev_b, 0));
    }
}

// Ghost cells of `buf` on every slab: x sides, halo rows, then y sides at the
// domain edges (grid.cpp:79-113 order).  A conserved field by default; the
// partial densities are ncomp = n_mat even-parity components (odd = -1).
// buf2 (optional): ncomp2 even-parity components (partial densities) filled in
// the same launch when the single-launch fill applies.
void fill_all(lf_handle* h, double* SlabState::*buf, int ncomp = 4, int odd_x = 1,
              int odd_y = 2, double* SlabState::*buf2 = nullptr, int ncomp2 = 0) {
  const int xbc[4] = {h->d.bc[0], h->d.bc[1], h->d.bc[2], h->d.bc[3]};
  bool one = true;  // the single-launch fill applies (every ghost source is interior)
  for (auto& s : h->slabs) one = one && s.L.nx >= NG && (!h->dim2 || s.L.ny >= NG);
  if (one) {
    // the y sides read only their own slab's rows, so they precede the halo
    // exchange (which carries the x ghosts of the neighbours' rows)
    for (auto& s : h->slabs) {
      CK(cudaSetDevice(s.device));
      const Field f2 = buf2 ? s.field(s.*buf2) : Field{};
      launch_fill_xy(s.field(s.*buf), s.L, xbc, s.sl, h->dim2, s.stream, ncomp, odd_x, odd_y,
                     buf2 ? &f2 : nullptr, ncomp2);
    }
    if (h->nccl) {
      nccl_exchange_halos(h, buf, ncomp);
      if (buf2) nccl_exchange_halos(h, buf2, ncomp2);
    } else {
      exchange_local(h, buf, ncomp);
      if (buf2) exchange_local(h, buf2, ncomp2);
    }
    CK(cudaGetLastError());
    return;
  }
  if (buf2) {
    fill_all(h, buf, ncomp, odd_x, odd_y);
    fill_all(h, buf2, ncomp2, -1, -1);
    return;
  }
  for (auto& s : h->slabs) {
    CK(cudaSetDevice(s.device));
    launch_fill_x(s.field(s.*buf), s.L, xbc, s.stream, ncomp, odd_x);
  }
  if (h->nccl)
    nccl_exchange_halos(h, buf, ncomp);
  else
    exchange_local(h, buf, ncomp);
  for (auto& s : h->slabs) {
    if (!h->dim2 || !(s.sl.fill_lo || s.sl.fill_hi)) continue;
    CK(cudaSetDevice(s.device));
    launch_fill_y_only(s.field(s.*buf), s.L, xbc, s.sl, s.stream, ncomp, odd_y);
  }
  CK(cudaGetLastError());
}

void fill_partials(lf_handle* h, double* SlabState::*buf) { fill_all(h, buf, h->mc.n, -1, -1); }

void sync_all(lf_handle* h) {
  for (auto& s : h->slabs) {
    CK(cudaSetDevice(s.device));
    CK(cudaStreamSynchronize(s.stream));
  }
}

// Read back scalars slot `slot` of every slab and combine them (max rate, min
// everything else) -- across ranks with one NCCL all-reduce.
Scalars combined_scalars(lf_handle* h, int slot) {
  Scalars r{};
  bool first = true;
  for (auto& s : h->slabs) {
    CK(cudaSetDevice(s.device));
    CK(cudaMemcpyAsync(&s.scal_host[slot], &s.scal[slot], sizeof(Scalars),
                       cudaMemcpyDeviceToHost, s.stream));
  }
  sync_all(h);
  for (auto& s : h->slabs) {
    const Scalars& x = s.scal_host[slot];
    if (first) {
      r = x;
      first = false;
      continue;
    }
    r.rate_bits = std::max(r.rate_bits, x.rate_bits);
    r.fail_dt = std::min(r.fail_dt, x.fail_dt);
    r.fail_prim = std::min(r.fail_prim, x.fail_prim);
    r.fail_trace = std::min(r.fail_trace, x.fail_trace);
    r.fail_update = std::min(r.fail_update, x.fail_update);
    r.min_rho_bits = std::min(r.min_rho_bits, x.min_rho_bits);
    r.min_eint_bits = std::min(r.min_eint_bits, x.min_eint_bits);
    r.fail_frac = std::min(r.fail_frac, x.fail_frac);
    r.min_p_key = std::min(r.min_p_key, x.min_p_key);
  }
  if (h->nccl) nccl_combine_scalars(h, &r);
  return r;
}

// Fetch the 4 components of local cell (i, j) of `buf` on the slab owning global row jg.
// Distributed handles: every rank reaches the error report (the failing index is
// all-reduced), only the owner holds the cell -- the owner's bits win an all-reduce
// max in which the other ranks contribute 0 (collective; +0.0 is all-zero bits).
static bool fetch_local(lf_handle* h, double* SlabState::*buf, int i, int jg, double v[4]) {
  for (auto& s : h->slabs) {
    int jl = jg - s.sl.y0;
    const bool inside = jl >= 0 && jl < s.L.ny;
    const bool ghost_lo = s.sl.fill_lo && jl >= -2 && jl < 0;
    const bool ghost_hi = s.sl.fill_hi && jl >= s.L.ny && jl < s.L.ny + 2;
    if (!(inside || ghost_lo || ghost_hi)) continue;
    CK(cudaSetDevice(s.device));
    for (int c = 0; c < 4; ++c)
      CK(cudaMemcpy(&v[c], (s.*buf) + s.L.origin() + c * s.L.fstride + (int64_t)jl * s.L.pitch + i,
                    sizeof(double), cudaMemcpyDeviceToHost));
    return true;
  }
  return false;
}

static bool owner_bits_to_all(lf_handle* h, bool found, double* v, int n) {
  if (!h->nccl) return found;
  unsigned long long u[4] = {0, 0, 0, 0};
  if (found)
    for (int c = 0; c < n; ++c) std::memcpy(&u[c], &v[c], sizeof(double));
  nccl_max_u64(h, u, n);
  for (int c = 0; c < n; ++c) std::memcpy(&v[c], &u[c], sizeof(double));
  return true;
}

bool fetch_cell(lf_handle* h, double* SlabState::*buf, int i, int jg, double v[4]) {
  const bool found = fetch_local(h, buf, i, jg, v);
  return owner_bits_to_all(h, found, v, 4);
}

// ---------------------------------------------------------------- error records
// The mixed-cell gamma of cell (i, jg) in slot gslot (collective like fetch_cell).
bool fetch_gamma(lf_handle* h, int gslot, int i, int jg, double* v) {
  bool found = false;
  for (auto& s : h->slabs) {
    const int jl = jg - s.sl.y0;
    const bool inside = jl >= 0 && jl < s.L.ny;
    const bool ghost_lo = s.sl.fill_lo && jl >= -2 && jl < 0;
    const bool ghost_hi = s.sl.fill_hi && jl >= s.L.ny && jl < s.L.ny + 2;
    if (!(inside || ghost_lo || ghost_hi)) continue;
    CK(cudaSetDevice(s.device));
    CK(cudaMemcpy(v, s.GC[gslot] + s.L.origin() + (int64_t)jl * s.L.pitch + i, sizeof(double),
                  cudaMemcpyDeviceToHost));
    found = true;
    break;
  }
  return owner_bits_to_all(h, found, v, 1);
}

int report_prim(lf_handle* h, double* SlabState::*buf, long long c, int64_t step, int gslot = 0) {
  const int gy = h->dim2 ? 2 : 0;
  const long long nxt = h->d.nx + 4;
  const long long ii = c % nxt - 2, jj = c / nxt - gy;
  double v[4] = {0, 0, 0, 0};
  fetch_cell(h, buf, (int)ii, (int)jj, v);
  // build_primitives reports with the cell's own EOS (solver.cpp:165-167)
  double gamma = h->d.gamma;
  if (h->mc.n) fetch_gamma(h, gslot, (int)ii, (int)jj, &gamma);
  // primitive_from_conserved with CellContext (euler.hpp:73-85)
  const char* what;
  double value;
  if (!(v[0] > 0.0)) {
    what = "non-positive density";
    value = v[0];
  } else {
    const double inv = 1.0 / v[0];
    const double kinetic = 0.5 * (v[1] * v[1] + v[2] * v[2]) * inv;
    value = (gamma - 1.0) * (v[3] - kinetic);
    what = "non-positive pressure";
  }
  char suffix[96];
  if (step >= 0)
    snprintf(suffix, sizeof suffix, " at cell (%lld,%lld) step %lld", ii, jj, (long long)step);
  else
    snprintf(suffix, sizeof suffix, " at cell (%lld,%lld)", ii, jj);
  set_err(h, LF_ERR_PRIMITIVE, "%s = %s%s", what, fmt_f(value).c_str(), suffix);
  h->err.i = ii;
  h->err.j = jj;
  h->err.step = step;
  h->err.value = value;
  return LF_ERR_PRIMITIVE;
}

int report_trace(lf_handle* h, long long code, int64_t step) {
  const long long nx = h->d.nx;
  const long long nex = (nx + 1) * h->d.ny;
  const bool is_x = code < nex;
  const long long e = is_x ? code : code - nex;
  const long long along = is_x ? nx + 1 : nx;
  set_err(h, LF_ERR_TRACE, "non-physical reconstructed trace at %s-face (%lld,%lld) step %lld",
          is_x ? "x" : "y", e % along, e / along, (long long)step);
  h->err.axis = is_x ? 0 : 1;
  h->err.i = e % along;
  h->err.j = e / along;
  h->err.step = step;
  return LF_ERR_TRACE;
}

int report_update(lf_handle* h, double* SlabState::*out, long long cc, int64_t step, double dt) {
  const long long nx = h->d.nx;
  const long long i = cc % nx, j = cc / nx;
  double v[4] = {0, 0, 0, 0};
  fetch_cell(h, out, (int)i, (int)j, v);
  const double r = v[0];
  const double eint = v[3] - 0.5 * (v[1] * v[1] + v[2] * v[2]) / r;
  set_err(h, LF_ERR_POSITIVITY,
          "update lost positivity at cell (%lld,%lld): rho = %s, internal energy density = %s, "
          "step %lld, dt %s",
          i, j, fmt_f(r).c_str(), fmt_f(eint).c_str(), (long long)step, fmt_f(dt).c_str());
  h->err.i = i;
  h->err.j = j;
  h->err.step = step;
  h->err.dt = dt;
  h->err.value = r;
  h->err.value2 = eint;
  return LF_ERR_POSITIVITY;
}

// fill_all_ghosts' fraction check (solver.cpp:122-127): smallest ghosted index
int report_frac(lf_handle* h, long long c) {
  const int gy = h->dim2 ? 2 : 0;
  const long long nxt = h->d.nx + 4;
  const long long i = c % nxt - 2, j = c / nxt - gy;
  set_err(h, LF_ERR_FRACTION, "mass fraction out of [0,1] beyond round-off at cell (%lld,%lld)", i, j);
  h->err.i = i;
  h->err.j = j;
  return LF_ERR_FRACTION;
}

// dt from the combined rate (solver.cpp:471-479)
int finish_dt(lf_handle* h, const Scalars& sc, double cfl, double time, double limit, double* dt) {
  if (sc.fail_dt != LLONG_MAX) {
    const long long nx = h->d.nx;
    set_err(h, LF_ERR_DT_STATE,
            "non-physical state while computing the time step at cell (%lld,%lld)",
            sc.fail_dt % nx, sc.fail_dt / nx);
    h->err.i = sc.fail_dt % nx;
    h->err.j = sc.fail_dt / nx;
    return LF_ERR_DT_STATE;
  }
  const double rate = bits_to_double(sc.rate_bits);
  double d = cfl / rate;
  if (time + d > limit) d = limit - time;
  if (!(d > 0.0)) {
    set_err(h, LF_ERR_DT_NONPOS, "non-positive time step (time limit already reached?)");
    h->err.dt = d;
    return LF_ERR_DT_NONPOS;
  }
  *dt = d;
  return 0;
}

// CFL rate of `buf` (ghosts not needed) into scalars slot 0.
// With materials: gamma_[0] of the last fill (solver.cpp:441), and when `part`
// is given the fraction closure of (buf, part) is computed first (heun_step's
// fill_all_ghosts(state.field, mat, 0), solver.cpp:491).
void launch_rate_all(lf_handle* h, double* SlabState::*buf, double* SlabState::*part = nullptr) {
  for (auto& s : h->slabs) {
    CK(cudaSetDevice(s.device));
    reset_scalars(&s.scal[0], s.stream);
    if (h->mc.n) {
      if (part)
        launch_mat_fractions(s.field(s.*buf), s.field(s.*part), s.field(s.Y[0]), s.field(s.GC[0]),
                             s.L, s.sl, h->mc, h->dim2, &s.scal[0], s.stream);
      launch_rate_g(s.field(s.*buf), s.field(s.GC[0]), s.L, s.sl, h->k, h->dim2, &s.scal[0],
                    s.stream);
    } else {
      launch_rate(s.field(s.*buf), s.L, s.sl, h->k, h->dim2, &s.scal[0], s.stream);
    }
  }
}

// One stage on every slab: prims(in) -> fluxes(set k) -> update(base, ...) -> out.
// With materials the stage uses the mixed-cell gamma of slot gslot; when
// `part` is given (the corrector's fill_all_ghosts(predictor_, &predictor_mat_,
// 1), solver.cpp:504) that slot's fractions are computed from (in, part) first.
void staged_stage(lf_handle* h, double* SlabState::*in, double* SlabState::*base,
                  double* SlabState::*out, int k, bool two, double dt, int slot,
                  double* SlabState::*part = nullptr, int gslot = 0) {
  fill_all(h, in);
  if (h->mc.n && part) fill_partials(h, part);
  for (auto& s : h->slabs) {
    CK(cudaSetDevice(s.device));
    reset_scalars(&s.scal[slot], s.stream);
    const FluxArr fx = s.fluxx(k), fy = s.fluxy(k);
    if (h->mc.n) {
      if (part)
        launch_mat_fractions(s.field(s.*in), s.field(s.*part), s.field(s.Y[gslot]),
                             s.field(s.GC[gslot]), s.L, s.sl, h->mc, h->dim2, &s.scal[slot],
                             s.stream);
      launch_prims_g(s.field(s.*in), s.field(s.W), s.field(s.GC[gslot]), s.L, s.sl, h->dim2,
                     &s.scal[slot], s.stream);
      launch_fluxes_g(s.field(s.W), s.field(s.GC[gslot]), fx, fy, s.ustx(k), s.usty(k), s.L,
                      s.sl, h->k, h->d.spatial_order >= 2, h->dim2, &s.scal[slot], s.stream);
    } else {
      launch_prims(s.field(s.*in), s.field(s.W), s.L, s.sl, h->k.gm1, h->dim2, &s.scal[slot],
                   s.stream);
      launch_fluxes(s.field(s.W), fx, fy, s.L, s.sl, h->k, h->d.spatial_order >= 2, h->dim2,
                    &s.scal[slot], s.stream);
    }
    const FluxArr fx0 = s.fluxx(0), fy0 = s.fluxy(0);
    launch_update(s.field(s.*base), fx0, fy0, two ? &fx : nullptr, two ? &fy : nullptr,
                  s.field(s.*out), s.L, s.sl, dt, h->d.dx, h->d.dy, h->dim2, &s.scal[slot],
                  s.stream);
  }
  CK(cudaGetLastError());
}

// accumulate_boundary_outflow (solver.cpp:406-432): ordered serial sums over
// the domain-boundary faces, gathered from every slab in global order.
void boundary_outflow(lf_handle* h, bool two, double dt, double* acc) {
  const int nx = h->d.nx, nyg = h->d.ny;
  std::vector<double> left(4 * (size_t)nyg), right(4 * (size_t)nyg), bot(4 * (size_t)nx),
      top(4 * (size_t)nx);
  for (auto& s : h->slabs) {
    CK(cudaSetDevice(s.device));
    launch_gather_boundary(s.fluxx(0), s.fluxy(0), two ? s.fluxx(1) : s.fluxx(0),
                           two ? s.fluxy(1) : s.fluxy(0), s.L, two, s.bnd, s.stream);
    const size_t nb = 4 * (size_t)(2 * s.L.ny + 2 * s.L.nx);
    CK(cudaMemcpyAsync(s.bnd_host, s.bnd, nb * sizeof(double), cudaMemcpyDeviceToHost, s.stream));
  }
  sync_all(h);
  for (auto& s : h->slabs) {
    const int ny = s.L.ny;
    const double* b = s.bnd_host;
    for (int c = 0; c < 4; ++c)
      for (int j = 0; j < ny; ++j) {
        left[(size_t)c * nyg + s.sl.y0 + j] = b[(size_t)c * ny + j];
        right[(size_t)c * nyg + s.sl.y0 + j] = b[4 * (size_t)ny + (size_t)c * ny + j];
      }
    if (s.sl.y0 == 0)
      for (int c = 0; c < 4; ++c)
        for (int i = 0; i < nx; ++i) bot[(size_t)c * nx + i] = b[8 * (size_t)ny + (size_t)c * nx + i];
    if (s.sl.y0 + ny == nyg)
      for (int c = 0; c < 4; ++c)
        for (int i = 0; i < nx; ++i)
          top[(size_t)c * nx + i] = b[8 * (size_t)ny + 4 * (size_t)nx + (size_t)c * nx + i];
  }
  if (h->nccl) nccl_gather_boundary(h, left.data(), right.data(), bot.data(), top.data());
  const double ax = dt * (h->dim2 ? h->d.dy : 1.0);
  for (int c = 0; c < 4; ++c) {
    double sum = 0.0;
    for (int j = 0; j < nyg; ++j) sum += right[(size_t)c * nyg + j] - left[(size_t)c * nyg + j];
    acc[c] += ax * sum;
  }
  if (h->dim2) {
    const double ay = dt * h->d.dx;
    for (int c = 0; c < 4; ++c) {
      double sum = 0.0;
      for (int i = 0; i < nx; ++i) sum += top[(size_t)c * nx + i] - bot[(size_t)c * nx + i];
      acc[c] += ay * sum;
    }
  }
}

void swap_state(lf_handle* h, double* SlabState::*a, double* SlabState::*b) {
  for (auto& s : h->slabs) std::swap(s.*a, s.*b);
}

// Check the stage scalars in the reference's order.
int check_stage(lf_handle* h, const Scalars& sc, double* SlabState::*in,
                double* SlabState::*out, int64_t step, double dt, int gslot = 0) {
  if (sc.fail_frac != LLONG_MAX) return report_frac(h, sc.fail_frac);
  if (sc.fail_prim != LLONG_MAX) return report_prim(h, in, sc.fail_prim, step, gslot);
  if (sc.fail_trace != LLONG_MAX) return report_trace(h, sc.fail_trace, step);
  if (sc.fail_update != LLONG_MAX) return report_update(h, out, sc.fail_update, step, dt);
  return 0;
}

// update_partials (solver.cpp:331-404) on every slab: out = base - flux of set
// 0 (fractions slot 0) [and set 1 (slot 1)].
void update_partials_all(lf_handle* h, double* SlabState::*base, double* SlabState::*out,
                         bool two, double dt) {
  for (auto& s : h->slabs) {
    CK(cudaSetDevice(s.device));
    const FluxArr fx1 = s.fluxx(1), fy1 = s.fluxy(1), ux1 = s.ustx(1), uy1 = s.usty(1);
    const Field y1 = s.field(s.Y[1]);
    launch_update_partials(s.field(s.*base), s.fluxx(0), s.fluxy(0), s.ustx(0), s.usty(0),
                           s.field(s.Y[0]), two ? &fx1 : nullptr, two ? &fy1 : nullptr,
                           two ? &ux1 : nullptr, two ? &uy1 : nullptr, two ? &y1 : nullptr,
                           s.field(s.*out), s.L, h->mc.n, dt, h->d.dx, h->d.dy, h->dim2,
                           s.stream);
  }
  CK(cudaGetLastError());
}

// solver.cpp:519-538: min over interior cells of e_int / sum_k y_k/(gamma_k - 1)
double material_min_p(lf_handle* h) {
  for (auto& s : h->slabs) {
    CK(cudaSetDevice(s.device));
    reset_scalars(&s.scal[3], s.stream);
    launch_mat_min_p(s.field(s.U), s.field(s.P), s.L, h->mc, &s.scal[3], s.stream);
  }
  const unsigned long long key = combined_scalars(h, 3).min_p_key;
  if (key == ~0ull) return std::numeric_limits<double>::infinity();  // min_p's initial value
  const unsigned long long b = (key >> 63) ? (key & 0x7fffffffffffffffull) : ~key;
  return bits_to_double(b);
}

int staged_heun(lf_handle* h, double cfl, double time, double limit, int64_t step,
                double* outflow, lf_step_out* out) {
  LF_TRACE("stage-wise heun step");
  const bool mat = h->mc.n > 0;
  if (mat && !h->partials_ready)
    return set_err(h, LF_ERR_CONFIG, "multimaterial step needs material storage");
  for (auto& s : h->slabs) alloc_staged(s);
  // fill_all_ghosts(state.field, mat, 0) then compute_dt (solver.cpp:491-492)
  fill_all(h, &SlabState::U);
  if (mat) fill_partials(h, &SlabState::P);
  launch_rate_all(h, &SlabState::U, mat ? &SlabState::P : nullptr);
  const Scalars s0 = combined_scalars(h, 0);
  if (s0.fail_frac != LLONG_MAX) return report_frac(h, s0.fail_frac);
  double dt = 0.0;
  int rc = finish_dt(h, s0, cfl, time, limit, &dt);
  if (rc) return rc;
  const bool hits = time + dt >= limit;

  // predictor: U -> Us with flux set 0 (solver.cpp:496-500)
  staged_stage(h, &SlabState::U, &SlabState::U, &SlabState::Us, 0, false, dt, 1);
  const Scalars s1 = combined_scalars(h, 1);
  rc = check_stage(h, s1, &SlabState::U, &SlabState::Us, step, dt);
  if (rc) return rc;
  if (mat) update_partials_all(h, &SlabState::P, &SlabState::Ps, false, dt);  // :501
  double min_rho = bits_to_double(s1.min_rho_bits), min_eint = bits_to_double(s1.min_eint_bits);
  double acc[4] = {0, 0, 0, 0};
  if (outflow) std::memcpy(acc, outflow, sizeof acc);

  if (h->d.time_order >= 2) {
    // corrector: Us -> U2 from U^n with 0.5*(F1 + F2) (solver.cpp:503-509)
    staged_stage(h, &SlabState::Us, &SlabState::U, &SlabState::U2, 1, true, dt, 2,
                 mat ? &SlabState::Ps : nullptr, 1);
    const Scalars s2 = combined_scalars(h, 2);
    if (s2.fail_frac != LLONG_MAX) return report_frac(h, s2.fail_frac);
    if (s2.fail_prim != LLONG_MAX) return report_prim(h, &SlabState::Us, s2.fail_prim, step, 1);
    if (s2.fail_trace != LLONG_MAX) return report_trace(h, s2.fail_trace, step);
    // the reference writes the corrector in place before it throws
    swap_state(h, &SlabState::U, &SlabState::U2);
    if (s2.fail_update != LLONG_MAX) return report_update(h, &SlabState::U, s2.fail_update, step, dt);
    if (mat) update_partials_all(h, &SlabState::P, &SlabState::P, true, dt);  // :508, in place
    min_rho = bits_to_double(s2.min_rho_bits);
    min_eint = bits_to_double(s2.min_eint_bits);
    boundary_outflow(h, true, dt, acc);
  } else {
    swap_state(h, &SlabState::U, &SlabState::Us);  // std::swap(state.field.comp, predictor_.comp)
    if (mat) swap_state(h, &SlabState::P, &SlabState::Ps);
    boundary_outflow(h, false, dt, acc);
  }
  h->rate_valid = false;
  fused_invalidate(h);
  if (outflow) std::memcpy(outflow, acc, sizeof acc);
  if (out) {
    out->dt = dt;
    out->hits_limit = hits;
    out->time = hits ? limit : time + dt;
    out->step = step + 1;
    out->min_rho = min_rho;
    out->min_p = mat ? material_min_p(h) : (h->d.gamma - 1.0) * min_eint;
  }
  return 0;
}

// LF_PATH_SMALL (small_step.cu): asked for, or LF_PATH_AUTO on a small grid
bool use_small(lf_handle* h) {
  return (h->path == LF_PATH_SMALL && small_supported(h)) || prefer_small(h);
}

bool use_fused(lf_handle* h) {
  if (h->path == LF_PATH_STAGED) return false;
  // the fast kernels' limiter (sweby_fast, fastmath.cuh) is the reference's for
  // beta >= 1 (make_limiter's range is [1, 2], but LagfluxSolver takes any
  // LimiterParams): other betas run the stage-wise kernels, which evaluate
  // sweby_limiter as written (reconstruct.hpp:24-30)
  if (!(h->d.beta >= 1.0)) return false;
  // materials: the two-pass material kernels for up to 8 materials, else stage-wise
  if (h->mc.n > 0 && (h->mc.n > TP_MAX_MATERIALS || h->path == LF_PATH_FUSED || !h->partials_ready))
    return false;
  // (the fused one-kernel step has no material transport: a slab beyond the
  // two-pass kernels' 32-bit offsets goes stage-wise)
  if (h->mc.n > 0) {
    for (auto& s : h->slabs)
      if (!tp_fits(s.L.pitch, s.L.ny)) return false;
    // ... and so does one whose two-pass scratch was vetoed (device memory)
    return fused_supported(h) && twopass_selected(h);
  }
  return fused_supported(h);
}

template <class F>
int guarded(lf_handle* h, F&& f) {
  if (!h) return LF_ERR_ARGUMENT;
  try {
    return f();
  } catch (const DeviceFail& e) {
    return set_err(h, LF_ERR_DEVICE, "%s", e.what.c_str());
  } catch (const std::bad_alloc&) {
    return set_err(h, LF_ERR_DEVICE, "host allocation failed");
  } catch (const std::exception& e) {
    return set_err(h, LF_ERR_DEVICE, "%s", e.what());
  }
}

}  // namespace

namespace lfb {
void fill_all_public(lf_handle* h, double* SlabState::*buf) { fill_all(h, buf); }
// fill_all's single-launch ghost fill without the halo exchange (the caller
// exchanges the halos itself, e.g. overlapped with interior work); false if the
// single-launch fill does not apply (then nothing was done)
bool fill_local_public(lf_handle* h, double* SlabState::*buf) {
  const int xbc[4] = {h->d.bc[0], h->d.bc[1], h->d.bc[2], h->d.bc[3]};
  for (auto& s : h->slabs)
    if (!(s.L.nx >= NG && (!h->dim2 || s.L.ny >= NG))) return false;
  for (auto& s : h->slabs) {
    CK(cudaSetDevice(s.device));
    launch_fill_xy(s.field(s.*buf), s.L, xbc, s.sl, h->dim2, s.stream, 4, 1, 2, nullptr, 0);
  }
  CK(cudaGetLastError());
  return true;
}
void fill_partials_public(lf_handle* h, double* SlabState::*buf) { fill_partials(h, buf); }
void fill_state_public(lf_handle* h, double* SlabState::*ubuf, double* SlabState::*pbuf) {
  fill_all(h, ubuf, 4, 1, 2, pbuf, h->mc.n);
}
void alloc_staged_public(lf_handle* h) {
  for (auto& s : h->slabs) alloc_staged(s);
}
Scalars rate_of_current(lf_handle* h) {
  if (h->mc.n) {
    // heun_step's fill_all_ghosts(state.field, mat, 0) before compute_dt
    fill_all(h, &SlabState::U);
    fill_partials(h, &SlabState::P);
    launch_rate_all(h, &SlabState::U, &SlabState::P);
  } else {
    launch_rate_all(h, &SlabState::U);
  }
  return combined_scalars(h, 0);
}
int staged_heun_public(lf_handle* h, double cfl, double time, double limit, int64_t step,
                       double* outflow, lf_step_out* out) {
  return staged_heun(h, cfl, time, limit, step, outflow, out);
}
}  // namespace lfb

// ====================================================================== C ABI
extern "C" {

int lf_abi_version(void) { return LF_ABI_VERSION; }

int lf_create(const lf_desc* desc, const int* devices, int ndev, lf_handle** out) {
  if (!desc || !out || ndev < 1) return LF_ERR_ARGUMENT;
  *out = nullptr;
  auto* h = new lf_handle;
  clear_err(&h->err);
  int rc = validate_desc(h, desc);
  if (rc) {
    *out = h;  // keep the handle so lf_last_error can report
    return rc;
  }
  init_common(h, desc);
  rc = guarded(h, [&] {
    if (ndev > 1 && !h->dim2) return set_err(h, LF_ERR_CONFIG, "y-slabs need a 2D grid");
    h->slabs.resize((size_t)ndev);
    const bool periodic = desc->bc[2] == LF_PERIODIC;
    for (int s = 0; s < ndev; ++s) {
      SlabState& sl = h->slabs[(size_t)s];
      sl.device = devices ? devices[s] : 0;
      int y0, rows;
      slab_rows(desc->ny, ndev, s, &y0, &rows);
      if (ndev > 1 && rows < NG)
        return set_err(h, LF_ERR_CONFIG, "each y-slab needs at least %d rows", NG);
      sl.L = Layout::make(desc->nx, rows);
      sl.sl.y0 = y0;
      sl.sl.ny_global = desc->ny;
      sl.sl.fill_lo = ndev == 1 || (!periodic && s == 0);
      sl.sl.fill_hi = ndev == 1 || (!periodic && s == ndev - 1);
      CK(cudaSetDevice(sl.device));
      // slabs sharing a device share one stream: stream order is the schedule
      if (s > 0 && sl.device == h->slabs[0].device) {
        sl.stream = h->slabs[0].stream;
      } else {
        CK(cudaStreamCreateWithFlags(&sl.own_stream, cudaStreamNonBlocking));
        sl.stream = sl.own_stream;
      }
      alloc_state(sl);
    }
    // enable peer access between distinct devices (in-process multi-GPU)
    for (auto& a : h->slabs)
      for (auto& b : h->slabs)
        if (a.device != b.device) {
          int can = 0;
          cudaDeviceCanAccessPeer(&can, a.device, b.device);
          if (can) {
            cudaSetDevice(a.device);
            cudaError_t e = cudaDeviceEnablePeerAccess(b.device, 0);
            if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
          }
        }
    sync_all(h);
    return 0;
  });
  *out = h;
  return rc;
}

int lf_nccl_unique_id(void* id128) { return nccl_unique_id(id128); }

int lf_create_dist(const lf_desc* desc, int device, int rank, int nranks, const void* nccl_id,
                   lf_handle** out) {
  if (!desc || !out || nranks < 1 || rank < 0 || rank >= nranks) return LF_ERR_ARGUMENT;
  *out = nullptr;
  auto* h = new lf_handle;
  clear_err(&h->err);
  int rc = validate_desc(h, desc);
  if (rc) {
    *out = h;
    return rc;
  }
  init_common(h, desc);
  rc = guarded(h, [&] {
    if (nranks > 1 && !h->dim2) return set_err(h, LF_ERR_CONFIG, "y-slabs need a 2D grid");
    h->rank = rank;
    h->nranks = nranks;
    h->slabs.resize(1);
    SlabState& sl = h->slabs[0];
    sl.device = device;
    int y0, rows;
    slab_rows(desc->ny, nranks, rank, &y0, &rows);
    if (nranks > 1 && rows < NG)
      return set_err(h, LF_ERR_CONFIG, "each y-slab needs at least %d rows", NG);
    const bool periodic = desc->bc[2] == LF_PERIODIC;
    sl.L = Layout::make(desc->nx, rows);
    sl.sl.y0 = y0;
    sl.sl.ny_global = desc->ny;
    sl.sl.fill_lo = nranks == 1 || (!periodic && rank == 0);
    sl.sl.fill_hi = nranks == 1 || (!periodic && rank == nranks - 1);
    CK(cudaSetDevice(device));
    CK(cudaStreamCreateWithFlags(&sl.own_stream, cudaStreamNonBlocking));
    sl.stream = sl.own_stream;
    alloc_state(sl);
    if (nranks > 1) {
      int e = nccl_init(h, nccl_id);
      if (e) return e;
    }
    sync_all(h);
    return 0;
  });
  *out = h;
  return rc;
}

int lf_wait_dumps(lf_handle* h);

void lf_destroy(lf_handle* h) {
  if (!h) return;
  lf_wait_dumps(h);   // asynchronous dumps still being written
  for (auto& s : h->slabs) {
    if (s.device >= 0) cudaSetDevice(s.device);
    if (s.stream) cudaStreamSynchronize(s.stream);
  }
  nccl_destroy(h);
  fused_release(h);
  small_release(h);
  for (auto& s : h->slabs) free_slab(s);
  delete h;
}

int lf_local_rows(lf_handle* h, int* row0, int* nrows) {
  if (!h || h->slabs.empty()) return LF_ERR_ARGUMENT;
  *row0 = h->slabs.front().sl.y0;
  *nrows = h->slabs.back().sl.y0 + h->slabs.back().L.ny - *row0;
  return 0;
}

int lf_upload(lf_handle* h, double* const field[4], int64_t ld) {
  LF_TRACE("lf_upload");
  return guarded(h, [&] {
    if (!field || ld < h->d.nx + 4) return set_err(h, LF_ERR_ARGUMENT, "bad field or ld");
    const int gy = h->dim2 ? 2 : 0;
    for (auto& s : h->slabs) {
      CK(cudaSetDevice(s.device));
      for (int c = 0; c < 4; ++c) {
        const double* src = field[c] + (int64_t)(s.sl.y0 + gy) * ld + 2;
        double* dst = s.U + s.L.origin() + c * s.L.fstride;
        CK(cudaMemcpy2DAsync(dst, s.L.pitch * sizeof(double), src, ld * sizeof(double),
                             (size_t)s.L.nx * sizeof(double), (size_t)s.L.ny, cudaMemcpyDefault,
                             s.stream));
      }
    }
    sync_all(h);
    h->tp_exact = 0;
    h->small_ieee = 0;  // a new state: the plain fast kernels first
    h->rate_valid = false;
    fused_invalidate(h);
    return 0;
  });
}

// ---- multimaterial (multimat.hpp; solver.cpp:61-88 MaterialSet argument) ----
int lf_set_materials(lf_handle* h, int n, const double* gammas) {
  return guarded(h, [&] {
    // make_material_set, multimat.cpp:7-15
    if (n < 1) return set_err(h, LF_ERR_CONFIG, "material set needs at least one material");
    if (n > MAX_MATERIALS) return set_err(h, LF_ERR_CONFIG, "at most 16 materials are supported");
    if (!gammas) return set_err(h, LF_ERR_ARGUMENT, "gammas is null");
    for (int k = 0; k < n; ++k)
      if (!(gammas[k] > 1.0) || !(gammas[k] <= 3.0))
        return set_err(h, LF_ERR_CONFIG, "material adiabatic index must lie in (1, 3], got %s",
                       fmt_f(gammas[k]).c_str());
    if (h->mc.n) return set_err(h, LF_ERR_CONFIG, "the material set is fixed at construction");
    h->mc.n = n;
    for (int k = 0; k < n; ++k) h->mc.gamma[k] = gammas[k];
    for (auto& s : h->slabs) {
      alloc_staged(s);
      CK(cudaSetDevice(s.device));
      const size_t kb = ((size_t)n * s.L.fstride + s.L.pitch) * sizeof(double);
      const size_t gb = ((size_t)s.L.fstride + s.L.pitch) * sizeof(double);
      CK(cudaMalloc(&s.P, kb));
      CK(cudaMalloc(&s.Ps, kb));
      CK(cudaMalloc(&s.P2, kb));
      CK(cudaMemsetAsync(s.P, 0, kb, s.stream));
      CK(cudaMemsetAsync(s.Ps, 0, kb, s.stream));
      CK(cudaMemsetAsync(s.P2, 0, kb, s.stream));
      if (n <= TP_MAX_MATERIALS) {  // the two-pass material kernels' stage-a fluxes
        CK(cudaMalloc(&s.MFX, (size_t)n * s.fx_stride * sizeof(double)));
        CK(cudaMalloc(&s.MFY, (size_t)n * s.fy_stride * sizeof(double)));
        CK(cudaMemsetAsync(s.MFX, 0, (size_t)n * s.fx_stride * sizeof(double), s.stream));
        CK(cudaMemsetAsync(s.MFY, 0, (size_t)n * s.fy_stride * sizeof(double), s.stream));
      }
      for (int k = 0; k < 2; ++k) {
        CK(cudaMalloc(&s.Y[k], kb));
        CK(cudaMemsetAsync(s.Y[k], 0, kb, s.stream));
        // gamma_[s].assign(cells, eos.gamma) (solver.cpp:81)
        CK(cudaMalloc(&s.GC[k], gb));
        fill_value(s.GC[k], (int64_t)(gb / sizeof(double)), h->d.gamma, s.stream);
        CK(cudaMalloc(&s.USX[k], (size_t)s.fx_stride * sizeof(double)));
        CK(cudaMalloc(&s.USY[k], (size_t)s.fy_stride * sizeof(double)));
        CK(cudaMemsetAsync(s.USX[k], 0, (size_t)s.fx_stride * sizeof(double), s.stream));
        CK(cudaMemsetAsync(s.USY[k], 0, (size_t)s.fy_stride * sizeof(double), s.stream));
      }
    }
    sync_all(h);
    fused_invalidate(h);
    return 0;
  });
}

int lf_upload_partials(lf_handle* h, double* const* partials, int64_t ld) {
  LF_TRACE("lf_upload_partials");
  return guarded(h, [&] {
    if (!h->mc.n) return set_err(h, LF_ERR_CONFIG, "no material set (lf_set_materials)");
    if (!partials || ld < h->d.nx + 4) return set_err(h, LF_ERR_ARGUMENT, "bad partials or ld");
    const int gy = h->dim2 ? 2 : 0;
    for (auto& s : h->slabs) {
      CK(cudaSetDevice(s.device));
      for (int k = 0; k < h->mc.n; ++k) {
        const double* src = partials[k] + (int64_t)(s.sl.y0 + gy) * ld + 2;
        double* dst = s.P + s.L.origin() + k * s.L.fstride;
        CK(cudaMemcpy2DAsync(dst, s.L.pitch * sizeof(double), src, ld * sizeof(double),
                             (size_t)s.L.nx * sizeof(double), (size_t)s.L.ny, cudaMemcpyDefault,
                             s.stream));
      }
    }
    sync_all(h);
    h->partials_ready = 1;
    // the cached CFL rate and fraction check came from the old partials (mixed-cell
    // gamma): a new material state, as in lf_upload
    h->tp_exact = 0;
    h->small_ieee = 0;
    h->rate_valid = false;
    fused_invalidate(h);
    return 0;
  });
}

int lf_download_partials(lf_handle* h, double* const* partials, int64_t ld) {
  LF_TRACE("lf_download_partials");
  return guarded(h, [&] {
    if (!h->mc.n) return set_err(h, LF_ERR_CONFIG, "no material set (lf_set_materials)");
    if (!partials || ld < h->d.nx + 4) return set_err(h, LF_ERR_ARGUMENT, "bad partials or ld");
    const int gy = h->dim2 ? 2 : 0;
    for (auto& s : h->slabs) {
      CK(cudaSetDevice(s.device));
      for (int k = 0; k < h->mc.n; ++k) {
        double* dst = partials[k] + (int64_t)(s.sl.y0 + gy) * ld + 2;
        const double* src = s.P + s.L.origin() + k * s.L.fstride;
        CK(cudaMemcpy2DAsync(dst, ld * sizeof(double), src, s.L.pitch * sizeof(double),
                             (size_t)s.L.nx * sizeof(double), (size_t)s.L.ny, cudaMemcpyDefault,
                             s.stream));
      }
    }
    sync_all(h);
    return 0;
  });
}

// ---- field dumps: field_csv (csv.cpp:26-83) + write_text_file (run.cpp:162-168) ----
namespace {
// format_g17 (csv.cpp:8-12): "%.17g".  std::to_chars(general, 17) is specified
// as printf's %.17g in the C locale (and is several times faster); tests compare
// the bytes against the reference's own field_csv.
inline void put_g17(std::string& out, double v) {
  char buf[32];
  const auto r = std::to_chars(buf, buf + sizeof buf, v, std::chars_format::general, 17);
  out.append(buf, (size_t)(r.ptr - buf));
}
}  // namespace

// A field_csv dump (csv.cpp:26-83) in two parts.  dump_derive (caller thread) derives
// the columns on the device into a snapshot buffer, in stream order with the steps;
// dump_finish copies them back, checks the fractions and formats / writes the file.
// lf_write_field_csv runs both; lf_write_field_csv_async runs dump_finish on a host
// thread, so the caller keeps stepping while the dump is copied, formatted and written.
struct DumpJob {
  std::string path;
  uint64_t digest = 0;
  double time = 0.0;
  int threads = 0;
  lf_desc d{};
  int dim2 = 1, n_mat = 0, ncols = 0, rows = 0, row0 = 0;
  struct Part {
    int device = 0, y0 = 0, ny = 0;
    double* dbuf = nullptr;             // ncols planes of nx * ny
    unsigned long long* dfail = nullptr;
    double* dcell = nullptr;            // the flagged cell's partials
    cudaStream_t copy = nullptr;        // the dump's own stream (async: off the step stream)
    cudaEvent_t ready = nullptr;        // the derive kernels done
  };
  std::vector<Part> parts;
  int rc = 0;
  int err_kind = 0;
  std::string err;
};

static void dump_release(DumpJob& job);

static std::unique_ptr<DumpJob> dump_derive(lf_handle* h, const char* path, uint64_t digest,
                                            double time, int threads) {
  auto job = std::make_unique<DumpJob>();
  job->path = path;
  job->digest = digest;
  job->time = time;
  job->threads = threads;
  job->d = h->d;
  job->dim2 = h->dim2;
  job->n_mat = h->mc.n;
  job->ncols = 5 + h->mc.n;
  // this process's rows (a distributed handle writes its slab rows only)
  job->row0 = h->slabs.front().sl.y0;
  job->rows = h->slabs.back().sl.y0 + h->slabs.back().L.ny - job->row0;
  try {
  for (auto& s : h->slabs) {
    CK(cudaSetDevice(s.device));
    DumpJob::Part pt;
    pt.device = s.device;
    pt.y0 = s.sl.y0;
    pt.ny = s.L.ny;
    const size_t plane = (size_t)h->d.nx * s.L.ny;
    // stream-ordered allocations (freed on the copy stream): neither side of the dump
    // synchronises the device, so the steps queued behind it keep running
    CK(cudaStreamCreateWithFlags(&pt.copy, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&pt.ready, cudaEventDisableTiming));
    job->parts.push_back(pt);
    DumpJob::Part& q = job->parts.back();
    CK(cudaMallocAsync(&q.dbuf, job->ncols * plane * sizeof(double), s.stream));
    CK(cudaMallocAsync(&q.dfail, sizeof(unsigned long long), s.stream));
    CK(cudaMallocAsync(&q.dcell, MAX_MATERIALS * sizeof(double), s.stream));
    CK(cudaMemsetAsync(q.dfail, 0xff, sizeof(unsigned long long), s.stream));
    launch_csv_derive(s.field(s.U), s.field(job->n_mat ? s.P : s.U), s.L, s.sl, h->d.gamma, h->mc,
                      q.dbuf, q.dfail, s.stream);
    if (job->n_mat) launch_csv_failcell(s.field(s.P), job->n_mat, s.L, s.sl, q.dfail, q.dcell, s.stream);
    CK(cudaEventRecord(q.ready, s.stream));
    CK(cudaStreamWaitEvent(q.copy, q.ready, 0));
  }
  } catch (...) {
    dump_release(*job);
    throw;
  }
  return job;
}

// (safe on a partly built job: CK may have thrown in dump_derive)
static void dump_release(DumpJob& job) {
  for (auto& pt : job.parts) {
    cudaSetDevice(pt.device);
    if (pt.copy) {
      if (pt.dbuf) cudaFreeAsync(pt.dbuf, pt.copy);
      if (pt.dfail) cudaFreeAsync(pt.dfail, pt.copy);
      if (pt.dcell) cudaFreeAsync(pt.dcell, pt.copy);
      cudaStreamSynchronize(pt.copy);
      cudaStreamDestroy(pt.copy);
    }
    if (pt.ready) cudaEventDestroy(pt.ready);
    pt = DumpJob::Part{};
  }
  job.parts.clear();
}

// (no CUDA error can throw out of here: a host thread may run it)
static void dump_finish(DumpJob& job) {
  const int nx = job.d.nx, rows = job.rows, row0 = job.row0, ncols = job.ncols;
  const int n_mat = job.n_mat;
  auto fail_job = [&](int kind, const std::string& msg) {
    job.rc = kind;
    job.err_kind = kind;
    job.err = msg;
  };
  std::vector<double> cols((size_t)ncols * nx * rows);
  unsigned long long fail_host = ~0ull;
  double cell[MAX_MATERIALS] = {0.0};
  for (auto& pt : job.parts) {
    const size_t plane = (size_t)nx * pt.ny;
    unsigned long long f = ~0ull;
    double pc[MAX_MATERIALS] = {0.0};
    bool ok = cudaSetDevice(pt.device) == cudaSuccess;   // (the copy stream waits on ready)
    for (int c = 0; ok && c < ncols; ++c)
      ok = cudaMemcpyAsync(&cols[((size_t)c * rows + (pt.y0 - row0)) * nx], pt.dbuf + c * plane,
                           plane * sizeof(double), cudaMemcpyDeviceToHost, pt.copy) == cudaSuccess;
    ok = ok && cudaMemcpyAsync(&f, pt.dfail, sizeof f, cudaMemcpyDeviceToHost, pt.copy) == cudaSuccess;
    if (n_mat)
      ok = ok && cudaMemcpyAsync(pc, pt.dcell, n_mat * sizeof(double), cudaMemcpyDeviceToHost,
                                 pt.copy) == cudaSuccess;
    ok = ok && cudaStreamSynchronize(pt.copy) == cudaSuccess;
    if (!ok) {
      dump_release(job);
      return fail_job(LF_ERR_DEVICE, std::string("field dump: ") + cudaGetErrorString(cudaGetLastError()));
    }
    if (f < fail_host) {
      fail_host = f;
      std::memcpy(cell, pc, sizeof cell);
    }
  }
  dump_release(job);
  if (fail_host != ~0ull) {
    // clamped_fraction's message for the first failing (cell, material), csv.cpp:49
    const int i = (int)(fail_host % (unsigned long long)nx);
    const int jl = (int)(fail_host / (unsigned long long)nx) - row0;
    const double rho = cols[(size_t)jl * nx + i];
    double y = 0.0;
    for (int k = 0; k < n_mat; ++k) {
      y = cell[k] / rho;
      if (!(y >= 0.0 && y <= 1.0) && (y < -1e-11 || y > 1.0 + 1e-11)) break;
    }
    return fail_job(LF_ERR_FRACTION, "mass fraction out of [0,1] beyond round-off = " + fmt_f(y));
  }
  // header and column names (csv.cpp:15-23, 33-36)
  std::string head;
  char hb[64];
  std::snprintf(hb, sizeof hb, "# config %016llx time ", (unsigned long long)job.digest);
  head += hb;
  put_g17(head, job.time);
  head += '\n';
  head += job.dim2 ? "x,y,rho,u,v,p,e_internal" : "x,rho,u,p,e_internal";
  for (int k = 1; k <= n_mat; ++k) head += ",y" + std::to_string(k);
  head += '\n';
  // rows formatted in parallel (row order kept), then written in order
  int nt = job.threads > 0 ? job.threads : (int)std::thread::hardware_concurrency();
  nt = std::max(1, std::min(nt, rows));
  std::vector<std::string> parts((size_t)nt);
  const size_t plane = (size_t)nx * rows;
  const lf_desc& d = job.d;
  const bool dim2 = job.dim2 != 0;
  auto work = [&](int t) {
    const int j0 = (int)((int64_t)rows * t / nt), j1 = (int)((int64_t)rows * (t + 1) / nt);
    std::string& out = parts[(size_t)t];
    out.reserve((size_t)(j1 - j0) * nx * (size_t)(ncols + 2) * 24);
    for (int jl = j0; jl < j1; ++jl) {
      const double y = d.y0 + ((jl + row0) + 0.5) * d.dy;  // CartesianGrid::yc
      for (int i = 0; i < nx; ++i) {
        const size_t c = (size_t)jl * nx + i;
        put_g17(out, d.x0 + (i + 0.5) * d.dx);               // CartesianGrid::xc
        if (dim2) {
          out += ',';
          put_g17(out, y);
        }
        out += ',';
        put_g17(out, cols[c]);
        out += ',';
        put_g17(out, cols[plane + c]);
        if (dim2) {
          out += ',';
          put_g17(out, cols[2 * plane + c]);
        }
        out += ',';
        put_g17(out, cols[3 * plane + c]);
        out += ',';
        put_g17(out, cols[4 * plane + c]);
        for (int k = 0; k < n_mat; ++k) {
          out += ',';
          put_g17(out, cols[(5 + k) * plane + c]);
        }
        out += '\n';
      }
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < nt; ++t) pool.emplace_back(work, t);
  work(0);
  for (auto& th : pool) th.join();
  FILE* fp = std::fopen(job.path.c_str(), "wb");
  if (!fp) return fail_job(LF_ERR_ARGUMENT, "cannot open " + job.path + " for writing");
  bool ok = std::fwrite(head.data(), 1, head.size(), fp) == head.size();
  for (auto& p : parts) ok = ok && std::fwrite(p.data(), 1, p.size(), fp) == p.size();
  ok = (std::fclose(fp) == 0) && ok;
  if (!ok) return fail_job(LF_ERR_ARGUMENT, "short write to " + job.path);
}

static int dump_check(lf_handle* h, const char* path) {
  if (!path) return set_err(h, LF_ERR_ARGUMENT, "path is null");
  if (h->mc.n && !h->partials_ready)
    return set_err(h, LF_ERR_CONFIG, "multimaterial dump needs material storage");
  return 0;
}

int lf_write_field_csv(lf_handle* h, const char* path, uint64_t digest, double time,
                       int threads) {
  LF_TRACE("lf_write_field_csv");
  return guarded(h, [&] {
    if (int rc = dump_check(h, path)) return rc;
    auto job = dump_derive(h, path, digest, time, threads);
    dump_finish(*job);
    return job->rc ? set_err(h, job->err_kind, "%s", job->err.c_str()) : 0;
  });
}

// Pending asynchronous dumps of a handle (joined by lf_wait_dumps / lf_destroy).
struct AsyncDump {
  std::unique_ptr<DumpJob> job;
  std::thread worker;
};
static std::mutex g_dumps_m;
static std::map<lf_handle*, std::vector<std::unique_ptr<AsyncDump>>> g_dumps;

int lf_write_field_csv_async(lf_handle* h, const char* path, uint64_t digest, double time,
                             int threads) {
  LF_TRACE("lf_write_field_csv_async");
  return guarded(h, [&] {
    if (int rc = dump_check(h, path)) return rc;
    auto ad = std::make_unique<AsyncDump>();
    ad->job = dump_derive(h, path, digest, time, threads);
    DumpJob* job = ad->job.get();
    ad->worker = std::thread([job] { dump_finish(*job); });
    std::lock_guard<std::mutex> lk(g_dumps_m);
    g_dumps[h].push_back(std::move(ad));
    return 0;
  });
}

int lf_wait_dumps(lf_handle* h) {
  LF_TRACE("lf_wait_dumps");
  if (!h) return LF_ERR_ARGUMENT;
  std::vector<std::unique_ptr<AsyncDump>> mine;
  {
    std::lock_guard<std::mutex> lk(g_dumps_m);
    auto it = g_dumps.find(h);
    if (it == g_dumps.end()) return 0;
    mine = std::move(it->second);
    g_dumps.erase(it);
  }
  int rc = 0;
  for (auto& ad : mine) {
    ad->worker.join();
    if (ad->job->rc && !rc) rc = set_err(h, ad->job->err_kind, "%s", ad->job->err.c_str());
  }
  return rc;
}

int lf_download(lf_handle* h, double* const field[4], int64_t ld, int fill_ghosts) {
  LF_TRACE("lf_download");
  return guarded(h, [&] {
    if (!field || ld < h->d.nx + 4) return set_err(h, LF_ERR_ARGUMENT, "bad field or ld");
    const int gy = h->dim2 ? 2 : 0;
    for (auto& s : h->slabs) {
      CK(cudaSetDevice(s.device));
      for (int c = 0; c < 4; ++c) {
        double* dst = field[c] + (int64_t)(s.sl.y0 + gy) * ld + 2;
        const double* src = s.U + s.L.origin() + c * s.L.fstride;
        CK(cudaMemcpy2DAsync(dst, ld * sizeof(double), src, s.L.pitch * sizeof(double),
                             (size_t)s.L.nx * sizeof(double), (size_t)s.L.ny, cudaMemcpyDefault,
                             s.stream));
      }
    }
    sync_all(h);
    if (fill_ghosts) host_apply_boundary(h->d, field, ld);
    return 0;
  });
}

int lf_download_ghosted(lf_handle* h, double* const field[4], int64_t ld) {
  LF_TRACE("lf_download_ghosted");
  return guarded(h, [&] {
    if (!field || ld < h->d.nx + 4) return set_err(h, LF_ERR_ARGUMENT, "bad field or ld");
    fill_all(h, &SlabState::U);
    const int gy = h->dim2 ? 2 : 0;
    for (auto& s : h->slabs) {
      CK(cudaSetDevice(s.device));
      // interior rows, plus the domain's y ghost rows on the edge slabs (filled
      // there, or received as halos when y is periodic over several slabs)
      const int r0 = h->dim2 && s.sl.y0 == 0 ? -2 : 0;
      const int r1 = s.L.ny + (h->dim2 && s.sl.y0 + s.L.ny == h->d.ny ? 2 : 0);
      for (int c = 0; c < 4; ++c) {
        double* dst = field[c] + (int64_t)(s.sl.y0 + gy + r0) * ld;
        const double* src = s.U + s.L.origin() + c * s.L.fstride + (int64_t)r0 * s.L.pitch - 2;
        CK(cudaMemcpy2DAsync(dst, ld * sizeof(double), src, s.L.pitch * sizeof(double),
                             (size_t)(s.L.nx + 4) * sizeof(double), (size_t)(r1 - r0),
                             cudaMemcpyDefault, s.stream));
      }
    }
    sync_all(h);
    return 0;
  });
}

int lf_init_fourier(lf_handle* h, uint64_t seed) {
  LF_TRACE("lf_init_fourier");
  return guarded(h, [&] {
    if (!h->dim2) return set_err(h, LF_ERR_CONFIG, "the Fourier initial state is 2D");
    std::vector<double> tx, ty, amp;
    fourier_tables(seed, h->d, tx, ty, amp);  // whole-grid tables (host, libm)
    // global maxima need every slab's raw values first
    std::vector<double*> dtx(h->slabs.size()), dty(h->slabs.size()), damp(h->slabs.size());
    for (size_t k = 0; k < h->slabs.size(); ++k) {
      SlabState& s = h->slabs[k];
      CK(cudaSetDevice(s.device));
      CK(cudaMalloc(&dtx[k], tx.size() * sizeof(double)));
      CK(cudaMalloc(&dty[k], 64 * (size_t)s.L.ny * sizeof(double)));
      CK(cudaMalloc(&damp[k], 32 * sizeof(double)));
      CK(cudaMemcpy(dtx[k], tx.data(), tx.size() * sizeof(double), cudaMemcpyHostToDevice));
      // this slab's rows of every y table
      std::vector<double> tyl(64 * (size_t)s.L.ny);
      for (int t = 0; t < 64; ++t)
        std::memcpy(&tyl[(size_t)t * s.L.ny], &ty[(size_t)t * h->d.ny + s.sl.y0],
                    (size_t)s.L.ny * sizeof(double));
      CK(cudaMemcpy(dty[k], tyl.data(), tyl.size() * sizeof(double), cudaMemcpyHostToDevice));
      CK(cudaMemcpy(damp[k], amp.data(), 32 * sizeof(double), cudaMemcpyHostToDevice));
      CK(cudaMemsetAsync(s.aux, 0, 4 * sizeof(unsigned long long), s.stream));
      launch_fourier_raw(s.field(s.U), s.L, dtx[k], dty[k], damp[k], s.stream);
      launch_absmax(s.field(s.U), s.L, s.aux, s.stream);
    }
    unsigned long long mx[4] = {0, 0, 0, 0};
    for (auto& s : h->slabs) {
      unsigned long long m[4];
      CK(cudaSetDevice(s.device));
      CK(cudaMemcpyAsync(m, s.aux, sizeof m, cudaMemcpyDeviceToHost, s.stream));
      CK(cudaStreamSynchronize(s.stream));
      for (int c = 0; c < 4; ++c) mx[c] = std::max(mx[c], m[c]);
    }
    if (h->nccl) nccl_max_u64(h, mx, 4);
    for (size_t k = 0; k < h->slabs.size(); ++k) {
      SlabState& s = h->slabs[k];
      CK(cudaSetDevice(s.device));
      CK(cudaMemcpyAsync(s.aux, mx, sizeof mx, cudaMemcpyHostToDevice, s.stream));
      launch_fourier_finish(s.field(s.U), s.L, s.aux, h->d.gamma, s.stream);
      CK(cudaStreamSynchronize(s.stream));
      cudaFree(dtx[k]);
      cudaFree(dty[k]);
      cudaFree(damp[k]);
    }
    CK(cudaGetLastError());
    h->tp_exact = 0;
    h->small_ieee = 0;  // a new state: the plain fast kernels first
    h->rate_valid = false;
    fused_invalidate(h);
    return 0;
  });
}

int lf_init_regions(lf_handle* h, const double* regions, int nreg) {
  LF_TRACE("lf_init_regions");
  return guarded(h, [&] {
    if (!regions || nreg < 1) return set_err(h, LF_ERR_ARGUMENT, "no regions");
    for (int r = 0; r < nreg; ++r) {
      const double* R = regions + 9 * r;
      const int m = (int)R[8];
      if (!(R[4] > 0.0) || !(R[7] > 0.0))  // conserved_from_primitive's checks (euler.hpp:89-90)
        return set_err(h, LF_ERR_PRIMITIVE, "%s = %s",
                       !(R[4] > 0.0) ? "non-positive density" : "non-positive pressure",
                       fmt_f(!(R[4] > 0.0) ? R[4] : R[7]).c_str());
      if (h->mc.n && (m < 1 || m > h->mc.n))
        return set_err(h, LF_ERR_CONFIG, "region material %d outside the material set", m);
    }
    unsigned long long fail = ~0ull;
    for (auto& s : h->slabs) {
      CK(cudaSetDevice(s.device));
      double* dreg = nullptr;
      unsigned long long* dfail = nullptr;
      CK(cudaMalloc(&dreg, 9 * (size_t)nreg * sizeof(double)));
      CK(cudaMalloc(&dfail, sizeof(unsigned long long)));
      CK(cudaMemcpyAsync(dreg, regions, 9 * (size_t)nreg * sizeof(double), cudaMemcpyHostToDevice,
                         s.stream));
      CK(cudaMemsetAsync(dfail, 0xff, sizeof(unsigned long long), s.stream));
      launch_init_regions(s.field(s.U), s.field(h->mc.n ? s.P : s.U), s.L, s.sl, h->d.x0, h->d.y0,
                          h->d.dx, h->d.dy, h->dim2, dreg, nreg, h->mc, h->d.gamma, dfail, s.stream);
      unsigned long long f;
      CK(cudaMemcpyAsync(&f, dfail, sizeof f, cudaMemcpyDeviceToHost, s.stream));
      CK(cudaStreamSynchronize(s.stream));
      fail = std::min(fail, f);
      cudaFree(dreg);
      cudaFree(dfail);
    }
    if (h->nccl) {  // min over ranks as max of the complement
      unsigned long long nf = ~fail;
      nccl_max_u64(h, &nf, 1);
      fail = ~nf;
    }
    if (fail != ~0ull) {
      // run.cpp:61-64 (the coordinate and the hit count of the first bad cell)
      const int i = (int)(fail % (unsigned long long)h->d.nx), j = (int)(fail / (unsigned long long)h->d.nx);
      const double x = h->d.x0 + (i + 0.5) * h->d.dx, y = h->d.y0 + (j + 0.5) * h->d.dy;
      int hits = 0;
      for (int r = 0; r < nreg; ++r) {
        const double* R = regions + 9 * r;
        hits += (x >= R[0] && x < R[1]) && (!h->dim2 || (y >= R[2] && y < R[3]));
      }
      return set_err(h, LF_ERR_CONFIG,
                     "cell center (%s,%s) is covered by %d regions; regions must tile the domain exactly",
                     fmt_f(x).c_str(), fmt_f(y).c_str(), hits);
    }
    if (h->mc.n) h->partials_ready = 1;
    h->tp_exact = 0;
    h->small_ieee = 0;  // a new state: the plain fast kernels first
    h->rate_valid = false;
    fused_invalidate(h);
    return 0;
  });
}

int lf_compute_dt(lf_handle* h, double cfl, double time, double limit_time, double* dt) {
  LF_TRACE("lf_compute_dt");
  return guarded(h, [&] {
    launch_rate_all(h, &SlabState::U);
    return finish_dt(h, combined_scalars(h, 0), cfl, time, limit_time, dt);
  });
}

int lf_edge_flux(int64_t n, const double* w_minus, const double* w_plus, const double* normals,
                 const double* gamma_minus, const double* gamma_plus, double* flux,
                 double* contact, int device, lf_error* err) {
  LF_TRACE("lf_edge_flux");
  if (err) clear_err(err);
  if (n < 0 || (n > 0 && (!w_minus || !w_plus || !normals || !gamma_minus || !gamma_plus || !flux)))
    return LF_ERR_ARGUMENT;
  if (n == 0) return 0;
  std::vector<void*> bufs;
  auto fail_dev = [&](const char* what) {
    for (void* p : bufs) cudaFree(p);
    if (err) {
      err->kind = LF_ERR_DEVICE;
      snprintf(err->message, sizeof err->message, "%s", what);
    }
    return LF_ERR_DEVICE;
  };
  if (cudaSetDevice(device) != cudaSuccess) return fail_dev("cudaSetDevice");
  const size_t sz[8] = {4, 4, 2, 1, 1, 4, 2, 0};
  double* d[7];
  for (int k = 0; k < 7; ++k) {
    if (cudaMalloc(&d[k], (size_t)n * sz[k] * sizeof(double)) != cudaSuccess) return fail_dev("cudaMalloc");
    bufs.push_back(d[k]);
  }
  unsigned long long* dfail = nullptr;
  if (cudaMalloc(&dfail, sizeof *dfail) != cudaSuccess) return fail_dev("cudaMalloc");
  bufs.push_back(dfail);
  const double* src[5] = {w_minus, w_plus, normals, gamma_minus, gamma_plus};
  for (int k = 0; k < 5; ++k)
    if (cudaMemcpy(d[k], src[k], (size_t)n * sz[k] * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess)
      return fail_dev("cudaMemcpy");
  if (cudaMemset(dfail, 0xff, sizeof *dfail) != cudaSuccess) return fail_dev("cudaMemset");
  launch_edge_flux(n, d[0], d[1], d[2], d[3], d[4], d[5], contact ? d[6] : nullptr, dfail, 0);
  unsigned long long f = 0;
  if (cudaMemcpy(&f, dfail, sizeof f, cudaMemcpyDeviceToHost) != cudaSuccess ||
      cudaMemcpy(flux, d[5], (size_t)n * 4 * sizeof(double), cudaMemcpyDeviceToHost) != cudaSuccess ||
      (contact && cudaMemcpy(contact, d[6], (size_t)n * 2 * sizeof(double), cudaMemcpyDeviceToHost) !=
                      cudaSuccess))
    return fail_dev("edge_flux kernel");
  for (void* p : bufs) cudaFree(p);
  if (f == ~0ull) return 0;
  // sound_speed's throw (euler.hpp:99-104) for the smallest failing face
  const int64_t i = (int64_t)(f / 4);
  const int which = (int)(f % 4);
  const double v = (which < 2 ? w_minus : w_plus)[4 * i + (which % 2 ? 3 : 0)];
  if (err) {
    err->kind = LF_ERR_PRIMITIVE;
    err->i = i;
    err->value = v;
    snprintf(err->message, sizeof err->message, "%s = %s",
             which % 2 ? "non-positive pressure" : "non-positive density", fmt_f(v).c_str());
  }
  return LF_ERR_PRIMITIVE;
}

int lf_interior_totals(lf_handle* h, double tot[4]) {
  LF_TRACE("lf_interior_totals");
  return guarded(h, [&] {
    if (!tot) return set_err(h, LF_ERR_ARGUMENT, "null totals");
    // slabs in row order; each continues the running sums of the one below
    std::vector<size_t> order(h->slabs.size());
    for (size_t k = 0; k < order.size(); ++k) order[k] = k;
    std::sort(order.begin(), order.end(),
              [&](size_t a, size_t b) { return h->slabs[a].sl.y0 < h->slabs[b].sl.y0; });
    double run[4] = {0.0, 0.0, 0.0, 0.0};
    for (size_t n = 0; n < order.size(); ++n) {
      SlabState& s = h->slabs[order[n]];
      CK(cudaSetDevice(s.device));
      double* d = nullptr;  // {in[4], out[4]}
      CK(cudaMalloc(&d, 8 * sizeof(double)));
      CK(cudaMemcpyAsync(d, run, sizeof run, cudaMemcpyHostToDevice, s.stream));
      if (h->nccl) nccl_recv_prev(h, d, 4);
      launch_interior_sums(s.U + s.L.origin(), s.L.fstride, (int)s.L.pitch, s.L.nx, s.L.ny, d,
                           d + 4, s.stream);
      if (h->nccl) {
        nccl_send_next(h, d + 4, 4);
        // the last rank holds the totals: every other rank contributes +0.0,
        // which leaves them unchanged (a running sum from +0.0 is never -0.0)
        if (h->rank != h->nranks - 1) CK(cudaMemsetAsync(d + 4, 0, 4 * sizeof(double), s.stream));
        nccl_sum_f64(h, d + 4, 4);
      }
      CK(cudaMemcpyAsync(run, d + 4, sizeof run, cudaMemcpyDeviceToHost, s.stream));
      CK(cudaStreamSynchronize(s.stream));
      cudaFree(d);
      CK(cudaGetLastError());
    }
    const double vol = h->dim2 ? h->d.dx * h->d.dy : h->d.dx;
    for (int c = 0; c < 4; ++c) tot[c] = run[c] * vol;
    return 0;
  });
}

int lf_max_rate(lf_handle* h, double* rate) {
  return guarded(h, [&] {
    launch_rate_all(h, &SlabState::U);
    *rate = bits_to_double(combined_scalars(h, 0).rate_bits);
    return 0;
  });
}

int lf_euler_stage(lf_handle* h, double dt, int64_t step) {
  LF_TRACE("lf_euler_stage");
  return guarded(h, [&] {
    for (auto& s : h->slabs) alloc_staged(s);
    staged_stage(h, &SlabState::U, &SlabState::U, &SlabState::Us, 0, false, dt, 1);
    const Scalars s1 = combined_scalars(h, 1);
    int rc = check_stage(h, s1, &SlabState::U, &SlabState::Us, step, dt);
    if (rc) return rc;
    swap_state(h, &SlabState::U, &SlabState::Us);
    h->rate_valid = false;
    fused_invalidate(h);
    return 0;
  });
}

int lf_heun_step(lf_handle* h, double cfl, double time, double limit_time, int64_t step,
                 double* boundary_outflow, lf_step_out* out) {
  LF_TRACE("lf_heun_step");
  return guarded(h, [&] {
    if (use_small(h)) return small_heun(h, cfl, time, limit_time, step, boundary_outflow, out);
    if (use_fused(h))
      return fused_heun(h, cfl, time, limit_time, step, boundary_outflow, out);
    return staged_heun(h, cfl, time, limit_time, step, boundary_outflow, out);
  });
}

int lf_advance(lf_handle* h, int nsteps, double cfl, double t_final, double* time,
               int64_t* step, double* outflow, lf_step_out* per_step, int* taken) {
  LF_TRACE("lf_advance");
  return guarded(h, [&] {
    if (use_small(h))
      return small_advance(h, nsteps, cfl, t_final, time, step, outflow, per_step, taken);
    if (use_fused(h))
      return fused_advance(h, nsteps, cfl, t_final, time, step, outflow, per_step, taken);
    // stage-wise fallback keeps the run.cpp loop on the host
    int k = 0;
    if (taken) *taken = 0;
    while (k < nsteps && *time < t_final) {
      lf_step_out o;
      int rc = staged_heun(h, cfl, *time, t_final, *step, outflow, &o);
      if (rc) return rc;
      *time = o.time;
      *step = o.step;
      if (per_step) per_step[k] = o;
      ++k;
      if (taken) *taken = k;
    }
    return 0;
  });
}

int lf_last_error(lf_handle* h, lf_error* err) {
  if (!h || !err) return LF_ERR_ARGUMENT;
  *err = h->err;
  return 0;
}

int lf_set_stream(lf_handle* h, void* stream) {
  if (!h) return LF_ERR_ARGUMENT;
  for (auto& s : h->slabs)
    s.stream = stream ? (cudaStream_t)stream
                      : (s.own_stream ? s.own_stream : h->slabs[0].own_stream);
  return 0;
}

int lf_set_path(lf_handle* h, int path) {
  if (!h || path < LF_PATH_AUTO || path > LF_PATH_SMALL) return LF_ERR_ARGUMENT;
  h->path = path;
  return 0;
}

int lf_resolved_path(lf_handle* h, int* path) {
  if (!h || !path) return LF_ERR_ARGUMENT;
  return guarded(h, [&] {
    *path = use_small(h)   ? LF_PATH_SMALL
            : !use_fused(h) ? LF_PATH_STAGED
            : twopass_selected(h) ? LF_PATH_TWOPASS
                                  : LF_PATH_FUSED;
    return 0;
  });
}

int lf_set_math(lf_handle* h, int math) {
  if (!h || (math != LF_MATH_EXACT && math != LF_MATH_CONTRACT)) return LF_ERR_ARGUMENT;
  h->math = math;
  return 0;
}

int lf_time_steps(lf_handle* h, int nsteps, double cfl, double* kernel_ms, double* step_ms,
                  int* kernel_launches) {
  LF_TRACE("lf_time_steps");
  return guarded(h, [&] {
    if (use_small(h)) return small_time_steps(h, nsteps, cfl, kernel_ms, step_ms, kernel_launches);
    if (!use_fused(h))
      return set_err(h, LF_ERR_ARGUMENT, "lf_time_steps times the fused / two-pass path");
    return fused_time_steps(h, nsteps, cfl, kernel_ms, step_ms, kernel_launches);
  });
}

int lf_device_bytes(lf_handle* h, int64_t* bytes) {
  if (!h || !bytes) return LF_ERR_ARGUMENT;
  int64_t b = 0;
  for (auto& s : h->slabs) {
    b += 2 * s.L.alloc * 8;
    if (s.Us) b += 2 * s.L.alloc * 8 + 2 * 4 * (s.fx_stride + s.fy_stride) * 8;
    if (s.P)
      b += (4 * ((int64_t)h->mc.n * s.L.fstride + s.L.pitch) + 2 * (s.L.fstride + s.L.pitch) +
            2 * (s.fx_stride + s.fy_stride)) * 8;
  }
  *bytes = b + fused_bytes(h);
  return 0;
}

}  // extern "C"

extern "C" int lf_launch_count(lf_handle* h, int64_t* launches) {
  if (!h || !launches) return LF_ERR_ARGUMENT;
  *launches = lfb::launch_count();
  return 0;
}

extern "C" int lf_slab_partition(int ny, int nranks, int rank, int* row0, int* nrows) {
  if (!row0 || !nrows || nranks < 1 || rank < 0 || rank >= nranks || ny < 1) return LF_ERR_ARGUMENT;
  slab_rows(ny, nranks, rank, row0, nrows);
  return LF_OK;
}
