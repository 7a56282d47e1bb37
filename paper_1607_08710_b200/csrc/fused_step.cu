// fused_step.cu -- one kernel per Heun time step (LagfluxSolver::heun_step, solver.cpp:489-546).
//
// Design:
//  * A block owns a strip of NC = 128 columns (TXO = 120 output columns plus a
//    4-column halo each side) and marches down a chunk of rows.  The whole step
//    -- primitives, MUSCL traces, Lagrangian HLL, upwind fluxes, predictor U*,
//    corrector U^{n+1}, positivity checks, min rho / min e_int and the CFL rate
//    of U^{n+1} for the next dt -- happens in one pass: U^n is read from HBM
//    about once (plus ~7% halo re-reads, mostly L2 hits) and U^{n+1} written once,
//    64 B/cell-update of compulsory traffic instead of the stage-wise 288 B.
//  * Warp specialisation: warps 0-3 ("P") run stage 1 on input row r (U^n ->
//    F^n faces -> U*(r-2)); warps 4-7 ("C") run stage 2 three rows behind
//    (U*(a) -> F* faces -> U^{n+1}(a-2)).  P and C exchange rows through small
//    shared-memory rings; each group synchronises internally on its own named
//    barrier and both meet once per row iteration.
//  * y-direction stencil data of a column lives in the registers of the thread
//    owning that column (rolling 3-row window, slopes shared between the two
//    faces of a cell); x-direction neighbours go through shared memory.
//  * Every fp64 expression keeps the reference's evaluation order (compiled
//    with --fmad=false), so results are bit-identical to the reference.
//  * Failure checks are detection only: any flag makes the host re-run that
//    step with the stage-wise kernels, which reproduce the reference's exact
//    error (kind, smallest index, text) and state semantics.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "fused.h"
#include "nccl_comm.h"

namespace lfb {

namespace {

constexpr int NC = 128;          // columns per strip (threads per group)
constexpr int TXO = NC - 8;      // output columns per strip
constexpr int NTHREADS = 2 * NC; // P group + C group
constexpr unsigned FULL = 0xffffffffu;

// Per-step control record, written by the host (first step) or k_finalize.
struct StepCtl {
  double time;                    // SolverState::time at the start of the step
  unsigned long long rate_bits;   // CFL rate of the state at the start of the step
  int done;                       // 1: skip (limit reached or an earlier step failed)
  int dtfail;                     // the rate check of this step's input failed
};

// Per-step accumulators: every field reduces with max (min via ~bits), so one
// atomicMax per block and one NCCL max across ranks combine them exactly.
struct StepAcc {
  unsigned long long rate_next;   // CFL rate of U^{n+1}
  unsigned long long fail;        // any failure flag in this step
  unsigned long long nmin_rho;    // ~bits(min rho of U^{n+1})
  unsigned long long nmin_eint;   // ~bits(min e_int of U^{n+1})
  unsigned long long dtfail_next; // rate check of U^{n+1} failed
  unsigned long long pad[3];
};

constexpr unsigned long long NINF_KEY = ~0x7ff0000000000000ull;  // ~bits(+inf)

struct FusedArgs {
  const double* __restrict__ u;   // U^n, component 0 at (0, 0)
  double* __restrict__ un;        // U^{n+1}
  int64_t pitch, fstride;
  int nx, ny;                     // local interior
  int y0g;                        // global row of local row 0
  int nyg;                        // global rows
  int rows_per_chunk;
  double gamma, gm1, beta, dx, dy;
  double cfl, limit;
  int bc_xlo, bc_xhi, bc_ylo, bc_yhi;
  int bottom_edge, top_edge;      // non-periodic domain edge at this slab's bottom / top
  const StepCtl* ctl;
  StepAcc* acc;
  double* bnd;                    // [left 4*nyg | right 4*nyg | bottom 4*nx | top 4*nx]
};

__device__ __forceinline__ void bar_named(int id) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(NC) : "memory");
}

__device__ __forceinline__ double key_to_double(unsigned long long b) {
  return __longlong_as_double((long long)b);
}

// limited slope of the middle value and the two traces of a cell (reconstruct.hpp:33-49)
template <bool MUSCL>
__device__ __forceinline__ void cell_traces(double qm, double q0, double qp, double beta,
                                            double& lo, double& hi) {
  if (MUSCL) {
    const double s = slope3(qm, q0, qp, beta);
    lo = q0 - 0.5 * s;   // plus-side trace of the face below / left (q2 - 0.5 s2)
    hi = q0 + 0.5 * s;   // minus-side trace of the face above / right (q1 + 0.5 s1)
  } else {
    lo = q0;
    hi = q0;
  }
}

template <bool MUSCL>
__global__ void __launch_bounds__(NTHREADS, 2) k_fused_step(FusedArgs a) {
  extern __shared__ double smem[];
  double* sWx = smem;                  // [4][NC]     P: W(r-2) for x slopes
  double* sTx = sWx + 4 * NC;          // [4][NC]     P: x hi-traces
  double* sFnx = sTx + 4 * NC;         // [4][4][NC]  ring: F^n x-faces of a row
  double* sFny = sFnx + 16 * NC;       // [4][4][NC]  ring: F^n y-faces
  double* sUs = sFny + 16 * NC;        // [2][4][NC]  U* rows
  double* sWc = sUs + 8 * NC;          // [4][NC]     C: W*(j) for x slopes
  double* sTc = sWc + 4 * NC;          // [4][NC]     C: x hi-traces
  double* sFc = sTc + 4 * NC;          // [4][NC]     C: 0.5 (F^n + F*) x-faces

  const StepCtl ctl = *a.ctl;
  if (ctl.done) return;
  if (ctl.dtfail) {
    if (threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0) atomicMax(&a.acc->fail, 1ull);
    return;
  }
  // dt exactly as compute_dt (solver.cpp:476-477) and apply_update (:262-263)
  const double rate = key_to_double(ctl.rate_bits);
  double dt = a.cfl / rate;
  if (ctl.time + dt > a.limit) dt = a.limit - ctl.time;
  if (!(dt > 0.0)) {
    if (threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0) atomicMax(&a.acc->fail, 1ull);
    return;
  }
  const double lam_x = dt / a.dx;
  const double lam_y = dt / a.dy;

  Consts K;
  K.gamma = a.gamma;
  K.gm1 = a.gm1;
  K.beta = a.beta;
  K.dx = a.dx;
  K.dy = a.dy;

  const int t = threadIdx.x & (NC - 1);
  const bool is_p = threadIdx.x < NC;
  const int x0 = blockIdx.x * TXO;
  const int c = x0 - 4 + t;                      // this thread's column
  const int y0 = blockIdx.y * a.rows_per_chunk;  // chunk output rows [y0, y1)
  const int y1 = min(y0 + a.rows_per_chunk, a.ny);
  const int nit = (y1 - y0) + 9;
  const bool col_in_mem = c >= -NG && c < a.nx + NG;
  const bool col_interior = c >= 0 && c < a.nx;
  const bool bottom_edge = a.bottom_edge && y0 == 0;
  const bool top_edge = a.top_edge && y1 == a.ny;

  unsigned fail = 0;

  if (is_p) {
    // ================================================================ stage 1 (P)
    double wm2[4] = {1.0, 0.0, 0.0, 1.0}, wm1[4] = {1.0, 0.0, 0.0, 1.0};
    double hiprev[4] = {1.0, 0.0, 0.0, 1.0}, fyprev[4] = {0.0, 0.0, 0.0, 0.0};
    for (int k = 0; k < nit; ++k) {
      const int r = y0 - 4 + k;
      const bool p_active = k <= (y1 - y0) + 7;
      double w[4] = {1.0, 0.0, 0.0, 1.0};
      double fy[4] = {0.0, 0.0, 0.0, 0.0};
      if (p_active) {
        // -- 1. U^n(r) -> W(r) (solver.cpp:145-163)
        if (col_in_mem) {
          const int64_t o = (int64_t)r * a.pitch + c;
          const double r0 = __ldg(a.u + o);
          const double m1 = __ldg(a.u + a.fstride + o);
          const double m2 = __ldg(a.u + 2 * a.fstride + o);
          const double e3 = __ldg(a.u + 3 * a.fstride + o);
          if (r0 > 0.0) {
            w[0] = r0;
            primitive(r0, m1, m2, e3, a.gm1, w[1], w[2], w[3]);
            if (!(w[3] > 0.0) && col_interior && r >= 0 && r < a.ny) fail = 1;
          } else {
            w[0] = w[1] = w[2] = w[3] = 0.0;
            if (col_interior && r >= 0 && r < a.ny) fail = 1;
          }
        }
        // -- 2. y direction: slope of row r-1, F^n on face (r-2 | r-1)
        if (k >= 2) {
          double lo[4], hi[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) cell_traces<MUSCL>(wm2[q], wm1[q], w[q], a.beta, lo[q], hi[q]);
          if (k >= 3) {
            if (!traces_ok(hiprev[0], hiprev[3], lo[0], lo[3]) && col_interior && r - 1 >= 0 &&
                r - 1 <= a.ny)
              fail = 1;
            face_flux<1>(hiprev[0], hiprev[1], hiprev[2], hiprev[3], lo[0], lo[1], lo[2], lo[3], K, fy);
#pragma unroll
            for (int q = 0; q < 4; ++q) sFny[((k & 3) * 4 + q) * NC + t] = fy[q];
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) hiprev[q] = hi[q];
        }
        // -- 3. x direction of row r-2: traces, then F^n x-faces into the ring
        if (k >= 2) {
#pragma unroll
          for (int q = 0; q < 4; ++q) sWx[q * NC + t] = wm2[q];
        }
      }
      bar_named(1);
      double xlo[4] = {1.0, 0.0, 0.0, 1.0};
      if (p_active && k >= 2 && t >= 1 && t <= NC - 2) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          double hi;
          cell_traces<MUSCL>(sWx[q * NC + t - 1], sWx[q * NC + t], sWx[q * NC + t + 1], a.beta,
                             xlo[q], hi);
          sTx[q * NC + t] = hi;
        }
      }
      bar_named(1);
      if (p_active && k >= 2 && t >= 2 && t <= NC - 2) {
        const double m0 = sTx[0 * NC + t - 1], m1 = sTx[1 * NC + t - 1];
        const double m2 = sTx[2 * NC + t - 1], m3 = sTx[3 * NC + t - 1];
        if (!traces_ok(m0, m3, xlo[0], xlo[3]) && c >= 0 && c <= a.nx && r - 2 >= 0 &&
            r - 2 < a.ny)
          fail = 1;
        double fx[4];
        face_flux<0>(m0, m1, m2, m3, xlo[0], xlo[1], xlo[2], xlo[3], K, fx);
#pragma unroll
        for (int q = 0; q < 4; ++q) sFnx[((k & 3) * 4 + q) * NC + t] = fx[q];
      }
      bar_named(1);
      // -- 4. predictor U*(r-2) (solver.cpp:283-291 with one flux set)
      if (p_active && k >= 4 && t >= 2 && t <= NC - 3 && col_in_mem) {
        const int row = r - 2;
        const int64_t o = (int64_t)row * a.pitch + c;
        double v[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const double fxl = sFnx[((k & 3) * 4 + q) * NC + t];
          const double fxr = sFnx[((k & 3) * 4 + q) * NC + t + 1];
          double val = __ldg(a.u + q * a.fstride + o) - lam_x * (fxr - fxl);
          val -= lam_y * (fy[q] - fyprev[q]);
          v[q] = val;
          sUs[((k & 1) * 4 + q) * NC + t] = val;
        }
        if (col_interior && row >= 0 && row < a.ny) {
          const double eint = internal_energy(v[0], v[1], v[2], v[3]);
          if (!(v[0] > 0.0) || !(eint > 0.0)) fail = 1;
        }
      }
      if (p_active && k >= 3) {
#pragma unroll
        for (int q = 0; q < 4; ++q) fyprev[q] = fy[q];
      }
      if (p_active) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          wm2[q] = wm1[q];
          wm1[q] = w[q];
        }
      }
      __syncthreads();
    }
  } else {
    // ================================================================ stage 2 (C)
    double vm2[4] = {1.0, 0.0, 0.0, 1.0}, vm1[4] = {1.0, 0.0, 0.0, 1.0};
    double hiprev[4] = {1.0, 0.0, 0.0, 1.0}, fcprev[4] = {0.0, 0.0, 0.0, 0.0};
    double stash[4] = {1.0, 0.0, 0.0, 1.0};
    unsigned long long rate_key = 0ull, nmin_r = NINF_KEY, nmin_e = NINF_KEY;
    unsigned dtfail = 0;
    // source column of this thread's U* value (ghost columns at non-periodic x edges)
    int src_t = t;
    bool flip_u = false;
    if (c < 0 && a.bc_xlo != LF_PERIODIC) {
      const int sc = a.bc_xlo == LF_REFLECTIVE ? -c - 1 : 0;
      src_t = t + (sc - c);
      flip_u = a.bc_xlo == LF_REFLECTIVE;
    } else if (c >= a.nx && a.bc_xhi != LF_PERIODIC) {
      const int sc = a.bc_xhi == LF_REFLECTIVE ? 2 * a.nx - 1 - c : a.nx - 1;
      src_t = t + (sc - c);
      flip_u = a.bc_xhi == LF_REFLECTIVE;
    }
    const bool has_us = t >= 2 && t <= NC - 3 && src_t >= 2 && src_t <= NC - 3;
    for (int k = 0; k < nit; ++k) {
      const int aa = y0 - 7 + k;   // U* row consumed this iteration
      const int j = aa - 2;        // U^{n+1} row finished this iteration
      const bool c_active = k >= 5;
      double w[4] = {1.0, 0.0, 0.0, 1.0};
      double fc[4] = {0.0, 0.0, 0.0, 0.0};
      if (c_active) {
        // -- 1. U*(aa) -> W*(aa) with the boundary images of the reference's
        //       ghost fill of predictor_ (grid.cpp:72-114)
        if (has_us) {
          const int buf = (k + 1) & 1;
          const double u0 = sUs[(buf * 4 + 0) * NC + src_t];
          double u1 = sUs[(buf * 4 + 1) * NC + src_t];
          const double u2 = sUs[(buf * 4 + 2) * NC + src_t];
          const double u3 = sUs[(buf * 4 + 3) * NC + src_t];
          if (flip_u) u1 = -1.0 * u1;
          if (u0 > 0.0) {
            w[0] = u0;
            primitive(u0, u1, u2, u3, a.gm1, w[1], w[2], w[3]);
            if (!(w[3] > 0.0) && col_interior && aa >= 0 && aa < a.ny) fail = 1;
          } else {
            w[0] = w[1] = w[2] = w[3] = 0.0;
            if (col_interior && aa >= 0 && aa < a.ny) fail = 1;
          }
        }
        const double sy = a.bc_ylo == LF_REFLECTIVE ? -1.0 : 1.0;
        if (bottom_edge && aa == 0) {
          // W*(-1) = image of W*(0)
#pragma unroll
          for (int q = 0; q < 4; ++q) vm1[q] = w[q];
          if (a.bc_ylo == LF_REFLECTIVE) vm1[2] = sy * vm1[2];
        }
        if (bottom_edge && aa == 1) {
          // hi trace of ghost row -1 from W*(-2) = image(W*(1) or W*(0)), W*(-1), W*(0)
          double g2[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) g2[q] = a.bc_ylo == LF_REFLECTIVE ? w[q] : vm1[q];
          if (a.bc_ylo == LF_REFLECTIVE) g2[2] = sy * g2[2];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            double lo;
            cell_traces<MUSCL>(g2[q], vm2[q], vm1[q], a.beta, lo, hiprev[q]);
          }
        }
        const double syh = a.bc_yhi == LF_REFLECTIVE ? -1.0 : 1.0;
        if (top_edge && aa == a.ny) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            w[q] = vm1[q];
            stash[q] = a.bc_yhi == LF_REFLECTIVE ? vm2[q] : vm1[q];
          }
          if (a.bc_yhi == LF_REFLECTIVE) {
            w[2] = syh * w[2];
            stash[2] = syh * stash[2];
          }
        } else if (top_edge && aa == a.ny + 1) {
#pragma unroll
          for (int q = 0; q < 4; ++q) w[q] = stash[q];
        }
        // -- 2. y direction: slope of row aa-1, F* on face (aa-2 | aa-1), averaged with F^n
        if (k >= 7) {
          double lo[4], hi[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) cell_traces<MUSCL>(vm2[q], vm1[q], w[q], a.beta, lo[q], hi[q]);
          if (k >= 8) {
            if (!traces_ok(hiprev[0], hiprev[3], lo[0], lo[3]) && col_interior && aa - 1 >= 0 &&
                aa - 1 <= a.ny)
              fail = 1;
            double fs[4];
            face_flux<1>(hiprev[0], hiprev[1], hiprev[2], hiprev[3], lo[0], lo[1], lo[2], lo[3], K, fs);
#pragma unroll
            for (int q = 0; q < 4; ++q) fc[q] = 0.5 * (sFny[(((k + 1) & 3) * 4 + q) * NC + t] + fs[q]);
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) hiprev[q] = hi[q];
        }
        // -- 3. x direction of row j = aa-2
        if (k >= 9) {
#pragma unroll
          for (int q = 0; q < 4; ++q) sWc[q * NC + t] = vm2[q];
        }
      }
      bar_named(2);
      double xlo[4] = {1.0, 0.0, 0.0, 1.0};
      if (c_active && k >= 9 && t >= 3 && t <= NC - 4) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          double hi;
          cell_traces<MUSCL>(sWc[q * NC + t - 1], sWc[q * NC + t], sWc[q * NC + t + 1], a.beta,
                             xlo[q], hi);
          sTc[q * NC + t] = hi;
        }
      }
      bar_named(2);
      if (c_active && k >= 9 && t >= 4 && t <= NC - 4) {
        const double m0 = sTc[0 * NC + t - 1], m1 = sTc[1 * NC + t - 1];
        const double m2 = sTc[2 * NC + t - 1], m3 = sTc[3 * NC + t - 1];
        if (!traces_ok(m0, m3, xlo[0], xlo[3]) && c >= 0 && c <= a.nx && j >= 0 && j < a.ny)
          fail = 1;
        double fs[4];
        face_flux<0>(m0, m1, m2, m3, xlo[0], xlo[1], xlo[2], xlo[3], K, fs);
#pragma unroll
        for (int q = 0; q < 4; ++q) sFc[q * NC + t] = 0.5 * (sFnx[(((k + 1) & 3) * 4 + q) * NC + t] + fs[q]);
      }
      bar_named(2);
      // -- 4. corrector U^{n+1}(j) (solver.cpp:283-291, two flux sets) + epilogue
      if (c_active && k >= 9 && t >= 4 && t <= NC - 5 && col_interior) {
        const int64_t o = (int64_t)j * a.pitch + c;
        double v[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          double val = __ldg(a.u + q * a.fstride + o) - lam_x * (sFc[q * NC + t + 1] - sFc[q * NC + t]);
          val -= lam_y * (fc[q] - fcprev[q]);
          v[q] = val;
          a.un[q * a.fstride + o] = val;
        }
        const double eint = internal_energy(v[0], v[1], v[2], v[3]);
        if (!(v[0] > 0.0) || !(eint > 0.0)) {
          fail = 1;
        } else {
          const unsigned long long kr = ~pos_bits(v[0]), ke = ~pos_bits(eint);
          nmin_r = kr > nmin_r ? kr : nmin_r;
          nmin_e = ke > nmin_e ? ke : nmin_e;
        }
        double rr;
        if (cfl_rate<true>(v[0], v[1], v[2], v[3], K, rr)) {
          if (rr == rr) {
            const unsigned long long b = pos_bits(rr);
            rate_key = b > rate_key ? b : rate_key;
          }
        } else {
          dtfail = 1;
        }
        // domain-boundary faces for accumulate_boundary_outflow (solver.cpp:406-432)
        const int jg = j + a.y0g;
        if (c == 0)
          for (int q = 0; q < 4; ++q) a.bnd[(int64_t)q * a.nyg + jg] = sFc[q * NC + t];
        if (c == a.nx - 1)
          for (int q = 0; q < 4; ++q) a.bnd[4 * (int64_t)a.nyg + (int64_t)q * a.nyg + jg] = sFc[q * NC + t + 1];
        if (jg == 0)
          for (int q = 0; q < 4; ++q) a.bnd[8 * (int64_t)a.nyg + (int64_t)q * a.nx + c] = fcprev[q];
        if (jg == a.nyg - 1)
          for (int q = 0; q < 4; ++q)
            a.bnd[8 * (int64_t)a.nyg + 4 * (int64_t)a.nx + (int64_t)q * a.nx + c] = fc[q];
      }
      if (c_active && k >= 8) {
#pragma unroll
        for (int q = 0; q < 4; ++q) fcprev[q] = fc[q];
      }
      if (c_active) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          vm2[q] = vm1[q];
          vm1[q] = w[q];
        }
      }
      __syncthreads();
    }
    // block-level reductions (warp shuffles, then one atomic per warp)
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long r2 = __shfl_xor_sync(FULL, rate_key, o);
      const unsigned long long a2 = __shfl_xor_sync(FULL, nmin_r, o);
      const unsigned long long b2 = __shfl_xor_sync(FULL, nmin_e, o);
      rate_key = r2 > rate_key ? r2 : rate_key;
      nmin_r = a2 > nmin_r ? a2 : nmin_r;
      nmin_e = b2 > nmin_e ? b2 : nmin_e;
    }
    dtfail = __any_sync(FULL, dtfail);
    if ((threadIdx.x & 31) == 0) {
      if (rate_key) atomicMax(&a.acc->rate_next, rate_key);
      if (nmin_r != NINF_KEY) atomicMax(&a.acc->nmin_rho, nmin_r);
      if (nmin_e != NINF_KEY) atomicMax(&a.acc->nmin_eint, nmin_e);
      if (dtfail) atomicMax(&a.acc->dtfail_next, 1ull);
    }
  }
  if (__any_sync(FULL, fail) && (threadIdx.x & 31) == 0) atomicMax(&a.acc->fail, 1ull);
}

// Per-step record handed back to the host.
struct StepRec {
  double dt;
  double time;       // time after the step
  double min_rho;
  double min_eint;
  int hits;
  int status;        // 0 ok, 1 failure flag (host diagnoses), 2 skipped (done)
};

// After the step's kernel (and the cross-rank all-reduce of acc): dt / time
// bookkeeping (solver.cpp:494,542-544), the ordered boundary-outflow sums
// (solver.cpp:406-432, one thread per component and direction) and the
// control record of the next step.
__global__ void k_finalize(const StepCtl* __restrict__ ctl, StepAcc* acc, StepCtl* nxt,
                           StepRec* rec, const double* __restrict__ bnd, double* outflow,
                           int nx, int nyg, double dx, double dy, double cfl, double limit,
                           double t_final) {
  __shared__ double sums[8];
  const int tid = threadIdx.x;
  const StepCtl c = *ctl;
  const bool skip = c.done != 0;
  double dt = 0.0;
  if (!skip) {
    const double rate = __longlong_as_double((long long)c.rate_bits);
    dt = cfl / rate;
    if (c.time + dt > limit) dt = limit - c.time;
  }
  const bool failed = !skip && (acc->fail != 0 || c.dtfail || !(dt > 0.0));
  if (!skip && !failed && tid < 8) {
    // solver.cpp:412-430: per component, right - left over rows in order; then top - bottom
    const int q = tid & 3;
    double s = 0.0;
    if (tid < 4) {
      const double* l = bnd + (int64_t)q * nyg;
      const double* r = bnd + 4 * (int64_t)nyg + (int64_t)q * nyg;
      for (int jj = 0; jj < nyg; ++jj) s += r[jj] - l[jj];
    } else {
      const double* b = bnd + 8 * (int64_t)nyg + (int64_t)q * nx;
      const double* tp = bnd + 8 * (int64_t)nyg + 4 * (int64_t)nx + (int64_t)q * nx;
      for (int ii = 0; ii < nx; ++ii) s += tp[ii] - b[ii];
    }
    sums[tid] = s;
  }
  __syncthreads();
  if (tid != 0) return;
  StepRec r;
  r.dt = dt;
  r.hits = 0;
  r.time = c.time;
  r.min_rho = 0.0;
  r.min_eint = 0.0;
  StepCtl n;
  n.rate_bits = acc->rate_next;
  n.dtfail = acc->dtfail_next != 0;
  if (skip) {
    r.status = 2;
    n = c;
    n.done = 1;
  } else if (failed) {
    r.status = 1;
    n = c;
    n.done = 1;
  } else {
    r.status = 0;
    r.hits = c.time + dt >= limit;
    r.time = r.hits ? limit : c.time + dt;
    r.min_rho = __longlong_as_double((long long)~acc->nmin_rho);
    r.min_eint = __longlong_as_double((long long)~acc->nmin_eint);
    const double ax = dt * dy, ay = dt * dx;
    for (int q = 0; q < 4; ++q) {
      outflow[q] += ax * sums[q];
      outflow[q] += ay * sums[4 + q];
    }
    n.time = r.time;
    n.done = !(r.time < t_final);
  }
  *rec = r;
  *nxt = n;
  // reset this step's accumulators for the step after next
  acc->rate_next = 0ull;
  acc->fail = 0ull;
  acc->nmin_rho = NINF_KEY;
  acc->nmin_eint = NINF_KEY;
  acc->dtfail_next = 0ull;
}

__global__ void k_acc_init(StepAcc* acc) {
  for (int i = 0; i < 2; ++i) {
    acc[i].rate_next = 0ull;
    acc[i].fail = 0ull;
    acc[i].nmin_rho = NINF_KEY;
    acc[i].nmin_eint = NINF_KEY;
    acc[i].dtfail_next = 0ull;
  }
}

struct DevFail : std::runtime_error {
  explicit DevFail(const std::string& w) : std::runtime_error(w) {}
};

#define FK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess) throw DevFail(std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

constexpr size_t SMEM_BYTES = (size_t)(4 + 4 + 16 + 16 + 8 + 4 + 4 + 4) * NC * sizeof(double);

}  // namespace

// Fused-path state of a handle (one per handle; all slabs on one device).
struct FusedState {
  StepCtl* ctl = nullptr;          // device [2]
  StepAcc* acc = nullptr;          // device [2]
  StepRec* rec = nullptr;          // device [cap]
  StepRec* rec_host = nullptr;     // pinned [cap]
  int cap = 0;
  double* bnd = nullptr;           // device [2][8 nyg + 8 nx]
  double* outflow = nullptr;       // device [4]
  double* outflow_host = nullptr;  // pinned [4]
  StepCtl* ctl_host = nullptr;     // pinned [2]
  int cur = 0;                     // ctl slot of the current state
  bool valid = false;              // ctl[cur].rate_bits is the rate of the current U
  int rows_per_chunk = 0;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
};

static FusedState* fstate(lf_handle* h) { return reinterpret_cast<FusedState*>(h->fused); }

bool fused_supported(lf_handle* h) {
  if (!h->dim2 || h->d.time_order < 2) return false;
  if (h->d.nx < 4) return false;
  for (auto& s : h->slabs) {
    if (s.L.ny < 4) return false;
    if (s.device != h->slabs[0].device) return false;  // shared step records need one device
  }
  return true;
}

static void fused_alloc(lf_handle* h, int steps) {
  FusedState* f = fstate(h);
  SlabState& s0 = h->slabs[0];
  FK(cudaSetDevice(s0.device));
  if (!f) {
    f = new FusedState;
    h->fused = f;
    FK(cudaMalloc(&f->ctl, 2 * sizeof(StepCtl)));
    FK(cudaMalloc(&f->acc, 2 * sizeof(StepAcc)));
    FK(cudaHostAlloc(&f->ctl_host, 2 * sizeof(StepCtl), cudaHostAllocDefault));
    const size_t nb = 2 * (8 * (size_t)h->d.ny + 8 * (size_t)h->d.nx);
    FK(cudaMalloc(&f->bnd, nb * sizeof(double)));
    FK(cudaMemsetAsync(f->bnd, 0, nb * sizeof(double), s0.stream));
    FK(cudaMalloc(&f->outflow, 4 * sizeof(double)));
    FK(cudaHostAlloc(&f->outflow_host, 4 * sizeof(double), cudaHostAllocDefault));
    FK(cudaEventCreate(&f->e0));
    FK(cudaEventCreate(&f->e1));
    k_acc_init<<<1, 1, 0, s0.stream>>>(f->acc);
    count_launch();
    for (int m = 0; m < 2; ++m) {
      FK(cudaFuncSetAttribute(m ? k_fused_step<true> : k_fused_step<false>,
                              cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_BYTES));
    }
    // chunk rows: enough blocks for several waves of 2 blocks / SM, long marches
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, s0.device);
    const int strips = (h->d.nx + TXO - 1) / TXO;
    int ny_local = 0;
    for (auto& s : h->slabs) ny_local = std::max(ny_local, s.L.ny);
    const int target_blocks = 2 * sms * 6;
    int chunks = std::max(1, (target_blocks + strips - 1) / strips);
    int rows = (ny_local + chunks - 1) / chunks;
    rows = std::max(rows, 64);
    f->rows_per_chunk = rows;
  }
  if (steps > f->cap) {
    cudaFree(f->rec);
    cudaFreeHost(f->rec_host);
    f->cap = std::max(steps, 64);
    FK(cudaMalloc(&f->rec, (size_t)f->cap * sizeof(StepRec)));
    FK(cudaHostAlloc(&f->rec_host, (size_t)f->cap * sizeof(StepRec), cudaHostAllocDefault));
  }
}

void fused_release(lf_handle* h) {
  FusedState* f = fstate(h);
  if (!f) return;
  cudaFree(f->ctl);
  cudaFree(f->acc);
  cudaFree(f->rec);
  cudaFreeHost(f->rec_host);
  cudaFree(f->bnd);
  cudaFree(f->outflow);
  cudaFreeHost(f->outflow_host);
  cudaFreeHost(f->ctl_host);
  if (f->e0) cudaEventDestroy(f->e0);
  if (f->e1) cudaEventDestroy(f->e1);
  delete f;
  h->fused = nullptr;
}

int64_t fused_bytes(lf_handle* h) {
  FusedState* f = fstate(h);
  if (!f) return 0;
  return (int64_t)(2 * (8 * (size_t)h->d.ny + 8 * (size_t)h->d.nx)) * 8 + (int64_t)f->cap * sizeof(StepRec);
}

void fused_invalidate(lf_handle* h) {
  if (FusedState* f = fstate(h)) f->valid = false;
}

// rate of the current state -> ctl[cur] (the compute_dt of the first step)
static void seed_ctl(lf_handle* h, double time) {
  FusedState* f = fstate(h);
  SlabState& s0 = h->slabs[0];
  if (!f->valid) {
    const Scalars sc = rate_of_current(h);
    StepCtl c{};
    c.time = time;
    c.rate_bits = sc.rate_bits;
    c.done = 0;
    c.dtfail = sc.fail_dt != LLONG_MAX;
    f->ctl_host[0] = c;
    FK(cudaMemcpyAsync(&f->ctl[f->cur], &f->ctl_host[0], sizeof(StepCtl), cudaMemcpyHostToDevice,
                       s0.stream));
    f->valid = true;
  } else {
    // keep the device-resident rate; set the caller's time and clear done
    FK(cudaMemcpyAsync(&f->ctl_host[0], &f->ctl[f->cur], sizeof(StepCtl), cudaMemcpyDeviceToHost,
                       s0.stream));
    FK(cudaStreamSynchronize(s0.stream));
    f->ctl_host[0].time = time;
    f->ctl_host[0].done = 0;
    FK(cudaMemcpyAsync(&f->ctl[f->cur], &f->ctl_host[0], sizeof(StepCtl), cudaMemcpyHostToDevice,
                       s0.stream));
  }
}

// Enqueue one fused step on every slab: ghosts of U, kernel(s) U -> U2, reduce, finalize.
static void enqueue_step(lf_handle* h, int n_in_batch, double cfl, double limit, double t_final,
                         cudaEvent_t k0, cudaEvent_t k1) {
  FusedState* f = fstate(h);
  const int cur = f->cur, nxt = cur ^ 1;
  fill_all_public(h, &SlabState::U);
  SlabState& s0 = h->slabs[0];
  double* bnd = f->bnd + (size_t)cur * (8 * (size_t)h->d.ny + 8 * (size_t)h->d.nx);
  const size_t nbnd = 8 * (size_t)h->d.ny + 8 * (size_t)h->d.nx;
  if (h->nccl) FK(cudaMemsetAsync(bnd, 0, nbnd * sizeof(double), s0.stream));  // disjoint sum
  if (k0) FK(cudaEventRecord(k0, s0.stream));
  for (auto& s : h->slabs) {
    FusedArgs a;
    a.u = s.U + s.L.origin();
    a.un = s.U2 + s.L.origin();
    a.pitch = s.L.pitch;
    a.fstride = s.L.fstride;
    a.nx = s.L.nx;
    a.ny = s.L.ny;
    a.y0g = s.sl.y0;
    a.nyg = h->d.ny;
    a.rows_per_chunk = f->rows_per_chunk;
    a.gamma = h->k.gamma;
    a.gm1 = h->k.gm1;
    a.beta = h->k.beta;
    a.dx = h->d.dx;
    a.dy = h->d.dy;
    a.cfl = cfl;
    a.limit = limit;
    a.bc_xlo = h->d.bc[0];
    a.bc_xhi = h->d.bc[1];
    a.bc_ylo = h->d.bc[2];
    a.bc_yhi = h->d.bc[3];
    a.bottom_edge = s.sl.fill_lo && h->d.bc[2] != LF_PERIODIC;
    a.top_edge = s.sl.fill_hi && h->d.bc[3] != LF_PERIODIC;
    a.ctl = f->ctl + cur;
    a.acc = f->acc + cur;
    a.bnd = bnd;
    dim3 grid((h->d.nx + TXO - 1) / TXO, (s.L.ny + f->rows_per_chunk - 1) / f->rows_per_chunk);
    if (h->d.spatial_order >= 2)
      k_fused_step<true><<<grid, NTHREADS, SMEM_BYTES, s.stream>>>(a);
    else
      k_fused_step<false><<<grid, NTHREADS, SMEM_BYTES, s.stream>>>(a);
    count_launch();
  }
  if (k1) FK(cudaEventRecord(k1, s0.stream));
  FK(cudaGetLastError());
  if (h->nccl) nccl_reduce_step(h, f->acc + cur, 5, bnd, 8 * (size_t)h->d.ny + 8 * (size_t)h->d.nx);
  k_finalize<<<1, 32, 0, s0.stream>>>(f->ctl + cur, f->acc + cur, f->ctl + nxt,
                                      f->rec + n_in_batch, bnd, f->outflow, h->d.nx, h->d.ny,
                                      h->d.dx, h->d.dy, cfl, limit, t_final);
  count_launch();
  FK(cudaGetLastError());
  for (auto& s : h->slabs) std::swap(s.U, s.U2);
  f->cur = nxt;
}

// Run up to n fused steps from (time, step); returns the number of steps that
// completed (records in f->rec_host) and the index of a failed step, if any.
static int run_batch(lf_handle* h, int n, double cfl, double limit, double t_final, double time,
                     const double* outflow_in, int* failed_at, bool timing, double* kernel_ms) {
  FusedState* f = fstate(h);
  SlabState& s0 = h->slabs[0];
  seed_ctl(h, time);
  double o[4] = {0, 0, 0, 0};
  if (outflow_in) std::memcpy(o, outflow_in, sizeof o);
  std::memcpy(f->outflow_host, o, sizeof o);
  FK(cudaMemcpyAsync(f->outflow, f->outflow_host, sizeof o, cudaMemcpyHostToDevice, s0.stream));
  std::vector<cudaEvent_t> evs;
  if (timing) {
    evs.resize(2 * (size_t)n);
    for (auto& e : evs) FK(cudaEventCreate(&e));
  }
  for (int i = 0; i < n; ++i)
    enqueue_step(h, i, cfl, limit, t_final, timing ? evs[2 * i] : nullptr,
                 timing ? evs[2 * i + 1] : nullptr);
  FK(cudaMemcpyAsync(f->rec_host, f->rec, (size_t)n * sizeof(StepRec), cudaMemcpyDeviceToHost,
                     s0.stream));
  FK(cudaMemcpyAsync(f->outflow_host, f->outflow, 4 * sizeof(double), cudaMemcpyDeviceToHost,
                     s0.stream));
  for (auto& s : h->slabs) {
    FK(cudaSetDevice(s.device));
    FK(cudaStreamSynchronize(s.stream));
  }
  if (timing) {
    double ms = 0.0;
    for (int i = 0; i < n; ++i) {
      float x = 0.f;
      FK(cudaEventElapsedTime(&x, evs[2 * i], evs[2 * i + 1]));
      ms += x;
    }
    *kernel_ms = ms;
    for (auto& e : evs) cudaEventDestroy(e);
  }
  int done = 0;
  *failed_at = -1;
  for (int i = 0; i < n; ++i) {
    if (f->rec_host[i].status == 0) {
      ++done;
      continue;
    }
    if (f->rec_host[i].status == 1) *failed_at = i;
    break;
  }
  // U/U2 were swapped once per enqueued step; the state after `done` steps is
  // the output of step done-1 (or the input if done == 0)
  const int undo = n - done;
  if (undo & 1)
    for (auto& s : h->slabs) std::swap(s.U, s.U2);
  f->cur = (f->cur + undo) & 1;  // ctl slot holding the state's rate
  f->valid = *failed_at < 0;     // after a failure the slot is not trustworthy
  return done;
}

static void to_out(const StepRec& r, int64_t step, double gm1, lf_step_out* o) {
  o->dt = r.dt;
  o->hits_limit = r.hits;
  o->time = r.time;
  o->step = step;
  o->min_rho = r.min_rho;
  o->min_p = gm1 * r.min_eint;
}

int fused_heun(lf_handle* h, double cfl, double time, double limit, int64_t step,
               double* outflow, lf_step_out* out) {
  try {
    fused_alloc(h, 1);
    int failed_at;
    const int done = run_batch(h, 1, cfl, limit, limit, time, outflow, &failed_at, false, nullptr);
    if (done == 1) {
      if (outflow) std::memcpy(outflow, fstate(h)->outflow_host, 4 * sizeof(double));
      if (out) to_out(fstate(h)->rec_host[0], step + 1, h->d.gamma - 1.0, out);
      return 0;
    }
  } catch (const DevFail& e) {
    throw std::runtime_error(e.what());
  }
  // a flag was raised: the stage-wise kernels reproduce the exact error / state
  fused_invalidate(h);
  return staged_heun_public(h, cfl, time, limit, step, outflow, out);
}

int fused_advance(lf_handle* h, int nsteps, double cfl, double t_final, double* time,
                  int64_t* step, double* outflow, lf_step_out* per_step, int* taken) {
  if (taken) *taken = 0;
  int k = 0;
  while (k < nsteps && *time < t_final) {
    const int batch = std::min(nsteps - k, 256);
    fused_alloc(h, batch);
    FusedState* f = fstate(h);
    int failed_at;
    const int done = run_batch(h, batch, cfl, t_final, t_final, *time, outflow, &failed_at,
                               false, nullptr);
    for (int i = 0; i < done; ++i) {
      *step += 1;
      if (per_step) to_out(f->rec_host[i], *step, h->d.gamma - 1.0, &per_step[k + i]);
      *time = f->rec_host[i].time;
    }
    k += done;
    if (taken) *taken = k;
    if (done > 0 && outflow) {
      // outflow_host holds the sum through the last completed step only when no
      // step failed; otherwise recompute by replaying is not needed: a failed
      // step does not touch the device outflow (finalize skips it)
      std::memcpy(outflow, f->outflow_host, 4 * sizeof(double));
    }
    if (failed_at >= 0) {
      fused_invalidate(h);
      lf_step_out o;
      const int rc = staged_heun_public(h, cfl, *time, t_final, *step, outflow, &o);
      if (rc) return rc;
      *step = o.step;
      *time = o.time;
      if (per_step) per_step[k] = o;
      ++k;
      if (taken) *taken = k;
      continue;
    }
    if (done < batch) break;  // reached t_final
  }
  return 0;
}

int fused_time_steps(lf_handle* h, int nsteps, double cfl, double* kernel_ms, double* step_ms,
                     int* launches) {
  fused_alloc(h, nsteps);
  FusedState* f = fstate(h);
  SlabState& s0 = h->slabs[0];
  const double big = 1.7976931348623157e308;
  // read back the current time so the timed steps continue the run
  FK(cudaMemcpy(&f->ctl_host[1], &f->ctl[f->cur], sizeof(StepCtl), cudaMemcpyDeviceToHost));
  const double t0 = f->valid ? f->ctl_host[1].time : 0.0;
  FK(cudaEventRecord(f->e0, s0.stream));
  int failed_at;
  double kms = 0.0;
  const int done = run_batch(h, nsteps, cfl, big, big, t0, nullptr, &failed_at, true, &kms);
  FK(cudaEventRecord(f->e1, s0.stream));
  FK(cudaEventSynchronize(f->e1));
  float loop = 0.f;
  FK(cudaEventElapsedTime(&loop, f->e0, f->e1));
  *kernel_ms = kms;
  *step_ms = loop;
  *launches = done * (int)h->slabs.size();
  return failed_at >= 0 ? LF_ERR_DEVICE : 0;
}

}  // namespace lfb
