// twopass_mat_kernel.cu -- the two-pass Heun step with multimaterial transport.
//
// The structure of twopass_kernel.cu (warp-independent 32-column strips
// marching down row chunks, y-stencils in per-lane register windows,
// x-neighbours through shuffles) extended by the reference's MaterialSet path:
//
//   fill_all_ghosts' closure (solver.cpp:100-121): per cell, the clamped mass
//     fractions y_k = P_k / rho and the mixed-cell gamma (pure cell: the last
//     material with y == 1; else 1 + 1 / sum_k y_k / (gamma_k - 1));
//   per-cell gamma in the primitives and each face side's own EOS in the
//     Riemann solve (solver.cpp:153-156, 228-233);
//   update_partials (solver.cpp:331-404): per-material face fluxes
//     mass * y_k(upwind cell) with the last material taking the complement, zero
//     on a u* == 0 face, combined as the reference accumulates them,
//     (0 + w F_a) + w F_b, then P_k - lam_x (fr - fl) - lam_y (ft - fb);
//   the diagnostics' min pressure from the fresh partials (solver.cpp:522-538).
//
// The predictor stores P* and its per-material face fluxes (the corrector's
// stage-a term); the corrector writes P^{n+1}, min p and the next step's CFL
// rate with the mixed-cell gamma of U^{n+1} (the next step's fill closure).
// The cell box of face_fast.cuh (with every cell's gamma checked as well) proves
// the face solves' fast divisions valid; the velocity-weighted u* quotient and
// the fraction quotients go through div_exact.  A clamp beyond round-off or a
// failed check flags the step and the stage-wise kernels recompute it exactly
// (errors included).
#include <cuda_runtime.h>

#include <cstdio>

#include "../../include/lagflux_b200.h"
#include "face_fast.cuh"
#include "fused_common.cuh"
#include "kernels.h"
#include "twopass.h"
#include "pdl.cuh"

// the multimaterial passes call div_exact at many sites: outline its cold path
#ifndef LF_MAT_DIV_OUTLINE
#define LF_MAT_DIV_OUTLINE 1
#endif
#if LF_MAT_DIV_OUTLINE
#define LF_MAT_DIV_EXACT div_exact_ol
#else
#define LF_MAT_DIV_EXACT div_exact
#endif

#ifdef LF_MAT_DEBUG
#define MFAIL(code)                                                                    \
  do {                                                                                 \
    fail = 1;                                                                          \
    if (atomicAdd(&dbg_count, 1u) < 40u)                                               \
      printf("FAIL %d corr=%d c=%d r=%d it=%d\n", (code), (int)CORR, c, r, it);         \
  } while (0)
__device__ unsigned dbg_count = 0;
#else
#define MFAIL(code) (fail = 1)
#endif

namespace lfb {

namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int LANES = 32;
constexpr int TXW = LANES - 4;

__device__ __forceinline__ double shup(double v) { return __shfl_up_sync(FULL, v, 1); }
__device__ __forceinline__ double shdn(double v) { return __shfl_down_sync(FULL, v, 1); }


struct MatK {
  int n;
  double gamma[TP_MAX_MATERIALS];
};

struct MatR {
  Recip rg[TP_MAX_MATERIALS];   // 1 / (gamma_k - 1.0), shared by every cell
};

// fill_all_ghosts' closure for one cell (solver.cpp:100-121) from the raw
// fractions raw_k = P_k / rho and their quotients q_k = raw_k / (gamma_k - 1);
// bad: a fraction beyond round-off.  The quotients go through div_exact:
// partial densities diffuse into arbitrarily small values (fronts decay
// geometrically) and the quotient must stay exact there.
template <int K>
__device__ __forceinline__ double closure_q(const double raw[K], const double q[K], const MatK& m,
                                            const MatR& mr, double y[K], bool& bad, bool& ok) {
  double ysum = 0.0;
  int pure = -1;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double yk = raw[k];
    double qk = q[k];
    if (yk < 0.0 || yk > 1.0) {
      if (raw[k] < -1e-11 || raw[k] > 1.0 + 1e-11) {
        bad = true;
        yk = 0.0;
      } else {
        yk = raw[k] < 0.0 ? 0.0 : 1.0;
      }
      qk = LF_MAT_DIV_EXACT(yk, mr.rg[k], ok);
    }
    y[k] = yk;
    if (yk == 1.0) pure = k;
    ysum += qk;
  }
  double gp = 0.0;
#pragma unroll
  for (int k = 0; k < K; ++k)
    if (pure == k) gp = m.gamma[k];
  return pure >= 0 ? gp : 1.0 + div1_fast(1.0, ysum, ok);
}

template <int K>
__device__ __forceinline__ double closure(const double* p, double rho, const MatK& m,
                                          const MatR& mr, double y[K], bool& bad, bool& ok) {
  const Recip rr = recip_of(rho);
  double raw[K], q[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    raw[k] = LF_MAT_DIV_EXACT(p[k], rr, ok);
    q[k] = LF_MAT_DIV_EXACT(raw[k], mr.rg[k], ok);
  }
  return closure_q<K>(raw, q, m, mr, y, bad, ok);
}

__device__ __forceinline__ bool gamma_in_box(double g) {
  const double gm1 = g - 1.0;
  return gm1 >= 0x1p-14 && gm1 < 0x1p6 && g < 0x1p7;
}

// face_fast with each side's own gamma (lagrangian_hll(wm, wp, n, el, er) and
// conserved_from_primitive with that side's EOS, riemann_hll.hpp:29-39).  The
// cell box of face_fast.cuh holds with per-side gammas too (every cell's gamma
// is checked: gamma - 1 in [2^-14, 2^6)), so only the velocity-weighted u*
// quotient needs div_exact; ok reports its range.  u* == 0: face_mean_g.
template <int AXIS>
__device__ __forceinline__ void face_g(const double m[4], const double p[4], double gl, double gr,
                                       double f[4], bool& ok, double& ps_out, double& us_out) {
  bool unused = true;
  const double ul = AXIS == 0 ? m[1] : m[2];
  const double ur = AXIS == 0 ? p[1] : p[2];
  const double cl = sqrt_fast(div1_fast(gl * m[3], m[0], unused), unused);
  const double cr = sqrt_fast(div1_fast(gr * p[3], p[0], unused), unused);
  const double cmax = pmax(cl, cr);
  const double rho_sum = m[0] + p[0];
  const Recip rs = recip_of(rho_sum);
  const double ps = div_fast(p[0] * m[3] + m[0] * p[3], rs, unused) -
                    div_fast(m[0] * p[0], rs, unused) * cmax * (ur - ul);
  const double us =
      LF_MAT_DIV_EXACT(m[0] * ul + p[0] * ur, rs, ok) - div1_fast(p[3] - m[3], cmax * rho_sum, unused);
  const bool pos = us > 0.0;
  const double s0 = pos ? m[0] : p[0], s1 = pos ? m[1] : p[1], s2 = pos ? m[2] : p[2];
  const double s3 = pos ? m[3] : p[3], gs = pos ? gl : gr;
  const double a1 = s0 * s1, a2 = s0 * s2;
  const double a3 = div1_fast(s3, gs - 1.0, unused) + 0.5 * s0 * (s1 * s1 + s2 * s2);
  f[0] = s0 * us;
  f[1] = AXIS == 0 ? a1 * us + ps : a1 * us;
  f[2] = AXIS == 1 ? a2 * us + ps : a2 * us;
  f[3] = a3 * us + ps * us;
  ps_out = ps;
  us_out = us;
}

// solver.cpp:33-41 mean state (u* == 0 or NaN) with each side's EOS
template <int AXIS>
__device__ __forceinline__ void face_mean_g(const double m[4], const double p[4], double gl,
                                            double gr, double ps, double us, double f[4]) {
  bool unused = true;
  const double m3c = div1_fast(m[3], gl - 1.0, unused) + 0.5 * m[0] * (m[1] * m[1] + m[2] * m[2]);
  const double p3c = div1_fast(p[3], gr - 1.0, unused) + 0.5 * p[0] * (p[1] * p[1] + p[2] * p[2]);
  const double a0 = 0.5 * (m[0] + p[0]);
  const double a1 = 0.5 * (m[0] * m[1] + p[0] * p[1]);
  const double a2 = 0.5 * (m[0] * m[2] + p[0] * p[2]);
  const double a3 = 0.5 * (m3c + p3c);
  f[0] = a0 * us;
  f[1] = AXIS == 0 ? a1 * us + ps : a1 * us;
  f[2] = AXIS == 1 ? a2 * us + ps : a2 * us;
  f[3] = a3 * us + ps * us;
}

// edge_material_flux (solver.cpp:345-357) from the face's mass flux and u* and
// the two candidate upwind fraction vectors
template <int K>
__device__ __forceinline__ void mat_face(double mass, double us, const double ylo[K],
                                         const double yhi[K], double out[K]) {
  const bool lo = us > 0.0;
  const bool zero = us == 0.0;
  double rest = mass;
#pragma unroll
  for (int k = 0; k < K - 1; ++k) {
    const double fk = zero ? 0.0 : mass * (lo ? ylo[k] : yhi[k]);
    out[k] = fk;
    rest -= fk;
  }
  out[K - 1] = zero ? 0.0 : rest;
}

// The update operands of a row (U^n, P^n and, in the corrector, the stage-a
// faces F^n and material fluxes) are staged one row ahead in shared memory with
// cp.async: at 8 warps/SM the loads issued at the top of their own iteration
// did not return before their use (ncu: long_scoreboard 25 % of the corrector),
// and in registers they would add 42 live registers to a 255-register kernel.
// Each lane copies and reads only its own elements, so the per-thread
// cp.async.wait_group orders them; absent operands are zero-filled (src-size 0).
#ifndef LF_MAT_ASYNC
#define LF_MAT_ASYNC 1
#endif
__device__ __forceinline__ void cp_async8(double* sdst, const double* gsrc, bool pred) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gsrc),
               "r"(pred ? 8 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_wait1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }

template <bool CORR, bool MUSCL, int K>
__global__ void __launch_bounds__(TP_THREADS, 2) k_pass_mat(PassArgs a, MatPassArgs m, MatK mk) {
  MatR mr;
#pragma unroll
  for (int k = 0; k < K; ++k) mr.rg[k] = recip_of(mk.gamma[k] - 1.0);
  pdl_wait();  // the previous kernel of the step chain (pdl.cuh)
  const StepCtl ctl = *a.ctl;
  if (ctl.done) return;
  if (ctl.dtfail) {
    if (threadIdx.x == 0 && blockIdx.x == 0) atomicMax(&a.acc->fail, 1ull);
    return;
  }
  const double rate = __longlong_as_double((long long)ctl.rate_bits);
  double dt = a.cfl / rate;
  if (ctl.time + dt > a.limit) dt = a.limit - ctl.time;
  if (!(dt > 0.0)) {
    if (threadIdx.x == 0 && blockIdx.x == 0) atomicMax(&a.acc->fail, 1ull);
    return;
  }
  const double lam_x = dt / a.dx;
  const double lam_y = dt / a.dy;
  const Recip rdx = recip_of(a.dx), rdy = recip_of(a.dy);

  const int lane = threadIdx.x & 31;
  const int warp = blockIdx.x * (TP_THREADS / 32) + (threadIdx.x >> 5);
  const int strip = warp % a.strips;
  const int chunk = warp / a.strips;
  const int y0 = chunk * a.rows_per_chunk;
  if (y0 >= a.ny) return;
  const int y1 = min(y0 + a.rows_per_chunk, a.ny);
  const int x0 = strip * TXW;
  const int c = x0 - 2 + lane;
  const bool col_in_mem = c >= -NG && c < a.nx + NG;
  const bool col_interior = c >= 0 && c < a.nx;
  const bool upd = lane >= 2 && lane <= LANES - 3 && col_interior;
  const bool store_fx = (lane >= 2 && lane <= LANES - 3 && c <= a.nx) || (lane == LANES - 2 && c == a.nx);
  const int nit = (y1 - y0) + 4;
  // this warp's strip holds the domain's first or last column
  const bool x_edge_warp = x0 - 2 <= 0 || x0 - 2 + LANES > a.nx - 1;

  unsigned fail = 0;
  unsigned long long rate_key = 0ull, nmin_r = NINF_KEY, nmin_e = NINF_KEY, nmin_p = NINF_KEY;
  unsigned dtfail = 0;

  const int P = (int)a.pitch;
  int o_in = (y0 - 2) * P + c;
#if LF_MAT_ASYNC
  // [warp][buffer][operand][lane]: bse 0-3, pbs 4.., fnx, fny, max_, may_
  constexpr int NOP = CORR ? 12 + 3 * K : 4 + K;
  // (dynamic: 5-8 materials need more than the 48 KB of static shared memory)
  extern __shared__ __align__(16) double stage_dyn[];
  double(*const st)[NOP][32] =
      reinterpret_cast<double(*)[NOP][32]>(stage_dyn + (threadIdx.x >> 5) * 2 * NOP * 32);
  auto issue = [&](int itn, int orow, int buf) {
    const bool pu = itn >= 4 && upd;
#pragma unroll
    for (int q = 0; q < 4; ++q)
      cp_async8(&st[buf][q][lane], pu ? a.base + q * a.fstride + orow : a.base, pu);
#pragma unroll
    for (int k = 0; k < K; ++k)
      cp_async8(&st[buf][4 + k][lane], pu ? m.pbase + k * a.fstride + orow : m.pbase, pu);
    if (CORR) {
      const bool px = a.heun && itn >= 4 && col_in_mem && c >= 0 && c <= a.nx;
      const bool py = a.heun && itn >= 3 && col_interior;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        cp_async8(&st[buf][4 + K + q][lane], px ? a.fx + q * a.fx_stride + orow : a.fx, px);
        cp_async8(&st[buf][8 + K + q][lane], py ? a.fy + q * a.fy_stride + (orow + P) : a.fy, py);
      }
#pragma unroll
      for (int k = 0; k < K; ++k) {
        cp_async8(&st[buf][12 + K + k][lane], px ? m.mfx + k * m.mfx_stride + orow : m.mfx, px);
        cp_async8(&st[buf][12 + 2 * K + k][lane], py ? m.mfy + k * m.mfy_stride + (orow + P) : m.mfy, py);
      }
    }
    cp_commit();
  };
  issue(0, o_in - 2 * P, 0);
#endif
  // the next input row (U and partials), loaded one iteration ahead
  double nxt[4] = {1.0, 0.0, 0.0, 1.0}, pnx[K];
#pragma unroll
  for (int k = 0; k < K; ++k) pnx[k] = k == 0 ? 1.0 : 0.0;
  if (col_in_mem) {
#pragma unroll
    for (int q = 0; q < 4; ++q) nxt[q] = __ldg(a.x + q * a.fstride + o_in);
#pragma unroll
    for (int k = 0; k < K; ++k) pnx[k] = __ldg(m.px + k * a.fstride + o_in);
  }
  // windows: W rows r-2, r-1; gamma rows r-2, r-1; fractions rows r-2, r-1
  double wm2[4] = {1.0, 0.0, 0.0, 1.0}, wm1[4] = {1.0, 0.0, 0.0, 1.0};
  double hiprev[4] = {1.0, 0.0, 0.0, 1.0}, fyprev[4] = {0.0, 0.0, 0.0, 0.0};
  double gm2 = mk.gamma[0], gm1c = mk.gamma[0];
  double ym2[K], ym1[K], myprev[K];   // myprev: material fluxes of the previous y-face
#pragma unroll
  for (int k = 0; k < K; ++k) ym2[k] = ym1[k] = myprev[k] = 0.0;

  for (int it = 0; it < nit; ++it) {
    const int r = y0 - 2 + it;
    const int row = r - 2;
    const int o_row = o_in - 2 * P;
    // -- input row r: U, partials -> fractions, gamma, W
    double w[4] = {1.0, 0.0, 0.0, 1.0}, yr[K], gr = mk.gamma[0];
#pragma unroll
    for (int k = 0; k < K; ++k) yr[k] = 0.0;
    double cur[4], pc[K];
#pragma unroll
    for (int q = 0; q < 4; ++q) cur[q] = nxt[q];
#pragma unroll
    for (int k = 0; k < K; ++k) pc[k] = pnx[k];
    if (it + 1 < nit && col_in_mem) {
#pragma unroll
      for (int q = 0; q < 4; ++q) nxt[q] = __ldg(a.x + q * a.fstride + o_in + P);
#pragma unroll
      for (int k = 0; k < K; ++k) pnx[k] = __ldg(m.px + k * a.fstride + o_in + P);
    }
    double bse[4] = {0.0, 0.0, 0.0, 0.0}, pbs[K];
    double fnx[4] = {0.0, 0.0, 0.0, 0.0}, fny[4] = {0.0, 0.0, 0.0, 0.0}, max_[K], may_[K];
#pragma unroll
    for (int k = 0; k < K; ++k) pbs[k] = max_[k] = may_[k] = 0.0;
#if LF_MAT_ASYNC
    // the next row's operands in flight during this row's work
    if (it + 1 < nit) issue(it + 1, o_row + P, (it + 1) & 1);
    else cp_commit();
#else
    // this iteration's update operands, issued early (their latency hides
    // behind the closure, traces and face solves)
    if (it >= 4 && upd) {
#pragma unroll
      for (int q = 0; q < 4; ++q) bse[q] = __ldg(a.base + q * a.fstride + o_row);
#pragma unroll
      for (int k = 0; k < K; ++k) pbs[k] = __ldg(m.pbase + k * a.fstride + o_row);
    }
    if (CORR && a.heun) {
      if (it >= 4 && col_in_mem && c >= 0 && c <= a.nx) {
#pragma unroll
        for (int q = 0; q < 4; ++q) fnx[q] = __ldg(a.fx + q * a.fx_stride + o_row);
#pragma unroll
        for (int k = 0; k < K; ++k) max_[k] = __ldg(m.mfx + k * m.mfx_stride + o_row);
      }
      if (it >= 3 && col_interior) {
#pragma unroll
        for (int q = 0; q < 4; ++q) fny[q] = __ldg(a.fy + q * a.fy_stride + (o_row + P));
#pragma unroll
        for (int k = 0; k < K; ++k) may_[k] = __ldg(m.mfy + k * m.mfy_stride + (o_row + P));
      }
    }
#endif
    if (col_in_mem) {
      bool bad = false, ok = true;
      gr = closure<K>(pc, cur[0], mk, mr, yr, bad, ok);
      prim_fast(cur[0], cur[1], cur[2], cur[3], gr - 1.0, w, ok);
      // the fill's closure covers the reference's ghosted cells; the state
      // checks the interior (ghosts are images of interior cells)
      const int rg_ = r + a.y0g;
      if (bad && c >= -2 && c < a.nx + 2 && rg_ >= -2 && rg_ < a.nyg + 2) MFAIL(1);
      if ((!ok || !cell_in_box(w) || !gamma_in_box(gr)) && col_interior && r >= 0 && r < a.ny)
        MFAIL(!ok ? 2 : (!cell_in_box(w) ? 3 : 4));
    }
    o_in += P;
    // -- traces (as twopass_kernel.cu)
    double ylo[4], yhi[4], xlo[4], xhi[4], xp[4], da[4], db[4], xmh[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) xp[q] = shdn(wm2[q]);
#pragma unroll
    for (int q = 0; q < 4; ++q) da[q] = xp[q] - wm2[q];
#pragma unroll
    for (int q = 0; q < 4; ++q) db[q] = shup(da[q]);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      cell_traces<MUSCL>(wm2[q], wm1[q], w[q], a.beta, ylo[q], yhi[q]);
      traces_ab<MUSCL>(da[q], db[q], wm2[q], a.beta, xlo[q], xhi[q]);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) xmh[q] = shup(xhi[q]);
    // -- faces: x (lane-1 | lane) of row r-2, y (r-2 | r-1)
    const double gl_x = shup(gm2);
    double fx[4], fy[4], psx, usx, psy, usy;
    bool okx = true, oky = true;
    face_g<0>(xmh, xlo, gl_x, gm2, fx, okx, psx, usx);
    face_g<1>(hiprev, ylo, gm2, gm1c, fy, oky, psy, usy);
    if (needs_mean(usx)) face_mean_g<0>(xmh, xlo, gl_x, gm2, psx, usx, fx);
    if (needs_mean(usy)) face_mean_g<1>(hiprev, ylo, gm2, gm1c, psy, usy, fy);
    const bool need_x = it >= 4 && lane >= 2 && lane <= LANES - 2 && c <= a.nx;
    const bool need_y = it >= 3 && lane >= 2 && lane <= LANES - 3 && col_interior;
    if ((need_x && !okx) || (need_y && !oky)) MFAIL(5);
    if (need_x && !traces_ok(xmh[0], xmh[3], xlo[0], xlo[3]) && c >= 0 && row >= 0 && row < a.ny)
      MFAIL(6);
    if (need_y && !traces_ok(hiprev[0], hiprev[3], ylo[0], ylo[3]) && r - 1 >= 0 && r - 1 <= a.ny)
      MFAIL(7);
    // -- material fluxes of this stage through the two faces
    double ylx[K], mfx_s[K], mfy_s[K];
#pragma unroll
    for (int k = 0; k < K; ++k) ylx[k] = shup(ym2[k]);
    mat_face<K>(fx[0], usx, ylx, ym2, mfx_s);
    mat_face<K>(fy[0], usy, ym2, ym1, mfy_s);
    // -- stage-a operands (corrector) and the Heun averages
#if LF_MAT_ASYNC
    cp_wait1();  // this row's group (the next row's may still be in flight)
    {
      const double(*const sb)[32] = st[it & 1];
#pragma unroll
      for (int q = 0; q < 4; ++q) bse[q] = sb[q][lane];
#pragma unroll
      for (int k = 0; k < K; ++k) pbs[k] = sb[4 + k][lane];
      if (CORR) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          fnx[q] = sb[4 + K + q][lane];
          fny[q] = sb[8 + K + q][lane];
        }
#pragma unroll
        for (int k = 0; k < K; ++k) {
          max_[k] = sb[12 + K + k][lane];
          may_[k] = sb[12 + 2 * K + k][lane];
        }
      }
    }
#endif
    double fxa[4], fya[4];
    if (CORR && a.heun) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        fxa[q] = 0.5 * (fnx[q] + fx[q]);
        fya[q] = 0.5 * (fny[q] + fy[q]);
      }
      // (0 + 0.5 F_a) + 0.5 F_b (solver.cpp:366-383)
#pragma unroll
      for (int k = 0; k < K; ++k) {
        mfx_s[k] = (0.0 + 0.5 * max_[k]) + 0.5 * mfx_s[k];
        mfy_s[k] = (0.0 + 0.5 * may_[k]) + 0.5 * mfy_s[k];
      }
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        fxa[q] = fx[q];
        fya[q] = fy[q];
      }
    }
    double fxr[4], mfxr[K];
#pragma unroll
    for (int q = 0; q < 4; ++q) fxr[q] = shdn(fxa[q]);
#pragma unroll
    for (int k = 0; k < K; ++k) mfxr[k] = shdn(mfx_s[k]);
    if (it >= 4) {
      if (!CORR) {
        if (store_fx) {
#pragma unroll
          for (int q = 0; q < 4; ++q) a.fxo[q * a.fx_stride + o_row] = fx[q];
#pragma unroll
          for (int k = 0; k < K; ++k) m.mfxo[k * m.mfx_stride + o_row] = mfx_s[k];
        }
        if (upd) {
#pragma unroll
          for (int q = 0; q < 4; ++q) a.fyo[q * a.fy_stride + (o_row + P)] = fy[q];
#pragma unroll
          for (int k = 0; k < K; ++k) m.mfyo[k * m.mfy_stride + (o_row + P)] = mfy_s[k];
        }
      }
      if (upd) {
        // hydro update (solver.cpp:283-291)
        double v[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          double val = bse[q] - lam_x * (fxr[q] - fxa[q]);
          val -= lam_y * (fya[q] - fyprev[q]);
          v[q] = val;
          a.out[q * a.fstride + o_row] = val;
        }
        // update_partials (solver.cpp:384-402); single stage: 0 + 1.0 t
        double pn[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const double fl = CORR ? mfx_s[k] : 0.0 + mfx_s[k];
          const double fr = CORR ? mfxr[k] : 0.0 + mfxr[k];
          const double fb = CORR ? myprev[k] : 0.0 + myprev[k];
          const double ft = CORR ? mfy_s[k] : 0.0 + mfy_s[k];
          double val = pbs[k] - lam_x * (fr - fl);
          val -= lam_y * (ft - fb);
          pn[k] = val;
          m.pout[k * a.fstride + o_row] = val;
        }
        if (!CORR) {
          // e_int > 0 (solver.cpp:300-302), conservative as in twopass_kernel.cu
          const double kin = 0.5 * (v[1] * v[1] + v[2] * v[2]);
          const double lhs = v[3] * v[0];
          if (!(v[0] > 0.0) || !(lhs > kin * (1.0 + 0x1p-48)) || !(lhs >= 0x1p-960)) MFAIL(8);
        } else {
          bool ok = true;
          const Recip r0 = recip_of(v[0]);
          const double kin = 0.5 * (v[1] * v[1] + v[2] * v[2]);
          const double eint = v[3] - LF_MAT_DIV_EXACT(kin, r0, ok);
          double rawn[K], qn[K];
          bool have_q = false;
          if (!(v[0] > 0.0) || !(eint > 0.0) || !ok) {
            MFAIL(9);
          } else {
            const unsigned long long kr = ~pos_bits(v[0]), ke = ~pos_bits(eint);
            nmin_r = kr > nmin_r ? kr : nmin_r;
            nmin_e = ke > nmin_e ? ke : nmin_e;
            // min p from the fresh partials (solver.cpp:526-536): no clamp here;
            // its quotients are the next step's closure quotients too
            double s = 0.0;
#pragma unroll
            for (int k = 0; k < K; ++k) {
              rawn[k] = LF_MAT_DIV_EXACT(pn[k], r0, ok);
              qn[k] = LF_MAT_DIV_EXACT(rawn[k], mr.rg[k], ok);
              s += qn[k];
            }
            have_q = true;
            const double pmin = LF_MAT_DIV_EXACT(eint, recip_of(s), ok);
            if (!ok) MFAIL(10);
            if (pmin == pmin) {
              if (pmin > 0.0) {
                const unsigned long long kp = ~pos_bits(pmin);
                nmin_p = kp > nmin_p ? kp : nmin_p;
              } else {
                MFAIL(11);   // a non-positive minimum is left to the stage-wise path
              }
            }
          }
          // the next step's CFL rate with its fill closure (solver.cpp:441-469)
          double yn[K];
          bool bad = false, okg = true;
          if (!have_q) {
#pragma unroll
            for (int k = 0; k < K; ++k) {
              rawn[k] = LF_MAT_DIV_EXACT(pn[k], r0, okg);
              qn[k] = LF_MAT_DIV_EXACT(rawn[k], mr.rg[k], okg);
            }
          }
          const double g = closure_q<K>(rawn, qn, mk, mr, yn, bad, okg);
          const double inv = div_fast(1.0, r0, okg);
          const double uu = v[1] * inv, vv = v[2] * inv;
          const double pp = (g - 1.0) * (v[3] - kin * inv);
          if (bad || !(v[0] > 0.0) || !(pp > 0.0)) {
            dtfail = 1;   // the next step's fill / compute_dt fails: stage-wise path
          } else {
            const double cs = sqrt_fast(g * pp * inv, okg);
            double rr = div_fast(abs_bits(uu) + cs, rdx, okg);
            rr += div_fast(abs_bits(vv) + cs, rdy, okg);
            if (!okg) MFAIL(12);
            if (rr == rr) {
              const unsigned long long b = pos_bits(rr);
              rate_key = b > rate_key ? b : rate_key;
            }
          }
          // boundary faces for accumulate_boundary_outflow (solver.cpp:406-432);
          // one warp-uniform test skips all four in the interior of the domain
          const int jg = row + a.y0g;
          if (x_edge_warp || jg == 0 || jg == a.nyg - 1) {
            if (c == 0)
              for (int q = 0; q < 4; ++q) a.bnd[(int64_t)q * a.nyg + jg] = fxa[q];
            if (c == a.nx - 1)
              for (int q = 0; q < 4; ++q) a.bnd[4 * (int64_t)a.nyg + (int64_t)q * a.nyg + jg] = fxr[q];
            if (jg == 0)
              for (int q = 0; q < 4; ++q) a.bnd[8 * (int64_t)a.nyg + (int64_t)q * a.nx + c] = fyprev[q];
            if (jg == a.nyg - 1)
              for (int q = 0; q < 4; ++q)
                a.bnd[8 * (int64_t)a.nyg + 4 * (int64_t)a.nx + (int64_t)q * a.nx + c] = fya[q];
          }
        }
      }
    } else if (!CORR && it == 3 && y0 == 0 && upd) {
      // the domain's first y-face (-1 | 0)
#pragma unroll
      for (int q = 0; q < 4; ++q) a.fyo[q * a.fy_stride + c] = fy[q];
#pragma unroll
      for (int k = 0; k < K; ++k) m.mfyo[k * m.mfy_stride + c] = mfy_s[k];
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      fyprev[q] = fya[q];
      hiprev[q] = yhi[q];
      wm2[q] = wm1[q];
      wm1[q] = w[q];
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
      myprev[k] = mfy_s[k];
      ym2[k] = ym1[k];
      ym1[k] = yr[k];
    }
    gm2 = gm1c;
    gm1c = gr;
  }
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long r2 = __shfl_xor_sync(FULL, rate_key, o);
    const unsigned long long a2 = __shfl_xor_sync(FULL, nmin_r, o);
    const unsigned long long b2 = __shfl_xor_sync(FULL, nmin_e, o);
    const unsigned long long c2 = __shfl_xor_sync(FULL, nmin_p, o);
    rate_key = r2 > rate_key ? r2 : rate_key;
    nmin_r = a2 > nmin_r ? a2 : nmin_r;
    nmin_e = b2 > nmin_e ? b2 : nmin_e;
    nmin_p = c2 > nmin_p ? c2 : nmin_p;
  }
  const unsigned anyfail = __any_sync(FULL, fail);
  dtfail = __any_sync(FULL, dtfail);
  if (lane == 0) {
    if (anyfail) atomicMax(&a.acc->fail, 1ull);
    if (CORR) {
      if (rate_key) atomicMax(&a.acc->rate_next, rate_key);
      if (nmin_r != NINF_KEY) atomicMax(&a.acc->nmin_rho, nmin_r);
      if (nmin_e != NINF_KEY) atomicMax(&a.acc->nmin_eint, nmin_e);
      if (nmin_p != NINF_KEY) atomicMax(&a.acc->nmin_p, nmin_p);
      if (dtfail) atomicMax(&a.acc->dtfail_next, 1ull);
    }
  }
}

// the corrector / predictor's operand staging (LF_MAT_ASYNC): [warp][buffer][operand][lane]
constexpr size_t stage_bytes(bool corr, int k) {
  return LF_MAT_ASYNC ? sizeof(double) * (TP_THREADS / 32) * 2 * (corr ? 12 + 3 * k : 4 + k) * 32
                      : 0;
}

template <bool CORR, bool MUSCL, int K>
void launch_one(const PassArgs& a, const MatPassArgs& m, const MatK& mk, unsigned blocks,
                cudaStream_t st) {
  constexpr size_t smem = stage_bytes(CORR, K);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(k_pass_mat<CORR, MUSCL, K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
  launch_chain(k_pass_mat<CORR, MUSCL, K>, dim3(blocks), dim3(TP_THREADS), smem, st, a, m, mk);
}

template <bool CORR, bool MUSCL>
void launch_k(const PassArgs& a, const MatPassArgs& m, const MatK& mk, unsigned blocks,
              cudaStream_t st) {
  switch (mk.n) {
    case 1: launch_one<CORR, MUSCL, 1>(a, m, mk, blocks, st); break;
    case 2: launch_one<CORR, MUSCL, 2>(a, m, mk, blocks, st); break;
    case 3: launch_one<CORR, MUSCL, 3>(a, m, mk, blocks, st); break;
    case 4: launch_one<CORR, MUSCL, 4>(a, m, mk, blocks, st); break;
    case 5: launch_one<CORR, MUSCL, 5>(a, m, mk, blocks, st); break;
    case 6: launch_one<CORR, MUSCL, 6>(a, m, mk, blocks, st); break;
    case 7: launch_one<CORR, MUSCL, 7>(a, m, mk, blocks, st); break;
    default: launch_one<CORR, MUSCL, 8>(a, m, mk, blocks, st); break;
  }
}

template <int K>
int resident_blocks() {
  constexpr size_t smem = stage_bytes(true, K);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(k_pass_mat<true, true, K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
  int b = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_pass_mat<true, true, K>, TP_THREADS,
                                                    smem) != cudaSuccess)
    b = 0;
  return b;
}

}  // namespace

int tp_resident_warps_mat(int nmat) {
  int b = 0;
  switch (nmat) {
    case 1: b = resident_blocks<1>(); break;
    case 2: b = resident_blocks<2>(); break;
    case 3: b = resident_blocks<3>(); break;
    case 4: b = resident_blocks<4>(); break;
    case 5: b = resident_blocks<5>(); break;
    case 6: b = resident_blocks<6>(); break;
    case 7: b = resident_blocks<7>(); break;
    default: b = resident_blocks<8>();
  }
  if (b < 1) b = 2;
  return b * (TP_THREADS / 32);
}

void launch_pass_mat(const PassArgs& a, const MatPassArgs& m, const MatConsts& mc, bool corr,
                     bool muscl, cudaStream_t st) {
  MatK mk{};
  mk.n = mc.n;
  for (int k = 0; k < TP_MAX_MATERIALS; ++k) mk.gamma[k] = k < mc.n ? mc.gamma[k] : 1.5;
  const int warps = a.strips * ((a.ny + a.rows_per_chunk - 1) / a.rows_per_chunk);
  const unsigned blocks = (unsigned)((warps + TP_THREADS / 32 - 1) / (TP_THREADS / 32));
  count_launch();
  if (corr) {
    if (muscl) launch_k<true, true>(a, m, mk, blocks, st);
    else launch_k<true, false>(a, m, mk, blocks, st);
  } else {
    if (muscl) launch_k<false, true>(a, m, mk, blocks, st);
    else launch_k<false, false>(a, m, mk, blocks, st);
  }
}

}  // namespace lfb
