// face_fast.cuh -- per-cell / per-face work of the fast Heun kernels.
//
// The reference's fp64 evaluation order throughout (compiled with
// --fmad=false); divisions and square roots through fastmath.cuh, whose
// results equal the IEEE operators bit for bit (up to the sign of a zero
// quotient) on their fast paths.  The face solves never evaluate the range
// checks: the cell box below proves them.  The per-cell epilogue still reports
// its checks through `ok`; the kernels turn any failure into a flag, and the
// host then recomputes the step with the stage-wise IEEE kernels, so no IEEE
// slow path (CALL, pinned registers) sits in the hot loops.  Shared by
// fused_kernel.cu and twopass_kernel.cu.
#pragma once

#include "fastmath.cuh"
#include "lagflux_device.cuh"

namespace lfb {

#ifdef __CUDACC__


struct FK {
  double gamma, gm1, beta;
  Recip rgm1, rdx, rdy;  // shared reciprocals of the constant divisors
};

__device__ __forceinline__ FK make_fk(double gamma, double gm1, double beta, double dx, double dy) {
  FK c;
  c.gamma = gamma;
  c.gm1 = gm1;
  c.beta = beta;
  c.rgm1 = recip_of(gm1);
  c.rdx = recip_of(dx);
  c.rdy = recip_of(dy);
  return c;
}

// Lagrange-flux face flux (riemann_hll.hpp:29-39, solver.cpp:26-43) on the fast
// paths, for u* != 0; ok &= every range check.  When needs_mean(us_out) the
// caller replaces f with face_mean (the reference's mean-state branch).
// TINY: some velocity of the stencil may lie in (0, 2^-500) (numerical
// precursors), so the velocity-weighted quotient of u* goes through div_exact;
// without such velocities the cell box proves the plain fast path valid.
template <int AXIS, bool TINY = true>
__device__ __forceinline__ void face_fast(double m0, double m1, double m2, double m3, double p0,
                                          double p1, double p2, double p3, const FK& c,
                                          double f[4], bool& ok, double& ps_out, double& us_out) {
  const double ul = AXIS == 0 ? m1 : m2;
  const double ur = AXIS == 0 ? p1 : p2;
  const double cl = sqrt_fast(div1_fast(c.gamma * m3, m0, ok), ok);
  const double cr = sqrt_fast(div1_fast(c.gamma * p3, p0, ok), ok);
  const double cmax = pmax(cl, cr);
  const double rho_sum = m0 + p0;
  const Recip rs = recip_of(rho_sum);
  const double ps = div_fast(p0 * m3 + m0 * p3, rs, ok) - div_fast(m0 * p0, rs, ok) * cmax * (ur - ul);
  const double un = TINY ? div_exact_ol(m0 * ul + p0 * ur, rs, ok) : div_fast(m0 * ul + p0 * ur, rs, ok);
  const double us = un - div1_fast(p3 - m3, cmax * rho_sum, ok);
  // upwind side, branch-free (u* > 0: minus trace, else plus trace); the mean
  // state of u* == 0 is patched afterwards by face_mean (rare), so the main
  // path stays one straight line the compiler can interleave with other faces
  const bool pos = us > 0.0;
  const double s0 = pos ? m0 : p0, s1 = pos ? m1 : p1, s2 = pos ? m2 : p2, s3 = pos ? m3 : p3;
  const double a1 = s0 * s1, a2 = s0 * s2;
  const double a3 = div_fast(s3, c.rgm1, ok) + 0.5 * s0 * (s1 * s1 + s2 * s2);
  f[0] = s0 * us;
  f[1] = AXIS == 0 ? a1 * us + ps : a1 * us;
  f[2] = AXIS == 1 ? a2 * us + ps : a2 * us;
  f[3] = a3 * us + ps * us;
  ps_out = ps;
  us_out = us;
}

__device__ __forceinline__ bool needs_mean(double us) { return !(us > 0.0 || us < 0.0); }

// u* == 0 (or NaN): the flux from the mean of the two conserved traces
// (solver.cpp:33-41), given the face's p* and u*.
template <int AXIS>
__device__ __forceinline__ void face_mean(double m0, double m1, double m2, double m3, double p0,
                                          double p1, double p2, double p3, double ps, double us,
                                          const FK& c, double f[4], bool& ok) {
  const double m3c = div_fast(m3, c.rgm1, ok) + 0.5 * m0 * (m1 * m1 + m2 * m2);
  const double p3c = div_fast(p3, c.rgm1, ok) + 0.5 * p0 * (p1 * p1 + p2 * p2);
  const double a0 = 0.5 * (m0 + p0);
  const double a1 = 0.5 * (m0 * m1 + p0 * p1);
  const double a2 = 0.5 * (m0 * m2 + p0 * p2);
  const double a3 = 0.5 * (m3c + p3c);
  f[0] = a0 * us;
  f[1] = AXIS == 0 ? a1 * us + ps : a1 * us;
  f[2] = AXIS == 1 ? a2 * us + ps : a2 * us;
  f[3] = a3 * us + ps * us;
}

// Cell traces (reconstruct.hpp:33-49): lo = q - 0.5 s (plus side of the face
// below/left), hi = q + 0.5 s (minus side of the face above/right).
template <bool MUSCL>
__device__ __forceinline__ void cell_traces(double qm, double q0, double qp, double beta,
                                            double& lo, double& hi) {
  if (MUSCL) {
    const double hs = 0.5 * sweby_fast(qp - q0, q0 - qm, beta);
    lo = q0 - hs;
    hi = q0 + hs;
  } else {
    lo = q0;
    hi = q0;
  }
}

// Traces from the two one-sided differences a = q+ - q0, b = q0 - q- (the
// caller shares them between neighbouring cells).
template <bool MUSCL>
__device__ __forceinline__ void traces_ab(double a, double b, double q0, double beta, double& lo,
                                          double& hi) {
  if (MUSCL) {
    const double hs = 0.5 * sweby_fast(a, b, beta);
    lo = q0 - hs;
    hi = q0 + hs;
  } else {
    lo = q0;
    hi = q0;
  }
}

// The cell box.  If every cell feeding a face has rho, p in [2^-100, 2^100) and
// |u|, |v| < 2^100, every division and square root of the face (face_fast /
// face_mean) is on its fast path -- except the velocity-weighted quotient of u*,
// which div_exact completes with the IEEE operator when needed -- so the
// kernels test the box once per cell instead of range-checking each operation:
//   * traces: rho0 - hs > 0 is either >= rho0/2 or, by Sterbenz, an exact
//     difference of two values >= 2^-101, hence >= 2^-153; all traces are below
//     2^101;
//   * dividends: p_R - p_L is 0 or >= 2^-205, every other dividend except
//     rho_L u_L + rho_R u_R (div_exact) is a product of traces >= 2^-306;
//   * divisors rho_L + rho_R, cmax (rho_L + rho_R), rho, gamma - 1 lie in
//     [2^-280, 2^233], so every quotient is in [2^-913, 2^400] -- normal, where
//     the fast path is exact (fastmath.cuh; gamma - 1 in [2^-14, 2^6) is checked
//     by const_in_box).
// A cell outside the box raises the failure flag: the stage-wise IEEE kernels
// then compute the step exactly (never for physical data).
__device__ __forceinline__ bool pos_in_box(double x) {
  // hi word of 2^-100 = 0x39b00000, of 2^100 = 0x46300000
  return ((unsigned)__double2hiint(x) - 0x39b00000u) < (0x46300000u - 0x39b00000u);
}
__device__ __forceinline__ bool vel_in_box(double x) {
  // |x| < 2^100 (hi word of 2^100 = 0x46300000); zero and subnormals included
  return ((unsigned)__double2hiint(x) & 0x7fffffffu) < 0x46300000u;
}
// a velocity in (0, 2^-500): the stencil needs the exact u* quotient (face_fast<.., true>)
__device__ __forceinline__ bool vel_tiny(double x) {
  const unsigned h = (unsigned)__double2hiint(x) & 0x7fffffffu;
  return h < 0x20b00000u && (h | (unsigned)__double2loint(x)) != 0u;
}
__device__ __forceinline__ bool cell_in_box(const double w[4]) {
  return pos_in_box(w[0]) && pos_in_box(w[3]) && vel_in_box(w[1]) && vel_in_box(w[2]);
}
__device__ __forceinline__ bool const_in_box(double gamma, double gm1) {
  return gm1 >= 0x1p-14 && gm1 < 0x1p6 && gamma < 0x1p7;
}

// Primitives (solver.cpp:153-157) with the fast reciprocal; ok &= range check.
__device__ __forceinline__ void prim_fast(double r, double mx, double my, double e, double gm1,
                                          double w[4], bool& ok) {
  const double inv = div1_fast(1.0, r, ok);
  w[0] = r;
  w[1] = mx * inv;
  w[2] = my * inv;
  w[3] = gm1 * (e - (0.5 * (mx * mx + my * my)) * inv);
}

// Epilogue of an updated cell, branch-free: the positivity test's internal
// energy (solver.cpp:300-302) and the CFL rate of the new state
// (solver.cpp:457-469) share 1/v0's reciprocal and the kinetic term
// kin = 0.5 (v1^2 + v2^2), which both reference expressions contain verbatim
// (kin / v0 and kin * inv).  ok_e / ok_r &= the range checks of each part;
// rate_ok is false for a non-physical cell (the reference's compute_dt failure).
__device__ __forceinline__ void cell_epilogue(const double v[4], const FK& c, double& eint,
                                              bool& ok_e, double& rr, bool& rate_ok,
                                              bool& ok_r) {
  const Recip r0 = recip_of(v[0]);
  const double kin = 0.5 * (v[1] * v[1] + v[2] * v[2]);
  eint = v[3] - div_exact(kin, r0, ok_e);
  const double inv = div_fast(1.0, r0, ok_r);
  const double uu = v[1] * inv, vv = v[2] * inv;
  const double p = c.gm1 * (v[3] - kin * inv);
  rate_ok = (v[0] > 0.0) && (p > 0.0);
  const double cs = sqrt_fast(c.gamma * p * inv, ok_r);
  rr = div_fast(abs_bits(uu) + cs, c.rdx, ok_r);
  rr += div_fast(abs_bits(vv) + cs, c.rdy, ok_r);
}

// cell_epilogue with its rate checks proved by a box instead of tested per
// operation.  If rho in [2^-100, 2^100), |m_x|, |m_y| < 2^100, p in [2^-400,
// 2^400) and dx, dy in [2^-100, 2^100) (dxy_box, once per launch): 1/rho is in
// (2^-100, 2^100]; gamma p / rho (gamma in [1, 2^7)) lies in [2^-500, 2^507], so
// the square root is on its fast path and cs in [2^-250, 2^254); |u| < 2^200;
// the rate dividends |u| + cs lie in [2^-250, 2^255) and the quotients by dx, dy
// in [2^-355, 2^355] -- all normal, where the fast paths are exact.  ok_r is
// then the box itself; a cell outside it flags the step (stage-wise re-run).
// The e_int quotient keeps div_exact and its own test (tiny kinetic energies).
// OL: the e_int quotient's tiny-dividend completion out of line (the exact
// kernels: smaller code, no spill; inline in the plain kernels, -1 % otherwise).
template <bool OL = false>
__device__ __forceinline__ void cell_epilogue_box(const double v[4], const FK& c, bool dxy_box,
                                                  double& eint, bool& ok_e, double& rr,
                                                  bool& rate_ok, bool& ok_r) {
  const Recip r0 = recip_of(v[0]);
  const double kin = 0.5 * (v[1] * v[1] + v[2] * v[2]);
  eint = v[3] - (OL ? div_exact_ol(kin, r0, ok_e) : div_exact(kin, r0, ok_e));
  bool dead = true;  // proved by the box
  const double inv = div_fast(1.0, r0, dead);
  const double uu = v[1] * inv, vv = v[2] * inv;
  const double p = c.gm1 * (v[3] - kin * inv);
  rate_ok = (v[0] > 0.0) && (p > 0.0);
  const double cs = sqrt_fast(c.gamma * p * inv, dead);
  rr = div_fast(abs_bits(uu) + cs, c.rdx, dead);
  rr += div_fast(abs_bits(vv) + cs, c.rdy, dead);
  // hi words: 2^-400 = 0x26f00000, 2^400 = 0x58f00000
  const bool p_box = ((unsigned)__double2hiint(p) - 0x26f00000u) < (0x58f00000u - 0x26f00000u);
  ok_r = ok_r && dxy_box && pos_in_box(v[0]) && vel_in_box(v[1]) && vel_in_box(v[2]) && p_box;
}

#endif  // __CUDACC__

}  // namespace lfb
