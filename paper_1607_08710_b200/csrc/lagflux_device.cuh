// lagflux_device.cuh -- per-cell / per-face fp64 arithmetic of the Lagrange-flux step.
//
// Every expression keeps the reference's operation order so that, compiled
// with --fmad=false (IEEE `/` and `sqrt` are the CUDA defaults for double),
// each value is bit-identical to the reference CPU build:
//   primitives        solver.cpp:153-157
//   sweby_limiter     reconstruct.hpp:24-30 (libstdc++ min/max tie semantics)
//   muscl_face_trace  reconstruct.hpp:44-49
//   lagrangian_hll    riemann_hll.hpp:27-40, sound_speed euler.hpp:99-104
//   upwind + flux     solver.cpp:26-43, conserved_from_primitive euler.hpp:87-97
//   update            solver.cpp:283-291, positivity solver.cpp:300-302
//   CFL rate          solver.cpp:457-469
// Axis normals are specialised (n = e_x or e_y): this changes only the sign of
// an exact zero (e.g. a -0.0 momentum flux), never a nonzero value, so parity
// is checked with == per element.
#pragma once

#include <cstdint>

namespace lfb {

struct Consts {
  double gamma;   // adiabatic index
  double gm1;     // gamma - 1.0 (the reference recomputes it inline: same value)
  double beta;    // Sweby coefficient
  double dx, dy;
};

#ifdef __CUDACC__
__device__ __forceinline__ double smin(double a, double b) { return (b < a) ? b : a; }
__device__ __forceinline__ double smax(double a, double b) { return (a < b) ? b : a; }

// reconstruct.hpp:24-30
__device__ __forceinline__ double sweby(double a, double b, double beta) {
  if (!(a * b > 0.0)) return 0.0;
  const double aa = fabs(a);
  const double ab = fabs(b);
  const double m = smax(smin(aa, beta * ab), smin(beta * aa, ab));
  return a > 0.0 ? m : -m;
}

// limited_slope(qm, q0, qp) = sweby(qp - q0, q0 - qm): reconstruct.hpp:33-35
__device__ __forceinline__ double slope3(double qm, double q0, double qp, double beta) {
  return sweby(qp - q0, q0 - qm, beta);
}

// primitives from conserved (solver.cpp:153-157).  Returns inv = 1/r.
__device__ __forceinline__ void primitive(double r, double mx, double my, double e, double gm1,
                                          double& u, double& v, double& p) {
  const double inv = 1.0 / r;
  u = mx * inv;
  v = my * inv;
  p = gm1 * (e - (0.5 * (mx * mx + my * my)) * inv);
}

// Lagrange-flux face flux for traces wm (low side) and wp (high side), w = (rho,u,v,p).
// AXIS 0: x-face (normal e_x), AXIS 1: y-face (normal e_y).
template <int AXIS>
__device__ __forceinline__ void face_flux(double wm0, double wm1, double wm2, double wm3,
                                          double wp0, double wp1, double wp2, double wp3,
                                          const Consts& k, double f[4]) {
  // lagrangian_hll (riemann_hll.hpp:29-39)
  const double ul = AXIS == 0 ? wm1 : wm2;
  const double ur = AXIS == 0 ? wp1 : wp2;
  const double cl = sqrt(k.gamma * wm3 / wm0);
  const double cr = sqrt(k.gamma * wp3 / wp0);
  const double cmax = smax(cl, cr);
  const double rho_sum = wm0 + wp0;
  const double ps = (wp0 * wm3 + wm0 * wp3) / rho_sum - (wm0 * wp0 / rho_sum) * cmax * (ur - ul);
  const double us = (wm0 * ul + wp0 * ur) / rho_sum - (wp3 - wm3) / (cmax * rho_sum);
  // upwind conserved interface state (solver.cpp:28-36, euler.hpp:91-95)
  double a0, a1, a2, a3;
  if (us > 0.0) {
    a0 = wm0;
    a1 = wm0 * wm1;
    a2 = wm0 * wm2;
    a3 = wm3 / k.gm1 + 0.5 * wm0 * (wm1 * wm1 + wm2 * wm2);
  } else if (us < 0.0) {
    a0 = wp0;
    a1 = wp0 * wp1;
    a2 = wp0 * wp2;
    a3 = wp3 / k.gm1 + 0.5 * wp0 * (wp1 * wp1 + wp2 * wp2);
  } else {
    const double m1 = wm0 * wm1, m2 = wm0 * wm2;
    const double m3 = wm3 / k.gm1 + 0.5 * wm0 * (wm1 * wm1 + wm2 * wm2);
    const double p1 = wp0 * wp1, p2 = wp0 * wp2;
    const double p3 = wp3 / k.gm1 + 0.5 * wp0 * (wp1 * wp1 + wp2 * wp2);
    a0 = 0.5 * (wm0 + wp0);
    a1 = 0.5 * (m1 + p1);
    a2 = 0.5 * (m2 + p2);
    a3 = 0.5 * (m3 + p3);
  }
  // contact_flux (solver.cpp:38-41) with n = e_AXIS
  f[0] = a0 * us;
  f[1] = AXIS == 0 ? a1 * us + ps : a1 * us;
  f[2] = AXIS == 1 ? a2 * us + ps : a2 * us;
  f[3] = a3 * us + ps * us;
}

// Trace positivity (solver.cpp:222).
__device__ __forceinline__ bool traces_ok(double wm0, double wm3, double wp0, double wp3) {
  return (wm0 > 0.0) && (wm3 > 0.0) && (wp0 > 0.0) && (wp3 > 0.0);
}

// Per-cell CFL rate (solver.cpp:457-468).  Returns false for a non-physical cell.
template <bool DIM2>
__device__ __forceinline__ bool cfl_rate(double r, double mx, double my, double e, const Consts& k,
                                         double& rate) {
  if (!(r > 0.0)) return false;
  const double inv = 1.0 / r;
  const double u = mx * inv;
  const double v = my * inv;
  const double p = k.gm1 * (e - 0.5 * (mx * mx + my * my) * inv);
  if (!(p > 0.0)) return false;
  const double c = sqrt(k.gamma * p * inv);
  double rr = (fabs(u) + c) / k.dx;
  if (DIM2) rr += (fabs(v) + c) / k.dy;
  rate = rr;
  return true;
}

// gamma-independent positivity of an updated cell (solver.cpp:300-302).
__device__ __forceinline__ double internal_energy(double v0, double v1, double v2, double v3) {
  return v3 - 0.5 * (v1 * v1 + v2 * v2) / v0;
}

// Order-preserving keys for atomic min/max on doubles.
__device__ __forceinline__ unsigned long long pos_bits(double x) {
  return (unsigned long long)__double_as_longlong(x);
}

#endif  // __CUDACC__

}  // namespace lfb
