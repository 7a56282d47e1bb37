// edge_flux.cu -- the reference's free edge_flux (solver.cpp:45-53) on the device,
// over a batch of faces with arbitrary unit normals and one EOS per side.
//
// The expressions are the reference's, in its order (compiled with --fmad=false,
// IEEE division and square root): lagrangian_hll (riemann_hll.hpp:27-45) with
// sound_speed's checks (euler.hpp:99-104), conserved_from_primitive
// (euler.hpp:87-97) and contact_flux (solver.cpp:26-43), normal products
// included -- unlike the step kernels, which specialise the axis normals, the
// results here equal the reference's bit for bit, signed zeros too.  A face
// whose state fails a check is reported like the reference's throw: the
// smallest such face, its first failing check (left rho, left p, right rho,
// right p -- the order lagrangian_hll evaluates them).
#include <cuda_runtime.h>

#include "kernels.h"

namespace lfb {

namespace {

__global__ void k_edge_flux(int64_t n, const double* __restrict__ wm, const double* __restrict__ wp,
                            const double* __restrict__ nrm, const double* __restrict__ gm,
                            const double* __restrict__ gp, double* __restrict__ flux,
                            double* __restrict__ contact, unsigned long long* fail) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double a0 = wm[4 * i], a1 = wm[4 * i + 1], a2 = wm[4 * i + 2], a3 = wm[4 * i + 3];
    const double b0 = wp[4 * i], b1 = wp[4 * i + 1], b2 = wp[4 * i + 2], b3 = wp[4 * i + 3];
    int bad = -1;
    if (!(a0 > 0.0)) bad = 0;
    else if (!(a3 > 0.0)) bad = 1;
    else if (!(b0 > 0.0)) bad = 2;
    else if (!(b3 > 0.0)) bad = 3;
    if (bad >= 0) {
      atomicMin(fail, (unsigned long long)i * 4 + (unsigned long long)bad);
      continue;
    }
    const double nx = nrm[2 * i], ny = nrm[2 * i + 1];
    const double gl = gm[i], gr = gp[i];
    // lagrangian_hll
    const double ul = a1 * nx + a2 * ny;
    const double ur = b1 * nx + b2 * ny;
    const double cl = sqrt(gl * a3 / a0);
    const double cr = sqrt(gr * b3 / b0);
    const double cmax = (cl < cr) ? cr : cl;  // std::max
    const double rho_sum = a0 + b0;
    const double ps = (b0 * a3 + a0 * b3) / rho_sum - (a0 * b0 / rho_sum) * cmax * (ur - ul);
    const double us = (a0 * ul + b0 * ur) / rho_sum - (b3 - a3) / (cmax * rho_sum);
    // conserved_from_primitive of both traces
    const double m1 = a0 * a1, m2 = a0 * a2;
    const double m3 = a3 / (gl - 1.0) + 0.5 * a0 * (a1 * a1 + a2 * a2);
    const double p1 = b0 * b1, p2 = b0 * b2;
    const double p3 = b3 / (gr - 1.0) + 0.5 * b0 * (b1 * b1 + b2 * b2);
    // contact_flux
    double u0, u1, u2, u3;
    if (us > 0.0) {
      u0 = a0, u1 = m1, u2 = m2, u3 = m3;
    } else if (us < 0.0) {
      u0 = b0, u1 = p1, u2 = p2, u3 = p3;
    } else {
      u0 = 0.5 * (a0 + b0);
      u1 = 0.5 * (m1 + p1);
      u2 = 0.5 * (m2 + p2);
      u3 = 0.5 * (m3 + p3);
    }
    flux[4 * i] = u0 * us;
    flux[4 * i + 1] = u1 * us + ps * nx;
    flux[4 * i + 2] = u2 * us + ps * ny;
    flux[4 * i + 3] = u3 * us + ps * us;
    if (contact) {
      contact[2 * i] = ps;
      contact[2 * i + 1] = us;
    }
  }
}

}  // namespace

void launch_edge_flux(int64_t n, const double* wm, const double* wp, const double* nrm,
                      const double* gm, const double* gp, double* flux, double* contact,
                      unsigned long long* fail, cudaStream_t st) {
  count_launch();
  const int64_t blocks = (n + 255) / 256;
  k_edge_flux<<<(unsigned)(blocks < 148 * 16 ? (blocks > 0 ? blocks : 1) : 148 * 16), 256, 0, st>>>(
      n, wm, wp, nrm, gm, gp, flux, contact, fail);
}

}  // namespace lfb
