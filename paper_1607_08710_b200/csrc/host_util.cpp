// host_util.cpp -- host helpers: ghost fill of downloaded fields and the
// 1D tables of the smooth-flow initial condition.
#include "host_util.h"

#include <cmath>
#include <random>

namespace lfb {

void host_apply_boundary(const lf_desc& d, double* const field[4], int64_t ld) {
  const int gx = 2, gy = d.dim == 2 ? 2 : 0;
  const int nx = d.nx, ny = d.ny;
  for (int c = 0; c < 4; ++c) {
    double* f = field[c];
    const double sx = c == 1 ? -1.0 : 1.0;
    const double sy = c == 2 ? -1.0 : 1.0;
    auto at = [&](int i, int j) -> double& { return f[(int64_t)j * ld + i]; };
    for (int j = gy; j < gy + ny; ++j)
      for (int l = 1; l <= gx; ++l) {
        const int lo = gx - l, hi = gx + nx - 1 + l;
        switch (d.bc[0]) {
          case LF_TRANSMISSIVE: at(lo, j) = at(gx, j); break;
          case LF_REFLECTIVE: at(lo, j) = sx * at(gx + l - 1, j); break;
          default: at(lo, j) = at(gx + ((nx - l) % nx + nx) % nx, j); break;
        }
        switch (d.bc[1]) {
          case LF_TRANSMISSIVE: at(hi, j) = at(gx + nx - 1, j); break;
          case LF_REFLECTIVE: at(hi, j) = sx * at(gx + nx - l, j); break;
          default: at(hi, j) = at(gx + (l - 1) % nx, j); break;
        }
      }
    if (gy == 0) continue;
    for (int i = 0; i < nx + 2 * gx; ++i)
      for (int l = 1; l <= gy; ++l) {
        const int lo = gy - l, hi = gy + ny - 1 + l;
        switch (d.bc[2]) {
          case LF_TRANSMISSIVE: at(i, lo) = at(i, gy); break;
          case LF_REFLECTIVE: at(i, lo) = sy * at(i, gy + l - 1); break;
          default: at(i, lo) = at(i, gy + ((ny - l) % ny + ny) % ny); break;
        }
        switch (d.bc[3]) {
          case LF_TRANSMISSIVE: at(i, hi) = at(i, gy + ny - 1); break;
          case LF_REFLECTIVE: at(i, hi) = sy * at(i, gy + ny - l); break;
          default: at(i, hi) = at(i, gy + (l - 1) % ny); break;
        }
      }
  }
}

void fourier_tables(uint64_t seed, const lf_desc& d, std::vector<double>& tx,
                    std::vector<double>& ty, std::vector<double>& amp) {
  const double two_pi = 6.283185307179586476925286766559;
  std::mt19937_64 rng(seed);
  tx.assign((size_t)64 * d.nx, 0.0);
  ty.assign((size_t)64 * d.ny, 0.0);
  amp.assign(32, 0.0);
  for (int k = 0; k < 4; ++k)
    for (int m = 0; m < 8; ++m) {
      const int kx = 1 + (int)(rng() % 8ULL);
      const int ky = 1 + (int)(rng() % 8ULL);
      const double a = (double)(rng() >> 11) * 0x1.0p-53;
      const double phi = two_pi * ((double)(rng() >> 11) * 0x1.0p-53);
      amp[(size_t)(k * 8 + m)] = a;
      double* sx = &tx[(size_t)(k * 8 + m) * 2 * d.nx];
      double* cx = sx + d.nx;
      for (int i = 0; i < d.nx; ++i) {
        const double x = d.x0 + (i + 0.5) * d.dx;
        const double arg = two_pi * (kx * x) + phi;
        sx[i] = std::sin(arg);
        cx[i] = std::cos(arg);
      }
      double* sy = &ty[(size_t)(k * 8 + m) * 2 * d.ny];
      double* cy = sy + d.ny;
      for (int j = 0; j < d.ny; ++j) {
        const double y = d.y0 + (j + 0.5) * d.dy;
        const double arg = two_pi * (ky * y);
        sy[j] = std::sin(arg);
        cy[j] = std::cos(arg);
      }
    }
}

}  // namespace lfb
