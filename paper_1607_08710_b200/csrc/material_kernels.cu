// material_kernels.cu -- multimaterial partial-density transport (stage-wise).
//
// The reference's MaterialSet path (solver.cpp:90-129, 131-171, 173-256,
// 331-404, 434-480, 519-540; multimat.cpp:17-44), one kernel per reference
// loop like stage_kernels.cu, so the failure semantics (smallest failing index,
// check order) carry over unchanged:
//   k_mat_fractions    fill_all_ghosts' closure: clamped fractions and the
//                      mixed-cell gamma of every ghosted cell
//   k_rate_g / k_prims_g / k_flux_g
//                      compute_dt / build_primitives / compute_fluxes with the
//                      per-cell gamma (each face side carries its own EOS) and
//                      the face u* stored for the material fluxes
//   k_update_partials  update_partials: per-material face fluxes from the mass
//                      flux and the upwind fractions (the last material takes
//                      the complement), the Heun weights applied as the
//                      reference accumulates them ((0 + w a) + w b)
//   k_mat_min_p        the diagnostics' min pressure from the fresh partials
// All arithmetic keeps the reference's operation order (--fmad=false).
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>

#include "kernels.h"
#include "reduce.cuh"

namespace lfb {

namespace {

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ long long warp_min_i64(long long v) {
  for (int o = 16; o > 0; o >>= 1) {
    const long long w = __shfl_xor_sync(FULL, v, o);
    v = w < v ? w : v;
  }
  return v;
}

// order-preserving key of a non-NaN double (unsigned compare == IEEE compare,
// -0.0 below +0.0)
__device__ __forceinline__ unsigned long long order_key(double x) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(x);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// ---------------------------------------------------------------- fractions
// solver.cpp:100-121 over the reference's ghosted cells (i in [-2, nx+2),
// j in [-gy, ny+gy)); the failure index is the reference's ghosted index.
__global__ void k_mat_fractions(Field u, Field part, Field y, Field gcell, int nx, int ny,
                                int gy_ref, Slab sl, MatConsts mc, Scalars* s) {
  const int i = (int)(blockIdx.x * blockDim.x + threadIdx.x) - 2;
  const int j = (int)(blockIdx.y * blockDim.y + threadIdx.y) - gy_ref;
  long long fail = LLONG_MAX;
  if (i < nx + 2 && j < ny + gy_ref) {
    const int64_t o = (int64_t)j * u.pitch + i;
    const double rho = u.p[o];
    double ysum_gamma = 0.0;
    int pure = -1;
    bool bad = false;
    for (int k = 0; k < mc.n; ++k) {
      const double raw = part.p[k * part.fstride + o] / rho;
      double yk = raw;
      if (yk < 0.0 || yk > 1.0) {
        if (raw < -1e-11 || raw > 1.0 + 1e-11) {
          bad = true;
          yk = 0.0;
        } else {
          yk = raw < 0.0 ? 0.0 : 1.0;
        }
      }
      y.p[k * y.fstride + o] = yk;
      if (yk == 1.0) pure = k;
      ysum_gamma += yk / (mc.gamma[k] - 1.0);
    }
    gcell.p[o] = pure >= 0 ? mc.gamma[pure] : 1.0 + 1.0 / ysum_gamma;
    const bool owned = (j >= 0 || sl.fill_lo) && (j < ny || sl.fill_hi);
    if (bad && owned) fail = (long long)(j + sl.y0 + gy_ref) * (nx + 4) + (i + 2);
  }
  fail = warp_min_i64(fail);
  if (((threadIdx.y * blockDim.x + threadIdx.x) & 31) == 0 && fail != LLONG_MAX)
    atomicMin(&s->fail_frac, fail);
}

// ---------------------------------------------------------------- CFL rate
// solver.cpp:449-470 with g = gamma_[0][cell]
template <bool DIM2>
__global__ void k_rate_g(Field u, Field gcell, int nx, int ny, int y0, Consts k, Scalars* s) {
  unsigned long long best = 0ull;
  long long fail = LLONG_MAX;
  const int64_t n = (int64_t)nx * ny;
  for (int64_t cc = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; cc < n;
       cc += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(cc % nx), j = (int)(cc / nx);
    const int64_t o = (int64_t)j * u.pitch + i;
    const double r = u.p[o];
    bool ok = r > 0.0;
    if (ok) {
      const double mx = u.p[u.fstride + o], my = u.p[2 * u.fstride + o];
      const double inv = 1.0 / r;
      const double uu = mx * inv;
      const double vv = my * inv;
      const double g = gcell.p[o];
      const double p = (g - 1.0) * (u.p[3 * u.fstride + o] - 0.5 * (mx * mx + my * my) * inv);
      ok = p > 0.0;
      if (ok) {
        const double c = sqrt(g * p * inv);
        double rr = (fabs(uu) + c) / k.dx;
        if (DIM2) rr += (fabs(vv) + c) / k.dy;
        if (rr == rr) {  // std::max(rate, rr) keeps rate for a NaN rr
          const unsigned long long b = pos_bits(rr);
          best = b > best ? b : best;
        }
      }
    }
    if (!ok) {
      const long long gidx = (long long)(j + y0) * nx + i;
      fail = gidx < fail ? gidx : fail;
    }
  }
  best = block_reduce(best, MaxOp(), 0ull);
  fail = block_reduce(fail, MinOp(), (long long)LLONG_MAX);
  if (threadIdx.x == 0) {
    if (best) atomicMax(&s->rate_bits, best);
    if (fail != LLONG_MAX) atomicMin(&s->fail_dt, fail);
  }
}

// ---------------------------------------------------------------- primitives
// solver.cpp:145-163 with g = gamma_[slot][c]
__global__ void k_prims_g(Field u, Field w, Field gcell, int nx, int ny, int gy_ref, Slab sl,
                          Scalars* s) {
  const int i = (int)(blockIdx.x * blockDim.x + threadIdx.x) - 2;
  const int j = (int)(blockIdx.y * blockDim.y + threadIdx.y) - gy_ref;
  long long fail = LLONG_MAX;
  if (i < nx + 2 && j < ny + gy_ref) {
    const int64_t o = (int64_t)j * u.pitch + i;
    const double r = u.p[o];
    double uu = 0.0, vv = 0.0, pp = 0.0, rr = 0.0;
    bool bad;
    if (!(r > 0.0)) {
      bad = true;
    } else {
      rr = r;
      primitive(r, u.p[u.fstride + o], u.p[2 * u.fstride + o], u.p[3 * u.fstride + o],
                gcell.p[o] - 1.0, uu, vv, pp);
      bad = !(pp > 0.0);
    }
    w.p[o] = rr;
    w.p[w.fstride + o] = uu;
    w.p[2 * w.fstride + o] = vv;
    w.p[3 * w.fstride + o] = pp;
    const bool owned = (j >= 0 || sl.fill_lo) && (j < ny || sl.fill_hi);
    if (bad && owned) fail = (long long)(j + sl.y0 + gy_ref) * (nx + 4) + (i + 2);
  }
  fail = warp_min_i64(fail);
  if (((threadIdx.y * blockDim.x + threadIdx.x) & 31) == 0 && fail != LLONG_MAX)
    atomicMin(&s->fail_prim, fail);
}

// ---------------------------------------------------------------- face fluxes
// solver.cpp:196-239 with el = gamma[clow], er = gamma[chigh]:
// lagrangian_hll(wm, wp, n, el, er), contact_flux(U(wm, el), U(wp, er), n, cs).
template <int AXIS>
__device__ __forceinline__ void face_flux_g(const double wm[4], const double wp[4], double el,
                                            double er, double f[4], double& us) {
  const double ul = AXIS == 0 ? wm[1] : wm[2];
  const double ur = AXIS == 0 ? wp[1] : wp[2];
  const double cl = sqrt(el * wm[3] / wm[0]);
  const double cr = sqrt(er * wp[3] / wp[0]);
  const double cmax = smax(cl, cr);
  const double rho_sum = wm[0] + wp[0];
  const double ps =
      (wp[0] * wm[3] + wm[0] * wp[3]) / rho_sum - (wm[0] * wp[0] / rho_sum) * cmax * (ur - ul);
  us = (wm[0] * ul + wp[0] * ur) / rho_sum - (wp[3] - wm[3]) / (cmax * rho_sum);
  double a0, a1, a2, a3;
  if (us > 0.0) {
    a0 = wm[0];
    a1 = wm[0] * wm[1];
    a2 = wm[0] * wm[2];
    a3 = wm[3] / (el - 1.0) + 0.5 * wm[0] * (wm[1] * wm[1] + wm[2] * wm[2]);
  } else if (us < 0.0) {
    a0 = wp[0];
    a1 = wp[0] * wp[1];
    a2 = wp[0] * wp[2];
    a3 = wp[3] / (er - 1.0) + 0.5 * wp[0] * (wp[1] * wp[1] + wp[2] * wp[2]);
  } else {
    const double m1 = wm[0] * wm[1], m2 = wm[0] * wm[2];
    const double m3 = wm[3] / (el - 1.0) + 0.5 * wm[0] * (wm[1] * wm[1] + wm[2] * wm[2]);
    const double p1 = wp[0] * wp[1], p2 = wp[0] * wp[2];
    const double p3 = wp[3] / (er - 1.0) + 0.5 * wp[0] * (wp[1] * wp[1] + wp[2] * wp[2]);
    a0 = 0.5 * (wm[0] + wp[0]);
    a1 = 0.5 * (m1 + p1);
    a2 = 0.5 * (m2 + p2);
    a3 = 0.5 * (m3 + p3);
  }
  f[0] = a0 * us;
  f[1] = AXIS == 0 ? a1 * us + ps : a1 * us;
  f[2] = AXIS == 1 ? a2 * us + ps : a2 * us;
  f[3] = a3 * us + ps * us;
}

template <int AXIS, bool MUSCL>
__global__ void k_flux_g(Field w, Field gcell, FluxArr fo, FluxArr uso, int nx, int ny, Slab sl,
                         Consts k, Scalars* s) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  const int b = blockIdx.y * blockDim.y + threadIdx.y;
  const int na = AXIS == 0 ? nx + 1 : nx;
  const int nb = AXIS == 0 ? ny : ny + 1;
  long long fail = LLONG_MAX;
  if (a < na && b < nb) {
    const int64_t st = AXIS == 0 ? 1 : w.pitch;
    const int64_t hi = (int64_t)b * w.pitch + a;
    const int64_t lo = hi - st;
    double wm[4], wp[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const double* q = w.p + c * w.fstride;
      if (MUSCL) {
        const double q0 = q[lo - st], q1 = q[lo], q2 = q[hi], q3 = q[hi + st];
        const double s1 = slope3(q0, q1, q2, k.beta);
        const double s2 = slope3(q1, q2, q3, k.beta);
        wm[c] = q1 + 0.5 * s1;
        wp[c] = q2 - 0.5 * s2;
      } else {
        wm[c] = q[lo];
        wp[c] = q[hi];
      }
    }
    double f[4] = {0.0, 0.0, 0.0, 0.0};
    double us = 0.0;
    if (traces_ok(wm[0], wm[3], wp[0], wp[3])) {
      face_flux_g<AXIS>(wm, wp, gcell.p[lo], gcell.p[hi], f, us);
    } else {
      const long long nex = (long long)(nx + 1) * sl.ny_global;
      fail = AXIS == 0 ? (long long)(b + sl.y0) * (nx + 1) + a
                       : nex + (long long)(b + sl.y0) * nx + a;
    }
    const int64_t fo_off = (int64_t)b * fo.pitch + a;
#pragma unroll
    for (int c = 0; c < 4; ++c) fo.p[c * fo.fstride + fo_off] = f[c];
    uso.p[fo_off] = us;
  }
  fail = warp_min_i64(fail);
  if (((threadIdx.y * blockDim.x + threadIdx.x) & 31) == 0 && fail != LLONG_MAX)
    atomicMin(&s->fail_trace, fail);
}

// ---------------------------------------------------------------- partials
// solver.cpp:341-403.  One face of one stage: its mass flux, u* and the
// fractions of the upwind cell; material k's flux (k < n-1: mass * y_k[up],
// the last: the complement), or 0 on a u* == 0 face.
struct EdgeMat {
  double mass, us, rest;
  const double* yup;     // fractions of the upwind cell, component 0
  int64_t ystride;
  __device__ __forceinline__ void init(double m, double u, const double* y_lo, const double* y_hi,
                                       int64_t ys) {
    mass = m;
    us = u;
    rest = m;
    yup = us > 0.0 ? y_lo : y_hi;
    ystride = ys;
  }
  __device__ __forceinline__ double next(int k, int n) {
    if (k < n - 1) {
      const double fk = us == 0.0 ? 0.0 : mass * yup[k * ystride];
      rest -= fk;
      return fk;
    }
    return us == 0.0 ? 0.0 : rest;
  }
};

template <bool TWO, bool DIM2>
__global__ void k_update_partials(Field base, FluxArr fxa, FluxArr fya, FluxArr usxa,
                                  FluxArr usya, Field ya, FluxArr fxb, FluxArr fyb,
                                  FluxArr usxb, FluxArr usyb, Field yb, Field out, int nx,
                                  int ny, int n_mat, double lam_x, double lam_y) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y * blockDim.y + threadIdx.y;
  if (i >= nx || j >= ny) return;
  const int64_t o = (int64_t)j * base.pitch + i;     // cell (fields and fractions)
  const int64_t ex = (int64_t)j * fxa.pitch + i;     // x-face left of the cell
  const int64_t ey = (int64_t)j * fya.pitch + i;     // y-face below the cell
  const int64_t P = base.pitch;
  // stage a: faces l, r, b, t
  EdgeMat la, ra, ba, ta, lb, rb, bb, tb;
  const double* yA = ya.p + o;
  la.init(fxa.p[ex], usxa.p[ex], yA - 1, yA, ya.fstride);
  ra.init(fxa.p[ex + 1], usxa.p[ex + 1], yA, yA + 1, ya.fstride);
  if (DIM2) {
    ba.init(fya.p[ey], usya.p[ey], yA - P, yA, ya.fstride);
    ta.init(fya.p[ey + fya.pitch], usya.p[ey + fya.pitch], yA, yA + P, ya.fstride);
  }
  if (TWO) {
    const double* yB = yb.p + o;
    lb.init(fxb.p[ex], usxb.p[ex], yB - 1, yB, yb.fstride);
    rb.init(fxb.p[ex + 1], usxb.p[ex + 1], yB, yB + 1, yb.fstride);
    if (DIM2) {
      bb.init(fyb.p[ey], usyb.p[ey], yB - P, yB, yb.fstride);
      tb.init(fyb.p[ey + fyb.pitch], usyb.p[ey + fyb.pitch], yB, yB + P, yb.fstride);
    }
  }
  const double w = TWO ? 0.5 : 1.0;
  for (int k = 0; k < n_mat; ++k) {
    // gather (solver.cpp:366-383): f += w * t, set a then set b, from 0.0
    double fl = 0.0, fr = 0.0, fbot = 0.0, ftop = 0.0;
    fl += w * la.next(k, n_mat);
    fr += w * ra.next(k, n_mat);
    if (DIM2) {
      fbot += w * ba.next(k, n_mat);
      ftop += w * ta.next(k, n_mat);
    }
    if (TWO) {
      fl += w * lb.next(k, n_mat);
      fr += w * rb.next(k, n_mat);
      if (DIM2) {
        fbot += w * bb.next(k, n_mat);
        ftop += w * tb.next(k, n_mat);
      }
    }
    double val = base.p[k * base.fstride + o] - lam_x * (fr - fl);
    if (DIM2) val -= lam_y * (ftop - fbot);
    out.p[k * out.fstride + o] = val;
  }
}

// ---------------------------------------------------------------- min p
__global__ void k_mat_min_p(Field u, Field part, int nx, int ny, MatConsts mc, Scalars* s) {
  unsigned long long best = ~0ull;
  const int64_t n = (int64_t)nx * ny;
  for (int64_t cc = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; cc < n;
       cc += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(cc % nx), j = (int)(cc / nx);
    const int64_t o = (int64_t)j * u.pitch + i;
    const double r = u.p[o];
    double sum = 0.0;
    for (int k = 0; k < mc.n; ++k) sum += (part.p[k * part.fstride + o] / r) / (mc.gamma[k] - 1.0);
    const double mx = u.p[u.fstride + o], my = u.p[2 * u.fstride + o];
    const double eint = u.p[3 * u.fstride + o] - 0.5 * (mx * mx + my * my) / r;
    const double x = eint / sum;
    if (x == x) {  // std::min(min_p, x) never picks a NaN x
      const unsigned long long key = order_key(x);
      best = key < best ? key : best;
    }
  }
  best = block_reduce(best, MinOp(), ~0ull);
  if (threadIdx.x == 0 && best != ~0ull) atomicMin(&s->min_p_key, best);
}

__global__ void k_fill_value(double* p, int64_t n, double v) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x)
    p[t] = v;
}

inline unsigned cdiv(int64_t a, int64_t b) { return (unsigned)((a + b - 1) / b); }

}  // namespace

void launch_mat_fractions(const Field& u, const Field& part, const Field& y, const Field& gcell,
                          const Layout& L, const Slab& sl, const MatConsts& mc, int dim2,
                          Scalars* s, cudaStream_t st) {
  const int gy = dim2 ? 2 : 0;
  dim3 blk(32, 8);
  dim3 grd(cdiv(L.nx + 4, 32), cdiv(L.ny + 2 * gy, 8));
  count_launch(), k_mat_fractions<<<grd, blk, 0, st>>>(u, part, y, gcell, L.nx, L.ny, gy, sl, mc, s);
}

void launch_rate_g(const Field& u, const Field& gcell, const Layout& L, const Slab& sl,
                   const Consts& k, int dim2, Scalars* s, cudaStream_t st) {
  const int64_t n = (int64_t)L.nx * L.ny;
  const unsigned blocks = (unsigned)std::min<int64_t>(cdiv(n, 256), 148 * 8);
  if (dim2)
    count_launch(), k_rate_g<true><<<blocks, 256, 0, st>>>(u, gcell, L.nx, L.ny, sl.y0, k, s);
  else
    count_launch(), k_rate_g<false><<<blocks, 256, 0, st>>>(u, gcell, L.nx, L.ny, sl.y0, k, s);
}

void launch_prims_g(const Field& u, const Field& w, const Field& gcell, const Layout& L,
                    const Slab& sl, int dim2, Scalars* s, cudaStream_t st) {
  const int gy = dim2 ? 2 : 0;
  dim3 blk(32, 8);
  dim3 grd(cdiv(L.nx + 4, 32), cdiv(L.ny + 2 * gy, 8));
  count_launch(), k_prims_g<<<grd, blk, 0, st>>>(u, w, gcell, L.nx, L.ny, gy, sl, s);
}

void launch_fluxes_g(const Field& w, const Field& gcell, const FluxArr& fx, const FluxArr& fy,
                     const FluxArr& usx, const FluxArr& usy, const Layout& L, const Slab& sl,
                     const Consts& k, int muscl, int dim2, Scalars* s, cudaStream_t st) {
  dim3 blk(32, 4);
  dim3 gx(cdiv(L.nx + 1, 32), cdiv(L.ny, 4));
  if (muscl)
    count_launch(), k_flux_g<0, true><<<gx, blk, 0, st>>>(w, gcell, fx, usx, L.nx, L.ny, sl, k, s);
  else
    count_launch(), k_flux_g<0, false><<<gx, blk, 0, st>>>(w, gcell, fx, usx, L.nx, L.ny, sl, k, s);
  if (!dim2) return;
  dim3 gy(cdiv(L.nx, 32), cdiv(L.ny + 1, 4));
  if (muscl)
    count_launch(), k_flux_g<1, true><<<gy, blk, 0, st>>>(w, gcell, fy, usy, L.nx, L.ny, sl, k, s);
  else
    count_launch(), k_flux_g<1, false><<<gy, blk, 0, st>>>(w, gcell, fy, usy, L.nx, L.ny, sl, k, s);
}

void launch_update_partials(const Field& base, const FluxArr& fxa, const FluxArr& fya,
                            const FluxArr& usxa, const FluxArr& usya, const Field& ya,
                            const FluxArr* fxb, const FluxArr* fyb, const FluxArr* usxb,
                            const FluxArr* usyb, const Field* yb, const Field& out,
                            const Layout& L, int n_mat, double dt, double dx, double dy,
                            int dim2, cudaStream_t st) {
  const double lam_x = dt / dx;  // solver.cpp:336-337 (divisions)
  const double lam_y = dt / dy;
  dim3 blk(32, 8);
  dim3 grd(cdiv(L.nx, 32), cdiv(L.ny, 8));
  const bool two = fxb != nullptr;
  const FluxArr xb = two ? *fxb : fxa, yb_ = two ? *fyb : fya;
  const FluxArr uxb = two ? *usxb : usxa, uyb = two ? *usyb : usya;
  const Field fb = two ? *yb : ya;
  if (two && dim2)
    count_launch(), k_update_partials<true, true><<<grd, blk, 0, st>>>(
        base, fxa, fya, usxa, usya, ya, xb, yb_, uxb, uyb, fb, out, L.nx, L.ny, n_mat, lam_x, lam_y);
  else if (two)
    count_launch(), k_update_partials<true, false><<<grd, blk, 0, st>>>(
        base, fxa, fya, usxa, usya, ya, xb, yb_, uxb, uyb, fb, out, L.nx, L.ny, n_mat, lam_x, lam_y);
  else if (dim2)
    count_launch(), k_update_partials<false, true><<<grd, blk, 0, st>>>(
        base, fxa, fya, usxa, usya, ya, xb, yb_, uxb, uyb, fb, out, L.nx, L.ny, n_mat, lam_x, lam_y);
  else
    count_launch(), k_update_partials<false, false><<<grd, blk, 0, st>>>(
        base, fxa, fya, usxa, usya, ya, xb, yb_, uxb, uyb, fb, out, L.nx, L.ny, n_mat, lam_x, lam_y);
}

void launch_mat_min_p(const Field& u, const Field& part, const Layout& L, const MatConsts& mc,
                      Scalars* s, cudaStream_t st) {
  const int64_t n = (int64_t)L.nx * L.ny;
  const unsigned blocks = (unsigned)std::min<int64_t>(cdiv(n, 256), 148 * 8);
  count_launch(), k_mat_min_p<<<blocks, 256, 0, st>>>(u, part, L.nx, L.ny, mc, s);
}

void fill_value(double* p, int64_t n, double v, cudaStream_t st) {
  const unsigned blocks = (unsigned)std::min<int64_t>(cdiv(n, 256), 148 * 8);
  count_launch(), k_fill_value<<<blocks, 256, 0, st>>>(p, n, v);
}


// ---------------------------------------------------------------- field dumps
// field_csv's per-cell quantities (csv.cpp:40-57), in its expression order:
//   u = mx / rho, v = my / rho, eint = E - 0.5 (mx^2 + my^2) / rho,
//   p = (gamma - 1) eint, e = eint / rho, y_k = clamped_fraction(partial_k, rho),
//   gamma = mixed_cell_gamma(y) (pure cells exact) or the eos gamma.
// out: ncols planes of nx * ny (row-major, local rows); the smallest failing
// interior index of the clamp (and its fraction value) -> fail / fail_val.
namespace {
__global__ void k_csv_derive(Field u, Field part, int nx, int ny, int y0, double gamma0,
                             MatConsts mc, double* out, unsigned long long* fail) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y * blockDim.y + threadIdx.y;
  if (i >= nx || j >= ny) return;
  const int64_t o = (int64_t)j * u.pitch + i;
  const int64_t plane = (int64_t)nx * ny, c = (int64_t)j * nx + i;
  const double rho = u.p[o], mx = u.p[u.fstride + o], my = u.p[2 * u.fstride + o];
  const double uu = mx / rho;
  const double vv = my / rho;
  double gamma = gamma0;
  if (mc.n > 0) {
    double s = 0.0;
    int pure = -1;
    for (int k = 0; k < mc.n; ++k) {
      const double y = part.p[k * part.fstride + o] / rho;
      double yk = y;
      if (!(y >= 0.0 && y <= 1.0)) {
        if (y < -1e-11 || y > 1.0 + 1e-11) {
          // the first failing cell in field_csv's row-major order; the host
          // recomputes its fraction for the message
          atomicMin(fail, (unsigned long long)((int64_t)(j + y0) * nx + i));
          yk = 0.0;
        } else {
          yk = y < 0.0 ? 0.0 : 1.0;
        }
      }
      out[(5 + k) * plane + c] = yk;
      // mixed_cell_gamma (multimat.cpp:25-32): the first pure material returns
      if (pure < 0) {
        if (yk == 1.0)
          pure = k;
        else
          s += yk / (mc.gamma[k] - 1.0);
      }
    }
    gamma = pure >= 0 ? mc.gamma[pure] : 1.0 + 1.0 / s;
  }
  const double eint = u.p[3 * u.fstride + o] - 0.5 * (mx * mx + my * my) / rho;
  out[c] = rho;
  out[plane + c] = uu;
  out[2 * plane + c] = vv;
  out[3 * plane + c] = (gamma - 1.0) * eint;
  out[4 * plane + c] = eint / rho;
}
}  // namespace

void launch_csv_derive(const Field& u, const Field& part, const Layout& L, const Slab& sl,
                       double gamma0, const MatConsts& mc, double* out, unsigned long long* fail,
                       cudaStream_t st) {
  dim3 blk(32, 8);
  dim3 grd(cdiv(L.nx, 32), cdiv(L.ny, 8));
  count_launch(), k_csv_derive<<<grd, blk, 0, st>>>(u, part, L.nx, L.ny, sl.y0, gamma0, mc, out, fail);
}

namespace {
// the partial densities of the cell k_csv_derive flagged (its failure message needs
// them), read in stream order so an asynchronous dump keeps the dump-time values
__global__ void k_csv_failcell(Field part, int n, int nx, int ny, int y0,
                               const unsigned long long* fail, double* out) {
  const unsigned long long f = *fail;
  if (f == ~0ull) return;
  const int i = (int)(f % (unsigned long long)nx), jl = (int)(f / (unsigned long long)nx) - y0;
  if (jl < 0 || jl >= ny) return;
  for (int k = 0; k < n; ++k) out[k] = part.p[k * part.fstride + (int64_t)jl * part.pitch + i];
}
}  // namespace

void launch_csv_failcell(const Field& part, int n, const Layout& L, const Slab& sl,
                         const unsigned long long* fail, double* out, cudaStream_t st) {
  count_launch(), k_csv_failcell<<<1, 1, 0, st>>>(part, n, L.nx, L.ny, sl.y0, fail, out);
}

}  // namespace lfb

// ---------------------------------------------------------------- region ICs
// initialize_hydro for InitKind::regions (run.cpp:29-78): each interior cell
// centre (CartesianGrid::xc/yc) must lie in exactly one region; the cell gets the
// region's primitive state converted with its material's gamma
// (conserved_from_primitive, euler.hpp:87-97) and, with materials, partial
// density rho in its material and 0 elsewhere.  Failures (not exactly one
// region) -> smallest row-major interior index in *fail.
namespace lfb {
namespace {
__global__ void k_init_regions(Field u, Field part, int nx, int ny, int y0g, double x0,
                               double yo, double dx, double dy, int dim2, const double* __restrict__ reg,
                               int nreg, MatConsts mc, double gamma0,
                               unsigned long long* fail) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y * blockDim.y + threadIdx.y;
  if (i >= nx || j >= ny) return;
  const double x = x0 + (i + 0.5) * dx;
  const double y = yo + ((j + y0g) + 0.5) * dy;
  int hits = 0, material = 0;
  double w0 = 0.0, w1 = 0.0, w2 = 0.0, w3 = 0.0;
  for (int r = 0; r < nreg; ++r) {
    const double* R = reg + 9 * r;  // x_min x_max y_min y_max rho u v p material(1-based)
    const bool in_x = x >= R[0] && x < R[1];
    const bool in_y = !dim2 || (y >= R[2] && y < R[3]);
    if (in_x && in_y) {
      ++hits;
      w0 = R[4];
      w1 = R[5];
      w2 = R[6];
      w3 = R[7];
      material = (int)R[8] - 1;
    }
  }
  if (hits != 1) {
    atomicMin(fail, (unsigned long long)((int64_t)(j + y0g) * nx + i));
    return;
  }
  const double gamma = mc.n > 0 ? mc.gamma[material] : gamma0;
  const int64_t o = (int64_t)j * u.pitch + i;
  u.p[o] = w0;
  u.p[u.fstride + o] = w0 * w1;
  u.p[2 * u.fstride + o] = w0 * w2;
  u.p[3 * u.fstride + o] = w3 / (gamma - 1.0) + 0.5 * w0 * (w1 * w1 + w2 * w2);
  for (int k = 0; k < mc.n; ++k) part.p[k * part.fstride + o] = k == material ? w0 : 0.0;
}
}  // namespace

void launch_init_regions(const Field& u, const Field& part, const Layout& L, const Slab& sl,
                         double x0, double y0, double dx, double dy, int dim2, const double* reg,
                         int nreg, const MatConsts& mc, double gamma0, unsigned long long* fail,
                         cudaStream_t st) {
  dim3 blk(32, 8);
  dim3 grd((unsigned)((L.nx + 31) / 32), (unsigned)((L.ny + 7) / 8));
  count_launch(), k_init_regions<<<grd, blk, 0, st>>>(u, part, L.nx, L.ny, sl.y0, x0, y0, dx, dy,
                                                     dim2, reg, nreg, mc, gamma0, fail);
}

}  // namespace lfb
